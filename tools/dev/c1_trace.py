"""Dev: C1 (N=2000 GbSB R=1000) one 20-step launch with the pair-kernel unit trace on."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant  # noqa: E402

with Solver(0) as s:
    s.gen_random_dense(2000, 1)
    s.init_state(1000, InitMode.small_uniform, 1, 7)
    cfg = SolverConfig(variant=Variant.gbsb, steps=1000, dt=1.25, c=1 / (2 * math.sqrt(2000)), a=0.2)
    s.advance(cfg, 0, 3)
    s.synchronize()
    os.environ["SBG_PAIR_TRACE"] = "1"
    s.advance(cfg, 3, 23)
    print("us/step", s.last_advance_ms() * 1e3 / 20)
