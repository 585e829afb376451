"""One resident-kernel launch at C2 (N=2000, R=8192, GdSB) for ncu."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
R = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
s = Solver(0)
s.gen_random_dense(2000, 1)
s.init_state(R, InitMode.small_uniform, 1, 7)
cfg = SolverConfig(variant=Variant.gdsb, steps=max(1000, steps + 10), dt=1.25, c=1 / (2 * math.sqrt(2000)), a=0.2)
s.advance(cfg, 0, 3)
s.synchronize()
s.advance(cfg, 3, 3 + steps)
print(f"{s.last_advance_ms() / steps * 1e3:.2f} us/step")
