"""C4 (SK N=4096, GbSB, R=2048, real J as fixed-point planes): a short advance for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402  (instance generator only)
from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
n = 4096
J = oracle.orc().gen_sk_f32(n, 1)
with Solver(0) as s:
    s.set_instance(J)
    cfg = SolverConfig(variant=Variant.gbsb, steps=1000, dt=1.25, c=0.5, a=0.2)
    s.init_state(2048, InitMode.small_uniform, 1, 7)
    s.advance(cfg, 0, 3)
    s.synchronize()
    s.advance(cfg, 3, 3 + steps)
    print(f"{s.last_advance_ms() / steps * 1e3:.2f} us/step")
