"""C3 (N=20000 ER d=10, GbSB, R=512): a short advance for an ncu capture of the CSR step kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402  (instance generator only)
from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
n, m = 20000, 100000
_, csr = oracle.orc().gen_er_csr(n, m, 1)
with Solver(0) as s:
    s.set_instance_csr(n, *csr)
    cfg = SolverConfig(variant=Variant.gbsb, steps=1000, dt=1.25, c=0.15810993011193192, a=0.2)
    s.init_state(512, InitMode.small_uniform, 1, 7)
    s.advance(cfg, 0, 3)
    s.synchronize()
    s.advance(cfg, 3, 3 + steps)
    print(f"{s.last_advance_ms() / steps * 1e3:.2f} us/step")
