"""Dev: where the e2e time goes at C2 (sbg_run with pinned x0/y0) vs the device-only advance."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, TuningResult, Variant  # noqa: E402

n, R, K = 2000, 8192, 200
c = 1 / (2 * math.sqrt(n))
s = Solver(0)
s.gen_random_dense(n, 1)
x0 = (torch.rand(R, n) * 0.2 - 0.1).pin_memory()
y0 = (torch.rand(R, n) * 0.2 - 0.1).pin_memory()
tun = TuningResult(c=c, dt=1.25)
for M in (K, 1000):
    cfg = SolverConfig(variant=Variant.gdsb, steps=M, dt=1.25, c=c, a=0.2)
    s.init_state(R, InitMode.small_uniform, 1, 7)
    s.advance(cfg, 0, K)
    s.synchronize()
    s.init_state(R, InitMode.small_uniform, 1, 7)
    s.advance(cfg, 0, K)
    print(f"advance M={M}: {s.last_advance_ms():.3f} ms / {K} steps")
cfg = SolverConfig(variant=Variant.gdsb, steps=K, dt=1.25, c=c, a=0.2)
for serial in ("0", "1"):
    os.environ["SBG_RUN_SERIAL"] = serial
    for _ in range(2):
        b = s.run_batch(cfg, tun, R, x0=x0.numpy(), y0=y0.numpy(), want_spins=False)
    print(f"run_batch serial={serial}: {b.timing}")
