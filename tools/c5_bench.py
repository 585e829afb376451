"""C5 on ONE GPU (world = 1): N = 100000 dense +-1 (gen_random_dense(100000, 1) in the
reference's exact draw order, generated on the device, 10 GB int8 + its 5 GB packed e2m1
copy), GdSB, R = 256, M = 5000 schedule; K timed steps in one persistent launch. Bound:
streaming J from HBM -- N^2 / 2 bytes per step on e2m1 operands (N^2 with SBG_Q4=0)."""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100000)
ap.add_argument("--R", type=int, default=256)
ap.add_argument("--steps", type=int, default=20)
args = ap.parse_args()
n, R = args.n, args.R
with Solver(0) as s:
    s.gen_random_dense(n, 1)
    s.init_state(R, InitMode.small_uniform, 1, 7)
    cfg = SolverConfig(variant=Variant.gdsb, steps=5000, dt=1.25, c=1 / (2 * math.sqrt(n)), a=0.2)
    s.advance(cfg, 0, 2)
    s.synchronize()
    s.advance(cfg, 2, 2 + args.steps)
    ms = s.last_advance_ms()
    us = ms / args.steps * 1e3
    fmt = s.operand_format
    jb = float(n) * n / (2.0 if fmt == "e2m1" else 1.0)
    sb = 24.0 * n * R
    out = {"n": n, "R": R, "operands": fmt, "us_per_step": us, "su_per_s": n * R / (us * 1e-6),
           "J_stream_gbs": jb / (us * 1e-6) / 1e9, "algorithmic_gbs": (jb + sb) / (us * 1e-6) / 1e9,
           "hbm_frac": (jb + sb) / (us * 1e-6) / 1e9 / 6553.0,
           "tensor_tops": 2.0 * n * n * R / (us * 1e-6) / 1e12}
    print(json.dumps(out))
