"""Runs the C2 step loop for profiling: N=2000, GdSB (or --variant), R replicas, K steps."""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2000)
ap.add_argument("--R", type=int, default=8192)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--variant", default="gdsb")
ap.add_argument("--warm", type=int, default=3, help="warm-up steps before the timed launch (clocks up)")
args = ap.parse_args()
s = Solver(0)
s.gen_random_dense(args.n, 1)
s.init_state(args.R, InitMode.small_uniform, 1, 7)
cfg = SolverConfig(variant=Variant[args.variant], steps=1000, dt=1.25, c=1 / (2 * math.sqrt(args.n)), a=0.2)
s.advance(cfg, 0, args.warm)  # warm-up: lazy module load + B-operand prep outside the timed launch
s.synchronize()
s.advance(cfg, args.warm, args.warm + args.steps)
s.synchronize()
ms = s.last_advance_ms()
print(f"{args.variant} n={args.n} R={args.R}: {ms / args.steps * 1e3:.1f} us/step, "
      f"{args.n * args.R * args.steps / (ms / 1e3):.3e} SU/s")
s.close()
