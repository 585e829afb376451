import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant
n, R = int(sys.argv[1]), int(sys.argv[2])
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
res = {}
for flag in ("1", "0"):
    os.environ["SBG_RESIDENT"] = flag
    with Solver(0) as s:
        s.gen_random_dense(n, 1)
        s.init_state(R, InitMode.small_uniform, 1, 7)
        cfg = SolverConfig(variant=Variant.gdsb, steps=100, dt=1.25, c=1 / (2 * math.sqrt(n)), a=0.2)
        s.advance(cfg, 0, steps)
        res[flag] = s.get_state()
x1, x0 = res["1"][0], res["0"][0]
bad = np.argwhere(x1 != x0)
print("mismatches", len(bad))
if len(bad):
    rr = np.unique(bad[:, 0]); ss = np.unique(bad[:, 1])
    print("replicas", rr[:20], len(rr), "mod160", np.unique(rr % 160)[:20])
    print("spins", ss[:20], len(ss), "spin blocks", np.unique(ss // 128))
