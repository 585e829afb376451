import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import oracle
from paper_2508_17655_b200 import Solver, SolverConfig, Variant
orc = oracle.orc()
n, R, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
J = orc.gen_dense_i8(n, 1)
x0, y0, p0 = orc.init_small_uniform(n, R, master=1)
c = 1 / (2 * math.sqrt(n))
mx, my, mp = orc.step_f32(3, J, x0, y0, p0, 0, 100, np.float32(1.25), np.float32(c), np.float32(0.2), steps)
for flag, cfgk in (("1", "0"), ("1", "11"), ("0", "0")):
    os.environ["SBG_RESIDENT"] = flag
    os.environ["SBG_RES_CFG"] = cfgk
    with Solver(0) as s:
        s.set_instance(J)
        s.set_state(x0, y0, p0)
        s.advance(SolverConfig(variant=Variant.gdsb, steps=100, dt=1.25, c=c, a=0.2), 0, steps)
        x, y, p = s.get_state()
    bad = np.argwhere(x != mx)
    print(f"resident={flag} cfg={cfgk}: mismatches vs mirror {len(bad)}", np.unique(bad[:, 0])[:5] if len(bad) else "")
os.environ["SBG_RESIDENT"] = "1"
os.environ["SBG_RES_CFG"] = "0"
with Solver(0) as s:
    s.set_instance(J)
    s.set_state(x0, y0, p0)
    s.advance(SolverConfig(variant=Variant.gdsb, steps=100, dt=1.25, c=c, a=0.2), 0, 1)
    x, y, p = s.get_state()
m1x, m1y, m1p = orc.step_f32(3, J, x0, y0, p0, 0, 100, np.float32(1.25), np.float32(c), np.float32(0.2), 1)
r = 960
print("x diff", np.abs(x[r] - m1x[r]).max(), "y diff", np.abs(y[r] - m1y[r]).max(), "p diff", np.abs(p[r] - m1p[r]).max())
print("x0 equal input?", (x[r] == x0[r]).all(), "p", p[r][:4], m1p[r][:4], "y", y[r][:4], m1y[r][:4])
# implied field from y: y1 = y0 - (p1 x0 - c F) dt  ->  F = ((y1 - y0)/dt + p1 x0)/c
Fg = ((y[r].astype(np.float64) - y0[r]) / 1.25 + p[r] * x0[r]) / c
Fm = ((m1y[r].astype(np.float64) - y0[r]) / 1.25 + m1p[r] * x0[r]) / c
print("implied F gpu", np.round(Fg[:8]), "mirror", np.round(Fm[:8]))
S = np.where(x0 >= 0, 1, -1)
print("F from S", (J[:8].astype(np.int64) @ S[r].astype(np.int64)))
