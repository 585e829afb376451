"""[needs the dev-hooks library: python paper_2508_17655_b200/build.py --devhooks, then
SBG_LIB_OVERRIDE=paper_2508_17655_b200/libsbgpu_dev.so]
Step periods of part 0 at the start of group 0 (SBG_RES_TRACE=1): how fast the four staggered
part chains of the TS kernel settle into the steady state."""
import sys
import numpy as np
d = np.loadtxt(sys.argv[1], dtype=np.int64)
row = lambda s, p: d[(d[:, 0] == s) & (d[:, 1] == p)][0, 2:]
dep = [row(s, 0)[0] / 1e3 for s in range(0, 40)]
per = np.diff(dep)
print("periods of steps 1..16:", " ".join(f"{x:.2f}" for x in per[:16]))
print(f"mean of steps 1..8 {per[:8].mean():.2f}  steps 20..39 {per[19:].mean():.2f} us")
