"""[needs the dev-hooks library: python paper_2508_17655_b200/build.py --devhooks, then
SBG_LIB_OVERRIDE=paper_2508_17655_b200/libsbgpu_dev.so]
Per-group timeline of the TS kernel (SBG_RES_GTRACE=1): for each replica group the median over CTAs
of group start (0), p loaded + G_0 handed over (1), first / second accumulator ready (2, 3), last step
done (4), p stored (5), helper done with the group's G_0 (6), all relative to the earliest stamp."""
import sys
import numpy as np
d = np.loadtxt(sys.argv[1], dtype=np.int64)  # cta group k time
t0 = d[:, 3].min()
names = ["start", "p+G0", "acc0", "acc1", "last", "p_st", "helper"]
for g in sorted(set(d[:, 1])):
    out = []
    for k in range(7):
        v = d[(d[:, 1] == g) & (d[:, 2] == k)][:, 3]
        out.append(f"{names[k]} {np.median(v - t0) / 1e3:7.1f}" if len(v) else f"{names[k]}     n/a")
    print(f"group {g}: " + " | ".join(out))
print(f"span {(d[:, 3].max() - t0) / 1e3:.1f} us")
