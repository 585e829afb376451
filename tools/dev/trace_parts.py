"""[needs the dev-hooks library: python paper_2508_17655_b200/build.py --devhooks, then
SBG_LIB_OVERRIDE=paper_2508_17655_b200/libsbgpu_dev.so]
Timeline of the parts kernel (SBG_RES_TRACE=1): pair 0's leader CTA, group 0, parts 0/1.
Prints, per part, the mean time of each event relative to part 0's G-dependency-met stamp of
the same step (us), and the step period."""
import sys
import numpy as np
d = np.loadtxt(sys.argv[1], dtype=np.int64)
names = {0: "dep met", 8: "loads issued", 6: "1st round landed", 7: "all landed", 9: "MMAs issued",
         1: "acc ready", 10: "tile free", 11: "1st chunk loaded", 12: "math done", 13: "st waited",
         2: "epilogue done", 3: "publisher has tile", 4: "store complete", 5: "released"}
order = [0, 8, 6, 7, 9, 1, 10, 11, 12, 13, 2, 3, 4, 5]
steps = sorted(set(d[:, 0]))[5:40]
ref = {s: d[(d[:, 0] == s) & (d[:, 1] == 0)][0, 2] for s in steps}
for part in (0, 1):
    rows = {s: d[(d[:, 0] == s) & (d[:, 1] == part)][0, 2:] for s in steps}
    out = []
    for k in order:
        v = np.mean([(rows[s][k] - ref[s]) / 1e3 for s in steps if rows[s][k] > 0])
        out.append(f"{names[k]} {v:+.2f}")
    print(f"part {part}: " + " | ".join(out))
per = np.mean(np.diff([ref[s] for s in steps])) / 1e3
print(f"period {per:.2f} us")
