"""[needs the dev-hooks library: python paper_2508_17655_b200/build.py --devhooks, then
SBG_LIB_OVERRIDE=paper_2508_17655_b200/libsbgpu_dev.so]
Every step of the traced group of the TS kernel (SBG_RES_TRACE = 1 + launch-relative group): per
part the dependency-met and released times relative to the group's first stamp, and part 0's period."""
import sys
import numpy as np
d = np.loadtxt(sys.argv[1], dtype=np.int64)
d = d[d[:, 2:].max(axis=1) > 0]
row = lambda s, p: d[(d[:, 0] == s) & (d[:, 1] == p)][0, 2:]
steps = sorted(set(d[:, 0]))
nparts = int(d[:, 1].max()) + 1
t0 = min(row(steps[0], p)[0] for p in range(nparts) if row(steps[0], p)[0] > 0)
prev = None
for s in steps:
    dep = [(row(s, p)[0] - t0) / 1e3 for p in range(nparts)]
    acc = [(row(s, p)[1] - t0) / 1e3 for p in range(nparts)]
    epi = [(row(s, p)[2] - t0) / 1e3 for p in range(nparts)]
    rel = [(row(s, p)[5] - t0) / 1e3 for p in range(nparts)]
    print(f"{s:3d} dep " + " ".join(f"{x:7.2f}" for x in dep) + " | acc " + " ".join(f"{x:7.2f}" for x in acc) +
          " | epi " + " ".join(f"{x:7.2f}" for x in epi) + " | rel " + " ".join(f"{x:7.2f}" for x in rel) +
          (f" | period {dep[0] - prev:.2f}" if prev is not None else ""))
    prev = dep[0]
