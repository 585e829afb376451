"""[needs the dev-hooks library: python paper_2508_17655_b200/build.py --devhooks, then
SBG_LIB_OVERRIDE=paper_2508_17655_b200/libsbgpu_dev.so]
Timeline of the TS kernel (SBG_RES_TRACE=1) over all four parts of pair 0's leader CTA, group 0:
for each part the mean time of every event relative to part 0's dependency-met stamp of the same
step, the epilogue's busy time per part, and how long the epilogue waited for each accumulator."""
import sys
import numpy as np
d = np.loadtxt(sys.argv[1], dtype=np.int64)
names = {0: "dep", 8: "ld_issued", 9: "mma_issued", 1: "acc_ready", 10: "tile_free", 11: "chunk0",
         12: "math_done", 2: "epi_done", 3: "pub_has", 4: "stored", 5: "released"}
order = [0, 8, 9, 1, 10, 11, 12, 2, 3, 4, 5]
steps = sorted(set(d[:, 0]))[8:48]
row = lambda s, p: d[(d[:, 0] == s) & (d[:, 1] == p)][0, 2:]
nparts = int(d[:, 1].max()) + 1
ref = {s: row(s, 0)[0] for s in steps}
for p in range(nparts):
    out = []
    for k in order:
        v = [(row(s, p)[k] - ref[s]) / 1e3 for s in steps if row(s, p)[k] > 0]
        out.append(f"{names[k]} {np.mean(v):+.2f}" if v else f"{names[k]} n/a")
    print(f"part {p}: " + " | ".join(out))
per = np.mean(np.diff([ref[s] for s in steps])) / 1e3
print(f"period {per:.2f} us")
# epilogue busy (acc_ready -> epi_done) per part, and its wait before each part (previous epi_done -> acc_ready)
busy = [np.mean([(row(s, p)[2] - row(s, p)[1]) / 1e3 for s in steps]) for p in range(nparts)]
seq = []
for s in steps:
    prev = None
    for p in range(nparts):
        r = row(s, p)
        if prev is not None:
            seq.append((p, (r[1] - prev) / 1e3))
        prev = r[2]
wait = [np.mean([w for q, w in seq if q == p]) for p in range(1, nparts)]
print("epilogue busy per part:", " ".join(f"{b:.2f}" for b in busy), f"sum {sum(busy):.2f}")
print("epilogue wait before parts 1..:", " ".join(f"{w:.2f}" for w in wait))
