"""Per-step timeline of pair 0, group 0, half 0 of the split resident kernel (SBG_RES_TRACE=1):
[0] producer's G dependency satisfied, [6] first operand stage landed (MMA issuer, leader),
[1] accumulator ready (epilogue), [2] epilogue done + tile handed over, [3] publisher has
the tile, [4] TMA store complete, [5] done[] released."""
import sys
import numpy as np
d = np.loadtxt(sys.argv[1], dtype=np.int64)
d0 = d[d[:, 1] == 0][5:40]
d1 = d[d[:, 1] == 1][5:40]
w, t1, t2, t3, t4, t5, t6, t7 = (d0[:, 2 + i] for i in range(8))
nxt = np.roll(w, -1)
sl = slice(0, -1)
f = lambda a: f"{np.mean(a[sl]) / 1e3:.2f}"  # noqa: E731
print(f"wait->first stage {f(t6 - w)}  first stage->acc ready {f(t1 - t6)}  epilogue {f(t2 - t1)}  "
      f"handover {f(t3 - t2)}  store {f(t4 - t3)}  proxy fence {f(t7 - t4)}  gpu fence+red {f(t5 - t7)}  release->next wait done {f(nxt - t5)}  "
      f"period {f(nxt - w)} us")
