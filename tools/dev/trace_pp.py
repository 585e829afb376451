import sys
import numpy as np
d = np.loadtxt(sys.argv[1], dtype=np.int64)
t0 = d[10, 2]
for row in d[10:22]:
    s, X, w, tf, ep, pub = row[:6]
    print(f"s{s} X{X}: G-ready {(w - t0) / 1e3:7.2f}  tfull {(tf - t0) / 1e3:7.2f}  epi-end {(ep - t0) / 1e3:7.2f}  "
          f"published {(pub - t0) / 1e3:7.2f}")
A = d[d[:, 1] == 0]
print("period (us):", np.diff(A[10:40, 2]).mean() / 1e3)
