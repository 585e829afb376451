import sys
import numpy as np
d = np.loadtxt(sys.argv[1], dtype=np.int64)
d = d[d[:, 1] == 0]
w, tf, ep, pub = d[5:35, 2], d[5:35, 3], d[5:35, 4], d[5:35, 5]
print(f"mma {np.mean(tf - w) / 1e3:.2f}  epi {np.mean(ep - tf) / 1e3:.2f}  publish {np.mean(pub - ep) / 1e3:.2f}  "
      f"period {np.mean(np.diff(w)) / 1e3:.2f} us")
if d.shape[1] > 6:
    l0, cl, sw = d[5:35, 6], d[5:35, 7], d[5:35, 8]
    print(f"  epi detail (warp 4): first ld {np.mean(l0 - tf) / 1e3:.2f}  chunks {np.mean(cl - l0) / 1e3:.2f}  "
          f"st wait {np.mean(sw - cl) / 1e3:.2f}  barrier {np.mean(ep - sw) / 1e3:.2f} us")
