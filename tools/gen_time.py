"""Times the device gen_random_dense (exact reference draw order) at n = 2000 .. 100000."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_17655_b200 import Solver  # noqa: E402
s = Solver(0)
for n in (2000, 20000, 100000):
    for rep in range(2):
        t = time.perf_counter(); s.gen_random_dense(n, 1); dt = time.perf_counter() - t
    print(f"gen_random_dense n={n}: {dt*1e3:.1f} ms (incl. alloc)", flush=True)
t = time.perf_counter(); s.gen_random_dense(100000, 1, 8, 1); print(f"shard 1/8: {(time.perf_counter()-t)*1e3:.1f} ms")
