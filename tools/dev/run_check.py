"""sbg_run pipelined (default) vs serial (SBG_RUN_SERIAL=1): identical results; e2e timing."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2508_17655_b200 import Solver, SolverConfig, TuningResult, Variant  # noqa: E402

orc = oracle.orc()
for n, R, M in [(2000, 8192, 200), (300, 1000, 50), (2000, 3000, 37)]:
    x0, y0, _ = orc.init_small_uniform(n, R, master=1)
    c = 1 / (2 * math.sqrt(n))
    cfg = SolverConfig(variant=Variant.gdsb, steps=M, dt=1.25, c=c, a=0.2)
    out = {}
    for mode in ("1", "0"):
        os.environ["SBG_RUN_SERIAL"] = mode
        with Solver(0) as s:
            s.gen_random_dense(n, 1)
            s.run_batch(cfg, TuningResult(c=c, dt=1.25), R, x0=x0, y0=y0, want_spins=False)
            t0 = time.perf_counter()
            b = s.run_batch(cfg, TuningResult(c=c, dt=1.25), R, x0=x0, y0=y0, want_x=True)
            dt = time.perf_counter() - t0
            out[mode] = (b, dt)
    a, bb = out["1"][0], out["0"][0]
    same = (a.x_final.view(np.uint32) == bb.x_final.view(np.uint32)).all() and (a.energies == bb.energies).all()
    print(f"n={n} R={R} M={M}: identical={same} serial {out['1'][1]*1e3:.2f} ms, pipelined {out['0'][1]*1e3:.2f} ms, "
          f"timing {bb.timing}")
