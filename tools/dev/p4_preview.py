"""Dev: GPU GdSB at M=21500 vs a (possibly partial) fp64-restatement fixture -- KS and P_S."""
import math
import sys

import numpy as np
from scipy.stats import ks_2samp

sys.path.insert(0, ".")
from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, TuningResult, Variant  # noqa: E402

d = np.load(sys.argv[1])
e_ref = d["energies"]
done = ~np.isnan(e_ref)
n, M = int(d["n"]), int(d["steps"])
c, dt, a = float(d["c"]), float(d["dt"]), float(d["a"])
with Solver(0) as s:
    s.gen_random_dense(n, int(d["instance_seed"]))
    cfg = SolverConfig(variant=Variant.gdsb, steps=M, dt=dt, c=c, a=a, init_mode=InitMode.uniform_random)
    b = s.run_batch(cfg, TuningResult(c=c, dt=dt), e_ref.size, master_seed=int(d["master"]), want_spins=False)
e_gpu = b.energies
er = e_ref[done]
print("trials", done.sum(), "KS p", ks_2samp(e_gpu, er).pvalue, "means", e_gpu.mean(), er.mean())
for t in (er.min(), np.percentile(er, 10), np.percentile(er, 50)):
    print("target", t, "P_S gpu", (e_gpu <= t).mean(), "ref", (er <= t).mean())
