"""Dev: summarise gpurun_out/pair_utrace.txt (SBG_PAIR_TRACE): per step, per unit kind (whole /
K part / last part), mean durations of MMA (start -> issued), epilogue (tfull -> done) and the
time from a pair's previous epilogue end to its next MMA start."""
import sys
import numpy as np
d = np.loadtxt(sys.argv[1], dtype=np.int64)
cta, slot, t0, t1, t2, t3, t4, t5, meta = d.T
# the MMA stamps (t0, t1, t5) exist only on the leader CTA of each pair (even CTA index)
t_min = t0[t0 > 0].min()
s = meta >> 40
kp = (meta >> 4) & 0xF
ks = meta & 0xF
for st in sorted(set(s))[:3]:
    m = (s == st) & (t2 > 0)
    print(f"step {st}: units {m.sum()}, epi-end span {(t4[m].min() - t_min) / 1e3:.1f} .. {(t4[m].max() - t_min) / 1e3:.1f} us")
    for name, mm in (("whole", m & (ks == 1)), ("part", m & (ks > 1) & (kp < ks - 1)), ("last", m & (ks > 1) & (kp == ks - 1))):
        if mm.sum() == 0:
            continue
        ld = mm & (cta % 2 == 0)
        mma = (t1[ld] - t0[ld]) / 1e3
        epi = (t4[mm] - t2[mm]) / 1e3
        wt = (t0[ld] - t5[ld]) / 1e3
        kd = np.where(t3[mm] > 0, (t3[mm] - t2[mm]) / 1e3, 0)
        print(f"  {name:5s} n={mm.sum():4d} wait-acc {wt.mean():7.1f}  mma {mma.mean():7.1f}  epi {epi.mean():6.1f} "
              f"(kdone wait {kd.mean():5.1f})  start {(t0[ld].min()-t_min)/1e3:7.1f}..{(t0[ld].max()-t_min)/1e3:7.1f}  "
              f"end {(t4[mm].min()-t_min)/1e3:7.1f}..{(t4[mm].max()-t_min)/1e3:7.1f}")
