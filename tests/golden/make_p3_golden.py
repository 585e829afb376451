"""P3 golden vectors at the BASELINE config sizes, from the REAL reference.

TEST INFRASTRUCTURE ONLY. Run in the build container (needs /root/reference and
`make -C oracle`):

    python tests/golden/make_p3_golden.py

Writes tests/golden/golden_p3.npz:

* C1/C2 geometry: gen_random_dense(2000, 1) (model.cpp:144-159), BASELINE init
  x0, y0 ~ U(-0.1, 0.1) fp32 for replicas r = 0, 1 (derive_seed(1, {7, r}); the
  device init the GPU uses, bit-exact with orc_init_small_uniform), p0 = 1.
  x after 30 steps of the reference's fp64 step() (engine.cpp:55-110, parity build
  -O3 -ffp-contract=off) for bsb, dsb, gbsb (A = 0.2, dt = 1.25, c = 1/(2 sqrt N),
  M = 1000 schedule).
* C4 geometry: the SK instance orc_gen_sk_f32(4096, 1) (J ~ N(0, 1/N) fp32,
  symmetric, zero diagonal; widened to fp64 for the reference), same init rule,
  x after 30 steps of bsb and gbsb with c = 0.5 (Wigner for sigma = 1/sqrt N).

The instances themselves are not stored: the GPU box regenerates them (device
generator / oracle restatement, both pinned bitwise to gen_random_dense).
GdSB has no reference step; its fp64 restatement (orc_step_f64 variant 3,
pinned at A = 0 to the reference dsb) is run by the test itself.
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_p3.npz")
STEPS, M, A, DT = 30, 1000, 0.2, 1.25


def main() -> None:
    R = oracle.ref("parity")
    orc = oracle.orc()
    g = {}
    for tag, n, variants, c, J in (
            ("pm1_n2000", 2000, (0, 1, 2), 1.0 / (2.0 * math.sqrt(2000)), None),
            ("sk_n4096", 4096, (0, 2), 0.5, None)):
        J = R.gen_random_dense(n, 1) if tag.startswith("pm1") else orc.gen_sk_f32(n, 1).astype(np.float64)
        x0, y0, _ = orc.init_small_uniform(n, 2, master=1, tag=7)
        g[f"{tag}_x0"] = x0
        g[f"{tag}_y0"] = y0
        g[f"{tag}_c"] = np.float64(c)
        for v in variants:
            # bsb (A = 0, no per-spin control) loses fp32 accuracy fastest: also kept at 20 steps
            for steps in ((20, STEPS) if v == 0 else (STEPS,)):
                xs = []
                for r in range(2):
                    x, _, _ = R.step_n(v, J, x0[r].astype(np.float64), y0[r].astype(np.float64), np.ones(n), 0, M, DT,
                                       c, A, steps)
                    xs.append(x)
                g[f"{tag}_v{v}_x{steps}"] = np.stack(xs)
            print(tag, v, flush=True)
    np.savez_compressed(OUT, steps=np.int64(STEPS), M=np.int64(M), a=np.float64(A), dt=np.float64(DT), **g)


if __name__ == "__main__":
    main()
