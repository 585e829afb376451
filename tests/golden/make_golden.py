"""Generate the committed golden vectors from the REAL reference.

Run in the build container (where /root/reference exists and `make -C oracle`
has built oracle/_ref/libsbopt_ref_parity.so, the unmodified reference core
compiled with -ffp-contract=off):

    python tests/golden/make_golden.py

Every array in golden_ref.npz is an output of the reference library itself
(rng.hpp, model.cpp, engine.cpp, kernels.hpp, spectral.cpp, bench.cpp) called
through oracle/ref_shim.cpp. Nothing here is computed by our restatement.
The GPU box has no /root/reference, so the tests read this file instead.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_ref.npz")


def uniform_symmetric_from_words(words: np.ndarray) -> np.ndarray:
    # rng.hpp:67-70 applied to raw next() words (exact in fp64).
    return 2.0 * ((words >> np.uint64(11)).astype(np.float64) * 2.0**-53) - 1.0


def main() -> None:
    R = oracle.ref("parity")
    g: dict[str, np.ndarray] = {}

    # rng.hpp: raw xoshiro256++ words and derive_seed folds
    g["xo_seed"] = np.array([0, 1, 12345, 2**63 + 7], np.uint64)
    g["xo_words"] = np.stack([R.xoshiro(int(s), 64) for s in g["xo_seed"]])
    keys = [(3, 0), (3, 1), (7, 0), (7, 8191), (1, 2, 3)]
    g["ds_master"] = np.array([0, 42, 2**40 + 3], np.uint64)
    g["ds_keys"] = np.array([list(k) + [0] * (3 - len(k)) for k in keys], np.uint64)
    g["ds_nkeys"] = np.array([len(k) for k in keys], np.int64)
    g["ds_out"] = np.array([[R.derive_seed(int(m), k) for k in keys] for m in g["ds_master"]], np.uint64)

    # model.cpp:144-159 dense +-1 instances (int8 is exact)
    for n, seed in [(2, 1), (37, 11), (130, 1)]:
        g[f"J_n{n}_s{seed}"] = R.gen_random_dense(n, seed).astype(np.int8)

    # kernels.hpp coupling_matvec on the tail-rule sizes, sign and real vectors
    J37 = g["J_n37_s11"].astype(np.float64)
    rng = np.random.default_rng(5)
    V = np.where(rng.random((4, 37)) < 0.5, -1.0, 1.0)
    Vr = rng.uniform(-1, 1, (4, 37))
    g["mv_v_sign"], g["mv_v_real"] = V, Vr
    g["mv_out_sign"] = np.stack([R.coupling_matvec(J37, v) for v in V])
    g["mv_out_real"] = np.stack([R.coupling_matvec(J37, v) for v in Vr])

    # model.cpp:112-123 energies
    S = np.where(rng.random((6, 37)) < 0.5, -1, 1).astype(np.int8)
    g["en_spins"] = S
    g["en_energy"] = np.array([R.ising_energy(J37, s) for s in S])

    # engine.cpp step: reference init_state and BASELINE-style injected init,
    # all three reference variants, trajectories at checkpoints.
    n = 37
    c, dt = R.auto_tune_wigner(J37, 1.25)
    g["tune_c"], g["tune_dt"] = np.array(c), np.array(dt)
    M, A = 200, 0.2
    checkpoints = [1, 10, 30, 50, 200]
    g["traj_checkpoints"] = np.array(checkpoints, np.int64)
    for seed in (1, 2):
        x0, y0, p0 = R.init_state(n, seed, False)
        g[f"init_ref_s{seed}_x"] = x0
        for variant in (0, 1, 2):
            xs, ys, ps = [], [], []
            x, y, p, m = x0, y0, p0, 0
            for cp in checkpoints:
                x, y, p = R.step_n(variant, J37, x, y, p, m, M, dt, c, A, cp - m)
                m = cp
                xs.append(x), ys.append(y), ps.append(p)
            g[f"traj_ref_v{variant}_s{seed}_x"] = np.stack(xs)
            g[f"traj_ref_v{variant}_s{seed}_y"] = np.stack(ys)
            g[f"traj_ref_v{variant}_s{seed}_p"] = np.stack(ps)
    # BASELINE init: replica r of master 9 draws x then y from
    # Xoshiro256pp(derive_seed(9, {7, r})), 0.1*uniform_symmetric rounded to fp32.
    for r in (0, 1):
        seed = R.derive_seed(9, [7, r])
        w = R.xoshiro(seed, 2 * n)
        u = uniform_symmetric_from_words(w)
        x0 = (0.1 * u[:n]).astype(np.float32).astype(np.float64)
        y0 = (0.1 * u[n:]).astype(np.float32).astype(np.float64)
        p0 = np.ones(n)
        g[f"init_small_r{r}_x"], g[f"init_small_r{r}_y"] = x0, y0
        for variant in (0, 1, 2):
            x, y, p = R.step_n(variant, J37, x0, y0, p0, 0, M, dt, c, A, 30)
            g[f"traj_small_v{variant}_r{r}_x30"] = x
            g[f"traj_small_v{variant}_r{r}_y30"] = y
            g[f"traj_small_v{variant}_r{r}_p30"] = p

    # engine.cpp run() and bench.cpp batch_best_of on a small instance
    J16 = R.gen_random_dense(16, 88)
    c16, dt16 = R.auto_tune_wigner(J16, 1.25)
    g["J_n16_s88"] = J16.astype(np.int8)
    g["bbo_c"], g["bbo_dt"] = np.array(c16), np.array(dt16)
    for variant in (0, 1, 2):
        s, e, seed = R.batch_best_of(variant, J16, 300, dt16, c16, 0.2, 6, 4242, 2)
        g[f"bbo_v{variant}_spins"], g[f"bbo_v{variant}_energy"], g[f"bbo_v{variant}_seed"] = (
            s, np.array(e), np.array(seed, np.uint64))
        energies = []
        for r in range(6):
            rs = R.derive_seed(4242, [3, r])
            _, er = R.run(variant, J16, 300, dt16, c16, 0.2, rs)
            energies.append(er)
        g[f"bbo_v{variant}_replica_energies"] = np.array(energies)

    # bench.cpp success / TTS (hits, n_rep, t_com) -> (p, dp, tts, dtts)
    cases = [(999, 1000, 0.010), (9, 10, 1.0), (500, 1000, 1.0), (99, 100, 1.0), (9899, 10000, 1.0),
             (1, 1000, 0.5)]
    g["tts_in"] = np.array(cases, np.float64)
    g["tts_out"] = np.array([R.success_tts(int(h), int(nr), t) for h, nr, t in cases])

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(g)} arrays) from {R.path}")


if __name__ == "__main__":
    main()
