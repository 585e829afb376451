"""Long-run reference fixtures for statistical parity and the TTS99 target (P4).

TEST INFRASTRUCTURE ONLY. Run in the build container, where /root/reference
exists and `make -C oracle` has built oracle/_ref:

    python tests/golden/make_tts_ref.py gbsb      # ~2.5 h on 8 cores
    python tests/golden/make_tts_ref.py gdsb      # ~5 min  (M=1000)
    python tests/golden/make_tts_ref.py gdsb_long # ~2.5 h  (M=21500)
    python tests/golden/make_tts_ref.py sk        # C4: SK N=4096 energy law, 256 trials

Instance: gen_random_dense(2000, 1) (model.cpp:144-159), the seeded stand-in
for K2000 (the G-set file is not in this container).
Settings are the paper's K2000 ones: A=0.2, dt=1.25, c=1/(2*sqrt(N))
(PAPER.md:463,471,366); Wigner tuning gives exactly this c and dt
(spectral.cpp:34-48).

Trials: r = 0..999 with seed_r = derive_seed(MASTER, {seed_stream::batch=3, r}),
exactly the replica seeding of batch_best_of (bench.cpp:77-82), each run
from the reference's own init_state(n, seed_r, uniform_random)
(engine.cpp:25-39).

* gbsb: every trial is the UNMODIFIED reference `run()` (engine.cpp:112-139),
  oracle/_ref timing flavour (the reference's -O3 with an AVX-512 ISA),
  M = 21500 steps.
* gdsb / gdsb_long: GdSB does not exist in the reference; the
  trials run the fp64 restatement `orc_step_f64` variant 3 (oracle/sbg_oracle.c,
  pinned at A=0 to the reference's dsb bitwise, tests/test_oracle.py) from the
  reference's own init_state words, M = 1000 / 21500.

Output: tests/golden/tts_ref_<tag>.npz with per-trial final energies (exact
integers for +-1 J), the seeds, and the settings. The file is written every
few completed trials so an interrupted run keeps its progress and resumes.
"""
from __future__ import annotations

import math
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
N, INST_SEED, MASTER, TRIALS = 2000, 1, 1, 1000
A, DT = 0.2, 1.25
C = 1.0 / (2.0 * math.sqrt(N))
JOBS = {"gbsb": (2, 21500), "gdsb": (3, 1000), "gdsb_long": (3, 21500)}


def sk_job() -> None:
    """C4 (BASELINE configs[3]) energy law: SK N=4096 (orc_gen_sk_f32(4096, 1), J ~ N(0, 1/N)
    fp32 widened to fp64), GbSB, A=0.2, dt=1.25, c=0.5 (Wigner for sigma = 1/sqrt N), M=1000,
    256 trials from the BASELINE init x0, y0 ~ U(-0.1, 0.1) of replicas r < 256
    (derive_seed(1, {7, r}), the states the GPU test injects); every trial is the UNMODIFIED
    reference step() (replica fan-out, ref_replica_fanout) and ising_energy (model.cpp:112-123)."""
    R = oracle.ref("timing")
    orc = oracle.orc()
    n, trials, M = 4096, 256, 1000
    J = orc.gen_sk_f32(n, 1).astype(np.float64)
    x0, y0, _ = orc.init_small_uniform(n, trials, master=1, tag=7)
    t0 = time.time()
    e, wall = R.replica_fanout(2, J, x0, y0, M, DT, 0.5, A, 0)
    print(f"sk: {trials} trials in {time.time() - t0:.0f} s", flush=True)
    np.savez_compressed(os.path.join(HERE, "tts_ref_sk_n4096.npz"), energies=e, variant=np.int64(2), steps=np.int64(M),
                        a=np.float64(A), dt=np.float64(DT), c=np.float64(0.5), n=np.int64(n), master=np.int64(1),
                        tag=np.int64(7), source=np.array("oracle/_ref step() fan-out (ref_replica_fanout)"))


def main(tag: str) -> None:
    if tag == "sk":
        return sk_job()
    variant, M = JOBS[tag]
    R = oracle.ref("timing")
    Rp = oracle.ref("parity")
    orc = oracle.orc()
    J = Rp.gen_random_dense(N, INST_SEED)
    J8 = J.astype(np.int8)
    seeds = np.array([Rp.derive_seed(MASTER, [3, r]) for r in range(TRIALS)], np.uint64)
    out = os.path.join(HERE, f"tts_ref_{tag}.npz")
    energies = np.full(TRIALS, np.nan)
    if os.path.exists(out):
        prev = np.load(out)
        energies[:] = prev["energies"]
    todo = [r for r in range(TRIALS) if np.isnan(energies[r])]
    print(f"{tag}: variant {variant}, M={M}, {len(todo)} of {TRIALS} trials to run", flush=True)

    def one(r: int) -> tuple[int, float]:
        seed = int(seeds[r])
        if variant == 2:
            _, e = R.run(variant, J, M, DT, C, A, seed)
            return r, e
        x, y, p = Rp.init_state(N, seed, False)
        x, y, p = orc.step_f64(variant, J, x, y, p, 0, M, DT, C, A, M)
        s = np.where(x >= 0, 1, -1).astype(np.int64)
        return r, -0.5 * float(s @ J8.astype(np.int64) @ s)

    def save() -> None:
        np.savez_compressed(
            out, energies=energies, seeds=seeds, variant=np.int64(variant), steps=np.int64(M), a=np.float64(A),
            dt=np.float64(DT), c=np.float64(C), n=np.int64(N), instance_seed=np.int64(INST_SEED),
            master=np.int64(MASTER), source=np.array("oracle/_ref run()" if variant == 2 else
                                                        "orc_step_f64 GdSB from reference init_state"))

    t0, done = time.time(), 0
    with ThreadPoolExecutor(int(os.environ.get("SBG_JOBS", os.cpu_count() or 1))) as ex:
        for r, e in ex.map(one, todo):
            energies[r] = e
            done += 1
            if done % 16 == 0 or done == len(todo):
                save()
                el = time.time() - t0
                print(f"{done}/{len(todo)} {el:.0f}s best {np.nanmin(energies):.0f}", flush=True)
    save()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gbsb")
