"""Protocol P4: long runs are chaotic, so they are matched in
distribution. >= 1000 trials of the same seeded instance and initial states on
the GPU (fp32, sm_100a) and on the reference's own fp64 step() (oracle/_ref;
the bitwise-pinned C restatement when _ref is absent); final energies compared
by a two-sample KS test and success probabilities against the best energy seen
by either side, within binomial confidence (success_from_counts, bench.cpp:15-26).
"""
import math

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def reference_final_energies(variant, J8, x0, y0, steps, dt, c, a):
    J = J8.astype(np.float64)
    if oracle.ref_available():
        e, _ = oracle.ref("timing").replica_fanout(variant, J, x0, y0, steps, dt, c, a, 0)
        return e
    orc = oracle.orc()
    out = []
    for r in range(x0.shape[0]):
        x, y, p = orc.step_f64(variant, J, x0[r].astype(np.float64), y0[r].astype(np.float64),
                               np.ones(J.shape[0]), 0, steps, dt, c, a, steps)
        s = np.where(x >= 0, 1, -1).astype(np.int64)
        out.append(-0.5 * float(s @ J8.astype(np.int64) @ s))
    return np.array(out)


def ks_2samp_pvalue(a, b):
    from scipy.stats import ks_2samp

    return ks_2samp(a, b).pvalue


@pytest.mark.parametrize("variant,name", [(2, "gbsb"), (1, "dsb")])
def test_final_energy_distribution_matches_reference(orc, variant, name):
    from paper_2508_17655_b200 import Solver, SolverConfig, TuningResult, Variant

    n, R, M = 100, 1200, 400
    J = orc.gen_dense_i8(n, 77)
    c, dt, a = 1 / (2 * math.sqrt(n)), 1.25, 0.2
    x0, y0, _ = orc.init_small_uniform(n, R, master=21)
    e_ref = reference_final_energies(variant, J, x0, y0, M, dt, c, a)
    with Solver(0) as s:
        s.set_instance(J)
        b = s.run_batch(SolverConfig(variant=Variant(variant), steps=M, dt=dt, c=c, a=a),
                        TuningResult(c=c, dt=dt), R, x0=x0, y0=y0, want_spins=False)
    e_gpu = b.energies
    assert ks_2samp_pvalue(e_gpu, e_ref) > 1e-3, (name, e_gpu.mean(), e_ref.mean())
    target = min(e_gpu.min(), e_ref.min())
    p1, p2 = (e_gpu <= target).mean(), (e_ref <= target).mean()
    pool = (p1 + p2) / 2
    sigma = math.sqrt(max(pool * (1 - pool), 1.0 / R) * 2 / R)
    assert abs(p1 - p2) <= 4 * sigma, (name, p1, p2)
    # at the short-horizon end the two are not independent samples: the first
    # steps agree (P3); here we only require the same law


# ----------------------------------------------------------------- long runs vs the reference (P4)

def _fixture(name):
    import os

    p = os.path.join(os.path.dirname(__file__), "golden", name)
    if not os.path.exists(p):
        pytest.skip(f"tests/golden/{name} not generated (tests/golden/make_tts_ref.py)")
    d = np.load(p)
    if np.isnan(d["energies"]).any():
        pytest.skip(f"tests/golden/{name} is incomplete")
    return d


def _binomial_agree(p1, n1, p2, n2, z=4.0):
    """|p1 - p2| within z standard errors of the difference (success_from_counts'
    binomial sigma, bench.cpp:15-26, per sample; floored at one hit in the larger sample)."""
    s = math.sqrt(max(p1 * (1 - p1), 1.0 / n1) / n1 + max(p2 * (1 - p2), 1.0 / n2) / n2)
    return abs(p1 - p2) <= z * s, s


@pytest.mark.parametrize("fixture,variant", [("tts_ref_gbsb.npz", "gbsb"), ("tts_ref_gdsb.npz", "gdsb"),
                                             ("tts_ref_gdsb_long.npz", "gdsb")])
def test_k2000_long_runs_match_reference(fixture, variant):
    """The north star's statistical pillar at the paper's K2000 settings (PAPER.md:463,471,366:
    M = 21500, A = 0.2, dt = 1.25, c = 1/(2 sqrt N)) on the N=2000 dense +-1 instance: 1000 GPU
    runs with the SAME seeds as the fixture's 1000 reference trials (derive_seed(1, {3, r}),
    batch_best_of's seeding, bench.cpp:77-82; reference init_state, engine.cpp:25-39).
    gbsb: the fixture is the unmodified reference run() (oracle/_ref). gdsb: GdSB does not exist
    in the reference; its fixture is the fp64 restatement (orc_step_f64 variant 3, pinned to
    the reference dsb at A = 0), M = 1000 and 21500.
    Checks: two-sample KS on the final-energy laws; P_S at the REFERENCE's best energy and at
    its 10th / 50th percentile energies within binomial confidence (4 sigma)."""
    from scipy.stats import ks_2samp

    from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, TuningResult, Variant

    d = _fixture(fixture)
    e_ref = d["energies"]
    n, M = int(d["n"]), int(d["steps"])
    c, dt, a = float(d["c"]), float(d["dt"]), float(d["a"])
    with Solver(0) as s:
        s.gen_random_dense(n, int(d["instance_seed"]))
        cfg = SolverConfig(variant=Variant[variant], steps=M, dt=dt, c=c, a=a, init_mode=InitMode.uniform_random)
        b = s.run_batch(cfg, TuningResult(c=c, dt=dt), e_ref.size, master_seed=int(d["master"]), want_spins=False)
    e_gpu = b.energies
    assert ks_2samp(e_gpu, e_ref).pvalue > 1e-3, (variant, M, e_gpu.mean(), e_ref.mean())
    best = float(e_ref.min())
    for tgt in (best, np.percentile(e_ref, 10), np.percentile(e_ref, 50)):
        p1, p2 = float((e_gpu <= tgt).mean()), float((e_ref <= tgt).mean())
        ok, sig = _binomial_agree(p1, e_gpu.size, p2, e_ref.size)
        assert ok, (variant, M, tgt, p1, p2, sig)


def test_c4_sk_energy_law_matches_reference():
    """C4 (BASELINE configs[3]): SK N=4096, J ~ N(0, 1/N), GbSB through the 24-bit fixed-point
    field, R=2048 replicas from the BASELINE init; the first 256 replicas' initial states are
    the fixture's 256 trials of the reference fp64 step() (tests/golden/tts_ref_sk_n4096.npz).
    Final energies (ising_energy, model.cpp:112-123, real J) compared in distribution: KS on
    all 2048 vs the 256 reference trials, and mean energies within 4 standard errors."""
    from scipy.stats import ks_2samp

    import oracle
    from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant

    d = _fixture("tts_ref_sk_n4096.npz")
    e_ref = d["energies"]
    n, M = int(d["n"]), int(d["steps"])
    J = oracle.orc().gen_sk_f32(n, 1)
    with Solver(0) as s:
        s.set_instance(J)
        s.init_state(2048, InitMode.small_uniform, int(d["master"]), int(d["tag"]))
        s.advance(SolverConfig(variant=Variant.gbsb, steps=M, dt=float(d["dt"]), c=float(d["c"]), a=float(d["a"])),
                  0, M)
        _, e_gpu, _, _ = s.readout()
    assert ks_2samp(e_gpu, e_ref).pvalue > 1e-3, (e_gpu.mean(), e_ref.mean())
    se = math.sqrt(e_gpu.var() / e_gpu.size + e_ref.var() / e_ref.size)
    assert abs(e_gpu.mean() - e_ref.mean()) <= 4 * se, (e_gpu.mean(), e_ref.mean(), se)
    # the first 256 GPU replicas ran from exactly the reference trials' initial states
    assert ks_2samp(e_gpu[:256], e_ref).pvalue > 1e-3
