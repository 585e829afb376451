"""Edge-of-chaos scan on the GPU (chaos.cpp:11-102): trajectory pairs
2e-6 apart as replica pairs of one launch with per-replica A. Final states bitwise
against the fp32 mirror; mean final delta against the reference's own fp64
chaos_scan within statistical error."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def test_paired_initial_conditions_match_reference():
    from paper_2508_17655_b200.solver import normalized_distance, paired_initial_conditions

    x1, x2 = paired_initial_conditions(64, 12345)
    if oracle.ref_available():
        rx, _, _ = oracle.ref().init_state(64, 12345, chaos_probe=True)
        assert (x1 == rx.astype(np.float32)).all()
    assert abs(normalized_distance(x1, x2) - 1e-6) < 1e-9  # test_chaos.cpp:22-39 (fp32-rounded pair)


def test_chaos_scan_bitwise_vs_mirror_and_statistics(orc):
    from paper_2508_17655_b200 import Solver, SolverConfig, TuningResult
    from paper_2508_17655_b200.solver import _derive_seed, chaos_scan, normalized_distance, paired_initial_conditions

    n, reps, M = 200, 40, 400
    J = orc.gen_dense_i8(n, 21)
    c, dt = 1 / (2 * np.sqrt(n)), 1.25
    a_values = [0.0, 1.0]
    with Solver(0) as s:
        s.set_instance(J)
        rows = chaos_scan(s, a_values, reps, SolverConfig(steps=M, seed=5), TuningResult(c=c, dt=dt))
    # bitwise: replay two pairs with the mirror
    for ai, a in enumerate(a_values):
        for r in (0, reps - 1):
            x1, x2 = paired_initial_conditions(n, _derive_seed(5, [4, ai, r]))
            x0 = np.stack([x1, x2])
            x, _, _ = orc.step_f32(2, J, x0, np.zeros_like(x0), np.ones_like(x0), 0, M, np.float32(dt), np.float32(c),
                                   np.float32(a), M)
            assert rows[ai].final_deltas[r] == normalized_distance(x[0], x[1])
    # statistics vs the reference's own fp64 chaos_scan on the same instance and seeds
    if oracle.ref_available():
        ref = oracle.ref("timing").chaos_scan(J.astype(np.float64), a_values, reps, M, dt, c, 5)
        for ai in range(len(a_values)):
            g, r_ = rows[ai].final_deltas, ref[ai]
            se = np.sqrt(g.var(ddof=1) / reps + r_.var(ddof=1) / reps) + 1e-3
            assert abs(g.mean() - r_.mean()) <= 4 * se, (a_values[ai], g.mean(), r_.mean())
