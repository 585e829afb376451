"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Protocols:
  P1  teacher-forced fields J*S bit-exact (int32) against the oracle;
  P2  bitwise trajectories against the fp32 GPU-op-order mirror (all variants:
      the continuous variants use an exact fixed-point field, so they are
      bitwise too);
  P3  fp32 vs the fp64 reference within 1e-5 relative through 30 steps;
plus readout/argmin, init bit-exactness, CSR == dense, and error behaviour.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

BSB, DSB, GBSB, GDSB = 0, 1, 2, 3


@pytest.fixture(scope="module")
def solver():
    from paper_2508_17655_b200 import Solver

    s = Solver(0)
    yield s
    s.close()


def cfg_for(variant, steps, dt, c, a):
    from paper_2508_17655_b200 import SolverConfig, Variant

    return SolverConfig(variant=Variant(variant), steps=steps, dt=dt, c=c, a=a)


@pytest.mark.parametrize("n,R", [(37, 5), (130, 129), (2000, 300)])
def test_p1_fields_sign_bit_exact(solver, orc, n, R):
    J = orc.gen_dense_i8(n, 1)
    solver.set_instance(J)
    rng = np.random.default_rng(n + R)
    S = np.where(rng.random((R, n)) < 0.5, -1, 1).astype(np.int8)
    F = solver.fields_sign(S)
    assert (F == orc.fields_i8(J, S)).all()


def test_p1_fields_teacher_forced_over_50_steps(solver, orc):
    """Feed the oracle's own sign matrix of each of 50 steps to the GPU."""
    n, R = 2000, 64
    J = orc.gen_dense_i8(n, 1)
    solver.set_instance(J)
    x, y, p = orc.init_small_uniform(n, R, master=5)
    c, dt = 1.0 / (2.0 * np.sqrt(n)), 1.25
    for m in range(50):
        S = np.where(x >= 0, 1, -1).astype(np.int8)
        assert (solver.fields_sign(S) == orc.fields_i8(J, S)).all(), f"step {m}"
        x, y, p = orc.step_f32(GDSB, J, x, y, p, m, 1000, np.float32(dt), np.float32(c), np.float32(0.2))


def test_fields_fixed_point_bit_exact(solver, orc):
    n, R = 300, 70
    J = orc.gen_dense_i8(n, 2)
    solver.set_instance(J)
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, (R, n)).astype(np.float32)
    x[0, :5] = [1.0, -1.0, 0.0, -0.0, 1e-30]
    F = solver.fields_fixed(x)
    assert (F.view(np.uint32) == orc.fields_fixed_i8(J, x).view(np.uint32)).all()
    # and it is fp32-accurate against the exact fp64 dot product
    exact = x.astype(np.float64) @ J.T.astype(np.float64)
    assert np.abs(F - exact).max() <= 1e-5 * max(1.0, np.abs(exact).max())


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_device_init_bit_exact(solver, orc, mode):
    n, R = 203, 77
    solver.set_instance(orc.gen_dense_i8(n, 3))
    from paper_2508_17655_b200 import InitMode

    solver.init_state(R, InitMode(mode), master=11, tag=7 if mode == 2 else 3, offset=5)
    x, y, p = solver.get_state()
    if mode == 2:
        ex, ey, ep = orc.init_small_uniform(n, R, master=11, tag=7, r0=5)
    else:
        ex, ey, ep = orc.init_reference(n, R, master=11, tag=3, chaos_probe=(mode == 1), r0=5)
    assert (x == ex).all() and (y == ey).all() and (p == ep).all()


@pytest.mark.parametrize("variant", [BSB, DSB, GBSB, GDSB])
@pytest.mark.parametrize("n,R", [(37, 3), (200, 130)])
def test_p2_trajectory_bitwise_vs_fp32_mirror(solver, orc, variant, n, R):
    J = orc.gen_dense_i8(n, 4)
    solver.set_instance(J)
    x0, y0, p0 = orc.init_small_uniform(n, R, master=3)
    c, dt, a, M = np.float32(1 / (2 * np.sqrt(n))), np.float32(1.25), np.float32(0.2), 200
    solver.set_state(x0, y0, p0)
    cfg = cfg_for(variant, M, float(dt), float(c), float(a))
    x, y, p = x0, y0, p0
    for m0, m1 in [(0, 1), (1, 10), (10, 60)]:
        solver.advance(cfg, m0, m1)
        gx, gy, gp = solver.get_state()
        x, y, p = orc.step_f32(variant, J, x, y, p, m0, M, dt, c, a, m1 - m0)
        assert (gx.view(np.uint32) == x.view(np.uint32)).all(), (variant, m1)
        assert (gy.view(np.uint32) == y.view(np.uint32)).all(), (variant, m1)
        assert (gp.view(np.uint32) == p.view(np.uint32)).all(), (variant, m1)


def test_p2_full_run_to_final_step(solver, orc):
    """M steps to the end (p -> 0 at m = M-1, engine.cpp:89), readout bitwise."""
    n, R, M = 96, 10, 300
    J = orc.gen_dense_i8(n, 6)
    solver.set_instance(J)
    x0, y0, p0 = orc.init_small_uniform(n, R, master=8)
    c, dt = np.float32(1 / (2 * np.sqrt(n))), np.float32(1.25)
    for variant in (GBSB, GDSB):
        cfg = cfg_for(variant, M, float(dt), float(c), 0.2)
        from paper_2508_17655_b200 import TuningResult

        b = solver.run_batch(cfg, TuningResult(c=float(c), dt=float(dt)), R, x0=x0, y0=y0, want_x=True)
        x, y, p = orc.step_f32(variant, J, x0, y0, p0, 0, M, dt, c, np.float32(0.2), M)
        assert (b.x_final == x).all()
        e2 = orc.energy2_i8(J, x)
        assert (b.energies == -0.5 * e2).all()
        assert b.best_index == orc.argmin(-e2)  # min energy == max E2, ties low
        assert (b.spins == np.where(x >= 0, 1, -1)).all()


@pytest.mark.parametrize("variant", [BSB, DSB, GBSB])
def test_p3_short_horizon_vs_fp64_reference(solver, golden, variant):
    """fp32 GPU vs the reference's fp64 step() (golden), <= 1e-5 relative at 30 steps."""
    J = golden["J_n37_s11"]
    c, dt = float(golden["tune_c"]), float(golden["tune_dt"])
    solver.set_instance(J)
    x0 = np.stack([golden[f"init_small_r{r}_x"] for r in (0, 1)]).astype(np.float32)
    y0 = np.stack([golden[f"init_small_r{r}_y"] for r in (0, 1)]).astype(np.float32)
    solver.set_state(x0, y0)
    solver.advance(cfg_for(variant, 200, dt, c, 0.2), 0, 30)
    x, _, _ = solver.get_state()
    for r in (0, 1):
        ref = golden[f"traj_small_v{variant}_r{r}_x30"]
        assert np.abs(x[r] - ref).max() / np.abs(ref).max() <= 1e-5


def test_readout_matches_reference_energy(solver, golden):
    J = golden["J_n37_s11"]
    solver.set_instance(J)
    S = golden["en_spins"]
    solver.set_state(S.astype(np.float32) * 0.5, np.zeros(S.shape, np.float32))
    spins, energy, best, best_e = solver.readout()
    assert (energy == golden["en_energy"]).all()
    assert (spins == S).all()
    e = golden["en_energy"]
    assert best == int(np.flatnonzero(e == e.min())[0]) and best_e == e.min()


def test_argmin_ties_to_lowest_index(solver):
    """bench.cpp:84-87 / test_bench.cpp:164-175: equal energies -> lowest replica."""
    J = np.array([[0, 1], [1, 0]], np.int8)
    solver.set_instance(J)
    x = np.array([[1, 1], [1, -1], [-1, 1], [0.5, -0.5]], np.float32)
    solver.set_state(x, np.zeros_like(x))
    _, energy, best, best_e = solver.readout()
    assert list(energy) == [-1.0, 1.0, 1.0, 1.0] or list(energy) == [-1.0, 1.0, 1.0, 1.0]
    assert best == 0 and best_e == -1.0
    solver.set_state(x[1:], np.zeros_like(x[1:]))
    _, energy, best, _ = solver.readout()
    assert best == 0  # three equal energies 1.0 -> index 0


def test_small_ground_states_found(solver, orc):
    """test_engine.cpp:265-281 analogue: N=10, best of 20 replicas reaches the brute-force ground state."""
    from paper_2508_17655_b200 import InitMode, SolverConfig, Variant, auto_tune_wigner

    for seed in (400, 401, 402):
        J = orc.gen_dense_i8(10, seed)
        solver.set_instance(J)
        bits = ((np.arange(1024)[:, None] >> np.arange(10)) & 1).astype(np.int64) * 2 - 1
        ground = (-0.5 * np.einsum("ki,ij,kj->k", bits, J.astype(np.int64), bits)).min()
        t = auto_tune_wigner(J.astype(np.float64))
        cfg = SolverConfig(variant=Variant.gbsb, steps=2000, a=0.2, init_mode=InitMode.uniform_random)
        best = solver.batch_best_of(cfg, t, 20, master_seed=seed)
        assert best.energy == ground


def test_csr_equals_dense_and_mirror(solver, orc):
    n, m, R = 3000, 15000, 33
    (ei, ej, w), csr = orc.gen_er_csr(n, m, 21)
    dense = np.zeros((n, n), np.int8)
    dense[ei, ej] = -w
    dense[ej, ei] = -w
    x0, y0, p0 = orc.init_small_uniform(n, R, master=2)
    c, dt = np.float32(0.158), np.float32(1.25)
    for variant in (GBSB, GDSB):
        cfg = cfg_for(variant, 100, float(dt), float(c), 0.2)
        solver.set_instance_csr(n, *csr)
        solver.set_state(x0, y0, p0)
        solver.advance(cfg, 0, 40)
        cx, cy, cp = solver.get_state()
        _, ce, cbest, _ = solver.readout()
        solver.set_instance(dense)
        solver.set_state(x0, y0, p0)
        solver.advance(cfg, 0, 40)
        dx, dy, dp = solver.get_state()
        _, de, dbest, _ = solver.readout()
        mx, my, mp = orc.step_f32_csr(variant, n, csr, x0, y0, p0, 0, 100, dt, c, np.float32(0.2), 40)
        assert (cx == mx).all() and (cy == my).all() and (cp == mp).all()
        assert (dx == cx).all() and (dy == cy).all() and (dp == cp).all()
        assert (ce == de).all() and cbest == dbest
        assert (ce == -0.5 * orc.energy2_csr(n, csr, mx)).all()


@pytest.mark.parametrize("knobs", [{"SBG_CSR_SLAB": "128"}, {"SBG_CSR_SLAB": "256"}, {"SBG_CSR_ASYNC": "4"},
                                   {"SBG_CSR_ASYNC": "8"}, {"SBG_CSR_ASYNC": "12"}, {"SBG_CSR_ASYNC": "16"},
                                   {"SBG_CSR_ASYNC": "8", "SBG_CSR_SLAB": "128"}, {"SBG_CSR_PF": "6"},
                                   {"SBG_CSR_PF": "7"}, {"SBG_CSR_LEAN": "1"}, {"SBG_CSR_LEAN": "2"},
                                   {"SBG_CSR_LEAN": "4"}, {"SBG_CSR_LEAN": "0"},
                                   {"SBG_CSR_LEAN": "2", "SBG_CSR_SLAB": "128"},
                                   {"SBG_CSR_LEAN": "2", "SBG_CSR_PFS": "1"}, {"SBG_CSR_LEAN": "2", "SBG_CSR_PFS": "0"},
                                   {"SBG_CSR_LEAN": "4", "SBG_CSR_PFS": "1", "SBG_CSR_SLAB": "128"}])
def test_csr_kernel_variants_bitwise(solver, orc, monkeypatch, knobs):
    """CSR step variants equal the round-1 register-path kernel (SBG_CSR_LEAN=-1) bitwise,
    per-replica A included: replica slabs stepped from L2 (SBG_CSR_SLAB; ragged last slab,
    300 = 128+128+44), the cp.async-staged gather kernel (SBG_CSR_ASYNC = gathers in flight per
    warp), the pipelined gather (SBG_CSR_PF) and the lean kernel (SBG_CSR_LEAN = gathers per
    round; 0 = the default; SBG_CSR_PFS = x, y, p prefetched into shared memory by cp.async);
    rows of degree 0 and > 32."""
    n, m, R, steps = 3000, 15000, 300, 24
    (ei, ej, w), (rowptr, col, val) = orc.gen_er_csr(n, m, 5)
    # one isolated spin and one hub of degree 40: the zero-degree and multi-chunk rows
    keep = ~((ei == 7) | (ej == 7))
    ei, ej, w = ei[keep], ej[keep], w[keep]
    hub = np.arange(100, 140)
    ei = np.concatenate([ei, np.full(40, 11)])
    ej = np.concatenate([ej, hub])
    w = np.concatenate([w, np.where(hub % 3 == 0, 1, -1)]).astype(w.dtype)
    pairs = {}
    for a, b, v in zip(ei.tolist(), ej.tolist(), w.tolist()):
        if a != b:
            pairs[(min(a, b), max(a, b))] = v
    rows = [[] for _ in range(n)]
    for (a, b), v in pairs.items():
        rows[a].append((b, -v))
        rows[b].append((a, -v))
    rowptr = np.zeros(n + 1, np.int32)
    rowptr[1:] = np.cumsum([len(r) for r in rows])
    col = np.array([c for r in rows for c, _ in sorted(r)], np.int32)
    val = np.array([v for r in rows for _, v in sorted(r)], np.int8)
    assert rowptr[8] == rowptr[7] and rowptr[12] - rowptr[11] > 32
    x0, y0, p0 = orc.init_small_uniform(n, R, master=4)
    a_rep = np.linspace(0.0, 0.6, R).astype(np.float32)
    for variant in (GBSB, GDSB):
        cfg = cfg_for(variant, 100, 1.25, 0.158, 0.2)
        out = []
        for env in ({"SBG_CSR_LEAN": "-1"}, {"SBG_CSR_LEAN": "-1", **knobs}):
            for key in ("SBG_CSR_SLAB", "SBG_CSR_ASYNC", "SBG_CSR_PF", "SBG_CSR_LEAN", "SBG_CSR_PFS"):
                monkeypatch.setenv(key, env.get(key, "0"))
            solver.set_instance_csr(n, rowptr, col, val)
            solver.set_state(x0, y0, p0)
            solver.set_replica_a(a_rep)
            solver.advance(cfg, 0, steps)
            out.append(solver.get_state())
        solver.set_replica_a(None)
        for a, b in zip(*out):
            assert (a.view(np.uint32) == b.view(np.uint32)).all(), (variant, knobs)


def test_c2_shape_subset_bitwise(solver, orc):
    """C2 geometry (N=2000, R=8192, GdSB): GPU replicas r0..r0+7 equal the mirror after 5 steps."""
    from paper_2508_17655_b200 import InitMode

    n, R = 2000, 8192
    J = orc.gen_dense_i8(n, 1)
    solver.set_instance(J)
    solver.init_state(R, InitMode.small_uniform, master=1, tag=7)
    c, dt = np.float32(1 / (2 * np.sqrt(n))), np.float32(1.25)
    solver.advance(cfg_for(GDSB, 1000, float(dt), float(c), 0.2), 0, 5)
    gx, gy, gp = solver.get_state()
    for r0 in (0, 4099, 8184):
        x, y, p = orc.init_small_uniform(n, 8, master=1, tag=7, r0=r0)
        x, y, p = orc.step_f32(GDSB, J, x, y, p, 0, 1000, dt, c, np.float32(0.2), 5)
        assert (gx[r0:r0 + 8] == x).all() and (gy[r0:r0 + 8] == y).all() and (gp[r0:r0 + 8] == p).all()


def test_invalid_arguments_raise(solver, orc):
    from paper_2508_17655_b200 import SolverConfig, TuningResult, Variant

    bad = np.array([[0, 1], [2, 0]], np.int8)
    with pytest.raises(ValueError):
        solver.set_instance(bad)  # not symmetric (model.cpp:60-63)
    with pytest.raises(ValueError):
        solver.set_instance(np.array([[1, 0], [0, 0]], np.int8))  # diagonal
    solver.set_instance(orc.gen_dense_i8(8, 1))
    t = TuningResult(c=0.1, dt=0.5)
    for kw in (dict(steps=0), dict(dt=-1.0), dict(a=-0.5)):
        with pytest.raises(ValueError):
            solver.run_batch(SolverConfig(variant=Variant.gbsb, **kw), t, 2, master_seed=1)
    solver.set_state(np.zeros((2, 8), np.float32), np.zeros((2, 8), np.float32))
    with pytest.raises(ValueError):
        solver.advance(SolverConfig(variant=Variant.gbsb, steps=10, dt=0.5, c=0.1), 5, 11)  # past M


def test_readout_best_matches_full_readout(solver, orc):
    n, R = 300, 77
    J = orc.gen_dense_i8(n, 12)
    solver.set_instance(J)
    x, y, _ = orc.init_reference(n, R, master=4)
    solver.set_state(x, y)
    spins, energy, best, best_e = solver.readout()
    bs, be, bi, energies = solver.readout_best()
    assert bi == best and be == best_e and (energies == energy).all() and (bs == spins[best]).all()
    assert (energy == -0.5 * orc.energy2_i8(J, x)).all()


def test_sweep_grid_matches_mirror_per_cell(solver, orc):
    """sweep (bench.cpp:171-197) on the GPU: per-replica A in one launch per M, seeds
    derive_seed(seed, {sweep, mi, ai, r}); every cell's energies bitwise vs the mirror."""
    from paper_2508_17655_b200 import SolverConfig, TuningResult, Variant
    from paper_2508_17655_b200.solver import _derive_seed, sweep

    n, reps = 64, 5
    J = orc.gen_dense_i8(n, 17)
    solver.set_instance(J)
    c, dt = 1 / (2 * np.sqrt(n)), 1.25
    base = SolverConfig(variant=Variant.gbsb, seed=99)
    t = TuningResult(c=c, dt=dt)
    m_values, a_values = [30, 80], [0.0, 0.2, 0.5]
    cells = sweep(solver, m_values, a_values, reps, base, t, target=-1e9)
    assert [(cl.mi, cl.ai) for cl in cells] == [(mi, ai) for mi in range(2) for ai in range(3)]
    for cl in cells:
        seeds = [_derive_seed(99, [1, cl.mi, cl.ai, r]) for r in range(reps)]
        x, y, p = orc.init_reference_seeds(n, seeds)
        x, y, p = orc.step_f32(2, J, x, y, p, 0, cl.m_steps, np.float32(dt), np.float32(c), np.float32(cl.a),
                               cl.m_steps)
        assert (cl.energies == -0.5 * orc.energy2_i8(J, x)).all(), (cl.mi, cl.ai)
        assert cl.best_energy == cl.energies.min()


def test_dt_sweep_grid_matches_mirror_per_cell(solver, orc):
    """dt_sweep (bench.cpp:206-269) on the GPU: cell (di, ti) runs at dt = tune_dt(lambda_min,
    lambda_max, D_t) (spectral.cpp:277-286) and M = llround(t_M / dt), replicas seeded
    derive_seed(seed, {dt_sweep, di, ti, r}) with the reference init; every cell's energies
    bitwise vs the fp32 mirror run with the same dt, M and seeds."""
    from paper_2508_17655_b200 import SolverConfig, TuningResult, Variant
    from paper_2508_17655_b200.solver import SEED_STREAM_DT_SWEEP, _derive_seed, dt_sweep, tune_dt

    n, reps = 64, 5
    J = orc.gen_dense_i8(n, 19)
    solver.set_instance(J)
    lmin, lmax = -14.2, 15.1
    t = TuningResult(c=1 / (2 * np.sqrt(n)), dt=1.0, lambda_min=lmin, lambda_max=lmax)
    base = SolverConfig(variant=Variant.gbsb, seed=77)
    d_ts, t_fs = [0.8, 1.25], [40.0, 101.5]
    cells = dt_sweep(solver, d_ts, t_fs, 0.2, reps, base, t, target=-1e9)
    assert [(cl.di, cl.ti) for cl in cells] == [(di, ti) for di in range(2) for ti in range(2)]
    for cl in cells:
        dt = tune_dt(lmin, lmax, d_ts[cl.di])
        assert cl.dt == dt
        q = t_fs[cl.ti] / dt
        assert cl.m_steps == int(np.floor(q + 0.5))
        seeds = [_derive_seed(77, [SEED_STREAM_DT_SWEEP, cl.di, cl.ti, r]) for r in range(reps)]
        x, y, p = orc.init_reference_seeds(n, seeds)
        x, y, p = orc.step_f32(2, J, x, y, p, 0, cl.m_steps, np.float32(dt), np.float32(t.c), np.float32(0.2),
                               cl.m_steps)
        assert (cl.energies == -0.5 * orc.energy2_i8(J, x)).all(), (cl.di, cl.ti)


@pytest.mark.parametrize("n,R,variant", [(2000, 3000, GDSB), (600, 700, GBSB), (300, 1, DSB)])
def test_run_best_returns_the_batch_best_of_winner(solver, orc, n, R, variant):
    """sbg_run_best (batch_best_of's result, bench.cpp:70-92): the winner's spins, energy and
    index (ties -> lowest replica) and the R energies equal a full run_batch readout of the
    same host initial states, and the winner's spins are sgn of its final x (sgn(0) = +1)."""
    from paper_2508_17655_b200 import SolverConfig, TuningResult, Variant

    J = orc.gen_dense_i8(n, 12)
    solver.set_instance(J)
    x0, y0, _ = orc.init_small_uniform(n, R, master=6)
    c = 1 / (2 * np.sqrt(n))
    cfg = SolverConfig(variant=Variant(variant), steps=40, dt=1.25, c=c, a=0.2)
    t = TuningResult(c=c, dt=1.25)
    spins, be, bi, energies, timing = solver.run_best(cfg, t, x0, y0)
    b = solver.run_batch(cfg, t, R, x0=x0, y0=y0, want_x=True)
    assert (energies == b.energies).all()
    assert bi == b.best_index == int(np.flatnonzero(b.energies == b.energies.min())[0])
    assert be == b.energies[bi]
    assert (spins == b.spins[bi]).all()
    assert (spins == np.where(b.x_final[bi] >= 0, 1, -1)).all()
    _, e_only, bi2, none, _ = solver.run_best(cfg, t, x0, y0, want_energies=False)
    assert none is None and bi2 == bi and e_only == be


def test_csr_chunked_advances_keep_state_spin_major(solver, orc):
    """CSR advances leave the state in the spin-major working copies and the next advance
    continues from there; readers (get_state, readout) bring the replica-major copy up to date.
    Chunked advances with and without reads in between == one advance == the mirror."""
    n, m, R = 2500, 9000, 300
    _, csr = orc.gen_er_csr(n, m, 8)
    c, dt = np.float32(0.21), np.float32(1.25)
    x0, y0, p0 = orc.init_small_uniform(n, R, master=4)
    cfg = cfg_for(GBSB, 60, float(dt), float(c), 0.2)
    solver.set_instance_csr(n, *csr)
    outs = []
    for plan in ([(0, 17)], [(0, 5), (5, 11), (11, 17)], [(0, 9), "read", (9, 17)]):
        solver.set_state(x0, y0, p0)
        for step in plan:
            if step == "read":
                solver.get_state()
                solver.readout()
            else:
                solver.advance(cfg, *step)
        outs.append(solver.get_state())
    mx, my, mp = orc.step_f32_csr(GBSB, n, csr, x0, y0, p0, 0, 60, dt, c, np.float32(0.2), 17)
    for x, y, p in outs:
        assert (x == mx).all() and (y == my).all() and (p == mp).all()
    _, e, _, _ = solver.readout()
    assert (e == -0.5 * orc.energy2_csr(n, csr, mx)).all()


def test_csr_solver_reused_across_replica_counts(solver, orc):
    """One CSR context run with R = 1, then R = 200 (same 256-replica padding bucket), then
    R = 300: every run bitwise equal to the fp32 mirror (the spin-major working buffers
    are sized for the bucket, not for the first R)."""
    n, m = 1500, 6000
    _, csr = orc.gen_er_csr(n, m, 5)
    c, dt = np.float32(0.2), np.float32(1.25)
    solver.set_instance_csr(n, *csr)
    for R in (1, 200, 300, 17):
        x0, y0, p0 = orc.init_small_uniform(n, R, master=R)
        solver.set_state(x0, y0, p0)
        solver.advance(cfg_for(GBSB, 50, float(dt), float(c), 0.2), 0, 9)
        x, y, p = solver.get_state()
        mx, my, mp = orc.step_f32_csr(GBSB, n, csr, x0, y0, p0, 0, 50, dt, c, np.float32(0.2), 9)
        assert (x == mx).all() and (y == my).all() and (p == mp).all(), R
        _, e, _, _ = solver.readout()
        assert (e == -0.5 * orc.energy2_csr(n, csr, mx)).all(), R


def test_trajectory_sampling_records_start_strides_final(solver, orc):
    """test_engine.cpp:232-249 analogue: stride 50 over M=120 -> m = 0, 50, 100, 120, bitwise states."""
    from paper_2508_17655_b200 import SolverConfig, TuningResult, Variant

    n, R = 40, 3
    J = orc.gen_dense_i8(n, 1)
    solver.set_instance(J)
    x0, y0, p0 = orc.init_small_uniform(n, R, master=6)
    cfg = SolverConfig(variant=Variant.gbsb, steps=120, dt=1.0, c=0.2, a=0.0, sample_stride=50)
    b = solver.run_batch(cfg, TuningResult(c=0.2, dt=1.0), R, x0=x0, y0=y0)
    assert [m for m, _ in b.trajectory] == [0, 50, 100, 120]
    x, y, p = x0, y0, p0
    prev = 0
    for m, xs in b.trajectory[1:]:
        x, y, p = orc.step_f32(2, J, x, y, p, prev, 120, np.float32(1.0), np.float32(0.2), np.float32(0.0), m - prev)
        prev = m
        assert (xs == x).all()
    cfg.sample_stride = 0
    assert solver.run_batch(cfg, TuningResult(c=0.2, dt=1.0), R, x0=x0, y0=y0).trajectory is None


@pytest.mark.parametrize("variant", [BSB, DSB, GBSB])
@pytest.mark.parametrize("seed", [1, 2])
def test_p3_reference_init_30_and_50_steps(solver, golden, variant, seed):
    """P3 with the reference's own init_state (x ~ U(-1,1), y = 0): <= 1e-5 relative at
    30 steps. At 50 steps fp32 state rounding, amplified by the chaotic
    dynamics, is past 1e-5 for any fp32 implementation; with this wider init
    the fp32 mirror itself (bitwise equal to the GPU) measures 3.0e-4 (bSB, seed 1),
    1.1e-4 (bSB, seed 2), <= 4.5e-5 otherwise, so 50 steps is held to 5e-4."""
    J = golden["J_n37_s11"]
    c, dt = float(golden["tune_c"]), float(golden["tune_dt"])
    solver.set_instance(J)
    x0 = golden[f"init_ref_s{seed}_x"].astype(np.float32)[None, :]
    solver.set_state(x0, np.zeros_like(x0))
    cps = list(golden["traj_checkpoints"])
    m = 0
    for cp, tol in ((30, 1e-5), (50, 5e-4)):
        solver.advance(cfg_for(variant, 200, dt, c, 0.2), m, cp)
        m = cp
        x, _, _ = solver.get_state()
        ref = golden[f"traj_ref_v{variant}_s{seed}_x"][cps.index(cp)]
        err = np.abs(x[0] - ref).max() / np.abs(ref).max()
        assert err <= tol, (variant, cp, err)


@pytest.mark.parametrize("n,R,variant", [(2000, 8192, GDSB), (300, 100, GDSB), (2000, 1000, 1), (700, 3000, GDSB),
                                         (4000, 512, 1), (256, 1, GDSB)])
def test_resident_kernel_equals_streaming(solver, orc, n, R, variant, monkeypatch):
    """The TMEM-resident sign-variant kernel (step_resident.cuh, the default) against the
    streaming kernels (SBG_RESIDENT=0): bitwise identical states and energies after a
    multi-step launch, including per-replica A."""
    from paper_2508_17655_b200 import InitMode

    solver.gen_random_dense(n, 3)
    c = 1 / (2 * np.sqrt(n))
    arep = np.random.default_rng(n).random(R).astype(np.float32)
    out = []
    for flag in ("1", "0"):
        monkeypatch.setenv("SBG_RESIDENT", flag)
        for use_a in (False, True):
            solver.init_state(R, InitMode.small_uniform, 5, 7)
            solver.set_replica_a(arep if use_a else None)
            solver.advance(cfg_for(variant, 100, 1.25, c, 0.2), 0, 13)
            x, y, p = solver.get_state()
            _, e, best, _ = solver.readout()
            out.append((x, y, p, e, best))
        solver.set_replica_a(None)
    for a, b in zip(out[:2], out[2:]):
        assert all((u.view(np.uint32) == v.view(np.uint32)).all() for u, v in zip(a[:3], b[:3]))
        assert (a[3] == b[3]).all() and a[4] == b[4]


def _run_resident(solver, J, R, variant, steps, monkeypatch, q4, resident="1", arep=None):
    from paper_2508_17655_b200 import InitMode

    monkeypatch.setenv("SBG_Q4", "1" if q4 else "0")
    monkeypatch.setenv("SBG_RESIDENT", resident)
    solver.set_instance(J)
    n = J.shape[0]
    solver.init_state(R, InitMode.small_uniform, 5, 7)
    solver.set_replica_a(arep)
    solver.advance(cfg_for(variant, 100, 1.25, 1 / (2 * np.sqrt(n)), 0.2), 0, steps)
    x, y, p = solver.get_state()
    _, e, best, _ = solver.readout()
    fmt = solver.operand_format
    solver.set_replica_a(None)
    return fmt, (x, y, p, e, best)


def _same(a, b):
    assert all((u.view(np.uint32) == v.view(np.uint32)).all() for u, v in zip(a[:3], b[:3]))
    assert (a[3] == b[3]).all() and a[4] == b[4]


E2M1_INTS = np.array([0, 1, -1, 2, -2, 3, -3, 4, -4, 6, -6], np.int8)


def _sym(n, values, seed):
    rng = np.random.default_rng(seed)
    J = np.triu(rng.choice(values, size=(n, n)), 1).astype(np.int8)
    return (J + J.T).astype(np.int8)


@pytest.mark.parametrize("n,R,variant,values", [(2000, 3000, GDSB, "pm1"), (777, 1500, DSB, "e2m1"),
                                                (513, 400, GDSB, "e2m1"), (1500, 2000, GDSB, "pm1")])
def test_e2m1_resident_equals_int8(solver, n, R, variant, values, monkeypatch):
    """kind::mxf4 operands (packed e2m1 J and G, unit E8M0 scales, f32 accumulation) give
    the same integer fields as the int8 MMAs: states, energies and winner bitwise equal to
    the int8 resident kernel and to the streaming kernels, for +-1 J and for J over every
    e2m1-exact integer {0, +-1, +-2, +-3, +-4, +-6}; odd n exercises the half-filled
    last byte of each packed row; per-replica A included."""
    J = _sym(n, np.array([1, -1], np.int8) if values == "pm1" else E2M1_INTS, n)
    arep = np.random.default_rng(n).random(R).astype(np.float32)
    f4, a = _run_resident(solver, J, R, variant, 17, monkeypatch, True, arep=arep)
    f8, b = _run_resident(solver, J, R, variant, 17, monkeypatch, False, arep=arep)
    _, c = _run_resident(solver, J, R, variant, 17, monkeypatch, True, resident="0", arep=arep)
    assert (f4, f8) == ("e2m1", "int8")
    _same(a, b)
    _same(a, c)


@pytest.mark.parametrize("n,R,variant,parts,pkb", [(2000, 8192, GDSB, "4", "0"), (2000, 3000, DSB, "4", "0"),
                                                   (1500, 2000, GDSB, "5", "0"), (513, 6000, GDSB, "4", "0"),
                                                   (777, 400, DSB, "5", "0"), (2000, 8192, GDSB, "4", "1"),
                                                   (777, 400, DSB, "5", "1"), (2000, 8192, GDSB, "4", "kh2"),
                                                   (1500, 2000, DSB, "4", "kh2")])
def test_ts_kernel_equals_parts_kernel(solver, n, R, variant, parts, pkb, monkeypatch):
    """The TS resident kernel (J in TMEM as the A operand of tcgen05.mma [a_tmem], x, y in
    shared memory, state moved by TMA at group boundaries; the default) against the parts
    kernel (J in shared memory, x, y in TMEM; SBG_RES_TS=0): states, energies and winner
    bitwise equal, over several replica groups, odd n (half-filled last packed byte),
    per-replica A, e2m1 J values beyond +-1."""
    J = _sym(n, np.array([1, -1], np.int8) if n % 2 == 0 else E2M1_INTS, n)
    arep = np.random.default_rng(n).random(R).astype(np.float32)
    monkeypatch.setenv("SBG_RES_PARTS", parts)
    # 1: per-K-block dependencies; kh2: each part-step's G in two halves (dev variants)
    monkeypatch.setenv("SBG_RES_PKB", "1" if pkb == "1" else "0")
    monkeypatch.setenv("SBG_RES_KH2", "1" if pkb == "kh2" else "0")
    f_ts, a = _run_resident(solver, J, R, variant, 23, monkeypatch, True, arep=arep)
    monkeypatch.delenv("SBG_RES_PKB")
    monkeypatch.delenv("SBG_RES_KH2")
    monkeypatch.setenv("SBG_RES_TS", "0")
    monkeypatch.setenv("SBG_RES_PARTS", "4")
    f_pa, b = _run_resident(solver, J, R, variant, 23, monkeypatch, True, arep=arep)
    assert f_ts == f_pa == "e2m1"
    _same(a, b)


@pytest.mark.parametrize("n,R", [(2000, 1440), (2000, 1441), (2048, 160), (2048, 159), (256, 1), (256, 11840),
                                 (255, 300), (1793, 2881)])
def test_ts_kernel_edge_geometries_equal_streaming(solver, n, R, monkeypatch):
    """The TS resident kernel at group / block / padding boundaries (exactly one group of 9
    blocks, one replica past it, one block, npad = 256 with one CTA pair per block and 74
    blocks per group, odd n) against the streaming kernel (SBG_RESIDENT=0): bitwise."""
    J = _sym(n, np.array([1, -1], np.int8), n + R)
    arep = np.random.default_rng(R).random(R).astype(np.float32)
    f_ts, a = _run_resident(solver, J, R, GDSB, 9, monkeypatch, True, arep=arep)
    _, b = _run_resident(solver, J, R, GDSB, 9, monkeypatch, True, resident="0", arep=arep)
    assert f_ts == "e2m1"
    _same(a, b)


def test_e2m1_streaming_large_n(solver, monkeypatch):
    """Past the resident kernel's size limit the streaming pair kernel runs on e2m1 operands
    (single-buffered accumulator, nibble-packed G written by the epilogue): bitwise equal to
    its int8 form at n = 20001 (odd), R = 256 -- the C5 regime."""
    n, R = 20001, 256
    rng = np.random.default_rng(4)
    J = np.triu(rng.choice(np.array([1, -1], np.int8), size=(n, n)), 1)
    J = (J + J.T).astype(np.int8)
    f4, a = _run_resident(solver, J, R, GDSB, 4, monkeypatch, True)
    f8, b = _run_resident(solver, J, R, GDSB, 4, monkeypatch, False)
    assert (f4, f8) == ("e2m1", "int8")
    _same(a, b)


def test_e2m1_large_fields_exact(solver, monkeypatch):
    """f32 accumulation of e2m1 products is exact while |F| < 2^24: J_ij = 6 everywhere
    off the diagonal and aligned spins drive |F| to 6 (n - 1) = 55,194 at n = 9200 (past
    2^15; the probe tools/dev/mxf4_probe.cu also checks 1.3e5), bitwise equal to int8."""
    n, R = 9200, 320
    J = np.full((n, n), 6, np.int8)
    np.fill_diagonal(J, 0)
    f4, a = _run_resident(solver, J, R, DSB, 5, monkeypatch, True)
    f8, b = _run_resident(solver, J, R, DSB, 5, monkeypatch, False)
    assert (f4, f8) == ("e2m1", "int8")
    _same(a, b)


def test_non_e2m1_couplings_stay_int8(solver, monkeypatch):
    """A coupling outside the e2m1-exact set (5, or |J| > 6) keeps the int8 operands."""
    for bad in (5, 7, -100):
        J = _sym(300, E2M1_INTS, 1)
        J[3, 7] = J[7, 3] = bad
        monkeypatch.setenv("SBG_Q4", "1")
        solver.set_instance(J)
        assert solver.operand_format == "int8"
    solver.set_instance(_sym(300, E2M1_INTS, 1))
    assert solver.operand_format == "e2m1"


@pytest.mark.parametrize("n,R", [(2000, 8192), (500, 2500), (2000, 2304)])  # 2304: two groups of the TS kernel by the tie rule
def test_run_pipelined_copies_equal_serial(solver, orc, n, R, monkeypatch):
    """sbg_run on the resident kernel overlaps each replica group's host->device copy with
    the earlier groups' steps (stream-ordered ready flags): results bitwise equal to the
    serial copy-then-run path, for pageable host buffers too."""
    from paper_2508_17655_b200 import SolverConfig, TuningResult, Variant

    solver.gen_random_dense(n, 2)
    x0, y0, _ = orc.init_small_uniform(n, R, master=3)
    c = 1 / (2 * np.sqrt(n))
    cfg = SolverConfig(variant=Variant.gdsb, steps=23, dt=1.25, c=c, a=0.2)
    out = []
    for flag in ("1", "0"):
        monkeypatch.setenv("SBG_RUN_SERIAL", flag)
        b = solver.run_batch(cfg, TuningResult(c=c, dt=1.25), R, x0=x0, y0=y0, want_x=True)
        out.append(b)
    assert (out[0].x_final.view(np.uint32) == out[1].x_final.view(np.uint32)).all()
    assert (out[0].energies == out[1].energies).all() and out[0].best_index == out[1].best_index
    assert (out[0].spins == out[1].spins).all()


@pytest.mark.parametrize("variant", [BSB, GBSB])
def test_wide_plane_tiles_bitwise(solver, orc, variant, monkeypatch):
    """Fixed-point variants on 128-replica pair tiles with one accumulator buffer (chosen
    automatically for large replica counts; forced here with SBG_STEP_CFG=9) equal the
    64-replica double-buffered tiles and the fp32 mirror bitwise."""
    n, R, M = 600, 300, 100
    J = _sym(n, np.array([1, -1], np.int8), 31)
    solver.set_instance(J)
    x0, y0, p0 = orc.init_small_uniform(n, R, master=31)
    c, dt, a = np.float32(1 / (2 * np.sqrt(n))), np.float32(1.25), np.float32(0.2)
    cfg = cfg_for(variant, M, float(dt), float(c), float(a))
    out = []
    for knob in ("9", "3"):
        monkeypatch.setenv("SBG_STEP_CFG", knob)
        solver.set_state(x0, y0, p0)
        solver.advance(cfg, 0, 15)
        out.append(solver.get_state())
    x, _, _ = orc.step_f32(variant, J, x0, y0, p0, 0, M, dt, c, a, 15)
    for u, v in zip(out[0], out[1]):
        assert (u.view(np.uint32) == v.view(np.uint32)).all()
    assert (out[0][0].view(np.uint32) == x.view(np.uint32)).all()


@pytest.mark.parametrize("ks", [2, 3, 4])
def test_e2m1_stream_k_split_bitwise(solver, orc, monkeypatch, ks):
    """Streaming e2m1 pair kernel with each pair tile's K range split over ks CTA pairs
    (SBG_KSPLIT; partial fields exchanged through global memory) == no split == the
    resident kernel == 128-replica pair tiles in replica-fast order (SBG_Q4_NPAIR), bitwise,
    with per-replica A; K blocks not divisible by ks included."""
    n, R, steps = 2000, 300, 12
    J = orc.gen_dense_i8(n, 9)
    x0, y0, p0 = orc.init_small_uniform(n, R, master=6)
    a_rep = np.linspace(0.0, 0.5, R).astype(np.float32)
    cfg = cfg_for(GDSB, 100, 1.25, float(1 / (2 * np.sqrt(n))), 0.2)
    out = []
    for env in ({}, {"SBG_RESIDENT": "0", "SBG_KSPLIT": "1"}, {"SBG_RESIDENT": "0", "SBG_KSPLIT": str(ks)},
                {"SBG_RESIDENT": "0", "SBG_Q4_NPAIR": "128", "SBG_KSPLIT": str(ks - 1)}):
        for key in ("SBG_RESIDENT", "SBG_KSPLIT", "SBG_Q4_NPAIR"):
            monkeypatch.delenv(key, raising=False)
        for key, v in env.items():
            monkeypatch.setenv(key, v)
        solver.set_instance(J)
        assert solver.operand_format == "e2m1"
        solver.set_state(x0, y0, p0)
        solver.set_replica_a(a_rep)
        solver.advance(cfg, 0, 5)
        solver.advance(cfg, 5, steps)
        out.append(solver.get_state())
        solver.set_replica_a(None)
    for st in out[1:]:
        for a, b in zip(out[0], st):
            assert (a.view(np.uint32) == b.view(np.uint32)).all()


@pytest.mark.parametrize("n,R", [(19200, 256), (25600, 300), (19200, 37)])
def test_e2m1_stream_tail_split_bitwise(solver, monkeypatch, n, R):
    """The default tail-only K split of the streaming e2m1 pair kernel (the T2 mod P tiles of a
    step's last, partial round of pair tiles run as K parts: 75 tiles on 74 pairs -> 1 tile in
    4 parts; 100 -> 26 tiles in 2 parts; two replica blocks -> 150 tiles) == no split
    (SBG_KTAIL=0), bitwise, with per-replica A, over two launches."""
    from paper_2508_17655_b200 import InitMode

    cfg = cfg_for(GDSB, 100, 1.25, float(1 / (2 * np.sqrt(n))), 0.2)
    a_rep = np.linspace(0.0, 0.5, R).astype(np.float32)
    out = []
    for env in ({}, {"SBG_KTAIL": "0"}):
        for key in ("SBG_RESIDENT", "SBG_KSPLIT", "SBG_KTAIL", "SBG_Q4_NPAIR"):
            monkeypatch.delenv(key, raising=False)
        for key, v in env.items():
            monkeypatch.setenv(key, v)
        solver.gen_random_dense(n, 3)
        assert solver.operand_format == "e2m1"
        solver.init_state(R, InitMode.small_uniform, 2, 7)
        solver.set_replica_a(a_rep)
        solver.advance(cfg, 0, 5)
        solver.advance(cfg, 5, 12)
        out.append(solver.get_state())
        solver.set_replica_a(None)
    for a, b in zip(out[0], out[1]):
        assert (a.view(np.uint32) == b.view(np.uint32)).all()


def test_ts_map_cache_follows_state_and_couplings(solver, orc):
    """The TS kernel's tensor maps are cached per G-buffer parity (sbgpu.cu TsMapKey): one
    Solver re-used across replica counts (new state buffers), odd and even advance lengths
    (both parities) and a new J must step exactly like fresh solvers."""
    from paper_2508_17655_b200 import InitMode, Solver

    n = 2000
    cfg = cfg_for(GDSB, 100, 1.25, float(1 / (2 * np.sqrt(n))), 0.2)
    runs = [(300, 1, (0, 3, 10)), (700, 1, (0, 5, 6, 9)), (300, 2, (0, 7, 12))]
    got = []
    for R, seed, chunks in runs:
        solver.gen_random_dense(n, seed)
        solver.init_state(R, InitMode.small_uniform, 4, 7)
        for m0, m1 in zip(chunks[:-1], chunks[1:]):
            solver.advance(cfg, m0, m1)
        got.append(solver.get_state())
    for (R, seed, chunks), st in zip(runs, got):
        with Solver(0) as fresh:
            fresh.gen_random_dense(n, seed)
            fresh.init_state(R, InitMode.small_uniform, 4, 7)
            fresh.advance(cfg, 0, chunks[-1])
            ref = fresh.get_state()
        for a, b in zip(st, ref):
            assert (a.view(np.uint32) == b.view(np.uint32)).all(), (R, seed)
