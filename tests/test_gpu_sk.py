"""Real-valued couplings (BASELINE configs[3], Sherrington-Kirkpatrick J ~ N(0, 1/N)):
the fixed-point coupling path, bitwise against the oracle's fp32 mirror and within
fp32 tolerance of the reference's fp64 step() and ising_energy()."""
import ctypes as C

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def solver():
    from paper_2508_17655_b200 import Solver

    s = Solver(0)
    yield s
    s.close()


def cfg_for(variant, steps, dt, c, a):
    from paper_2508_17655_b200 import SolverConfig, Variant

    return SolverConfig(variant=Variant(variant), steps=steps, dt=dt, c=c, a=a)


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
def test_sk_trajectory_bitwise_vs_mirror(solver, orc, variant):
    n, R, M = 300, 70, 200
    J = orc.gen_sk_f32(n, 9)
    planes, shift = orc.fx_quantize(J)
    solver.set_instance(J)
    assert solver._L.sbg_coupling_scale_exp(solver._h) == shift
    x0, y0, p0 = orc.init_small_uniform(n, R, master=13)
    c, dt, a = np.float32(0.5), np.float32(1.25), np.float32(0.2)
    solver.set_state(x0, y0, p0)
    cfg = cfg_for(variant, M, float(dt), float(c), float(a))
    x, y, p = x0, y0, p0
    for m0, m1 in [(0, 1), (1, 25)]:
        solver.advance(cfg, m0, m1)
        gx, gy, gp = solver.get_state()
        x, y, p = orc.step_f32_fx(variant, planes, shift, x, y, p, m0, M, dt, c, a, m1 - m0)
        assert (gx.view(np.uint32) == x.view(np.uint32)).all(), (variant, m1)
        assert (gy.view(np.uint32) == y.view(np.uint32)).all()
        assert (gp.view(np.uint32) == p.view(np.uint32)).all()
    _, energy, best, _ = solver.readout()
    e_ref = orc.energy_fx(planes, shift, gx)
    assert (energy == e_ref).all()


def test_sk_short_horizon_vs_fp64_reference(solver, orc):
    """P3 on real J: <= 1e-5 relative through 30 steps against the reference step() in fp64."""
    n, R = 256, 4
    J = orc.gen_sk_f32(n, 4)
    solver.set_instance(J)
    x0, y0, _ = orc.init_small_uniform(n, R, master=2)
    c, dt = 0.5, 1.25
    solver.set_state(x0, y0)
    for variant in (0, 1, 2):
        solver.set_state(x0, y0)
        solver.advance(cfg_for(variant, 200, dt, c, 0.2), 0, 30)
        gx, _, _ = solver.get_state()
        for r in range(R):
            if oracle.ref_available():
                rx, _, _ = oracle.ref().step_n(variant, J.astype(np.float64), x0[r], y0[r], np.ones(n), 0, 200, dt,
                                               c, 0.2, 30)
            else:
                rx, _, _ = orc.step_f64(variant, J.astype(np.float64), x0[r], y0[r], np.ones(n), 0, 200, dt, c, 0.2,
                                        30)
            assert np.abs(gx[r] - rx).max() / np.abs(rx).max() <= 1e-5, (variant, r)


def test_sk_energy_vs_reference_ising_energy(solver, orc):
    n, R = 400, 33
    J = orc.gen_sk_f32(n, 5)
    solver.set_instance(J)
    x, y, _ = orc.init_reference(n, R, master=8)
    solver.set_state(x, y)
    _, energy, _, _ = solver.readout()
    J64 = J.astype(np.float64)
    s = np.where(x >= 0, 1.0, -1.0)
    e_ref = -0.5 * np.einsum("ri,ij,rj->r", s, J64, s)
    assert np.abs(energy - e_ref).max() <= 1e-6 * np.abs(e_ref).max()


@pytest.mark.parametrize("variant", [0, 2])
def test_sk_tile_widths_bitwise(solver, orc, variant, monkeypatch):
    """The real-J step on 64-replica tiles (one accumulator buffer, drained before the state
    update; the default) and on 32-replica tiles (double-buffered; SBG_FX_BN=32) agree
    bitwise with each other and with the fp32 mirror, replica count not a tile multiple."""
    n, R, M = 384, 200, 100
    J = orc.gen_sk_f32(n, 21)
    planes, shift = orc.fx_quantize(J)
    solver.set_instance(J)
    x0, y0, p0 = orc.init_small_uniform(n, R, master=21)
    c, dt, a = np.float32(0.5), np.float32(1.25), np.float32(0.2)
    cfg = cfg_for(variant, M, float(dt), float(c), float(a))
    out = []
    for bn in ("64", "32"):
        monkeypatch.setenv("SBG_FX_BN", bn)
        solver.set_state(x0, y0, p0)
        solver.advance(cfg, 0, 12)
        out.append(solver.get_state())
    x, y, p = orc.step_f32_fx(variant, planes, shift, x0, y0, p0, 0, M, dt, c, a, 12)
    for g in out:
        assert (g[0].view(np.uint32) == x.view(np.uint32)).all()
        assert (g[1].view(np.uint32) == y.view(np.uint32)).all()
        assert (g[2].view(np.uint32) == p.view(np.uint32)).all()
