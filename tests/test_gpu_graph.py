"""Graph / JSON ingestion straight to the device (sbg_set_couplings_graph /
sbg_set_couplings_entries_f64) on the GPU: the G-set text of a MAX-CUT graph lands as
the same CSR the oracle builds (trajectories bitwise vs the fp32 CSR mirror), cuts
from the device energies equal the reference's own cut_value on the device spins,
and JSON documents reach the same device image as the dense setters."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

GBSB, GDSB = 2, 3


@pytest.fixture(scope="module")
def solver():
    from paper_2508_17655_b200 import Solver

    s = Solver(0)
    yield s
    s.close()


def cfg(variant, M, dt, c, a):
    from paper_2508_17655_b200 import SolverConfig, Variant

    return SolverConfig(variant=Variant(variant), steps=M, dt=dt, c=c, a=a)


def torus(L, seed):
    """G-set-style toroidal grid (L x L, 4-regular) with +-1 weights."""
    rng = np.random.default_rng(seed)
    ei, ej = [], []
    for r in range(L):
        for c in range(L):
            v = r * L + c
            ei += [v, v]
            ej += [r * L + (c + 1) % L, ((r + 1) % L) * L + c]
    return np.array(ei), np.array(ej), np.where(rng.random(len(ei)) < 0.5, 1, -1)


def test_gset_text_to_device_csr_bitwise(solver, orc):
    from paper_2508_17655_b200 import TuningResult, parse_gset, serialize_gset
    from paper_2508_17655_b200.instances import CutGraph

    n, m, R = 2000, 9000, 40
    (ei, ej, w), csr = orc.gen_er_csr(n, m, 8)
    g = parse_gset(serialize_gset(CutGraph(n, ei, ej, w.astype(np.int64))))
    solver.set_graph(g)
    assert solver.total_weight == int(w.astype(np.int64).sum())
    x0, y0, p0 = orc.init_small_uniform(n, R, master=4)
    c, dt = np.float32(0.17), np.float32(1.25)
    for variant in (GBSB, GDSB):
        solver.set_state(x0, y0, p0)
        solver.advance(cfg(variant, 300, float(dt), float(c), 0.2), 0, 30)
        x, y, p = solver.get_state()
        mx, my, mp = orc.step_f32_csr(variant, n, csr, x0, y0, p0, 0, 300, dt, c, np.float32(0.2), 30)
        assert (x == mx).all() and (y == my).all() and (p == mp).all()
    b = solver.run_batch(cfg(GBSB, 400, 1.25, float(c), 0.2), TuningResult(c=float(c), dt=1.25), R, x0=x0, y0=y0)
    if oracle.ref_available():
        for r in range(0, R, 7):
            assert b.cuts[r] == oracle.ref().cut_value(n, g.i, g.j, g.w, b.spins[r])


def test_torus_cut_matches_reference(solver):
    from paper_2508_17655_b200 import TuningResult
    from paper_2508_17655_b200.instances import CutGraph, cut_value

    ei, ej, w = torus(40, 3)
    g = CutGraph(1600, ei, ej, w)
    solver.set_graph(g)
    t = solver.auto_tune("wigner")
    b = solver.run_batch(cfg(GBSB, 2000, t.dt, t.c, 0.2), t, 64, master_seed=9)
    for r in range(64):
        assert b.cuts[r] == cut_value(g, b.spins[r])
        if oracle.ref_available() and r % 16 == 0:
            assert b.cuts[r] == oracle.ref().cut_value(1600, g.i, g.j, g.w, b.spins[r])
    assert isinstance(t, TuningResult)


def test_json_entries_reach_the_same_device_image(solver, orc):
    from paper_2508_17655_b200 import instance_from_json
    from paper_2508_17655_b200.instances import entries_from_dense, instance_to_json

    n, R = 300, 16
    x0, y0, p0 = orc.init_small_uniform(n, R, master=6)
    c = 1 / (2 * np.sqrt(n))
    cases = [orc.gen_dense_i8(n, 2).astype(np.float64)]  # dense +-1: dense int8 path
    sparse = np.zeros((n, n))
    (ei, ej, w), _ = orc.gen_er_csr(n, 900, 1)
    sparse[ei, ej] = -w
    sparse[ej, ei] = -w
    cases.append(sparse)  # sparse integer: CSR path
    real = orc.gen_sk_f32(n, 4).astype(np.float64)
    cases.append(real)  # real-valued: fixed-point path
    for J in cases:
        e = instance_from_json(instance_to_json(entries_from_dense(J)))
        out = []
        for setter in (lambda: solver.set_instance_entries(e), lambda: solver.set_instance(J)):
            setter()
            solver.set_state(x0, y0, p0)
            solver.advance(cfg(GBSB, 100, 1.25, c, 0.2), 0, 20)
            out.append(solver.get_state()[0])
        assert (out[0] == out[1]).all()


def test_graph_errors(solver):
    from paper_2508_17655_b200._lib import SbgError
    from paper_2508_17655_b200.instances import CutGraph

    g = CutGraph(3, np.array([0]), np.array([1]), np.array([200]))
    with pytest.raises(SbgError, match="int8"):
        solver.set_graph(g)
