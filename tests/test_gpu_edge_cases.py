"""Edge cases the reference's own tests pin (proj/tests/test_engine.cpp), run through
the C ABI on the GPU: single oscillator, walls, sign-only field of dSB, magnitude
field of bSB, |x| <= 1, the linear p schedule at A = 0, monotone p for A <= 1,
single replica / single step, odd sizes."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BSB, DSB, GBSB, GDSB = 0, 1, 2, 3


@pytest.fixture(scope="module")
def solver():
    from paper_2508_17655_b200 import Solver

    s = Solver(0)
    yield s
    s.close()


def cfg(variant, steps, dt, c, a=0.0):
    from paper_2508_17655_b200 import SolverConfig, Variant

    return SolverConfig(variant=Variant(variant), steps=steps, dt=dt, c=c, a=a)


def test_single_oscillator_step_by_hand(solver):
    """test_engine.cpp:80-93: M=1, x=0.5 -> p=0, y=0, x=0.5; a second step throws."""
    solver.set_instance(np.zeros((1, 1), np.int8))
    solver.set_state(np.array([[0.5]], np.float32), np.zeros((1, 1), np.float32))
    solver.advance(cfg(GBSB, 1, 1.0, 1.0), 0, 1)
    x, y, p = solver.get_state()
    assert (p[0, 0], y[0, 0], x[0, 0]) == (0.0, 0.0, 0.5)
    with pytest.raises(ValueError):
        solver.advance(cfg(GBSB, 1, 1.0, 1.0), 1, 2)


@pytest.mark.parametrize("x0,y0,want", [(0.9, 2.0, 1.0), (-0.9, -2.0, -1.0)])
def test_wall_clamps_and_zeroes_momentum(solver, x0, y0, want):
    """test_engine.cpp:95-122."""
    solver.set_instance(np.zeros((1, 1), np.int8))
    solver.set_state(np.array([[x0]], np.float32), np.array([[y0]], np.float32))
    solver.advance(cfg(GBSB, 1000, 0.1, 1.0), 0, 1)
    x, y, _ = solver.get_state()
    assert x[0, 0] == want and y[0, 0] == 0.0
    solver.set_state(np.array([[0.2]], np.float32), np.array([[0.3]], np.float32))
    solver.advance(cfg(GBSB, 1000, 0.1, 1.0), 0, 1)
    x, y, _ = solver.get_state()
    assert abs(x[0, 0]) < 1.0 and y[0, 0] != 0.0


def test_dsb_sees_signs_bsb_sees_magnitudes(solver):
    """test_engine.cpp:182-210."""
    solver.set_instance(np.array([[0, 1], [1, 0]], np.int8))
    a = np.array([[0.5, -0.25]], np.float32)
    b = np.array([[0.5, -0.75]], np.float32)
    ys = []
    for variant in (DSB, BSB):
        out = []
        for x0 in (a, b):
            solver.set_state(x0, np.zeros_like(x0))
            solver.advance(cfg(variant, 10, 0.1, 1.0), 0, 1)
            out.append(solver.get_state()[1][0, 0])
        ys.append(out)
    assert ys[0][0] == ys[0][1]  # dSB: oscillator 0 saw only sgn(x_1)
    assert ys[1][0] != ys[1][1]  # bSB: magnitudes


@pytest.mark.parametrize("variant", [BSB, DSB, GBSB, GDSB])
def test_positions_stay_inside_walls(solver, orc, variant):
    """test_engine.cpp:139-149 (every step boundary)."""
    n = 30
    solver.set_instance(orc.gen_dense_i8(n, 8))
    x0, _, _ = orc.init_reference(n, 4, master=4)
    solver.set_state(x0, np.zeros_like(x0))
    c = cfg(variant, 400, 1.25, 1.0 / (2.0 * np.sqrt(30.0)), 0.3)
    for m in range(0, 400, 40):
        solver.advance(c, m, m + 40)
        x, _, _ = solver.get_state()
        assert np.abs(x).max() <= 1.0


def test_linear_schedule_at_a0(solver, orc):
    """test_engine.cpp:151-162: p = 1 - m/M. The reference checks 1e-12 in fp64; the fp32
    iteration accumulates one rounding per step (<= m * 2^-24), so 2e-5 here; the last
    step (inv = 1) still lands on exactly 0."""
    n, M = 5, 1000
    solver.set_instance(orc.gen_dense_i8(n, 2))
    x0, _, _ = orc.init_reference(n, 1, master=3)
    solver.set_state(x0, np.zeros_like(x0))
    for m in range(0, M, 100):
        solver.advance(cfg(BSB, M, 0.5, 0.1), m, m + 100)
        _, _, p = solver.get_state()
        assert np.abs(p - (1.0 - (m + 100) / M)).max() <= 2e-5
    assert np.abs(p).max() == 0.0


@pytest.mark.parametrize("a", [0.3, 1.0])
def test_p_non_increasing_in_unit_interval(solver, orc, a):
    """test_engine.cpp:164-180."""
    n = 20
    solver.set_instance(orc.gen_dense_i8(n, 6))
    x0, _, _ = orc.init_reference(n, 3, master=9)
    solver.set_state(x0, np.zeros_like(x0))
    prev = np.ones((3, n), np.float32)
    for m in range(0, 300, 30):
        solver.advance(cfg(GBSB, 300, 1.0, 1.0 / (2.0 * np.sqrt(20.0)), a), m, m + 30)
        _, _, p = solver.get_state()
        assert (p <= prev).all() and (p >= 0).all() and (p <= 1).all()
        prev = p


@pytest.mark.parametrize("n,R", [(1, 1), (2, 1), (129, 1), (257, 3), (1000, 257)])
def test_odd_sizes_bitwise(solver, orc, n, R):
    J = orc.gen_dense_i8(n, 5) if n > 1 else np.zeros((1, 1), np.int8)
    solver.set_instance(J)
    x0, y0, p0 = orc.init_small_uniform(n, R, master=1)
    c = 1 / (2 * np.sqrt(max(n, 2)))
    for variant in (GDSB, GBSB):
        solver.set_state(x0, y0)
        solver.advance(cfg(variant, 7, 1.25, c, 0.2), 0, 7)
        x, y, p = solver.get_state()
        ex, ey, ep = orc.step_f32(variant, J, x0, y0, p0, 0, 7, np.float32(1.25), np.float32(c), np.float32(0.2), 7)
        assert (x == ex).all() and (y == ey).all() and (p == ep).all(), (variant, n, R)


@pytest.mark.parametrize("kind", ["dense_pm1", "sk", "csr"])
def test_empty_advance_is_a_no_op(solver, orc, kind):
    """advance(m, m) steps nothing (engine.cpp:55-110 is never called) on every kernel family,
    including the resident kernels and the CSR path's spin-major working copies."""
    n, R = 400, 50
    if kind == "dense_pm1":
        solver.set_instance(orc.gen_dense_i8(n, 3))
    elif kind == "sk":
        solver.set_instance(orc.gen_sk_f32(n, 3))
    else:
        _, csr = orc.gen_er_csr(n, 1500, 3)
        solver.set_instance_csr(n, *csr)
    x0, y0, p0 = orc.init_small_uniform(n, R, master=5)
    solver.set_state(x0, y0, p0)
    for v in (GDSB, GBSB):
        solver.advance(cfg(v, 20, 1.25, 0.05, 0.2), 7, 7)
    x, y, p = solver.get_state()
    assert (x == x0).all() and (y == y0).all() and (p == p0).all()
    solver.advance(cfg(GDSB, 20, 1.25, 0.05, 0.2), 0, 3)
    x3, _, _ = solver.get_state()
    solver.advance(cfg(GDSB, 20, 1.25, 0.05, 0.2), 3, 3)
    x3b, _, _ = solver.get_state()
    assert (x3 == x3b).all()
