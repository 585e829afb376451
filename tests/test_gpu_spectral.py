"""Device extreme_eigenvalues / auto_tune (spectral.cuh) against the reference's own
extreme_eigenvalues / auto_tune (spectral.cpp:207-326, compiled in oracle/_ref with
-ffp-contract=off): bitwise eigenvalue estimates, iteration counts and eigenvectors
for integer couplings (dense int8 and CSR), including the ConvergenceError path
(the reference's N >= 40 dense +-1 instances hit the 10 n cap),
the n == 2 closed form and the n <= 32 Jacobi branch."""
import time

import numpy as np
import pytest

import oracle

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not oracle.ref_available(), reason="needs oracle/_ref (the compiled reference)")]


@pytest.fixture(scope="module")
def solver():
    from paper_2508_17655_b200 import Solver

    s = Solver(0)
    yield s
    s.close()


@pytest.fixture(scope="module")
def ref():
    return oracle.ref("parity")


def dense_from_csr(n, rp, col, val):
    J = np.zeros((n, n), np.int8)
    for i in range(n):
        J[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    return J


def planted(n, seed):
    u = np.sign(np.random.default_rng(seed).standard_normal(n)).astype(np.int8)
    J = -np.outer(u, u).astype(np.int8)
    np.fill_diagonal(J, 0)
    return J


def check_same(solver, ref, J, tol=1e-6, max_iters=0):
    from paper_2508_17655_b200 import ConvergenceError

    rc, want, vmax, vmin = ref.extreme_eigenvalues(J.astype(np.float64), tol, max_iters)
    if rc == 7:
        with pytest.raises(ConvergenceError) as ei:
            solver.extreme_eigenvalues(tol, max_iters, want_vectors=True)
        got = ei.value.last_estimate
        assert str(ei.value) == ref.last_error()
    else:
        got = solver.extreme_eigenvalues(tol, max_iters, want_vectors=True)
    assert got.lambda_max == want["lambda_max"]
    assert (np.isnan(got.lambda_min) and np.isnan(want["lambda_min"])) or got.lambda_min == want["lambda_min"]
    assert got.iterations == want["iterations"]
    assert got.method == ["power_iteration", "wigner", "exact_small"][want["method"]]
    assert (got.v_max == vmax).all()
    if not np.isnan(want["lambda_min"]):
        assert (got.v_min == vmin).all()
    return rc, got


@pytest.mark.parametrize("n,seed", [(3, 1), (10, 4000), (17, 2), (31, 9), (32, 5)])
def test_jacobi_small_bitwise(solver, orc, ref, n, seed):
    solver.set_instance(orc.gen_dense_i8(n, seed))
    check_same(solver, ref, orc.gen_dense_i8(n, seed))


@pytest.mark.parametrize("c01", [1, -1, 5])
def test_two_by_two_closed_form(solver, ref, c01):
    J = np.array([[0, c01], [c01, 0]], np.int8)
    solver.set_instance(J)
    check_same(solver, ref, J)


@pytest.mark.parametrize("n,seed,max_iters", [(40, 3, 0), (100, 1, 0), (200, 7, 20000), (333, 4, 0)])
def test_dense_power_iteration_bitwise(solver, orc, ref, n, seed, max_iters):
    """Includes the non-converging cap (ConvergenceError with the carried estimate) and,
    at n = 200 with 100 n iterations, convergence of both ends after stall perturbations."""
    J = orc.gen_dense_i8(n, seed)
    solver.set_instance(J)
    check_same(solver, ref, J, max_iters=max_iters)


def test_planted_dense(solver, ref):
    J = planted(300, 1)
    solver.set_instance(J)
    rc, got = check_same(solver, ref, J)
    assert rc == 0 and abs(got.lambda_min + 299) < 1e-9


@pytest.mark.parametrize("n,m,seed", [(300, 900, 5), (1001, 3000, 2)])
def test_csr_power_iteration_bitwise(solver, orc, ref, n, m, seed):
    """CSR row_dot with the dense lane rule (j mod 8, tail into lane 0) == dense fp64."""
    _, (rp, col, val) = orc.gen_er_csr(n, m, seed)
    solver.set_instance_csr(n, rp, col, val)
    J = dense_from_csr(n, rp, col, val)
    check_same(solver, ref, J)
    solver.set_instance(J)  # same instance through the dense int8 path
    check_same(solver, ref, J)


def test_c3_shape_csr_speed(solver, orc, ref):
    """ER n = 2000, mean degree 10: ~16k power iterations; GPU vs the reference's own."""
    n, m = 2000, 10000
    _, (rp, col, val) = orc.gen_er_csr(n, m, 9)
    solver.set_instance_csr(n, rp, col, val)
    t0 = time.perf_counter()
    got = solver.extreme_eigenvalues()
    t_gpu = time.perf_counter() - t0
    J = dense_from_csr(n, rp, col, val).astype(np.float64)
    t0 = time.perf_counter()
    rc, want, _, _ = ref.extreme_eigenvalues(J)
    t_ref = time.perf_counter() - t0
    print(f"\nextreme_eigenvalues ER n=2000: {want['iterations']} iterations, gpu {t_gpu:.3f} s, reference {t_ref:.2f} s")
    assert rc == 0 and (got.lambda_max, got.lambda_min, got.iterations) == (
        want["lambda_max"], want["lambda_min"], want["iterations"])


def test_auto_tune_numerical_and_wigner(solver, orc, ref):
    from paper_2508_17655_b200 import ConvergenceError

    J = orc.gen_dense_i8(200, 7)
    solver.set_instance(J)
    t = solver.auto_tune("numerical", 1.25, 1e-6, 20000)
    rc, want = ref.auto_tune(J.astype(np.float64), True, 1.25, 1e-6, 20000)
    assert rc == 0 and (t.c, t.dt, t.lambda_max, t.lambda_min) == want and t.converged
    w = solver.auto_tune("wigner", 1.1)
    rc, want = ref.auto_tune(J.astype(np.float64), False, 1.1)
    assert rc == 0 and (w.c, w.dt, w.lambda_max, w.lambda_min) == want and w.method == "wigner"
    # lambda_max misses the cap: the reference's auto_tune rethrows (spectral.cpp:311-316)
    J = orc.gen_dense_i8(100, 1)
    solver.set_instance(J)
    assert ref.auto_tune(J.astype(np.float64), True)[0] == 7
    with pytest.raises(ConvergenceError):
        solver.auto_tune("numerical")


def test_auto_tune_real_couplings_tolerance(solver, orc, ref):
    """SK fp32 J lives on the device as a 24-bit fixed-point image, so only a tolerance
    holds (|dJ| <= 2^-24 max|J| per entry)."""
    n = 300
    J = orc.gen_sk_f32(n, 3)
    solver.set_instance(J)
    t = solver.auto_tune("wigner")
    rc, want = ref.auto_tune(J.astype(np.float64), False)
    assert rc == 0 and abs(t.c / want[0] - 1) < 1e-6
    got = solver.extreme_eigenvalues(1e-6, 100000)
    rc, w, _, _ = ref.extreme_eigenvalues(J.astype(np.float64), 1e-6, 100000)
    assert rc == 0
    assert abs(got.lambda_max - w["lambda_max"]) < 1e-5 * abs(w["lambda_max"])
    assert abs(got.lambda_min - w["lambda_min"]) < 1e-5 * abs(w["lambda_min"])


def test_argument_errors(solver, ref):
    solver.set_instance(np.zeros((1, 1), np.int8))
    with pytest.raises(ValueError, match="n >= 2"):
        solver.extreme_eigenvalues()
    solver.set_instance(np.zeros((5, 5), np.int8))
    with pytest.raises(ValueError, match="degenerate"):
        solver.extreme_eigenvalues()
    with pytest.raises(ValueError, match="degenerate"):
        solver.auto_tune("wigner")
    solver.set_instance(np.array([[0, 1], [1, 0]], np.int8))
    with pytest.raises(ValueError, match="tolerance"):
        solver.extreme_eigenvalues(0.0)
    with pytest.raises(ValueError, match="d_t_factor"):
        solver.auto_tune("numerical", 0.0)
