"""TEST INFRASTRUCTURE ONLY — the CPU checker for the sbgpu hot path.

Two libraries are exposed through ctypes:

* ``ref``  — the UNMODIFIED reference core (``/root/reference/proj/core/src/*.cpp``)
  compiled by ``oracle/Makefile`` into ``oracle/_ref/`` with a thin extern "C"
  shim (``oracle/ref_shim.cpp``). Parity flavour: ``-O3 -ffp-contract=off``.
* ``orc``  — our plain-C restatement (``oracle/sbg_oracle.c``) of the same
  algorithm for what the reference cannot run (GdSB, BASELINE initial states,
  int8/CSR/SK instances, the fp32 op-order mirror of the CUDA epilogue).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference leg may import this package, and only as the checker. The product
(``paper_2508_17655_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import platform
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

_i64, _u64, _i32, _f64, _f32 = C.c_int64, C.c_uint64, C.c_int32, C.c_double, C.c_float
_P = C.c_void_p


def build() -> None:
    """Compile the restatement (always) and oracle/_ref (when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "-j4"], check=True)


def _ptr(a: np.ndarray) -> C.c_void_p:
    assert a.flags["C_CONTIGUOUS"], "arrays passed to the oracle must be C-contiguous"
    return C.c_void_p(a.ctypes.data)


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
    return C.CDLL(path)


def _cpu_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    fl = line.split()
                    return all(x in fl for x in ("avx512f", "avx512bw", "avx512vl", "avx512dq", "avx512cd"))
    except OSError:
        pass
    return False


class _Ref:
    """ctypes view of the compiled reference (oracle/_ref)."""

    def __init__(self, flavour: str = "parity"):
        if flavour == "timing":
            name = "libsbopt_ref_v4.so" if _cpu_has_avx512() else "libsbopt_ref_v3.so"
        else:
            name = "libsbopt_ref_parity.so"
        self.path = os.path.join(REF_DIR, name)
        L = self.lib = _load(self.path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_derive_seed.restype = _u64
        L.ref_derive_seed.argtypes = [_u64, _P, C.c_int]
        L.ref_xoshiro_next.argtypes = [_u64, _i64, _P]
        L.ref_gen_random_dense.argtypes = [_i64, _u64, _P]
        L.ref_init_state.argtypes = [_i64, _u64, C.c_int, _P, _P, _P]
        L.ref_step_n.argtypes = [C.c_int, _i64, _P, _P, _P, _P, _u64, _u64, _f64, _f64, _f64, _u64]
        L.ref_coupling_matvec.argtypes = [_i64, _P, _P, _P]
        L.ref_ising_energy.argtypes = [_i64, _P, _P, _P]
        L.ref_auto_tune_wigner.argtypes = [_i64, _P, _f64, _P, _P]
        L.ref_extreme_eigenvalues.argtypes = [_i64, _P, _f64, _u64, _P, _P, _P]
        L.ref_auto_tune.argtypes = [_i64, _P, C.c_int, _f64, _f64, _u64, _P]
        L.ref_parse_gset.argtypes = [C.c_char_p, _P, _P, _i64, _P, _P, _P]
        L.ref_cut_value.argtypes = [_i64, _i64, _P, _P, _P, _P, _P]
        L.ref_instance_from_json.argtypes = [C.c_char_p, _i64, _P, _P]
        L.ref_instance_to_json.restype = _i64
        L.ref_instance_to_json.argtypes = [_i64, _P, C.c_char_p, _i64]
        L.ref_run.argtypes = [C.c_int, _i64, _P, _u64, _f64, _f64, _f64, _u64, _P, _P, _P]
        L.ref_batch_best_of.argtypes = [C.c_int, _i64, _P, _u64, _f64, _f64, _f64, _i64, _u64,
                                        C.c_uint, _P, _P, _P]
        L.ref_success_tts.argtypes = [_i64, _i64, _f64, _P, _P, _P, _P]
        L.ref_replica_fanout.argtypes = [C.c_int, _i64, _P, _i64, _P, _P, _u64, _f64, _f64, _f64,
                                         C.c_uint, _P, _P]
        L.ref_effective_workers.restype = C.c_uint
        L.ref_effective_workers.argtypes = [C.c_uint]
        L.ref_chaos_scan.argtypes = [_i64, _P, _P, _i64, _i64, _u64, _f64, _f64, _u64, C.c_uint, _P]

    def _check(self, rc: int) -> None:
        if rc != 0:
            raise ValueError(self.lib.ref_last_error().decode())

    def derive_seed(self, master: int, keys) -> int:
        k = np.asarray(list(keys), dtype=np.uint64)
        return int(self.lib.ref_derive_seed(master, _ptr(k), len(k)))

    def xoshiro(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.uint64)
        self.lib.ref_xoshiro_next(seed, count, _ptr(out))
        return out

    def gen_random_dense(self, n: int, seed: int) -> np.ndarray:
        J = np.empty((n, n), np.float64)
        self._check(self.lib.ref_gen_random_dense(n, seed, _ptr(J)))
        return J

    def init_state(self, n: int, seed: int, chaos_probe: bool = False):
        x, y, p = (np.empty(n, np.float64) for _ in range(3))
        self._check(self.lib.ref_init_state(n, seed, int(chaos_probe), _ptr(x), _ptr(y), _ptr(p)))
        return x, y, p

    def step_n(self, variant: int, J: np.ndarray, x, y, p, m0: int, steps: int, dt: float, c: float,
               a: float, nsteps: int):
        J = np.ascontiguousarray(J, np.float64)
        x, y, p = (np.array(v, np.float64, copy=True) for v in (x, y, p))
        self._check(self.lib.ref_step_n(variant, J.shape[0], _ptr(J), _ptr(x), _ptr(y), _ptr(p), m0,
                                        steps, dt, c, a, nsteps))
        return x, y, p

    def coupling_matvec(self, J: np.ndarray, v: np.ndarray) -> np.ndarray:
        J = np.ascontiguousarray(J, np.float64)
        v = np.ascontiguousarray(v, np.float64)
        out = np.empty(J.shape[0], np.float64)
        self._check(self.lib.ref_coupling_matvec(J.shape[0], _ptr(J), _ptr(v), _ptr(out)))
        return out

    def ising_energy(self, J: np.ndarray, spins: np.ndarray) -> float:
        J = np.ascontiguousarray(J, np.float64)
        s = np.ascontiguousarray(spins, np.int8)
        e = np.zeros(1, np.float64)
        self._check(self.lib.ref_ising_energy(J.shape[0], _ptr(J), _ptr(s), _ptr(e)))
        return float(e[0])

    def auto_tune_wigner(self, J: np.ndarray, d_t: float = 1.25):
        J = np.ascontiguousarray(J, np.float64)
        c, dt = np.zeros(1), np.zeros(1)
        self._check(self.lib.ref_auto_tune_wigner(J.shape[0], _ptr(J), d_t, _ptr(c), _ptr(dt)))
        return float(c[0]), float(dt[0])

    def run(self, variant: int, J: np.ndarray, steps: int, dt: float, c: float, a: float, seed: int):
        J = np.ascontiguousarray(J, np.float64)
        n = J.shape[0]
        s = np.empty(n, np.int8)
        e = np.zeros(1)
        dummy = np.zeros(1)
        self._check(self.lib.ref_run(variant, n, _ptr(J), steps, dt, c, a, seed, _ptr(s), _ptr(e), _ptr(dummy)))
        return s, float(e[0])

    def batch_best_of(self, variant: int, J: np.ndarray, steps: int, dt: float, c: float, a: float,
                      n_batch: int, master: int, workers: int = 1):
        J = np.ascontiguousarray(J, np.float64)
        n = J.shape[0]
        s = np.empty(n, np.int8)
        e = np.zeros(1)
        seed = np.zeros(1, np.uint64)
        self._check(self.lib.ref_batch_best_of(variant, n, _ptr(J), steps, dt, c, a, n_batch, master,
                                               workers, _ptr(s), _ptr(e), _ptr(seed)))
        return s, float(e[0]), int(seed[0])

    def success_tts(self, hits: int, n_rep: int, t_com: float):
        out = [np.zeros(1) for _ in range(4)]
        self._check(self.lib.ref_success_tts(hits, n_rep, t_com, *(_ptr(o) for o in out)))
        return tuple(float(o[0]) for o in out)

    def replica_fanout(self, variant: int, J: np.ndarray, x0: np.ndarray, y0: np.ndarray, steps: int,
                       dt: float, c: float, a: float, workers: int = 0):
        J = np.ascontiguousarray(J, np.float64)
        x0 = np.ascontiguousarray(x0, np.float32)
        y0 = np.ascontiguousarray(y0, np.float32)
        R = x0.shape[0]
        e = np.empty(R, np.float64)
        wall = np.zeros(1)
        self._check(self.lib.ref_replica_fanout(variant, J.shape[0], _ptr(J), R, _ptr(x0), _ptr(y0), steps,
                                                dt, c, a, workers, _ptr(e), _ptr(wall)))
        return e, float(wall[0])

    def chaos_scan(self, J, a_values, reps, steps, dt, c, seed, workers=0):
        J = np.ascontiguousarray(J, np.float64)
        a = np.ascontiguousarray(a_values, np.float64)
        out = np.empty((len(a), reps))
        self._check(self.lib.ref_chaos_scan(J.shape[0], _ptr(J), _ptr(a), len(a), reps, steps, dt, c, seed,
                                            workers, _ptr(out)))
        return out

    def extreme_eigenvalues(self, J, tol: float = 1e-6, max_iters: int = 0):
        """-> (rc, dict(lambda_max, lambda_min, iterations, method, tolerance, converged), v_max, v_min);
        rc 0 ok, 7 ConvergenceError (carried estimate), 1 invalid argument (ValueError raised)."""
        J = np.ascontiguousarray(J, np.float64)
        n = J.shape[0]
        out = np.zeros(6)
        vmax, vmin = np.full(n, np.nan), np.full(n, np.nan)
        rc = self.lib.ref_extreme_eigenvalues(n, _ptr(J), tol, max_iters, _ptr(out), _ptr(vmax), _ptr(vmin))
        if rc == 1:
            raise ValueError(self.lib.ref_last_error().decode())
        keys = ["lambda_max", "lambda_min", "iterations", "method", "tolerance", "converged"]
        d = dict(zip(keys, out.tolist()))
        d["iterations"], d["method"] = int(d["iterations"]), int(d["method"])
        return rc, d, vmax, vmin

    def auto_tune(self, J, numerical: bool, d_t: float = 1.25, tol: float = 1e-6, max_iters: int = 0):
        """-> (rc, (c, dt, lambda_max, lambda_min)); rc 7 = ConvergenceError propagated."""
        J = np.ascontiguousarray(J, np.float64)
        out = np.zeros(4)
        rc = self.lib.ref_auto_tune(J.shape[0], _ptr(J), int(numerical), d_t, tol, max_iters, _ptr(out))
        if rc == 1:
            raise ValueError(self.lib.ref_last_error().decode())
        return rc, tuple(out.tolist())

    def parse_gset(self, text: str):
        """-> (n, i, j, w) 0-based, or raises ValueError(message) like the reference's ParseError."""
        n, m = np.zeros(1, np.int64), np.zeros(1, np.int64)
        cap = max(1, text.count("\n") + 1)
        ei, ej, w = (np.zeros(cap, np.int64) for _ in range(3))
        if self.lib.ref_parse_gset(text.encode(), _ptr(n), _ptr(m), cap, _ptr(ei), _ptr(ej), _ptr(w)):
            raise ValueError(self.lib.ref_last_error().decode())
        k = int(m[0])
        return int(n[0]), ei[:k], ej[:k], w[:k]

    def cut_value(self, n, ei, ej, w, spins) -> int:
        ei, ej, w = (np.ascontiguousarray(a, np.int64) for a in (ei, ej, w))
        spins = np.ascontiguousarray(spins, np.int8)
        out = C.c_longlong()
        self._check(self.lib.ref_cut_value(n, len(ei), _ptr(ei), _ptr(ej), _ptr(w), _ptr(spins), C.byref(out)))
        return int(out.value)

    def instance_from_json(self, text: str, cap: int = 1 << 22):
        n = np.zeros(1, np.int64)
        J = np.zeros(cap)
        if self.lib.ref_instance_from_json(text.encode(), cap, _ptr(n), _ptr(J)):
            raise ValueError(self.lib.ref_last_error().decode())
        k = int(n[0])
        return J[:k * k].reshape(k, k)

    def instance_to_json(self, J) -> str:
        J = np.ascontiguousarray(J, np.float64)
        cap = 64 + 48 * J.size
        buf = C.create_string_buffer(cap)
        if self.lib.ref_instance_to_json(J.shape[0], _ptr(J), buf, cap) < 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return buf.value.decode()

    def last_error(self) -> str:
        return self.lib.ref_last_error().decode()

    def effective_workers(self, requested: int = 0) -> int:
        return int(self.lib.ref_effective_workers(requested))


class _Orc:
    """ctypes view of the C restatement (oracle/libsbg_oracle.so)."""

    def __init__(self):
        L = self.lib = _load(os.path.join(HERE, "libsbg_oracle.so"))
        L.orc_derive_seed.restype = _u64
        L.orc_derive_seed.argtypes = [_u64, _P, C.c_int]
        L.orc_xoshiro_next_n.argtypes = [_u64, _i64, _P]
        L.orc_gen_dense_i8.argtypes = [_i64, _u64, _P]
        L.orc_gen_dense_i8_rows.argtypes = [_i64, _u64, _i64, _i64, _P]
        L.orc_gen_hash_pm1_rows.argtypes = [_i64, _u64, _i64, _i64, _P]
        L.orc_gen_er_edges.restype = _i64
        L.orc_gen_er_edges.argtypes = [_i64, _i64, _u64, _P, _P, _P]
        L.orc_edges_to_csr.argtypes = [_i64, _i64, _P, _P, _P, _P, _P, _P]
        L.orc_gen_sk_f32.argtypes = [_i64, _u64, _P]
        L.orc_init_small_uniform.argtypes = [_i64, _i64, _i64, _i64, _u64, _u64, _P, _P, _P]
        L.orc_init_reference.argtypes = [_i64, _i64, _i64, _i64, _u64, _u64, C.c_int, _P, _P, _P]
        L.orc_matvec_lanes_f64.argtypes = [_i64, _P, _P, _P]
        L.orc_csr_matvec_lanes_f64.argtypes = [_i64, _P, _P, _P, _P, _P]
        L.orc_step_f64.argtypes = [C.c_int, _i64, _P, _P, _P, _P, _u64, _u64, _f64, _f64, _f64]
        L.orc_fields_i8.argtypes = [_i64, _P, _i64, _i64, _P, _P]
        L.orc_fields_fixed_i8.argtypes = [_i64, _P, _i64, _i64, _P, _P]
        L.orc_step_f32.argtypes = [C.c_int, _i64, _P, _i64, _i64, _P, _P, _P, _u64, _u64, _f32, _f32, _f32]
        L.orc_step_f32_csr.argtypes = [C.c_int, _i64, _P, _P, _P, _i64, _i64, _P, _P, _P, _u64, _u64,
                                       _f32, _f32, _f32]
        L.orc_energy2_i8.argtypes = [_i64, _P, _i64, _i64, _P, _P]
        L.orc_energy2_csr.argtypes = [_i64, _P, _P, _P, _i64, _i64, _P, _P]
        L.orc_argmin_i64.restype = _i64
        L.orc_argmin_i64.argtypes = [_i64, _P]
        L.orc_success_tts.argtypes = [_i64, _i64, _f64, _P, _P, _P, _P]
        L.orc_fx_quantize.restype = C.c_int
        L.orc_fx_quantize.argtypes = [_i64, _P, _P]
        L.orc_step_f32_fx.argtypes = [C.c_int, _i64, _P, C.c_int, _i64, _i64, _P, _P, _P, _u64, _u64, _f32, _f32,
                                      _f32]
        L.orc_energy2_fx.argtypes = [_i64, _P, _i64, _i64, _P, _P]
        L.orc_fields_fx.argtypes = [C.c_int, _i64, _P, C.c_int, _i64, _i64, _P, _P]
        L.orc_init_reference_seeds.argtypes = [_i64, _i64, _i64, _P, C.c_int, _P, _P, _P]
        L.orc_phase_batch_f32.argtypes = [_i64, _P, _P, _P, _P, _f32, _f32, _f32, _u64, _u64]

    def derive_seed(self, master: int, keys) -> int:
        k = np.asarray(list(keys), dtype=np.uint64)
        return int(self.lib.orc_derive_seed(master, _ptr(k), len(k)))

    def xoshiro(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.uint64)
        self.lib.orc_xoshiro_next_n(seed, count, _ptr(out))
        return out

    def gen_dense_i8(self, n: int, seed: int) -> np.ndarray:
        J = np.empty((n, n), np.int8)
        self.lib.orc_gen_dense_i8(n, seed, _ptr(J))
        return J

    def gen_dense_i8_rows(self, n: int, seed: int, row0: int, rows: int) -> np.ndarray:
        J = np.empty((rows, n), np.int8)
        self.lib.orc_gen_dense_i8_rows(n, seed, row0, rows, _ptr(J))
        return J

    def gen_hash_pm1_rows(self, n: int, seed: int, row0: int, rows: int) -> np.ndarray:
        J = np.empty((rows, n), np.int8)
        self.lib.orc_gen_hash_pm1_rows(n, seed, row0, rows, _ptr(J))
        return J

    def gen_er_csr(self, n: int, m: int, seed: int):
        ei, ej = np.empty(m, np.int32), np.empty(m, np.int32)
        w = np.empty(m, np.int8)
        got = self.lib.orc_gen_er_edges(n, m, seed, _ptr(ei), _ptr(ej), _ptr(w))
        if got != m:
            raise ValueError("ER generator: m too large for n")
        rowptr = np.empty(n + 1, np.int32)
        col, val = np.empty(2 * m, np.int32), np.empty(2 * m, np.int8)
        self.lib.orc_edges_to_csr(n, m, _ptr(ei), _ptr(ej), _ptr(w), _ptr(rowptr), _ptr(col), _ptr(val))
        return (ei, ej, w), (rowptr, col, val)

    def gen_sk_f32(self, n: int, seed: int) -> np.ndarray:
        J = np.empty((n, n), np.float32)
        self.lib.orc_gen_sk_f32(n, seed, _ptr(J))
        return J

    def init_small_uniform(self, n: int, R: int, master: int, tag: int = 7, r0: int = 0, ld: int | None = None):
        ld = n if ld is None else ld
        x, y, p = (np.empty((R, ld), np.float32) for _ in range(3))
        self.lib.orc_init_small_uniform(n, ld, r0, R, master, tag, _ptr(x), _ptr(y), _ptr(p))
        return x, y, p

    def init_reference(self, n: int, R: int, master: int, tag: int = 3, chaos_probe: bool = False,
                       r0: int = 0, ld: int | None = None):
        ld = n if ld is None else ld
        x, y, p = (np.empty((R, ld), np.float32) for _ in range(3))
        self.lib.orc_init_reference(n, ld, r0, R, master, tag, int(chaos_probe), _ptr(x), _ptr(y), _ptr(p))
        return x, y, p

    def init_reference_seeds(self, n: int, seeds, chaos_probe: bool = False):
        seeds = np.ascontiguousarray(seeds, np.uint64)
        R = len(seeds)
        x, y, p = (np.empty((R, n), np.float32) for _ in range(3))
        self.lib.orc_init_reference_seeds(n, n, R, _ptr(seeds), int(chaos_probe), _ptr(x), _ptr(y), _ptr(p))
        return x, y, p

    def matvec_lanes_f64(self, J, v):
        J = np.ascontiguousarray(J, np.float64)
        v = np.ascontiguousarray(v, np.float64)
        out = np.empty(J.shape[0])
        self.lib.orc_matvec_lanes_f64(J.shape[0], _ptr(J), _ptr(v), _ptr(out))
        return out

    def csr_matvec_lanes_f64(self, n, rowptr, col, val, v):
        val = np.ascontiguousarray(val, np.float64)
        v = np.ascontiguousarray(v, np.float64)
        out = np.empty(n)
        self.lib.orc_csr_matvec_lanes_f64(n, _ptr(rowptr), _ptr(col), _ptr(val), _ptr(v), _ptr(out))
        return out

    def step_f64(self, variant, J, x, y, p, m, M, dt, c, a, nsteps: int = 1):
        J = np.ascontiguousarray(J, np.float64)
        x, y, p = (np.array(v, np.float64, copy=True) for v in (x, y, p))
        for k in range(nsteps):
            self.lib.orc_step_f64(variant, J.shape[0], _ptr(J), _ptr(x), _ptr(y), _ptr(p), m + k, M, dt, c, a)
        return x, y, p

    def fields_i8(self, J, S):
        J = np.ascontiguousarray(J, np.int8)
        S = np.ascontiguousarray(S, np.int8)
        F = np.empty(S.shape, np.int32)
        self.lib.orc_fields_i8(J.shape[0], _ptr(J), S.shape[0], S.shape[1], _ptr(S), _ptr(F))
        return F

    def fields_fixed_i8(self, J, x):
        J = np.ascontiguousarray(J, np.int8)
        x = np.ascontiguousarray(x, np.float32)
        F = np.empty(x.shape, np.float32)
        self.lib.orc_fields_fixed_i8(J.shape[0], _ptr(J), x.shape[0], x.shape[1], _ptr(x), _ptr(F))
        return F

    def step_f32(self, variant, J, x, y, p, m, M, dt, c, a, nsteps: int = 1):
        """fp32 GPU-op-order mirror over [R][ld] states; returns new copies."""
        J = np.ascontiguousarray(J, np.int8)
        x, y, p = (np.array(v, np.float32, copy=True) for v in (x, y, p))
        for k in range(nsteps):
            self.lib.orc_step_f32(variant, J.shape[0], _ptr(J), x.shape[0], x.shape[1], _ptr(x), _ptr(y),
                                  _ptr(p), m + k, M, dt, c, a)
        return x, y, p

    def step_f32_csr(self, variant, n, csr, x, y, p, m, M, dt, c, a, nsteps: int = 1):
        rowptr, col, val = csr
        x, y, p = (np.array(v, np.float32, copy=True) for v in (x, y, p))
        for k in range(nsteps):
            self.lib.orc_step_f32_csr(variant, n, _ptr(rowptr), _ptr(col), _ptr(val), x.shape[0], x.shape[1],
                                      _ptr(x), _ptr(y), _ptr(p), m + k, M, dt, c, a)
        return x, y, p

    def energy2_i8(self, J, x):
        J = np.ascontiguousarray(J, np.int8)
        x = np.ascontiguousarray(x, np.float32)
        E2 = np.empty(x.shape[0], np.int64)
        self.lib.orc_energy2_i8(J.shape[0], _ptr(J), x.shape[0], x.shape[1], _ptr(x), _ptr(E2))
        return E2

    def energy2_csr(self, n, csr, x):
        rowptr, col, val = csr
        x = np.ascontiguousarray(x, np.float32)
        E2 = np.empty(x.shape[0], np.int64)
        self.lib.orc_energy2_csr(n, _ptr(rowptr), _ptr(col), _ptr(val), x.shape[0], x.shape[1], _ptr(x), _ptr(E2))
        return E2

    def argmin(self, v):
        v = np.ascontiguousarray(v, np.int64)
        return int(self.lib.orc_argmin_i64(len(v), _ptr(v)))

    def phase_batch(self, F, x, y, p, a, c, dt, m, M):
        """In-place fp32 phase update (GPU op order) of contiguous float32 arrays."""
        F = np.ascontiguousarray(F, np.float32)
        for v in (x, y, p):
            assert v.dtype == np.float32 and v.flags["C_CONTIGUOUS"]
        self.lib.orc_phase_batch_f32(F.size, _ptr(F), _ptr(x), _ptr(y), _ptr(p), a, c, dt, m, M)

    def fx_quantize(self, J):
        J = np.ascontiguousarray(J, np.float32)
        n = J.shape[0]
        planes = np.empty((3, n, n), np.uint8)
        shift = self.lib.orc_fx_quantize(n, _ptr(J), _ptr(planes))
        return planes, int(shift)

    def step_f32_fx(self, variant, planes, shift, x, y, p, m, M, dt, c, a, nsteps: int = 1):
        planes = np.ascontiguousarray(planes, np.uint8)
        n = planes.shape[1]
        x, y, p = (np.array(v, np.float32, copy=True) for v in (x, y, p))
        for k in range(nsteps):
            self.lib.orc_step_f32_fx(variant, n, _ptr(planes), shift, x.shape[0], x.shape[1], _ptr(x), _ptr(y),
                                     _ptr(p), m + k, M, dt, c, a)
        return x, y, p

    def fields_fx(self, variant, planes, shift, x):
        """The GPU's fixed-point field of real J (9 plane products for the continuous variants)."""
        planes = np.ascontiguousarray(planes, np.uint8)
        x = np.ascontiguousarray(x, np.float32)
        F = np.empty_like(x)
        self.lib.orc_fields_fx(variant, planes.shape[1], _ptr(planes), shift, x.shape[0], x.shape[1], _ptr(x), _ptr(F))
        return F

    def energy_fx(self, planes, shift, x):
        planes = np.ascontiguousarray(planes, np.uint8)
        x = np.ascontiguousarray(x, np.float32)
        E2 = np.empty(x.shape[0], np.int64)
        self.lib.orc_energy2_fx(planes.shape[1], _ptr(planes), x.shape[0], x.shape[1], _ptr(x), _ptr(E2))
        return -0.5 * E2.astype(np.float64) * 2.0 ** -shift

    def success_tts(self, hits, n_rep, t_com):
        out = [np.zeros(1) for _ in range(4)]
        rc = self.lib.orc_success_tts(hits, n_rep, t_com, *(_ptr(o) for o in out))
        if rc != 0:
            raise ValueError(f"success/TTS undefined (code {rc})")
        return tuple(float(o[0]) for o in out)


_cache: dict = {}


def ref(flavour: str = "parity") -> _Ref:
    key = ("ref", flavour)
    if key not in _cache:
        _cache[key] = _Ref(flavour)
    return _cache[key]


def orc() -> _Orc:
    if "orc" not in _cache:
        _cache["orc"] = _Orc()
    return _cache["orc"]


def ref_available() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "libsbopt_ref_parity.so"))


def host_description() -> str:
    model = platform.processor() or "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model
