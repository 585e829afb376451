"""Host-side mirror of the reference solver API for the GSB hot path.

Names, argument meaning and error behaviour follow sbopt
(/root/reference/proj/core/include/sbopt/{engine,bench,spectral}.hpp) so that
parity tests read like the reference's own tests; every call goes through the
sbgpu C ABI (include/sbgpu.h) to the sm_100a kernels. There is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import math
from typing import Optional

import numpy as np

from . import _lib
from ._lib import ptr, raise_for


class Variant(enum.IntEnum):  # engine.hpp:26 (+ gdsb)
    bsb = _lib.BSB
    dsb = _lib.DSB
    gbsb = _lib.GBSB
    gdsb = _lib.GDSB


class InitMode(enum.IntEnum):  # engine.hpp:27 (+ the BASELINE small-uniform init)
    uniform_random = _lib.INIT_UNIFORM_RANDOM
    chaos_probe = _lib.INIT_CHAOS_PROBE
    small_uniform = _lib.INIT_SMALL_UNIFORM


SEED_STREAM_BATCH = 3  # rng.hpp:36 seed_stream::batch
SEED_STREAM_GPU_INIT = 7  # BASELINE "gpu_init" stream


@dataclasses.dataclass
class SolverConfig:  # engine.hpp:29-38
    variant: Variant = Variant.gbsb
    steps: int = 1000
    dt: Optional[float] = None
    c: Optional[float] = None
    a: float = 0.0
    seed: int = 0
    init_mode: InitMode = InitMode.uniform_random
    sample_stride: int = 0  # 0 = record the final state only (engine.hpp:37)


@dataclasses.dataclass
class SpectralEstimate:  # spectral.hpp:19-27
    lambda_max: float = 0.0
    lambda_min: float = 0.0
    method: str = "power_iteration"  # power_iteration | wigner | exact_small (SpectralMethod)
    tolerance: float = 0.0
    v_max: Optional[np.ndarray] = None
    v_min: Optional[np.ndarray] = None
    iterations: int = 0


class ConvergenceError(RuntimeError):
    """spectral.hpp:38-47: iterative estimation missed the residual target; the
    carried estimate is attached."""

    def __init__(self, message: str, last_estimate: SpectralEstimate):
        super().__init__(message)
        self.last_estimate = last_estimate


_SPECTRAL_METHODS = {0: "power_iteration", 1: "wigner", 2: "exact_small"}


@dataclasses.dataclass
class TuningResult:  # spectral.hpp:28-33
    c: float = 0.0
    dt: float = 0.0
    d_t_factor: float = 0.0
    lambda_max: float = float("nan")
    lambda_min: float = float("nan")
    method: str = "wigner"
    source: Optional[SpectralEstimate] = None
    converged: bool = True  # False: tuned from a carried estimate (the reference's stderr warning)


@dataclasses.dataclass
class RunResult:  # engine.hpp:56-64 (batched: one per replica)
    final_spins: np.ndarray
    energy: float
    cut: Optional[int] = None
    wall_time_s: float = 0.0
    config_echo: Optional[SolverConfig] = None
    tuning_echo: Optional[TuningResult] = None


def resolve_config(cfg: SolverConfig, tuning: TuningResult) -> SolverConfig:
    """engine.cpp:48-53 + validate() :16-21 (raises ValueError like std::invalid_argument)."""
    out = dataclasses.replace(cfg)
    if out.dt is None:
        out.dt = tuning.dt
    if out.c is None:
        out.c = tuning.c
    if out.steps < 1:
        raise ValueError("step count M must be >= 1")
    if not out.dt > 0.0:
        raise ValueError("dt must be positive")
    if not out.c > 0.0:
        raise ValueError("c must be positive")
    if not out.a >= 0.0:
        raise ValueError("A must be >= 0")
    return out


def auto_tune_wigner(J: np.ndarray, d_t_factor: float = 1.25) -> TuningResult:
    """auto_tune(TuneMode::wigner) (spectral.cpp:294-326) via the C ABI."""
    J = np.ascontiguousarray(J, np.float64)
    c, dt = C.c_double(), C.c_double()
    rc = _lib.lib().sbg_tune_wigner_f64(J.shape[0], ptr(J), d_t_factor, C.byref(c), C.byref(dt))
    if rc:
        raise ValueError("degenerate instance: all couplings zero")
    edge = 1.0 / c.value
    return TuningResult(c=c.value, dt=dt.value, d_t_factor=d_t_factor, lambda_max=edge, lambda_min=-edge)


@dataclasses.dataclass
class SuccessStats:  # bench.hpp:22-28
    p_s: float
    delta_p_s: float
    n_rep: int
    target_value: float
    hit_count: int


@dataclasses.dataclass
class TtsResult:  # bench.hpp:41-46
    tts_s: float
    delta_tts_s: float
    t_com_s: float
    stats: SuccessStats


def success_from_counts(hit_count: int, n_rep: int, target: float) -> SuccessStats:
    out = (C.c_double * 4)()
    rc = _lib.lib().sbg_success_tts(hit_count, n_rep, 1.0, out)
    if rc and not (n_rep > 0 and 0 <= hit_count <= n_rep):
        raise ValueError("success probability needs n_rep >= 1 and hits <= n_rep")
    return SuccessStats(out[0], out[1], n_rep, target, hit_count)


def success_probability(energies, target: float) -> SuccessStats:
    """bench.cpp:28-36: hit = energy <= target (exact)."""
    e = np.asarray(energies, np.float64)
    if e.size == 0:
        raise ValueError("no results")
    return success_from_counts(int((e <= target).sum()), int(e.size), target)


def success_probability_cut(cuts, target: float) -> SuccessStats:
    """bench.cpp:38-50 with HitKind::cut_max: hit = cut >= target."""
    c = np.asarray(cuts, np.float64)
    if c.size == 0:
        raise ValueError("no results")
    return success_from_counts(int((c >= target).sum()), int(c.size), target)


def time_to_solution(t_com_s: float, stats: SuccessStats) -> TtsResult:
    """bench.cpp:52-68."""
    if not t_com_s > 0.0:
        raise ValueError("t_com must be positive")
    if not stats.p_s > 0.0:
        raise ValueError("TTS undefined for p_s = 0")
    out = (C.c_double * 4)()
    raise_for(_lib.lib().sbg_success_tts(stats.hit_count, stats.n_rep, t_com_s, out), "tts")
    return TtsResult(out[2], out[3], t_com_s, stats)


class Solver:
    """One sbgpu context on one CUDA device (replaces ThreadPool + per-run state)."""

    def __init__(self, device: int = 0):
        self._L = _lib.lib()
        h = C.c_void_p()
        rc = self._L.sbg_create(device, C.byref(h))
        if rc:
            raise _lib.SbgError(rc, f"sbg_create(device={device}) failed: {self._L.sbg_strerror(rc).decode()}")
        self._h = h
        self.device = device
        self.n = self.n_global = 0
        self.total_weight: Optional[int] = None

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.sbg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, rc: int) -> None:
        if rc:
            raise_for(rc, self._L.sbg_last_error(self._h).decode())

    @property
    def device_name(self) -> str:
        return self._L.sbg_device_name(self._h).decode()

    @property
    def operand_format(self) -> str:
        """'e2m1' when the dense couplings carry a packed FP4 copy (sign variants then run
        kind::mxf4 MMAs), else 'int8'."""
        return "e2m1" if self._L.sbg_couplings_e2m1(self._h) else "int8"

    @property
    def sm_count(self) -> int:
        return self._L.sbg_device_sm_count(self._h)

    @property
    def kernel_launches(self) -> int:
        return self._L.sbg_kernel_launches(self._h)

    # ----------------------------------------------------------- instances
    def set_instance(self, J: np.ndarray, graph_total_weight: Optional[int] = None) -> None:
        """IsingInstance (model.hpp:46-70), dense integer J (int8 or integral fp64)."""
        J = np.ascontiguousarray(J)
        n = J.shape[0]
        if J.dtype == np.int8:
            self._check(self._L.sbg_set_couplings_dense_i8(self._h, n, ptr(J)))
        elif J.dtype == np.float32:
            self._check(self._L.sbg_set_couplings_dense_f32(self._h, n, ptr(J)))
        else:
            J = np.ascontiguousarray(J, np.float64)
            self._check(self._L.sbg_set_couplings_dense_f64(self._h, n, ptr(J)))
        self.n = self.n_global = n
        if not np.all(np.equal(np.mod(J, 1), 0)):
            self.total_weight = graph_total_weight  # real couplings: no implied MAX-CUT graph
            return
        # cut via the bridge (model.hpp:103-104): J = -w  =>  W = -sum_{i<j} J_ij
        self.total_weight = graph_total_weight if graph_total_weight is not None else int(
            -np.triu(J.astype(np.int64), 1).sum())

    def set_graph(self, graph) -> None:
        """MAX-CUT graph (instances.CutGraph) straight to device CSR: maxcut_to_ising
        (model.cpp:134-142) without the dense fp64 matrix; cut = (W - E) / 2."""
        W = C.c_int64()
        self._check(self._L.sbg_set_couplings_graph(self._h, graph.n, graph.m, ptr(graph.i), ptr(graph.j),
                                                    ptr(graph.w), C.byref(W)))
        self.n = self.n_global = graph.n
        self.total_weight = int(W.value)

    def set_instance_entries(self, entries, graph_total_weight: Optional[int] = None) -> None:
        """IsingInstance::from_entries (model.cpp:70-86) from instances.CouplingEntries."""
        i = np.ascontiguousarray(entries.i, np.int64)
        j = np.ascontiguousarray(entries.j, np.int64)
        v = np.ascontiguousarray(entries.value, np.float64)
        self._check(self._L.sbg_set_couplings_entries_f64(self._h, entries.n, len(i), ptr(i), ptr(j), ptr(v)))
        self.n = self.n_global = entries.n
        integral = bool(np.all(np.mod(v, 1) == 0))
        self.total_weight = graph_total_weight if graph_total_weight is not None else (
            int(-v.astype(np.int64).sum()) if integral else None)

    # ------------------------------------------------------- spectrum / tuning

    def extreme_eigenvalues(self, tol: float = 1e-6, max_iters: int = 0, want_vectors: bool = False):
        """extreme_eigenvalues (spectral.cpp:207-246) on the device couplings. Raises
        ConvergenceError (estimate attached) like the reference."""
        st = _lib.Spectral()
        vmax = np.full(self.n, np.nan) if want_vectors else None
        vmin = np.full(self.n, np.nan) if want_vectors else None
        rc = self._L.sbg_extreme_eigenvalues(self._h, tol, max_iters, C.byref(st),
                                             ptr(vmax) if want_vectors else None, ptr(vmin) if want_vectors else None)
        est = SpectralEstimate(st.lambda_max, st.lambda_min, _SPECTRAL_METHODS[st.method], st.tolerance,
                               vmax, vmin, int(st.iterations))
        if rc == _lib.SBG_ERR_CONVERGENCE:
            raise ConvergenceError(self._L.sbg_last_error(self._h).decode(), est)
        self._check(rc)
        return est

    def auto_tune(self, mode: str = "numerical", d_t_factor: float = 1.25, tol: float = 1e-6,
                  max_iters: int = 0) -> TuningResult:
        """auto_tune (spectral.cpp:294-326) on the device couplings; mode "wigner" | "numerical"."""
        st = _lib.Spectral()
        m = {"wigner": 0, "numerical": 1}[mode]
        rc = self._L.sbg_auto_tune(self._h, m, d_t_factor, tol, max_iters, C.byref(st))
        est = SpectralEstimate(st.lambda_max, st.lambda_min, _SPECTRAL_METHODS[st.method], st.tolerance,
                               None, None, int(st.iterations))
        if rc == _lib.SBG_ERR_CONVERGENCE:
            raise ConvergenceError(self._L.sbg_last_error(self._h).decode(), est)
        self._check(rc)
        return TuningResult(c=st.c, dt=st.dt, d_t_factor=st.d_t_factor, lambda_max=st.lambda_max,
                            lambda_min=st.lambda_min, method=est.method, source=est, converged=bool(st.converged))

    # ------------------------------------------------------- row sharding (C5)
    def set_instance_rows(self, J_rows: np.ndarray, n_global: int, world: int, rank: int) -> None:
        """This rank's rows of J (rows x n_global int8; rows as sbg_set_couplings_rows_i8 assigns)."""
        J_rows = np.ascontiguousarray(J_rows, np.int8)
        self._check(self._L.sbg_set_couplings_rows_i8(self._h, n_global, world, rank, ptr(J_rows)))
        info = self.shard_info()
        self.n = info["rows_valid"]
        self.n_global = n_global
        self.total_weight = None

    def gen_hash_pm1(self, n_global: int, seed: int, world: int = 1, rank: int = 0) -> None:
        """Device-generated +-1 couplings (large-N throughput runs; not gen_random_dense's order)."""
        self._check(self._L.sbg_gen_couplings_hash_pm1(self._h, n_global, world, rank, seed))
        self.n = self.shard_info()["rows_valid"] if world > 1 else n_global
        self.n_global = n_global
        self.total_weight = None

    def shard_info(self) -> dict:
        vals = [C.c_int64() for _ in range(4)]
        self._check(self._L.sbg_shard_info(self._h, *(C.byref(v) for v in vals)))
        return dict(zip(["row0", "rows_valid", "rows_padded", "kpad"], (v.value for v in vals)))

    def shard_buffers(self):
        g0, g1, d = C.c_void_p(), C.c_void_p(), C.c_void_p()
        self._check(self._L.sbg_shard_buffers(self._h, C.byref(g0), C.byref(g1), C.byref(d)))
        return g0.value, g1.value, d.value

    def shard_set_peers(self, peers) -> None:
        """peers: list of (g0, g1, done) device pointers of the OTHER ranks."""
        n = len(peers)
        arr = [(C.c_void_p * max(n, 1))(*[p[k] for p in peers]) for k in range(3)]
        self._check(self._L.sbg_shard_set_peers(self._h, n, arr[0], arr[1], arr[2]))

    def shard_prepare(self, variant) -> None:
        self._check(self._L.sbg_shard_prepare(self._h, int(variant)))

    def shard_push_slab(self) -> None:
        self._check(self._L.sbg_shard_push_slab(self._h))

    def shard_ipc_export(self) -> bytes:
        buf = (C.c_char * 192)()
        self._check(self._L.sbg_shard_ipc_export(self._h, buf))
        return bytes(buf)

    def shard_ipc_open(self, handles: bytes):
        g0, g1, d = C.c_void_p(), C.c_void_p(), C.c_void_p()
        self._check(self._L.sbg_shard_ipc_open(self._h, handles, C.byref(g0), C.byref(g1), C.byref(d)))
        return g0.value, g1.value, d.value

    def readout_partial(self) -> np.ndarray:
        e2 = np.empty(self.R, np.int64)
        self._check(self._L.sbg_readout_partial(self._h, ptr(e2)))
        return e2

    def gen_random_dense(self, n: int, seed: int, world: int = 1, rank: int = 0, shard: bool = False) -> None:
        """gen_random_dense (model.cpp:144-159) generated on the device in the reference's
        exact draw order; world > 1 (or shard=True) keeps only this rank's rows (row sharding)."""
        if world == 1 and not shard:
            self._check(self._L.sbg_gen_couplings_dense_pm1(self._h, n, seed))
            self.n = n
        else:
            self._check(self._L.sbg_gen_couplings_dense_pm1_rows(self._h, n, world, rank, seed))
            self.n = self.shard_info()["rows_valid"]
        self.n_global = n
        self.total_weight = None

    def get_couplings(self, row_begin: int = 0, rows: Optional[int] = None) -> np.ndarray:
        """Rows of the device int8 couplings (all n columns; local rows for a shard)."""
        rows = self.n - row_begin if rows is None else rows
        out = np.empty((rows, self.n_global), np.int8)
        self._check(self._L.sbg_get_couplings_i8(self._h, row_begin, rows, ptr(out)))
        return out

    def set_instance_csr(self, n: int, rowptr, col, val, total_weight: Optional[int] = None) -> None:
        rowptr = np.ascontiguousarray(rowptr, np.int32)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.int8)
        self._check(self._L.sbg_set_couplings_csr_i8(self._h, n, len(col), ptr(rowptr), ptr(col), ptr(val)))
        self.n = self.n_global = n
        self.total_weight = total_weight if total_weight is not None else int(-val.astype(np.int64).sum() // 2)

    # -------------------------------------------------------------- states
    def set_state(self, x: np.ndarray, y: np.ndarray, p: Optional[np.ndarray] = None) -> None:
        x = np.ascontiguousarray(x, np.float32)
        y = np.ascontiguousarray(y, np.float32)
        if p is not None:
            p = np.ascontiguousarray(p, np.float32)
        self._check(self._L.sbg_set_state(self._h, x.shape[0], ptr(x), ptr(y), ptr(p)))
        self.R = x.shape[0]

    def init_state(self, R: int, mode: InitMode, master: int, tag: int, offset: int = 0) -> None:
        self._check(self._L.sbg_init_state(self._h, R, int(mode), master, tag, offset))
        self.R = R

    def init_state_seeds(self, seeds, mode: InitMode) -> None:
        seeds = np.ascontiguousarray(seeds, np.uint64)
        self._check(self._L.sbg_init_state_seeds(self._h, len(seeds), int(mode), ptr(seeds)))
        self.R = len(seeds)

    def set_replica_a(self, a) -> None:
        """Per-replica A (gbsb/gdsb); None clears."""
        if a is None:
            self._check(self._L.sbg_set_replica_a(self._h, 0, None))
            return
        a = np.ascontiguousarray(a, np.float32)
        self._check(self._L.sbg_set_replica_a(self._h, len(a), ptr(a)))

    def get_state(self):
        x, y, p = (np.empty((self.R, self.n), np.float32) for _ in range(3))
        self._check(self._L.sbg_get_state(self._h, ptr(x), ptr(y), ptr(p)))
        return x, y, p

    @staticmethod
    def params(cfg: SolverConfig) -> _lib.Params:
        return _lib.Params(int(cfg.variant), 0, int(cfg.steps), float(cfg.dt), float(cfg.c), float(cfg.a))

    def advance(self, cfg: SolverConfig, m_begin: int, m_end: int) -> None:
        """step() (engine.cpp:55-110) for m = m_begin .. m_end-1 of an M-step run."""
        prm = self.params(cfg)
        self._check(self._L.sbg_advance(self._h, C.byref(prm), m_begin, m_end))

    def synchronize(self) -> None:
        self._check(self._L.sbg_synchronize(self._h))

    def last_advance_ms(self) -> float:
        return self._L.sbg_last_advance_ms(self._h)

    def readout(self):
        """(spins R x n int8, energies R, best_index, best_energy)."""
        spins = np.empty((self.R, self.n), np.int8)
        energy = np.empty(self.R, np.float64)
        best = C.c_int64()
        best_e = C.c_double()
        self._check(self._L.sbg_readout(self._h, ptr(spins), ptr(energy), C.byref(best), C.byref(best_e)))
        return spins, energy, int(best.value), float(best_e.value)

    def readout_best(self):
        """(best_spins n int8, best_energy, best_index, energies R)."""
        spins = np.empty(self.n, np.int8)
        energy = np.empty(self.R, np.float64)
        best = C.c_int64()
        best_e = C.c_double()
        self._check(self._L.sbg_readout_best(self._h, ptr(spins), C.byref(best_e), C.byref(best), ptr(energy)))
        return spins, float(best_e.value), int(best.value), energy

    def fields_sign(self, S: np.ndarray) -> np.ndarray:
        S = np.ascontiguousarray(S, np.int8)
        F = np.empty(S.shape, np.int32)
        self._check(self._L.sbg_fields_sign(self._h, S.shape[0], ptr(S), ptr(F)))
        return F

    def fields_fixed(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        F = np.empty(x.shape, np.float32)
        self._check(self._L.sbg_fields_fixed(self._h, x.shape[0], ptr(x), ptr(F)))
        return F

    # ---------------------------------------------------------------- runs
    def run_batch(self, cfg: SolverConfig, tuning: TuningResult, R: int, x0: Optional[np.ndarray] = None,
                  y0: Optional[np.ndarray] = None, master_seed: int = 0, tag: int = SEED_STREAM_BATCH,
                  replica_offset: int = 0, want_x: bool = False, want_spins: bool = True):
        """run() (engine.cpp:112-139) for R replicas in one device pass.

        Initial states: host x0/y0 (R x n fp32), or generated on the device from
        derive_seed(master_seed, {tag, replica_offset + r}) with cfg.init_mode.
        Returns (list-free) arrays: spins, energies, cuts, best index, timing dict, x_final.
        """
        rcfg = resolve_config(cfg, tuning)
        if rcfg.sample_stride > 0:
            return self._run_batch_sampled(rcfg, tuning, R, x0, y0, master_seed, tag, replica_offset, want_spins)
        prm = self.params(rcfg)
        spins = np.empty((R, self.n), np.int8) if want_spins else None
        energy = np.empty(R, np.float64)
        best = C.c_int64()
        timing = _lib.Timing()
        x_final = np.empty((R, self.n), np.float32) if want_x else None
        if x0 is not None:
            x0 = np.ascontiguousarray(x0, np.float32)
            y0 = np.ascontiguousarray(y0 if y0 is not None else np.zeros_like(x0), np.float32)
            self._check(self._L.sbg_run(self._h, C.byref(prm), R, ptr(x0), ptr(y0), ptr(x_final), ptr(spins),
                                        ptr(energy), C.byref(best), C.byref(timing)))
        else:
            self._check(self._L.sbg_run_seeded(self._h, C.byref(prm), R, int(rcfg.init_mode), master_seed, tag,
                                               replica_offset, ptr(spins), ptr(energy), C.byref(best),
                                               C.byref(timing)))
        self.R = R
        cuts = None
        if self.total_weight is not None:
            # cut = (W - E) / 2 (model.hpp:103-104), exact integers
            cuts = ((self.total_weight - energy) / 2).astype(np.int64)
        return BatchResult(spins, energy, cuts, int(best.value), timing.as_dict(), x_final, rcfg, tuning)

    def run_best(self, cfg: SolverConfig, tuning: TuningResult, x0: np.ndarray, y0: Optional[np.ndarray] = None,
                 want_energies: bool = True):
        """batch_best_of's result (bench.cpp:70-92) for R = len(x0) replicas from host initial
        states in one call (sbg_run_best): H2D, M steps, readout, and D2H of only the winner's
        spins, energy and index (+ the R energies if want_energies).
        Returns (best_spins, best_energy, best_index, energies | None, timing dict)."""
        rcfg = resolve_config(cfg, tuning)
        prm = self.params(rcfg)
        x0 = np.ascontiguousarray(x0, np.float32)
        y0 = np.ascontiguousarray(y0 if y0 is not None else np.zeros_like(x0), np.float32)
        R = x0.shape[0]
        spins = np.empty(self.n, np.int8)
        be = C.c_double()
        bi = C.c_int64()
        energies = np.empty(R, np.float64) if want_energies else None
        timing = _lib.Timing()
        self._check(self._L.sbg_run_best(self._h, C.byref(prm), R, ptr(x0), ptr(y0), ptr(spins), C.byref(be),
                                         C.byref(bi), ptr(energies), C.byref(timing)))
        self.R = R
        return spins, float(be.value), int(bi.value), energies, timing.as_dict()

    def _run_batch_sampled(self, rcfg, tuning, R, x0, y0, master_seed, tag, replica_offset, want_spins):
        """run() with sample_stride (engine.cpp:117-133): x recorded at m = 0, every
        stride steps and at the final step; trajectory[k] = (m, x of all replicas)."""
        import time

        t0 = time.perf_counter()
        if x0 is not None:
            self.set_state(x0, y0 if y0 is not None else np.zeros_like(x0))
        else:
            self.init_state(R, rcfg.init_mode, master_seed, tag, replica_offset)
        traj = [(0, self.get_state()[0])]
        m = 0
        while m < rcfg.steps:
            nxt = min(m + rcfg.sample_stride, rcfg.steps)
            self.advance(rcfg, m, nxt)
            m = nxt
            if m % rcfg.sample_stride == 0 or m == rcfg.steps:
                traj.append((m, self.get_state()[0]))
        spins, energies, best, _ = self.readout()
        cuts = None
        if self.total_weight is not None:
            cuts = ((self.total_weight - energies) / 2).astype(np.int64)
        timing = {"total_ms": (time.perf_counter() - t0) * 1e3}
        b = BatchResult(spins if want_spins else None, energies, cuts, best, timing, traj[-1][1], rcfg, tuning)
        b.trajectory = traj
        return b

    def run(self, cfg: SolverConfig, tuning: TuningResult) -> RunResult:
        """run() (engine.cpp:112-139) for one replica: init_state(n, cfg.seed, cfg.init_mode),
        M steps, readout; wall time covers init + steps + readout."""
        import time

        rcfg = resolve_config(cfg, tuning)
        t0 = time.perf_counter()
        self.init_state_seeds(np.array([rcfg.seed], np.uint64), rcfg.init_mode)
        self.advance(rcfg, 0, int(rcfg.steps))
        spins, energy, _, _ = self.readout()
        wall = time.perf_counter() - t0
        cut = None if self.total_weight is None else cut_from_energy(self.total_weight, float(energy[0]))
        return RunResult(final_spins=spins[0].copy(), energy=float(energy[0]), cut=cut, wall_time_s=wall,
                         config_echo=rcfg, tuning_echo=tuning)

    def batch_best_of(self, cfg: SolverConfig, tuning: TuningResult, n_batch: int, master_seed: int) -> RunResult:
        """bench.cpp:70-92: replicas seeded derive_seed(master, {batch, r}); min energy, ties -> lowest r."""
        if n_batch < 1:
            raise ValueError("batch size must be >= 1")
        b = self.run_batch(cfg, tuning, n_batch, master_seed=master_seed, tag=SEED_STREAM_BATCH)
        w = b.best_index
        echo = dataclasses.replace(b.config, seed=_derive_seed(master_seed, [SEED_STREAM_BATCH, w]))
        return RunResult(final_spins=b.spins[w].copy(), energy=float(b.energies[w]),
                         cut=None if b.cuts is None else int(b.cuts[w]),
                         wall_time_s=b.timing["total_ms"] / 1e3, config_echo=echo, tuning_echo=tuning)


@dataclasses.dataclass
class BatchResult:
    spins: np.ndarray
    energies: np.ndarray
    cuts: Optional[np.ndarray]
    best_index: int
    timing: dict
    x_final: Optional[np.ndarray]
    config: SolverConfig
    tuning: TuningResult
    trajectory: Optional[list] = None  # [(m, x[R][n])] when config.sample_stride > 0


def _mix64(z: int) -> int:
    M = (1 << 64) - 1
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def _derive_seed(master: int, keys) -> int:
    """rng.hpp:26-31 (host bookkeeping for config echoes only)."""
    M = (1 << 64) - 1
    h = _mix64((master + 0x9E3779B97F4A7C15) & M)
    for k in keys:
        h = _mix64(h ^ ((k + 0x9E3779B97F4A7C15) & M))
    return h


def cut_from_energy(total_weight: int, energy: float) -> int:
    return int(math.floor((total_weight - energy) / 2 + 0.5))


SEED_STREAM_SWEEP = 1  # rng.hpp:34 seed_stream::sweep


@dataclasses.dataclass
class SweepCell:  # bench.hpp:72-80
    mi: int
    ai: int
    m_steps: int
    a: float
    stats: SuccessStats
    mean_energy: float
    best_energy: float
    energies: np.ndarray


def sweep(solver: "Solver", m_values, a_values, reps: int, cfg_base: SolverConfig, tuning: TuningResult,
          target: float):
    """sbopt::sweep (bench.cpp:171-197) on the GPU: one launch per M value covering every
    A cell x reps replicas (per-replica A); replica r of cell (mi, ai) is seeded
    derive_seed(cfg_base.seed, {sweep, mi, ai, r}) with cfg_base.init_mode, as
    run_sweep_cell does (bench.cpp:159). Cells row-major, M outer, A inner."""
    if len(m_values) == 0 or len(a_values) == 0:
        raise ValueError("empty sweep axes")
    if reps < 1:
        raise ValueError("sweep needs reps >= 1")
    cells = []
    na = len(a_values)
    for mi, m_steps in enumerate(m_values):
        cfg = resolve_config(dataclasses.replace(cfg_base, steps=int(m_steps)), tuning)
        seeds = np.array([_derive_seed(cfg_base.seed, [SEED_STREAM_SWEEP, mi, ai, r])
                          for ai in range(na) for r in range(reps)], np.uint64)
        solver.init_state_seeds(seeds, cfg.init_mode)
        solver.set_replica_a(np.repeat(np.asarray(a_values, np.float32), reps))
        solver.advance(cfg, 0, int(m_steps))
        _, energies, _, _ = solver.readout()
        solver.set_replica_a(None)
        for ai, a in enumerate(a_values):
            e = energies[ai * reps:(ai + 1) * reps]
            cells.append(SweepCell(mi, ai, int(m_steps), float(a), success_probability(e, target),
                                   float(e.mean()), float(e.min()), e.copy()))
    return cells


SEED_STREAM_DT_SWEEP = 2  # rng.hpp:35 seed_stream::dt_sweep
SEED_STREAM_BENCH = 6  # rng.hpp:39 seed_stream::bench


def tune_dt(lambda_min: float, lambda_max: float, d_t_factor: float) -> float:
    """spectral.cpp:277-286: dt = D_t sqrt(2 / (1 - lambda_min / lambda_max))."""
    if not lambda_max > 0.0:
        raise ValueError("lambda_max must be positive")
    if not lambda_min < 0.0:
        raise ValueError("lambda_min must be negative")
    if not d_t_factor > 0.0:
        raise ValueError("d_t_factor must be positive")
    return d_t_factor * math.sqrt(2.0 / (1.0 - lambda_min / lambda_max))


def stability_limit(lambda_min: float, lambda_max: float) -> float:
    """spectral.cpp:288-292."""
    if not lambda_max > 0.0:
        raise ValueError("lambda_max must be positive")
    if not lambda_min < 0.0:
        raise ValueError("lambda_min must be negative")
    return 2.0 / math.sqrt(1.0 - lambda_min / lambda_max)


@dataclasses.dataclass
class DtSweepCell:  # bench.hpp:114-124
    di: int
    ti: int
    d_t_factor: float
    t_final: float
    dt: float
    m_steps: int
    stats: SuccessStats
    mean_energy: float
    best_energy: float
    energies: np.ndarray


def dt_sweep(solver: "Solver", d_t_values, t_final_values, a: float, reps: int, cfg_base: SolverConfig,
             tuning: TuningResult, target: float):
    """sbopt::dt_sweep (bench.cpp:208-269) on the GPU: cell (di, ti) runs reps replicas at
    dt = tune_dt(lambda_min, lambda_max, D_t) and M = llround(t_M / dt), replica r seeded
    derive_seed(cfg_base.seed, {dt_sweep, di, ti, r}); one device launch per cell."""
    if len(d_t_values) == 0 or len(t_final_values) == 0:
        raise ValueError("empty sweep axes")
    if reps < 1:
        raise ValueError("sweep needs reps >= 1")
    if any(not v > 0.0 for v in d_t_values):
        raise ValueError("D_t values must be positive")
    if any(not v > 0.0 for v in t_final_values):
        raise ValueError("t_M values must be positive")
    cells = []
    for di, d_t in enumerate(d_t_values):
        dt = tune_dt(tuning.lambda_min, tuning.lambda_max, d_t)
        for ti, t_final in enumerate(t_final_values):
            q = t_final / dt  # std::llround: half away from zero
            m_steps = int(math.floor(q + 0.5)) if q >= 0 else -int(math.floor(-q + 0.5))
            if m_steps == 0:
                raise ValueError(f"t_M = {t_final:f} rounds to zero steps at dt = {dt:f}")
            cfg = resolve_config(dataclasses.replace(cfg_base, steps=m_steps, dt=dt, a=a), tuning)
            seeds = np.array([_derive_seed(cfg_base.seed, [SEED_STREAM_DT_SWEEP, di, ti, r]) for r in range(reps)],
                             np.uint64)
            solver.init_state_seeds(seeds, cfg.init_mode)
            solver.advance(cfg, 0, m_steps)
            _, e, _, _ = solver.readout()
            cells.append(DtSweepCell(di, ti, float(d_t), float(t_final), dt, m_steps, success_probability(e, target),
                                     float(e.mean()), float(e.min()), e.copy()))
    return cells


SEED_STREAM_CHAOS = 4  # rng.hpp:37
SEED_STREAM_CHAOS_PERTURB = 5  # rng.hpp:38


class _HostXoshiro:
    """rng.hpp:44-77 on the host, for building explicit initial states (chaos pairs)."""

    M64 = (1 << 64) - 1

    def __init__(self, seed: int):
        z = seed
        self.s = []
        for _ in range(4):
            z = (z + 0x9E3779B97F4A7C15) & self.M64
            self.s.append(_mix64(z))

    def next(self) -> int:
        s0, s1, s2, s3 = self.s
        M = self.M64
        result = ((((s0 + s3) & M) << 23 | ((s0 + s3) & M) >> 41) & M) + s0 & M
        t = (s1 << 17) & M
        s2 ^= s0
        s3 ^= s1
        s1 ^= s2
        s0 ^= s3
        s2 ^= t
        s3 = ((s3 << 45) | (s3 >> 19)) & M
        self.s = [s0, s1, s2, s3]
        return result

    def random_sign(self) -> float:
        return -1.0 if (self.next() >> 63) else 1.0


def paired_initial_conditions(n: int, seed: int):
    """chaos.cpp:11-18 rounded to fp32: x1 = +-0.1 (init_state chaos_probe), x2 = x1 +
    2e-6 * random_sign from Xoshiro(derive_seed(seed, {chaos_perturb})); y = 0, p = 1."""
    g = _HostXoshiro(seed)
    x1 = np.array([0.1 * g.random_sign() for _ in range(n)])
    h = _HostXoshiro(_derive_seed(seed, [SEED_STREAM_CHAOS_PERTURB]))
    x2 = x1 + np.array([2e-6 * h.random_sign() for _ in range(n)])
    return x1.astype(np.float32), x2.astype(np.float32)


def normalized_distance(x1, x2) -> float:
    """chaos.cpp:20-29: sqrt(sum (x1 - x2)^2 / (4 N))."""
    d = np.asarray(x1, np.float64) - np.asarray(x2, np.float64)
    return float(np.sqrt((d * d).sum() / (4.0 * d.size)))


@dataclasses.dataclass
class ChaosScanRow:  # chaos.hpp:44-51
    a: float
    mean_final_delta: float
    std_error: float
    reps: int
    seed: int
    final_deltas: np.ndarray


def chaos_scan(solver: "Solver", a_values, reps: int, cfg_base: SolverConfig, tuning: TuningResult):
    """sbopt::chaos_scan (chaos.cpp:65-102) on the GPU: all len(a_values) x reps
    trajectory PAIRS run as 2 x that many replicas of one launch (per-replica A),
    pair (ai, r) seeded derive_seed(cfg_base.seed, {chaos, ai, r})."""
    if reps < 1:
        raise ValueError("chaos scan needs reps >= 1")
    cfg = resolve_config(dataclasses.replace(cfg_base, variant=Variant.gbsb), tuning)
    n = solver.n
    xs, a_rep = [], []
    for ai, a in enumerate(a_values):
        for r in range(reps):
            x1, x2 = paired_initial_conditions(n, _derive_seed(cfg_base.seed, [SEED_STREAM_CHAOS, ai, r]))
            xs += [x1, x2]
            a_rep += [a, a]
    x0 = np.stack(xs)
    solver.set_state(x0, np.zeros_like(x0))
    solver.set_replica_a(np.asarray(a_rep, np.float32))
    solver.advance(cfg, 0, int(cfg.steps))
    x, _, _ = solver.get_state()
    solver.set_replica_a(None)
    rows = []
    for ai, a in enumerate(a_values):
        d = np.array([normalized_distance(x[2 * (ai * reps + r)], x[2 * (ai * reps + r) + 1]) for r in range(reps)])
        mean = float(d.mean())
        se = float(np.sqrt(((d - mean) ** 2).sum() / (reps - 1) / reps)) if reps > 1 else 0.0
        rows.append(ChaosScanRow(float(a), mean, se, reps, cfg_base.seed, d))
    return rows
