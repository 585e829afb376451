"""ctypes binding of the sbgpu C ABI (include/sbgpu.h), libsbgpu.so in-tree.

There is no fallback: if the CUDA library is missing or no sm_100 device is
present, calls raise. The library is built by ``paper_2508_17655_b200.build``
(``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SBG_LIB_OVERRIDE") or os.path.join(HERE, "libsbgpu.so")  # dev A/B builds

SBG_OK, SBG_ERR_INVALID_ARGUMENT, SBG_ERR_OUT_OF_MEMORY, SBG_ERR_CUDA, SBG_ERR_NCCL, SBG_ERR_STATE, \
    SBG_ERR_UNSUPPORTED, SBG_ERR_CONVERGENCE = range(8)
BSB, DSB, GBSB, GDSB = 0, 1, 2, 3
INIT_UNIFORM_RANDOM, INIT_CHAOS_PROBE, INIT_SMALL_UNIFORM = 0, 1, 2

EXPORTS = [
    "sbg_abi_version", "sbg_strerror", "sbg_create", "sbg_destroy", "sbg_last_error", "sbg_device_sm_count",
    "sbg_device_name", "sbg_couplings_e2m1",
    "sbg_set_couplings_dense_i8", "sbg_set_couplings_dense_f64", "sbg_set_couplings_dense_f32",
    "sbg_coupling_scale_exp", "sbg_gen_couplings_dense_pm1",
    "sbg_set_couplings_csr_i8", "sbg_n", "sbg_set_state", "sbg_init_state", "sbg_get_state", "sbg_advance",
    "sbg_readout", "sbg_readout_best", "sbg_fields_sign", "sbg_fields_fixed", "sbg_run", "sbg_run_best", "sbg_run_seeded", "sbg_synchronize",
    "sbg_kernel_launches", "sbg_state_device", "sbg_last_advance_ms", "sbg_success_tts", "sbg_tune_wigner_f64",
    "sbg_set_couplings_rows_i8", "sbg_shard_info", "sbg_shard_buffers", "sbg_shard_set_peers", "sbg_shard_prepare",
    "sbg_shard_push_slab", "sbg_shard_advance_fused", "sbg_shard_ipc_export", "sbg_shard_ipc_open",
    "sbg_readout_partial",
    "sbg_gen_couplings_hash_pm1", "sbg_set_replica_a", "sbg_init_state_seeds",
    "sbg_gen_couplings_dense_pm1_rows", "sbg_get_couplings_i8", "sbg_extreme_eigenvalues", "sbg_auto_tune",
    "sbg_set_couplings_graph", "sbg_set_couplings_entries_f64",
]


class SbgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"sbgpu error {code}: {msg}")
        self.code = code


class SbgInvalidArgument(SbgError, ValueError):
    """Mirrors std::invalid_argument thrown by the reference (engine.cpp:16-21, :57-60)."""


class Params(C.Structure):
    _fields_ = [("variant", C.c_int32), ("reserved", C.c_int32), ("steps", C.c_uint64), ("dt", C.c_double),
                ("c", C.c_double), ("a", C.c_double)]


class Spectral(C.Structure):  # sbg_spectral
    _fields_ = [("lambda_max", C.c_double), ("lambda_min", C.c_double), ("c", C.c_double), ("dt", C.c_double),
                ("d_t_factor", C.c_double), ("tolerance", C.c_double), ("iterations", C.c_uint64),
                ("method", C.c_int32), ("converged", C.c_int32)]


class Timing(C.Structure):
    _fields_ = [("h2d_ms", C.c_double), ("init_ms", C.c_double), ("steps_ms", C.c_double),
                ("readout_ms", C.c_double), ("d2h_ms", C.c_double), ("total_ms", C.c_double),
                ("kernel_launches", C.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    P, i64, u64, i32, f64 = C.c_void_p, C.c_int64, C.c_uint64, C.c_int32, C.c_double
    L.sbg_strerror.restype = C.c_char_p
    L.sbg_last_error.restype = C.c_char_p
    L.sbg_last_error.argtypes = [P]
    L.sbg_create.argtypes = [C.c_int, C.POINTER(P)]
    L.sbg_destroy.argtypes = [P]
    L.sbg_destroy.restype = None
    L.sbg_device_sm_count.argtypes = [P]
    L.sbg_device_name.argtypes = [P]
    L.sbg_device_name.restype = C.c_char_p
    L.sbg_couplings_e2m1.argtypes = [P]
    L.sbg_set_couplings_dense_i8.argtypes = [P, i64, P]
    L.sbg_set_couplings_dense_f64.argtypes = [P, i64, P]
    L.sbg_gen_couplings_dense_pm1.argtypes = [P, i64, u64]
    L.sbg_set_couplings_dense_f32.argtypes = [P, i64, P]
    L.sbg_coupling_scale_exp.argtypes = [P]
    L.sbg_set_couplings_csr_i8.argtypes = [P, i64, i64, P, P, P]
    L.sbg_n.restype = i64
    L.sbg_n.argtypes = [P]
    L.sbg_set_state.argtypes = [P, i64, P, P, P]
    L.sbg_init_state.argtypes = [P, i64, i32, u64, u64, i64]
    L.sbg_get_state.argtypes = [P, P, P, P]
    L.sbg_advance.argtypes = [P, C.POINTER(Params), u64, u64]
    L.sbg_readout.argtypes = [P, P, P, P, P]
    L.sbg_readout_best.argtypes = [P, P, P, P, P]
    L.sbg_fields_sign.argtypes = [P, i64, P, P]
    L.sbg_fields_fixed.argtypes = [P, i64, P, P]
    L.sbg_run.argtypes = [P, C.POINTER(Params), i64, P, P, P, P, P, P, C.POINTER(Timing)]
    L.sbg_run_best.argtypes = [P, C.POINTER(Params), i64, P, P, P, P, P, P, C.POINTER(Timing)]
    L.sbg_run_seeded.argtypes = [P, C.POINTER(Params), i64, i32, u64, u64, i64, P, P, P, C.POINTER(Timing)]
    L.sbg_synchronize.argtypes = [P]
    L.sbg_kernel_launches.restype = i64
    L.sbg_kernel_launches.argtypes = [P]
    L.sbg_state_device.argtypes = [P, P, P, P, P, P]
    L.sbg_last_advance_ms.restype = f64
    L.sbg_last_advance_ms.argtypes = [P]
    L.sbg_success_tts.argtypes = [i64, i64, f64, P]
    L.sbg_tune_wigner_f64.argtypes = [i64, P, f64, P, P]
    L.sbg_set_couplings_rows_i8.argtypes = [P, i64, i32, i32, P]
    L.sbg_shard_info.argtypes = [P, P, P, P, P]
    L.sbg_shard_buffers.argtypes = [P, P, P, P]
    L.sbg_shard_set_peers.argtypes = [P, i32, P, P, P]
    L.sbg_shard_prepare.argtypes = [P, i32]
    L.sbg_shard_push_slab.argtypes = [P]
    if hasattr(L, "sbg_shard_advance_fused"):  # (dev A/B against builds that predate it)
        L.sbg_shard_advance_fused.argtypes = [P, i32, P, u64, u64]
    L.sbg_shard_ipc_export.argtypes = [P, P]
    L.sbg_shard_ipc_open.argtypes = [P, P, P, P, P]
    L.sbg_readout_partial.argtypes = [P, P]
    L.sbg_gen_couplings_hash_pm1.argtypes = [P, i64, i32, i32, u64]
    L.sbg_gen_couplings_dense_pm1_rows.argtypes = [P, i64, i32, i32, u64]
    L.sbg_get_couplings_i8.argtypes = [P, i64, i64, P]
    L.sbg_extreme_eigenvalues.argtypes = [P, C.c_double, u64, C.POINTER(Spectral), P, P]
    L.sbg_auto_tune.argtypes = [P, i32, C.c_double, C.c_double, u64, C.POINTER(Spectral)]
    L.sbg_set_couplings_graph.argtypes = [P, i64, i64, P, P, P, P]
    L.sbg_set_couplings_entries_f64.argtypes = [P, i64, i64, P, P, P]
    L.sbg_set_replica_a.argtypes = [P, i64, P]
    L.sbg_init_state_seeds.argtypes = [P, i64, i32, P]
    _lib = L
    return L


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return C.c_void_p(a.ctypes.data)


def raise_for(code: int, msg: str) -> None:
    if code == SBG_OK:
        return
    if code == SBG_ERR_INVALID_ARGUMENT:
        raise SbgInvalidArgument(code, msg)
    raise SbgError(code, msg)
