"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, host-only entry points (statistics, tuning) match the
reference, and device calls fail cleanly without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2508_17655_b200 import build as b

    b.build()
    from paper_2508_17655_b200 import _lib

    return _lib.lib()


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "sbgpu.h")).read()
    return sorted(set(re.findall(r"\b(sbg_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    from paper_2508_17655_b200 import _lib

    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_every_declared_symbol_exported(L):
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert L.sbg_abi_version() == 1


def test_success_tts_kats(L, golden):
    out = (C.c_double * 4)()
    for (h, nr, t), ref in zip(golden["tts_in"], golden["tts_out"]):
        assert L.sbg_success_tts(int(h), int(nr), float(t), out) == 0
        assert list(out) == list(ref)
    assert L.sbg_success_tts(0, 10, 1.0, out) == 1  # TTS undefined for p_s = 0
    assert L.sbg_success_tts(11, 10, 1.0, out) == 1  # hits > n_rep


def test_python_mirror_stats(golden):
    from paper_2508_17655_b200 import success_from_counts, success_probability, time_to_solution

    st = success_from_counts(500, 1000, 0.0)
    tts = time_to_solution(1.0, st)
    assert abs(tts.tts_s - 6.6439) / 6.6439 < 1e-4 and abs(tts.delta_tts_s - 0.3031) / 0.3031 < 1e-3
    assert time_to_solution(0.010, success_from_counts(999, 1000, 0.0)).tts_s == 0.010
    with pytest.raises(ValueError):
        time_to_solution(1.0, success_from_counts(0, 10, 0.0))
    st = success_probability([-3.0, -5.0, -5.0, -4.0], -5.0)
    assert st.hit_count == 2 and st.p_s == 0.5


def test_wigner_tuning_matches_reference(golden):
    from paper_2508_17655_b200 import auto_tune_wigner

    t = auto_tune_wigner(golden["J_n37_s11"].astype(np.float64))
    assert t.c == float(golden["tune_c"]) and t.dt == float(golden["tune_dt"])


def test_config_resolution_mirrors_reference():
    from paper_2508_17655_b200 import SolverConfig, TuningResult, resolve_config

    t = TuningResult(c=0.25, dt=1.25)
    r = resolve_config(SolverConfig(), t)
    assert (r.c, r.dt) == (0.25, 1.25)
    assert resolve_config(SolverConfig(dt=0.5), t).dt == 0.5
    for kw in (dict(steps=0), dict(dt=-1.0), dict(a=-0.5)):
        with pytest.raises(ValueError):
            resolve_config(SolverConfig(**kw), t)


def test_create_without_gpu_fails_cleanly(L):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    assert L.sbg_create(0, C.byref(h)) != 0 and not h.value
