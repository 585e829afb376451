"""The C++ host mirror (include/sbgpu.hpp): compiles here, runs on the GPU."""
import json
import os
import subprocess

import numpy as np

import oracle
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "api_demo.cpp")
LIBDIR = os.path.join(ROOT, "paper_2508_17655_b200")


def build(out):
    from paper_2508_17655_b200 import build as b

    b.build()
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), SRC, "-o", out,
           "-L", LIBDIR, "-lsbgpu", f"-Wl,-rpath,{LIBDIR}"]
    subprocess.run(cmd, check=True)


def test_cpp_api_compiles(tmp_path):
    build(str(tmp_path / "api_demo"))


@pytest.mark.gpu
def test_cpp_api_matches_oracle(tmp_path, orc):
    exe = str(tmp_path / "api_demo")
    build(exe)
    out = json.loads(subprocess.run([exe], check=True, capture_output=True, text=True).stdout)
    assert out["invalid_caught"] == 2
    assert out["convergence_caught"] == 1
    n, R = out["n"], out["R"]
    # rebuild the demo's instance and run the fp32 mirror from the same seeded states
    J = np.zeros((n, n), np.int8)
    z = 12345
    M64 = (1 << 64) - 1
    from paper_2508_17655_b200.solver import _mix64

    for i in range(n):
        for j in range(i + 1, n):
            z = _mix64((z + 1) & M64)
            J[i, j] = J[j, i] = -1 if (z >> 63) else 1
    assert out["c"] == 1 / (2 * np.sqrt(n)) and out["dt"] == 1.25
    x, y, p = orc.init_small_uniform(n, R, master=7, tag=7)
    x, y, p = orc.step_f32(3, J, x, y, p, 0, 100, np.float32(out["dt"]), np.float32(out["c"]), np.float32(0.2), 100)
    e = -0.5 * orc.energy2_i8(J, x)
    assert out["energies"] == list(e)
    W = -int(np.triu(J.astype(np.int64), 1).sum())
    assert out["cuts"] == [int((W - v) // 2) for v in e]
    assert abs(out["tts_mid"] - 6.6439) < 1e-3
    assert out["wigner_c"] == out["c"]
    # batch_best_of from host initial states (sbg_run_best): the same winner, spins included
    bi = int(np.flatnonzero(e == e.min())[0])
    assert out["states_best_index"] == bi and out["states_best_energy"] == e[bi]
    assert out["states_best_spins_match"] == 1
    if oracle.ref_available():  # device power iteration == the reference's, bitwise
        rc, want, _, _ = oracle.ref().extreme_eigenvalues(J.astype(np.float64), 1e-6, 100000)
        assert rc == 0 and (out["lambda_max"], out["lambda_min"], out["iterations"]) == (
            want["lambda_max"], want["lambda_min"], want["iterations"])
