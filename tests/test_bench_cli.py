"""bench.py's launcher contract on CPU (no GPU needed): --gpus N outside torchrun
re-executes itself under torch.distributed.run with N ranks (rank 0 alone prints the
reference arm's line), and a launcher whose WORLD_SIZE disagrees with --gpus is refused."""
import json
import os
import subprocess
import sys

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra, timeout=300):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], env=env, capture_output=True,
                          text=True, timeout=timeout, cwd=ROOT)


def test_world_size_mismatch_is_refused():
    r = _run(["--gpus", "3", "--impl", "reference"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "--gpus 3" in r.stderr


@pytest.mark.skipif(not oracle.ref_available(), reason="needs oracle/_ref (the compiled reference)")
def test_gpus_2_relaunches_under_torchrun():
    r = _run(["--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "3"],
             {"SBG_BENCH_REF_BUDGET": "0.2", "OMP_NUM_THREADS": "1"})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["steps"] == 1
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
