"""The sbopt CLI on the GPU (python -m paper_2508_17655_b200): every subcommand end to
end on small instances, output documents checked against the oracle (energies from
the reported spins, cuts via the reference's cut_value) and the reference's formats
(manifest keys, CSV headers, exit codes)."""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def run(*args):
    p = subprocess.run([sys.executable, "-m", "paper_2508_17655_b200", *map(str, args)], capture_output=True,
                       text=True, cwd=str(ROOT), timeout=600)
    return p.returncode, p.stdout, p.stderr


def torus_gset(L, seed):
    rng = np.random.default_rng(seed)
    lines = []
    for r in range(L):
        for c in range(L):
            v = r * L + c + 1
            for u in (r * L + (c + 1) % L + 1, ((r + 1) % L) * L + c + 1):
                lines.append(f"{v} {u} {1 if rng.random() < 0.5 else -1}")
    return f"{L * L} {len(lines)}\n" + "\n".join(lines) + "\n"


def test_gen_then_solve_json(tmp_path, orc):
    rc, out, err = run("gen", "--n", 60, "--seed", 3)
    assert rc == 0, err
    doc = json.loads(out)
    assert doc["label"] == "dense-n60-s3" and doc["n"] == 60
    J = orc.gen_dense_i8(60, 3)
    assert all(J[i, j] == v for i, j, v in doc["edges"]) and len(doc["edges"]) == 60 * 59 // 2
    f = tmp_path / "inst.json"
    f.write_text(out)
    rc, out, err = run("solve", f, "--tune", "wigner", "--M", 500, "--seed", 5, "--variant", "gdsb")
    assert rc == 0, err
    m = json.loads(out)
    assert set(m) == {"tool", "instance", "config", "tuning", "energy", "cut", "wall_time_s", "spins", "device"}
    s = np.array(m["spins"], np.int64)
    assert m["energy"] == -0.5 * s @ J.astype(np.int64) @ s and m["cut"] is None
    assert m["config"]["variant"] == "gdsb" and m["tuning"]["method"] == "wigner"
    assert m["instance"] == {"label": "dense-n60-s3", "n": 60}


def test_solve_gset_batch_and_rle(tmp_path):
    from paper_2508_17655_b200.instances import cut_value, parse_gset

    f = tmp_path / "torus.txt"
    f.write_text(torus_gset(12, 1))
    g = parse_gset(f.read_text())
    rc, out, err = run("solve", "--gset", f, "--tune", "wigner", "--batch", 32, "--M", 800, "--seed", 2,
                       "--rle-spins")
    assert rc == 0, err
    m = json.loads(out)
    s = np.concatenate([np.full(c, v, np.int8) for v, c in m["spins_rle"]])
    assert m["cut"] == cut_value(g, s)
    if oracle.ref_available():
        assert m["cut"] == oracle.ref().cut_value(g.n, g.i, g.j, g.w, s)


def test_bench_sweep_chaos(tmp_path):
    f = tmp_path / "torus.txt"
    f.write_text(torus_gset(10, 2))
    rc, out, err = run("bench", f, "--tune", "wigner", "--reps", 64, "--M", 500, "--target-cut", 40)
    assert rc == 0, err
    b = json.loads(out)
    assert b["reps"] == 64 and 0 <= b["p_s"] <= 1 and b["hits"] == round(b["p_s"] * 64)
    csv = tmp_path / "sweep.csv"
    rc, _, err = run("sweep", f, "--tune", "wigner", "--M-grid", "200,400", "--A-grid", "0:0.4:0.2", "--reps", 16,
                     "--target-energy", -60, "--out", csv)
    assert rc == 0, err
    lines = csv.read_text().strip().split("\n")
    assert lines[0] == "m,a,reps,hits,p_s,delta_p_s,mean_energy,best_energy" and len(lines) == 7
    summary = json.loads((tmp_path / "sweep.csv.json").read_text())
    assert summary["axis_m"] == [200, 400] and len(summary["cells"]) == 6
    rc, _, err = run("sweep", f, "--tune", "wigner", "--M-grid", "200,400", "--A-grid", "0:0.4:0.2", "--reps", 16,
                     "--target-energy", -60, "--out", csv, "--resume")
    assert rc == 0 and len(csv.read_text().strip().split("\n")) == 7
    dcsv = tmp_path / "dt.csv"
    rc, _, err = run("sweep", f, "--tune", "wigner", "--Dt-grid", "0.8,1.2", "--tM-grid", "100,300", "--reps", 8,
                     "--target-energy", -60, "--out", dcsv)
    assert rc == 0, err
    rows = dcsv.read_text().strip().split("\n")
    assert rows[0].startswith("d_t,t_final,dt,m") and len(rows) == 5
    rc, out, err = run("chaos", f, "--tune", "wigner", "--A-grid", "0,0.5", "--reps", 4, "--M", 200)
    assert rc == 0, err
    rows = out.strip().split("\n")
    assert rows[0] == "a,mean_final_delta,stderr,reps,seed" and len(rows) == 3


def test_runtime_and_parse_errors(tmp_path):
    rc, _, err = run("solve", "--dense", 100, "--tune", "numerical")  # lambda_max misses the 10 n cap
    assert rc == 1 and "did not converge" in err
    bad = tmp_path / "bad.txt"
    bad.write_text("3 2\n1 2 1\n2 1 1\n")
    rc, _, err = run("solve", bad)
    assert rc == 2 and "line 3: duplicate edge (2, 1)" in err
    rc, _, err = run("bench", "--dense", 20, "--tune", "wigner", "--target-cut", 3)
    assert rc == 2 and "needs a graph instance" in err
