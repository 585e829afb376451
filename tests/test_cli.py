"""CLI host logic (cli.py, mirroring tools/sbopt.cpp): exit codes and messages of the
usage paths, grid parsing, CSV row formatting, the FPGA cycle model -- everything that
runs before the device is touched. CPU only; tests/test_gpu_cli.py runs the commands."""
import subprocess
import sys

import pytest

from paper_2508_17655_b200 import cli


def run(*args):
    p = subprocess.run([sys.executable, "-m", "paper_2508_17655_b200", *args], capture_output=True, text=True,
                       cwd=str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    return p.returncode, p.stdout, p.stderr


def test_usage_errors_exit_2():
    rc, _, err = run("solve")
    assert rc == 2 and "sbopt: no instance given" in err
    rc, _, err = run("solve", "--dense", "10", "--gset", "x.txt")
    assert rc == 2 and "exactly one instance source" in err
    rc, _, err = run("solve", "/nonexistent/file.txt")
    assert rc == 2 and "no such file" in err
    rc, _, _ = run("solve", "--variant", "nope", "--dense", "10")
    assert rc == 2
    rc, _, _ = run("frobnicate")
    assert rc == 2


def test_cycles_model():
    rc, out, _ = run("cycles", "--n", "2048", "--pr", "8", "--pc", "8", "--pb", "8", "--latency", "100",
                     "--fsys", "3e8")
    assert rc == 0
    lines = out.split()
    assert int(lines[0]) == 2048 * 2048 // 512 + 8 + 100 and lines[1] == "step_time_us"
    rc, _, err = run("cycles", "--n", "10", "--pr", "3", "--pc", "1", "--pb", "1", "--latency", "0")
    assert rc == 2 and "not divisible" in err


def test_parse_grid():
    assert cli.parse_grid("0:1:0.25") == [0.0, 0.25, 0.5, 0.75, 1.0]
    assert cli.parse_grid("0.1,0.2,,0.3") == [0.1, 0.2, 0.3]
    assert cli.parse_int_grid("100:300:100") == [100, 200, 300]
    for bad in ("1:2", "1:2:0", "", "a:b:c"):
        with pytest.raises(cli.UsageError):
            cli.parse_grid(bad)
    with pytest.raises(cli.UsageError):
        cli.parse_int_grid("0,1")


def test_csv_rows_printf_format():
    from types import SimpleNamespace as NS
    c = NS(m_steps=1000, a=0.15, stats=NS(n_rep=50, hit_count=7, p_s=0.14, delta_p_s=0.04907137658554119),
           mean_energy=-1234.5678901234, best_energy=-1300.0)
    assert cli.sweep_csv_row(c) == "1000,0.15,50,7,0.14,0.04907137659,-1234.56789,-1300"
    assert cli.SWEEP_HEADER == "m,a,reps,hits,p_s,delta_p_s,mean_energy,best_energy"


def test_targets():
    from paper_2508_17655_b200.instances import CutGraph
    import numpy as np

    p = cli.Problem("maxcut", 3, CutGraph(3, np.array([0, 1]), np.array([1, 2]), np.array([2, 3])))
    assert cli.resolve_energy_target(p, None, 4) == 5 - 8
    with pytest.raises(cli.UsageError):
        cli.resolve_energy_target(p, 1.0, 2.0)
    with pytest.raises(cli.UsageError):
        cli.resolve_energy_target(cli.Problem("x", 3), None, 2.0)
