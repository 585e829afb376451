"""`python -m paper_2508_17655_b200` -- the sbopt command line (tools/sbopt.cpp) with
the solver on the GPU.

Same subcommands, options, output documents and exit codes as the reference CLI
(solve / bench / sweep / chaos / gen / cycles; exit 2 for usage, parse and
invalid-argument errors, 1 for runtime errors, messages "sbopt: ..." on stderr).
Differences, all deliberate: instances are loaded straight to the device (G-set and
sparse JSON as CSR, no dense fp64), tuning runs on the device, replicas of a
bench/sweep/chaos run share one device launch, and every output document carries a
"device" echo (GPU name, SM count, arithmetic) next to the reference's fields.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time
from typing import Optional

import numpy as np

from . import solver as S
from .instances import ParseError, entries_from_dense, instance_from_json, instance_to_json, parse_gset

VERSION = "0.1.0"
ARITHMETIC = "fp32 state; exact integer fields (int8 tensor cores, s32 accumulate)"


class UsageError(Exception):
    pass


# --------------------------------------------------------------------------- options

def add_instance_options(p):  # sbopt.cpp:63-70
    p.add_argument("instance", nargs="?", default="", help="instance file (G-set text or JSON, sniffed)")
    p.add_argument("--gset", default="", help="G-set graph file")
    p.add_argument("--json", default="", help="JSON instance file")
    p.add_argument("--dense", type=int, default=0, help="generate a random dense +-1 instance of this size")
    p.add_argument("--dense-seed", type=int, default=1, help="seed for --dense [1]")


def add_solver_options(p):  # sbopt.cpp:71-86
    p.add_argument("--variant", default="gbsb", choices=["bsb", "dsb", "gbsb", "gdsb"],
                   help="bsb | dsb | gbsb | gdsb [gbsb]")
    p.add_argument("--A", type=float, default=0.2, help="nonlinear-control strength A [0.2]")
    p.add_argument("--M", type=int, default=1000, help="number of time-evolution steps M [1000]")
    p.add_argument("--Dt", type=float, default=1.25, help="time-step factor D_t [1.25]")
    p.add_argument("--dt", type=float, default=None, help="explicit time step (skips dt tuning)")
    p.add_argument("--c", type=float, default=None, help="explicit coupling scale (skips c tuning)")
    p.add_argument("--tune", default="numerical", choices=["wigner", "numerical"], help="wigner | numerical")
    p.add_argument("--seed", type=int, default=0, help="master seed [0]")
    p.add_argument("--sample-stride", type=int, default=0, help="trajectory sampling stride (0 = final only)")
    p.add_argument("--workers", type=int, default=0, help="accepted for compatibility (the GPU runs all replicas)")
    p.add_argument("--device", default="gpu", choices=["gpu"], help="execution device [gpu]")
    p.add_argument("--gpu", type=int, default=0, help="CUDA device index [0]")


class Problem:
    def __init__(self, label: str, n: int, graph=None):
        self.label, self.n, self.graph = label, n, graph


def read_file(path: str) -> str:  # sbopt.cpp:88-97
    if not os.path.exists(path):
        raise UsageError(f"no such file: {path}")
    try:
        with open(path, "rb") as f:
            return f.read().decode()
    except OSError:
        raise UsageError(f"cannot open {path}") from None


def looks_like_json(text: str) -> bool:
    s = text.lstrip(" \t\r\n")
    return s.startswith("{")


def load_problem(solver, a) -> Problem:  # sbopt.cpp:104-131, straight to the device
    sources = int(bool(a.instance)) + int(bool(a.gset)) + int(bool(a.json)) + int(a.dense > 0)
    if sources == 0:
        raise UsageError("no instance given (positional path, --gset, --json or --dense)")
    if sources > 1:
        raise UsageError("give exactly one instance source")
    if a.dense > 0:
        if a.dense < 2:
            raise ValueError("random dense instance needs n >= 2")
        solver.gen_random_dense(a.dense, a.dense_seed)
        return Problem(f"dense-n{a.dense}-s{a.dense_seed}", a.dense)
    text = read_file(a.json or a.gset or a.instance)
    if a.json or (a.instance and looks_like_json(text)):
        e = instance_from_json(text)
        solver.set_instance_entries(e)
        solver.total_weight = None  # a JSON instance carries no graph (cut = null)
        return Problem(e.label, e.n)
    g = parse_gset(text)
    solver.set_graph(g)
    return Problem("maxcut", g.n, g)


def make_config(a) -> S.SolverConfig:  # sbopt.cpp:139-149
    return S.SolverConfig(variant=S.Variant[a.variant], steps=a.M, dt=a.dt, c=a.c, a=a.A, seed=a.seed,
                          sample_stride=a.sample_stride)


def make_tuning(solver, a) -> S.TuningResult:  # sbopt.cpp:151-166
    if a.dt is not None and a.c is not None:
        return S.TuningResult(c=a.c, dt=a.dt, d_t_factor=0.0, lambda_max=math.nan, lambda_min=math.nan,
                              method="wigner")
    return solver.auto_tune(a.tune, a.Dt)


def write_output(path: str, text: str) -> None:  # sbopt.cpp:168-176
    if not path or path == "-":
        sys.stdout.write(text + "\n")
        sys.stdout.flush()
        return
    try:
        with open(path, "w") as f:
            f.write(text + "\n")
    except OSError:
        raise UsageError(f"cannot write {path}") from None


def parse_grid(spec: str):  # sbopt.cpp:179-203
    values = []
    if ":" in spec:
        parts = spec.split(":")
        try:
            if len(parts) != 3:
                raise ValueError
            lo, hi, step = (float(x) for x in parts)
        except ValueError:
            raise UsageError(f"bad grid spec '{spec}' (want lo:hi:step)") from None
        if not step > 0.0:
            raise UsageError(f"bad grid spec '{spec}' (want lo:hi:step)")
        v = lo
        while v <= hi + step * 0.5:
            values.append(0.0 if abs(v) < step * 1e-9 else v)
            v += step
    else:
        for tok in spec.split(","):
            if tok:
                try:
                    values.append(float(tok))
                except ValueError:
                    raise UsageError(f"bad grid value '{tok}'") from None
    if not values:
        raise UsageError(f"empty grid spec '{spec}'")
    return values


def parse_int_grid(spec: str):  # sbopt.cpp:205-213
    out = []
    for v in parse_grid(spec):
        i = int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))
        if i < 1:
            raise UsageError(f"grid values must be >= 1 in '{spec}'")
        out.append(i)
    return out


def resolve_energy_target(problem: Problem, target_energy, target_cut) -> float:  # sbopt.cpp:215-224
    if target_energy is not None and target_cut is not None:
        raise UsageError("give one of --target-energy/--target-cut")
    if target_energy is not None:
        return float(target_energy)
    if target_cut is None:
        raise UsageError("a target is required (--target-energy or --target-cut)")
    if problem.graph is None:
        raise UsageError("--target-cut needs a graph instance (G-set)")
    return float(problem.graph.total_weight()) - 2.0 * target_cut


def _num(x):
    return None if isinstance(x, float) and not math.isfinite(x) else x


def device_json(solver) -> dict:
    return {"kind": "gpu", "name": solver.device_name, "sms": solver.sm_count, "arithmetic": ARITHMETIC}


def config_json(cfg: S.SolverConfig) -> dict:  # engine.cpp:187-198
    return {"variant": cfg.variant.name, "M": int(cfg.steps), "dt": _num(cfg.dt), "c": _num(cfg.c), "A": cfg.a,
            "seed": int(cfg.seed), "init_mode": cfg.init_mode.name, "sample_stride": int(cfg.sample_stride)}


def tuning_json(t: S.TuningResult) -> dict:  # engine.cpp:200-209
    j = {"c": t.c, "dt": t.dt, "D_t": t.d_t_factor, "method": t.method}
    if math.isfinite(t.lambda_max):
        j["lambda_max"] = t.lambda_max
    if math.isfinite(t.lambda_min):
        j["lambda_min"] = t.lambda_min
    return j


def rle_encode(spins):  # engine.cpp rle_encode: runs of equal values
    runs = []
    for v in spins.tolist():
        if runs and runs[-1][0] == v:
            runs[-1][1] += 1
        else:
            runs.append([v, 1])
    return runs


def run_manifest_json(res: S.RunResult, label: str, rle: bool, solver) -> str:  # engine.cpp:213-235
    doc = {"tool": "sbopt", "instance": {"label": label, "n": int(len(res.final_spins))},
           "config": config_json(res.config_echo), "tuning": tuning_json(res.tuning_echo), "energy": res.energy,
           "cut": res.cut, "wall_time_s": res.wall_time_s, "device": device_json(solver)}
    if rle:
        doc["spins_rle"] = rle_encode(res.final_spins)
    else:
        doc["spins"] = [int(v) for v in res.final_spins]
    return json.dumps(doc, sort_keys=True, separators=(",", ":"))


# -------------------------------------------------------------------------- commands

def cmd_solve(solver, a) -> int:  # sbopt.cpp:228-246
    problem = load_problem(solver, a)
    tuning = make_tuning(solver, a)
    cfg = make_config(a)
    if a.batch > 1:
        res = solver.batch_best_of(cfg, tuning, a.batch, a.seed)
    else:
        res = solver.run(cfg, tuning)
    if problem.graph is None:
        res.cut = None
    write_output(a.out, run_manifest_json(res, problem.label, a.rle_spins, solver))
    return 0


def cmd_bench(solver, a) -> int:  # sbopt.cpp:248-310; all reps x batch replicas in one launch
    problem = load_problem(solver, a)
    target = resolve_energy_target(problem, a.target_energy, a.target_cut)
    tuning = make_tuning(solver, a)
    cfg = S.resolve_config(make_config(a), tuning)
    reps, batch = a.reps, a.batch
    if reps < 1:
        raise ValueError("success probability needs n_rep >= 1")
    rep_seeds = [S._derive_seed(a.seed, [S.SEED_STREAM_BENCH, r]) for r in range(reps)]
    if batch > 1:
        seeds = [S._derive_seed(rs, [S.SEED_STREAM_BATCH, b]) for rs in rep_seeds for b in range(batch)]
    else:
        seeds = rep_seeds
    t0 = time.perf_counter()
    solver.init_state_seeds(np.array(seeds, np.uint64), cfg.init_mode)
    solver.advance(cfg, 0, int(cfg.steps))
    _, e, _, _ = solver.readout()
    t_batch = time.perf_counter() - t0
    energies = e.reshape(reps, batch).min(axis=1)
    stats = S.success_probability(energies, target)
    t_com = t_batch / reps  # amortised machine time per repetition
    doc = {"tool": "sbopt", "instance": problem.label, "reps": reps, "batch": batch, "seed": a.seed,
           "target_energy": target, "p_s": stats.p_s, "delta_p_s": stats.delta_p_s, "hits": stats.hit_count,
           "t_com_s": t_com, "t_batch_s": t_batch, "best_energy": float(energies.min()),
           "mean_energy": float(energies.mean()),
           "config": {"variant": a.variant, "M": a.M, "A": a.A, "dt": tuning.dt if a.dt is None else a.dt,
                      "c": tuning.c if a.c is None else a.c, "D_t": tuning.d_t_factor},
           "device": device_json(solver)}
    if stats.p_s > 0.0:
        tts = S.time_to_solution(t_com, stats)
        doc["tts_s"], doc["delta_tts_s"] = tts.tts_s, tts.delta_tts_s
    else:
        doc["tts_s"], doc["delta_tts_s"] = None, None
    write_output(a.out, json.dumps(doc, sort_keys=True, indent=2))
    return 0


SWEEP_HEADER = "m,a,reps,hits,p_s,delta_p_s,mean_energy,best_energy"  # bench.cpp:271-273
DT_SWEEP_HEADER = "d_t,t_final,dt,m,reps,hits,p_s,delta_p_s,mean_energy,best_energy"


def _g(x) -> str:  # printf("%.10g")
    return "%.10g" % x


def sweep_csv_row(c) -> str:
    return ",".join([str(c.m_steps), _g(c.a), str(c.stats.n_rep), str(c.stats.hit_count), _g(c.stats.p_s),
                     _g(c.stats.delta_p_s), _g(c.mean_energy), _g(c.best_energy)])


def dt_sweep_csv_row(c) -> str:
    return ",".join([_g(c.d_t_factor), _g(c.t_final), _g(c.dt), str(c.m_steps), str(c.stats.n_rep),
                     str(c.stats.hit_count), _g(c.stats.p_s), _g(c.stats.delta_p_s), _g(c.mean_energy),
                     _g(c.best_energy)])


def _stats_json(st) -> dict:
    return {"p_s": st.p_s, "delta_p_s": st.delta_p_s, "n_rep": st.n_rep, "hits": st.hit_count, "target": st.target_value}


def _base_config_json(cfg: S.SolverConfig) -> dict:
    return {"variant": cfg.variant.name, "dt": _num(cfg.dt), "c": _num(cfg.c), "seed": int(cfg.seed),
            "init_mode": cfg.init_mode.name}


def read_done_keys(path: str, header: str):  # sbopt.cpp:334-352
    keys = []
    if not os.path.exists(path):
        return keys
    with open(path) as f:
        lines = f.read().split("\n")
    if not lines or lines[0] != header:
        raise UsageError(f"existing output {path} does not match the expected CSV schema")
    for line in lines[1:]:
        if line:
            parts = line.split(",")
            if len(parts) >= 2:
                keys.append((float(parts[0]), float(parts[1])))
    return keys


def cmd_sweep(solver, a) -> int:  # sbopt.cpp:354-421
    dt_mode = bool(a.Dt_grid) or bool(a.tM_grid)
    if dt_mode and (not a.Dt_grid or not a.tM_grid):
        raise UsageError("dt-sweep mode needs both --Dt-grid and --tM-grid")
    if not dt_mode and (not a.M_grid or not a.A_grid):
        raise UsageError("sweep needs --M-grid and --A-grid (or --Dt-grid/--tM-grid)")
    if not a.out:
        raise UsageError("sweep needs --out CSV path")
    problem = load_problem(solver, a)
    target = resolve_energy_target(problem, a.target_energy, a.target_cut)
    tuning = make_tuning(solver, a)
    base = make_config(a)
    header = DT_SWEEP_HEADER if dt_mode else SWEEP_HEADER
    done = read_done_keys(a.out, header) if a.resume and os.path.exists(a.out) else []

    def is_done(k1, k2):
        return any(abs(p - k1) < 1e-9 and abs(q - k2) < 1e-9 for p, q in done)

    fresh = not a.resume or not os.path.exists(a.out)
    try:
        out = open(a.out, "w" if fresh else "a")
    except OSError:
        raise UsageError(f"cannot write {a.out}") from None
    with out:
        if fresh:
            out.write(header + "\n")
        if dt_mode:
            cells = S.dt_sweep(solver, parse_grid(a.Dt_grid), parse_grid(a.tM_grid), a.A, a.reps, base, tuning, target)
            for c in cells:
                if not is_done(c.d_t_factor, c.t_final):
                    out.write(dt_sweep_csv_row(c) + "\n")
                    print(f"sweep: D_t={c.d_t_factor:g} t_M={c.t_final:g} p_s={c.stats.p_s:g}", file=sys.stderr)
            summary = {"instance": problem.label, "axis_d_t": parse_grid(a.Dt_grid),
                       "axis_t_final": parse_grid(a.tM_grid), "reps": a.reps, "target": target,
                       "cells": [{"d_t": c.d_t_factor, "t_final": c.t_final, "dt": c.dt, "m": c.m_steps,
                                  "stats": _stats_json(c.stats), "mean_energy": c.mean_energy,
                                  "best_energy": c.best_energy} for c in cells]}
        else:
            m_grid, a_grid = parse_int_grid(a.M_grid), parse_grid(a.A_grid)
            cells = [c for c in S.sweep(solver, m_grid, a_grid, a.reps, base, tuning, target)
                     if not is_done(float(c.m_steps), c.a)]
            for c in cells:
                out.write(sweep_csv_row(c) + "\n")
                print(f"sweep: M={c.m_steps} A={c.a:g} p_s={c.stats.p_s:g}", file=sys.stderr)
            summary = {"instance": problem.label, "axis_m": m_grid, "axis_a": a_grid, "reps": a.reps,
                       "target": target,
                       "cells": [{"m": c.m_steps, "a": c.a, "stats": _stats_json(c.stats),
                                  "mean_energy": c.mean_energy, "best_energy": c.best_energy} for c in cells]}
    summary["config"] = _base_config_json(base)
    summary["environment"] = {"workers": 0, "arithmetic": ARITHMETIC, "tool": "sbopt", "device": device_json(solver)}
    write_output(a.summary or a.out + ".json", json.dumps(summary, sort_keys=True, indent=2))
    return 0


def cmd_chaos(solver, a) -> int:  # sbopt.cpp:423-440
    problem = load_problem(solver, a)
    del problem
    tuning = make_tuning(solver, a)
    base = make_config(a)
    rows = S.chaos_scan(solver, parse_grid(a.A_grid), a.reps, base, tuning)
    lines = ["a,mean_final_delta,stderr,reps,seed"]
    lines += [",".join([_g(r.a), _g(r.mean_final_delta), _g(r.std_error), str(r.reps), str(r.seed)]) for r in rows]
    write_output(a.out, "\n".join(lines))
    return 0


def cmd_cycles(a) -> int:  # sbopt.cpp:442-450 over bench.cpp:94-121 (FPGA cycle model)
    n, pr, pc, pb = a.n, a.pr, a.pc, a.pb
    if n < 1 or pr < 1 or pc < 1 or pb < 1:
        raise ValueError("counts must be >= 1")
    mac = pr * pc * pb
    if (n * n) % mac:
        raise ValueError(f"N^2 = {n * n} is not divisible by P_r*P_c*P_b = {mac}")
    if (pb * pr) % pc:
        raise ValueError(f"P_b*P_r = {pb * pr} is not divisible by P_c = {pc}")
    n_cyc = (n * n) // mac + (pb * pr) // pc + a.latency
    print(n_cyc)
    if a.fsys is not None:
        if not a.fsys > 0.0:
            raise ValueError("clock frequency must be positive")
        print(f"step_time_us {n_cyc / a.fsys * 1e6:g}")
    return 0


def cmd_gen(solver, a) -> int:  # sbopt.cpp:452-458, generated on the device
    if a.n < 2:
        raise ValueError("random dense instance needs n >= 2")
    solver.gen_random_dense(a.n, a.seed)
    J = solver.get_couplings()
    label = a.label or f"dense-n{a.n}-s{a.seed}"
    write_output(a.out, instance_to_json(entries_from_dense(J, label)))
    return 0


def build_parser() -> argparse.ArgumentParser:
    app = argparse.ArgumentParser(prog="sbopt", description="simulated-bifurcation Ising/MAX-CUT solver "
                                  "and benchmark harness (GPU)")
    app.add_argument("--version", action="version", version=f"sbopt {VERSION} (sm_100a)")
    sub = app.add_subparsers(dest="cmd", required=True)
    solve = sub.add_parser("solve", help="run the solver once (or batch best-of)")
    add_instance_options(solve)
    add_solver_options(solve)
    solve.add_argument("--batch", type=int, default=1, help="replicas per solve, best energy wins [1]")
    solve.add_argument("--rle-spins", action="store_true", help="run-length encode spins in the manifest")
    solve.add_argument("--out", default="", help="output path (default stdout)")
    bench = sub.add_parser("bench", help="success probability and time-to-solution")
    add_instance_options(bench)
    add_solver_options(bench)
    bench.add_argument("--reps", type=int, default=100, help="repetitions for estimating P_S [100]")
    bench.add_argument("--batch", type=int, default=1, help="batch size per repetition [1]")
    bench.add_argument("--target-energy", type=float, default=None, help="hit when energy <= this")
    bench.add_argument("--target-cut", type=float, default=None, help="hit when cut >= this (graph instances)")
    bench.add_argument("--out", default="", help="output path (default stdout)")
    sweep = sub.add_parser("sweep", help="(M, A) or (D_t, t_M) success-probability grid")
    add_instance_options(sweep)
    add_solver_options(sweep)
    sweep.add_argument("--M-grid", dest="M_grid", default="", help="M values, 'lo:hi:step' or comma list")
    sweep.add_argument("--A-grid", dest="A_grid", default="", help="A values, 'lo:hi:step' or comma list")
    sweep.add_argument("--Dt-grid", dest="Dt_grid", default="", help="D_t values (dt-sweep mode)")
    sweep.add_argument("--tM-grid", dest="tM_grid", default="", help="t_M values (dt-sweep mode)")
    sweep.add_argument("--reps", type=int, default=100, help="repetitions per cell [100]")
    sweep.add_argument("--target-energy", type=float, default=None)
    sweep.add_argument("--target-cut", type=float, default=None)
    sweep.add_argument("--out", default="", help="CSV output path")
    sweep.add_argument("--summary", default="", help="JSON summary path [<out>.json]")
    sweep.add_argument("--resume", action="store_true", help="skip cells already present in --out")
    chaos = sub.add_parser("chaos", help="paired-trajectory divergence scan over A")
    add_instance_options(chaos)
    add_solver_options(chaos)
    chaos.add_argument("--A-grid", dest="A_grid", default="0:1:0.05", help="A values [0:1:0.05]")
    chaos.add_argument("--reps", type=int, default=100, help="paired runs per A value [100]")
    chaos.add_argument("--out", default="", help="CSV output path (default stdout)")
    cycles = sub.add_parser("cycles", help="clock cycles per time-evolution step")
    for k in ("n", "pr", "pc", "pb", "latency"):
        cycles.add_argument(f"--{k}", type=int, required=True)
    cycles.add_argument("--fsys", type=float, default=None)
    gen = sub.add_parser("gen", help="generate a random dense +-1 instance (JSON)")
    gen.add_argument("--n", type=int, required=True, help="spin count")
    gen.add_argument("--seed", type=int, default=1, help="generator seed [1]")
    gen.add_argument("--label", default="", help="instance label")
    gen.add_argument("--out", default="", help="output path (default stdout)")
    gen.add_argument("--gpu", type=int, default=0)
    return app


def main(argv: Optional[list] = None) -> int:  # sbopt.cpp:461-557
    app = build_parser()
    try:
        a = app.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    try:
        if a.cmd == "cycles":
            return cmd_cycles(a)
        if a.cmd != "gen":  # argument-only checks before touching the device
            sources = int(bool(a.instance)) + int(bool(a.gset)) + int(bool(a.json)) + int(a.dense > 0)
            if sources == 0:
                raise UsageError("no instance given (positional path, --gset, --json or --dense)")
            if sources > 1:
                raise UsageError("give exactly one instance source")
            for path in (a.instance, a.gset, a.json):
                if path and not os.path.exists(path):
                    raise UsageError(f"no such file: {path}")
        with S.Solver(getattr(a, "gpu", 0)) as solver:
            return {"solve": cmd_solve, "bench": cmd_bench, "sweep": cmd_sweep, "chaos": cmd_chaos,
                    "gen": cmd_gen}[a.cmd](solver, a)
    except (UsageError, ParseError, ValueError) as e:
        print(f"sbopt: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # runtime errors (device, convergence, IO)
        print(f"sbopt: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
