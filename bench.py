"""bench.py — GSB spin-updates/s on the BASELINE workload (configs[1], "C2").

Workload (BASELINE.json configs[1]): N=2000 dense +-1 MAX-CUT instance
(gen_random_dense draw order, seed 1), GdSB (sign-discretised field, per-spin
nonlinear control A=0.2), dt=1.25, c=1/(2 sqrt N) (Wigner), M=1000 schedule,
R=8192 replicas in total sharded over the ranks (replica r keeps its global
index and seed), x0,y0 ~ U(-0.1,0.1) fp32 from derive_seed(1, {7, r}).
A "step" = one GSB time step of every replica = one launch of the tcgen05
step kernel. value = N * R * steps / device time (max over ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU implementation
(oracle/_ref: the unmodified sbopt core, cmd_bench's replica fan-out over a
ThreadPool with all host threads) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_SPINS = 2000
R_TOTAL = 8192
M_SCHED = 1000
A_CTRL = 0.2
DT = 1.25
INSTANCE_SEED = 1
MASTER = 1
INIT_TAG = 7
L2_BYTES = 126 * 1024 * 1024
METRIC = "GSB spin-updates/s (N*R*steps/s), N=2000 dense +-1 MAX-CUT, GdSB, R=8192"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_reference_sample(workers: int, budget_s: float, J64: np.ndarray, rng_states, label: str):
    """Time the reference's replica fan-out on a bounded sample; returns SU/s and description."""
    import oracle

    ref = oracle.ref("timing")
    threads = ref.effective_workers(workers)
    R_s = 2 * threads
    x0, y0 = rng_states(R_s)
    c = 1.0 / (2.0 * math.sqrt(N_SPINS))
    # calibrate: 5 steps, then size the sample to the budget
    _, w = ref.replica_fanout(1, J64, x0, y0, 5, DT, c, A_CTRL, threads)
    per_step = max(w / 5, 1e-6)
    m_s = int(max(5, min(M_SCHED, budget_s / per_step)))
    energies, wall = ref.replica_fanout(1, J64, x0, y0, m_s, DT, c, A_CTRL, threads)
    su = N_SPINS * R_s * m_s / wall
    sample = (f"{R_s} replicas x {m_s} steps of the reference dsb step() (GdSB does not exist in the reference; "
              f"same per-step cost: sign field + phases), N={N_SPINS}, {label}, {os.path.basename(ref.path)}")
    return su, threads, sample, wall


def host_states(orc, R, r0=0):
    x, y, _ = orc.init_small_uniform(N_SPINS, R, master=MASTER, tag=INIT_TAG, r0=r0)
    return x, y


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle

    oracle.build()
    orc = oracle.orc()
    J64 = orc.gen_dense_i8(N_SPINS, INSTANCE_SEED).astype(np.float64)
    total = args.steps + args.warmup
    budget = max(0.5, min(5.0, 150.0 / max(total, 1)))
    vals = []
    threads, sample, walls = 0, "", []
    for it in range(total):
        su, threads, sample, wall = cpu_reference_sample(0, budget, J64, lambda R: host_states(orc, R),
                                                         "all host threads")
        if it >= args.warmup:
            vals.append(su)
            walls.append(wall)
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "spin-updates/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(walls),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded gen_random_dense instance, BASELINE U(-0.1,0.1) init)",
        "config": {"workload": "C2: N=2000 dense +-1, R=8192 (reference timed on a bounded replica sample)",
                   "n": N_SPINS, "replicas": R_TOTAL, "M": M_SCHED, "A": A_CTRL, "dt": DT},
        "cpu_baseline": {"value": value, "unit": "spin-updates/s", "cores": threads, "kind": "reference",
                         "sample": sample, "host": oracle.host_description()},
        "e2e": {"value": value, "unit": "spin-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    rank, world, local = dist_env()
    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, TuningResult, Variant

    if R_TOTAL % world:
        raise SystemExit("R must divide evenly over the ranks")
    R = R_TOTAL // world
    r0 = rank * R
    c = 1.0 / (2.0 * math.sqrt(N_SPINS))
    cfg = SolverConfig(variant=Variant.gdsb, steps=M_SCHED, dt=DT, c=c, a=A_CTRL, init_mode=InitMode.small_uniform)
    s = Solver(local)
    s.gen_random_dense(N_SPINS, INSTANCE_SEED)
    s.init_state(R, InitMode.small_uniform, MASTER, INIT_TAG, offset=r0)
    state_bytes = 12 * N_SPINS * R
    flush = state_bytes < 1.5 * L2_BYTES  # state could largely sit in L2: flush between timed steps
    flush_buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device="cuda") if flush else None

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()

    # warm-up (also builds the B operand once)
    m = 0
    s.advance(cfg, m, m + args.warmup)
    m += args.warmup
    s.synchronize()
    launches0 = s.kernel_launches
    barrier()
    with ClockSampler(local) as clk:
        if not flush:
            s.advance(cfg, m, m + args.steps)
            dev_ms = s.last_advance_ms()
        else:
            dev_ms = 0.0
            for k in range(args.steps):
                flush_buf.zero_()
                torch.cuda.synchronize()
                s.advance(cfg, m + k, m + k + 1)
                dev_ms += s.last_advance_ms()
        s.synchronize()
    barrier()
    m += args.steps
    launches = s.kernel_launches - launches0
    if world > 1:
        t = torch.tensor([dev_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dev_ms = float(t.item())
    su_total = N_SPINS * R_TOTAL * args.steps
    value = su_total / (dev_ms / 1e3)
    ms_per_step = dev_ms / args.steps

    # ---- end to end through the public API: host (pinned) x0,y0 -> run() -> spins/energies on host
    x0h, y0h = init_host_states(local, R, r0)
    e2e_steps = args.steps
    cfg_e2e = SolverConfig(variant=Variant.gdsb, steps=e2e_steps, dt=DT, c=c, a=A_CTRL)
    tun = TuningResult(c=c, dt=DT)
    s.run_batch(cfg_e2e, tun, R, x0=x0h, y0=y0h)  # warm
    barrier()
    t0 = time.perf_counter()
    b = s.run_batch(cfg_e2e, tun, R, x0=x0h, y0=y0h)
    barrier()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_val = N_SPINS * R_TOTAL * e2e_steps / e2e_s
    h2d = 2 * 4 * N_SPINS * R  # x0, y0 fp32
    d2h = N_SPINS * R + 8 * R + 8  # spins int8 + energies + best index

    if rank != 0:
        s.close()
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (the step kernel; one launch per step)
    hbm_peak, peak_src = peaks()
    bytes_per_launch = 24 * N_SPINS * R + N_SPINS * N_SPINS  # 24 B/SU state + J (int8) once
    achieved = bytes_per_launch / (ms_per_step / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "step_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"R{R}")
        except Exception:
            traffic = None
    ops_per_launch = 2 * N_SPINS * N_SPINS * R

    line = {
        "metric": METRIC, "value": value, "unit": "spin-updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "i8 field (tcgen05 kind::i8, s32 acc) / f32 state",
        "data": "synthetic (seeded gen_random_dense N=2000 instance; x0,y0~U(-0.1,0.1) from derive_seed(1,{7,r}))",
        "config": {"workload": "C2 (BASELINE configs[1]): N=2000 dense +-1, GdSB, R=8192 sharded over ranks",
                   "n": N_SPINS, "replicas": R_TOTAL, "replicas_per_gpu": R, "M": M_SCHED, "A": A_CTRL,
                   "dt": DT, "c": c, "parallelism": f"replicas/{world}",
                   "l2": ("flushed (256 MB write) between timed steps" if flush else
                          f"state {state_bytes / 2**20:.0f} MB per GPU > 126 MB L2 (inputs larger than L2)")},
        "e2e": {"value": e2e_val, "unit": "spin-updates/s", "h2d_bytes_per_step": h2d / e2e_steps,
                "d2h_bytes_per_step": d2h / e2e_steps,
                "note": f"one run() of M={e2e_steps} steps per call: H2D x0,y0 from pinned host, M steps, "
                        "readout (energy+argmin), D2H spins/energies; wall clock, max over ranks",
                "device_breakdown_ms": b.timing},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bytes_per_launch,
                     "tensor_tops": ops_per_launch / (ms_per_step / 1e3) / 1e12},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        import oracle

        oracle.build()
        orc = oracle.orc()
        J64 = orc.gen_dense_i8(N_SPINS, INSTANCE_SEED).astype(np.float64)
        su, threads, sample, _ = cpu_reference_sample(0, 20.0, J64, lambda RR: host_states(orc, RR),
                                                      "all host threads")
        line["cpu_baseline"] = {"value": su, "unit": "spin-updates/s", "cores": threads, "kind": "reference",
                                "sample": sample, "host": oracle.host_description()}
    print(json.dumps(line), flush=True)
    s.close()


def init_host_states(device: int, R: int, r0: int):
    """Initial states in pinned host memory (generated on the GPU, copied once, outside timing)."""
    import torch

    from paper_2508_17655_b200 import InitMode, Solver

    with Solver(device) as t:
        t.gen_random_dense(N_SPINS, INSTANCE_SEED)
        t.init_state(R, InitMode.small_uniform, MASTER, INIT_TAG, offset=r0)
        x, y, _ = t.get_state()
    xp = torch.empty((R, N_SPINS), dtype=torch.float32, pin_memory=True)
    yp = torch.empty((R, N_SPINS), dtype=torch.float32, pin_memory=True)
    xp.numpy()[:] = x
    yp.numpy()[:] = y
    return xp.numpy(), yp.numpy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    global M_SCHED
    M_SCHED = max(M_SCHED, args.warmup + args.steps)  # per-step cost does not depend on M
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
