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
R_PER_GPU = 8192
TTS_POOL = 8
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


DTYPES = {"e2m1": "e2m1 operands (tcgen05 kind::mxf4, unit E8M0 scales, f32 acc: exact integer field) / f32 state",
          "int8": "i8 operands (tcgen05 kind::i8, s32 acc) / f32 state"}
KERNELS = {"e2m1": "gsb_resident_parts_kernel<3,true,4> (four interleaved column-part chains per 160-replica block, "
                   "J resident in shared memory, one 3D TMA load of G per part-step, p in registers)",
           "int8": "gsb_resident_pair_kernel<5,16,4,160,false>"}


def tensor_peak(fmt):
    """Dense tensor peak of the pipe the resident kernel multiplies on, measured on this pool's
    B200 as SURVEY 8(d) asks: e2m1 -> tools/fp4_peak.py (cuBLASLt FP4 GEMM 8192^3, burst),
    int8 -> tools/int8_peak.py (cuBLASLt int8 GEMM 8192^3, burst); the datasheet dense
    figure (9000 / 4500 TOPS) if the measurement file is missing."""
    name, key, nominal = ("fp4_peak.json", "fp4_tops_burst", 9000.0) if fmt == "e2m1" else \
        ("int8_peak.json", "int8_tops_burst", 4500.0)
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return float(json.load(f)[key]), f"measured (profiles/{name}, cuBLASLt 8192^3 burst)"
    except Exception:
        return nominal, f"nominal (datasheet dense {fmt})"


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
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded gen_random_dense instance, BASELINE U(-0.1,0.1) init)",
        "config": {"workload": "C2 (BASELINE configs[1]): N=2000 dense +-1, GdSB, R=8192 replicas per GPU "
                               "(reference timed on a bounded replica sample on rank 0's host)",
                   "n": N_SPINS, "replicas_per_gpu": R_PER_GPU, "M": M_SCHED, "A": A_CTRL, "dt": DT},
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

    # Weak scaling over replicas: every rank owns R_PER_GPU whole
    # replicas with global indices rank*R .. rank*R+R-1 (seeds do not depend on
    # the rank count); no data-path collective.
    R = R_PER_GPU
    r0 = rank * R
    R_all = R * world
    c = 1.0 / (2.0 * math.sqrt(N_SPINS))
    cfg = SolverConfig(variant=Variant.gdsb, steps=M_SCHED, dt=DT, c=c, a=A_CTRL, init_mode=InitMode.small_uniform)
    s = Solver(local)
    s.gen_random_dense(N_SPINS, INSTANCE_SEED)
    fmt = s.operand_format  # e2m1 for +-1 J: the resident kernel runs kind::mxf4 MMAs
    s.init_state(R, InitMode.small_uniform, MASTER, INIT_TAG, offset=r0)
    state_bytes = 12 * N_SPINS * R
    assert state_bytes > L2_BYTES, "per-GPU state must exceed L2 (timing protocol)"

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()

    # warm-up steps (own launch; also builds the B operand once)
    s.advance(cfg, 0, args.warmup)
    s.synchronize()
    launches0 = s.kernel_launches
    barrier()
    with ClockSampler(local) as clk:
        s.advance(cfg, args.warmup, args.warmup + args.steps)  # K steps, persistent multi-step kernel
        dev_ms = s.last_advance_ms()
        s.synchronize()
    barrier()
    launches = s.kernel_launches - launches0
    if world > 1:
        t = torch.tensor([dev_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dev_ms = float(t.item())
    su_total = N_SPINS * R_all * args.steps
    value = su_total / (dev_ms / 1e3)
    ms_per_step = dev_ms / args.steps

    # ---- end to end through the public API: pinned host x0,y0 -> run() -> spins/energies on host
    x0h, y0h = init_host_states(local, R, r0)
    e2e_steps = M_SCHED  # one whole run of the C2 schedule (M = 1000), as the reference's run() does
    cfg_e2e = SolverConfig(variant=Variant.gdsb, steps=e2e_steps, dt=DT, c=c, a=A_CTRL)
    tun = TuningResult(c=c, dt=DT)
    s.run_batch(cfg_e2e, tun, R, x0=x0h, y0=y0h, want_spins=False)  # warm
    barrier()
    t0 = time.perf_counter()
    b = s.run_batch(cfg_e2e, tun, R, x0=x0h, y0=y0h, want_spins=False)
    barrier()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_val = N_SPINS * R_all * e2e_steps / e2e_s
    h2d = 2 * 4 * N_SPINS * R  # x0, y0 fp32
    d2h = 8 * R + 8  # per-replica energies + best index (batch_best_of result)

    tts = None
    if world == 1 and not args.no_tts:
        tts = measure_tts(s, local)

    if rank != 0:
        s.close()
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    # ---- roofline of the dominant (only) kernel of the timed region: gsb_resident_pair_kernel
    # keeps x, y, p in TMEM for the whole launch, so the 24 B/SU state stream of the
    # streaming formulation never reaches HBM; "if the kernel keeps state on-chip
    # across steps and beats the HBM term, report the tensor-only fraction and say so".
    hbm_peak, hbm_src = peaks()
    t_peak, t_src = tensor_peak(fmt)
    ops_per_step = 2 * N_SPINS * N_SPINS * R  # 2N ops per spin-update
    tops = ops_per_step / (ms_per_step / 1e3) / 1e12
    stream_bytes = 24 * N_SPINS * R + N_SPINS * N_SPINS  # the streaming formulation's HBM bytes per step
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "step_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"resident_gdsb_n2000_R8192_{fmt}_dram_bytes_per_step")
        except Exception:
            traffic = None

    line = {
        "metric": METRIC, "value": value, "unit": "spin-updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": DTYPES[fmt],
        "data": "synthetic (seeded gen_random_dense N=2000 instance; x0,y0~U(-0.1,0.1) from derive_seed(1,{7,r}))",
        "config": {"workload": "C2 (BASELINE configs[1]): N=2000 dense +-1, GdSB, R=8192 replicas per GPU",
                   "n": N_SPINS, "replicas_per_gpu": R, "replicas_total": R_all, "M": M_SCHED, "A": A_CTRL,
                   "dt": DT, "c": c, "parallelism": f"replica-sharded x{world} (no collective)",
                   "timed": f"{args.steps} steps in one persistent multi-step launch, CUDA events, max over ranks",
                   "l2": f"inputs larger than L2: state {state_bytes / 2**20:.0f} MiB per GPU > 126 MB L2"},
        "e2e": {"value": e2e_val, "unit": "spin-updates/s", "h2d_bytes_per_step": h2d / e2e_steps,
                "d2h_bytes_per_step": d2h / e2e_steps,
                "note": f"one sbg_run() of M={e2e_steps} steps per rank: H2D x0,y0 from pinned host, M steps, "
                        "readout (energy+argmin), D2H energies+best index; wall clock, max over ranks",
                "device_breakdown_ms": b.timing},
        "roofline": {"bound": "tensor", "achieved": tops, "peak": t_peak, "unit": "TFLOP/s",
                     "frac": tops / t_peak, "traffic": traffic, "peak_source": t_src,
                     "op_type": f"{fmt} tensor ops (2 per MAC), 2*N*N*R per step",
                     "kernel": KERNELS[fmt] + "; all timed steps in one launch, x, y in TMEM",
                     "streaming_equivalent": {"bytes_per_step": stream_bytes,
                                              "gbs": stream_bytes / (ms_per_step / 1e3) / 1e9,
                                              "hbm_peak_gbs": hbm_peak, "hbm_peak_source": hbm_src,
                                              "note": "the 24 B/SU state stream a non-resident kernel must move; "
                                                      "above the HBM peak = faster than any streaming design"}},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if tts is not None:
        line["tts99"] = tts["gbsb"]
        line["tts99_gdsb"] = tts["gdsb"]
        line["tts99_common_target"] = tts["common_target"]
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


def measure_tts(s, device, variants=("gbsb", "gdsb")):
    """TTS99 on the N=2000 dense +-1 instance, paper K2000 settings:
    GbSB and GdSB, M=21500, A=0.2, dt=1.25, c=1/(2 sqrt N), R=1000 replicas per batch (C1
    shape), reference init (x~U(-1,1), y=0; batch_best_of seeds). Per variant the target is
    the best energy over TTS_POOL of its own batches (the K2000 file is absent);
    P_S from a fresh batch; TTS via the reference's time_to_solution (bench.cpp:52-68). The
    fresh batches are also scored against the best target over all variants."""
    from paper_2508_17655_b200 import (InitMode, SolverConfig, TuningResult, Variant, success_probability,
                                       time_to_solution)

    c = 1.0 / (2.0 * math.sqrt(N_SPINS))
    tun = TuningResult(c=c, dt=DT)
    out, fresh = {}, {}
    for v in variants:
        cfg = SolverConfig(variant=Variant[v], steps=21500, dt=DT, c=c, a=A_CTRL, init_mode=InitMode.uniform_random)
        target_e = float(min(s.run_batch(cfg, tun, 1000, master_seed=1000 + k).energies.min()
                             for k in range(TTS_POOL)))
        t0 = time.perf_counter()
        b = s.run_batch(cfg, tun, 1000, master_seed=999)
        t_batch = time.perf_counter() - t0
        fresh[v] = (b.energies, t_batch)
        st = success_probability(b.energies, target_e)
        r = {"variant": v, "M": 21500, "A": A_CTRL, "replicas_per_batch": 1000, "target_energy": target_e,
             "target": f"best energy over {TTS_POOL} GPU batches x 1000 runs of this variant",
             "p_s": st.p_s, "delta_p_s": st.delta_p_s, "t_batch_s": t_batch, "device_ms_batch": b.timing["total_ms"]}
        if st.p_s > 0:
            run = time_to_solution(t_batch, st)
            amort = time_to_solution(t_batch / 1000, st)
            r.update({"tts99_run_ms": run.tts_s * 1e3, "delta_tts99_run_ms": run.delta_tts_s * 1e3,
                      "tts99_amortised_ms": amort.tts_s * 1e3})
        else:
            r["tts99_run_ms"] = None
        out[v] = r
    common = min(r["target_energy"] for r in out.values())
    out["common_target"] = {"target_energy": common,
                            "p_s": {v: success_probability(e, common).p_s for v, (e, _) in fresh.items()}}
    return out


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
    ap.add_argument("--no-tts", action="store_true")
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
