"""bench.py — GSB spin-updates/s on the BASELINE workload (configs[1], "C2").

Workload (BASELINE.json configs[1]): N=2000 dense +-1 MAX-CUT instance
(gen_random_dense draw order, seed 1), GdSB (sign-discretised field, per-spin
nonlinear control A=0.2), dt=1.25, c=1/(2 sqrt N) (Wigner), M=1000 schedule,
R=8192 replicas per GPU (weak scaling; replica r keeps its global index and seed),
x0,y0 ~ U(-0.1,0.1) fp32 from derive_seed(1, {7, r}).
A "step" = one GSB time step of every replica. value = N * R * steps / device time
(CUDA events around one persistent launch of K steps, max over ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--gpus N without torchrun re-executes itself under torch.distributed.run with N ranks
(127.0.0.1); under torchrun WORLD_SIZE must equal N. One process per GPU; replicas are
sharded with no data-path collective ("weak" scaling).

Extra keys of the N=1 line (each measured in this run):
  e2e          one sbg_run_best (the batch_best_of result) from pinned host x0, y0:
               H2D, M steps, readout, D2H of the winner's spins/energy/index + R energies;
  tts99        GbSB and GdSB at the paper's K2000 settings, P_S against the REFERENCE's
               best energy over its 1000 run() trials (tests/golden/tts_ref_gbsb.npz),
               same seeds as those trials; with the CPU reference's own P_S and TTS;
  configs      C1, C3, C4 and C5 (single GPU) of BASELINE.json: us/step, SU/s, roofline
               on SURVEY 8(d)'s algorithmic ops/bytes (and the executed plane ops), DRAM
               traffic from a committed ncu capture, and a CPU baseline each;
  cpu_baseline the reference's step() fanned out over all host threads, bounded sample.
N>1 (one rank per GPU) adds c5_row_shards: N=100000 row-sharded over the ranks, the
fused NVLink all-gather inside one multi-step launch (device-side peer-wait timeout).

--impl reference times the reference's own CPU implementation (oracle/_ref: the
unmodified sbopt core compiled from its sources; cmd_bench's replica fan-out over a
ThreadPool with all host threads) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
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
M_SCHED = 1000
A_CTRL = 0.2
DT = 1.25
INSTANCE_SEED = 1
MASTER = 1
INIT_TAG = 7
L2_BYTES = 126 * 1024 * 1024
METRIC = "GSB spin-updates/s (N*R*steps/s), N=2000 dense +-1 MAX-CUT, GdSB, R=8192"
TTS_M = 21500  # PAPER.md:463 (K2000 settings: M=21500, A=0.2, dt=1.25, c=1/(2 sqrt N))
TTS_REF = os.path.join(ROOT, "tests", "golden", "tts_ref_gbsb.npz")
TRAFFIC = os.path.join(ROOT, "profiles", "r02_traffic.json")


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(args) -> None:
    """--gpus N > 1 outside torchrun: re-execute this command with N ranks (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


DTYPES = {"e2m1": "e2m1 operands (tcgen05 kind::mxf4, unit E8M0 scales, f32 acc: exact integer field) / f32 state",
          "int8": "i8 operands (tcgen05 kind::i8, s32 acc) / f32 state"}
KERNELS = {"e2m1": "gsb_resident_ts_kernel<2,4> (four interleaved column-part chains per 160-replica block; J in TMEM "
                   "as the A operand of TS-form kind::mxf4 MMAs; x, y in shared memory, moved by TMA at group "
                   "boundaries; p in registers; one 3D TMA load of G per part-step; later groups' G_0 published "
                   "ahead by a helper warp)",
           "int8": "gsb_resident_pair_kernel<5,16,4,160,false>"}


def tensor_peak(fmt):
    """Dense tensor peak of the pipe a kernel multiplies on, measured on this pool's B200 as
    SURVEY 8(d) asks: e2m1 -> tools/fp4_peak.py (cuBLASLt FP4 GEMM 8192^3, burst), int8 ->
    tools/int8_peak.py (cuBLASLt int8 GEMM 8192^3, burst); the datasheet dense figure if the
    measurement file is missing."""
    name, key, nominal = ("fp4_peak.json", "fp4_tops_burst", 9000.0) if fmt == "e2m1" else \
        ("int8_peak.json", "int8_tops_burst", 4500.0)
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return float(json.load(f)[key]), f"measured (profiles/{name}, cuBLASLt 8192^3 burst)"
    except Exception:
        return nominal, f"nominal (datasheet dense {fmt})"


def traffic_for(key: str, steps: int):
    """DRAM bytes per launch of `steps` steps from the committed ncu captures
    (profiles/r02_traffic.json: dram__bytes_read.sum + dram__bytes_write.sum of the
    timed launch, captured at two step counts): the capture at this step count, or the
    two-point line fixed + per_step * steps through the captures, labelled as such."""
    try:
        with open(TRAFFIC) as f:
            t = json.load(f)[key]
    except Exception:
        return None
    caps = {int(k): float(v) for k, v in t["launch_bytes"].items()}
    if steps in caps:
        return {"bytes_per_launch": caps[steps], "steps": steps, "source": f"ncu capture at {steps} steps"}
    (k1, b1), (k2, b2) = sorted(caps.items())[:2]
    per = (b2 - b1) / (k2 - k1)
    fixed = b1 - per * k1
    return {"bytes_per_launch": fixed + per * steps, "steps": steps,
            "source": f"line through ncu captures at {k1} and {k2} steps (fixed {fixed:.3e} B + {per:.3e} B/step)"}


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


# ------------------------------------------------------------------ CPU (reference) legs

def cpu_fanout_sample(variant: int, J64: np.ndarray, x0: np.ndarray, y0: np.ndarray, c: float, budget_s: float,
                      m_max: int = M_SCHED):
    """The reference's replica fan-out (cmd_bench, sbopt.cpp:265-272: run/step per replica
    over a ThreadPool of all host threads, pool=nullptr inside) on len(x0) replicas,
    calibrated to ~budget_s. Returns (SU/s, threads, steps, wall)."""
    import oracle

    ref = oracle.ref("timing")
    threads = ref.effective_workers(0)
    n = J64.shape[0]
    _, w = ref.replica_fanout(variant, J64, x0, y0, 2, DT, c, A_CTRL, threads)
    per_step = max(w / 2, 1e-6)
    m_s = int(max(2, min(m_max, budget_s / per_step)))
    _, wall = ref.replica_fanout(variant, J64, x0, y0, m_s, DT, c, A_CTRL, threads)
    return n * x0.shape[0] * m_s / wall, threads, m_s, wall, os.path.basename(ref.path)


def cpu_reference_c2(budget_s: float):
    import oracle

    orc = oracle.orc()
    J64 = orc.gen_dense_i8(N_SPINS, INSTANCE_SEED).astype(np.float64)
    threads = oracle.ref("timing").effective_workers(0)
    x0, y0, _ = orc.init_small_uniform(N_SPINS, 2 * threads, master=MASTER, tag=INIT_TAG)
    su, threads, m_s, wall, lib = cpu_fanout_sample(1, J64, x0, y0, 1.0 / (2.0 * math.sqrt(N_SPINS)), budget_s)
    sample = (f"{x0.shape[0]} replicas x {m_s} steps of the reference dsb step() (GdSB does not exist in the "
              f"reference; same per-step cost: sign field + phases), N={N_SPINS}, all host threads, {lib}")
    return su, threads, sample, wall


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle

    oracle.build()
    total = args.steps + args.warmup
    budget = max(0.5, min(5.0, 150.0 / max(total, 1)))
    if os.environ.get("SBG_BENCH_REF_BUDGET"):  # tests: a shorter sample per timed step
        budget = float(os.environ["SBG_BENCH_REF_BUDGET"])
    vals = []
    threads, sample = 0, ""
    for it in range(total):
        su, threads, sample, _ = cpu_reference_c2(budget)
        if it >= args.warmup:
            vals.append(su)
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "spin-updates/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        # one step of the whole per-GPU workload (N x R spin-updates) at the measured rate
        "ms_per_step": 1e3 * N_SPINS * R_PER_GPU / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded gen_random_dense instance, BASELINE U(-0.1,0.1) init)",
        "config": {"workload": "C2 (BASELINE configs[1]): N=2000 dense +-1, GdSB, R=8192 replicas per GPU "
                               "(reference timed on a bounded replica sample on rank 0's host; each of the K timed "
                               "'steps' is one such sample, ms_per_step = N*R/value)",
                   "n": N_SPINS, "replicas_per_gpu": R_PER_GPU, "M": M_SCHED, "A": A_CTRL, "dt": DT},
        "cpu_baseline": {"value": value, "unit": "spin-updates/s", "cores": threads, "kind": "reference",
                         "sample": sample, "host": oracle.host_description()},
        "e2e": {"value": value, "unit": "spin-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm

def timed_advance(s, cfg, warmup: int, steps: int):
    """W warm-up steps in their own launch, then K steps in one persistent launch; device ms."""
    s.advance(cfg, 0, warmup)
    s.synchronize()
    s.advance(cfg, warmup, warmup + steps)
    ms = s.last_advance_ms()
    s.synchronize()
    return ms


def run_ours(args):
    rank, world, local = dist_env()
    import torch

    if torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} ranks need {world} GPUs; this box has {torch.cuda.device_count()}")
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, TuningResult, Variant

    # Weak scaling over replicas: every rank owns R_PER_GPU whole replicas with
    # global indices rank*R .. rank*R+R-1 (seeds do not depend on the rank count); no
    # data-path collective.
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

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

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
    dev_ms = max_over_ranks(dev_ms)
    su_total = N_SPINS * R_all * args.steps
    value = su_total / (dev_ms / 1e3)
    ms_per_step = dev_ms / args.steps

    # ---- end to end through the public API: pinned host x0,y0 -> sbg_run_best -> the
    # batch_best_of result (winner spins, energy, index) + all energies on the host
    x0h, y0h = init_host_states(local, R, r0)
    e2e_steps = M_SCHED  # one whole run of the C2 schedule (M = 1000), as the reference's run() does
    cfg_e2e = SolverConfig(variant=Variant.gdsb, steps=e2e_steps, dt=DT, c=c, a=A_CTRL)
    tun = TuningResult(c=c, dt=DT)
    s.run_best(cfg_e2e, tun, x0h, y0h)  # warm
    barrier()
    t0 = time.perf_counter()
    _, _, _, _, e2e_timing = s.run_best(cfg_e2e, tun, x0h, y0h)
    barrier()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e_val = N_SPINS * R_all * e2e_steps / e2e_s
    h2d = 2 * 4 * N_SPINS * R  # x0, y0 fp32
    d2h = N_SPINS + 8 + 8 + 8 * R  # winner spins (int8), energy, index + the R energies

    extra = {}
    if world == 1:
        if not args.no_tts:
            extra.update(measure_tts(s))
    else:
        extra["c5_row_shards"] = c5_leg_in_children(args, rank, world)
    s.close()

    if world == 1 and not args.no_configs:
        extra["configs"] = measure_configs(args, local)

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    # ---- roofline of the dominant (only) kernel of the timed region. The resident kernel keeps
    # x, y, p on chip for the launch, so the 24 B/SU state stream of the streaming formulation
    # never reaches HBM; "if the kernel keeps state on-chip across steps and beats
    # the HBM term, report the tensor-only fraction and say so".
    hbm_peak, hbm_src = peaks()
    t_peak, t_src = tensor_peak(fmt)
    ops_per_step = 2 * N_SPINS * N_SPINS * R  # 2N ops per spin-update
    tops = ops_per_step / (ms_per_step / 1e3) / 1e12
    stream_bytes = 24 * N_SPINS * R + N_SPINS * N_SPINS  # the streaming formulation's HBM bytes per step
    tr = traffic_for(f"c2_resident_{fmt}", args.steps)

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
                "note": f"one sbg_run_best() of M={e2e_steps} steps per rank (batch_best_of's result): H2D x0,y0 "
                        "from pinned host, M steps, readout (energies + argmin), D2H of the winner's spins, energy, "
                        "index and the R energies; wall clock, max over ranks",
                "device_breakdown_ms": e2e_timing},
        "roofline": {"bound": "tensor", "achieved": tops, "peak": t_peak, "unit": "TFLOP/s",
                     "frac": tops / t_peak,
                     "traffic": tr["bytes_per_launch"] if tr else None,
                     "traffic_source": (tr["source"] + " (bytes per launch of the timed K steps)") if tr else None,
                     "peak_source": t_src,
                     "op_type": f"{fmt} tensor ops (2 per MAC), 2*N*N*R per step",
                     "kernel": KERNELS[fmt] + "; all timed steps in one launch",
                     "streaming_equivalent": {"bytes_per_step": stream_bytes,
                                              "gbs": stream_bytes / (ms_per_step / 1e3) / 1e9,
                                              "hbm_peak_gbs": hbm_peak, "hbm_peak_source": hbm_src,
                                              "note": "the 24 B/SU state stream a non-resident kernel must move; "
                                                      "above the HBM peak = faster than any streaming design"}},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    line.update(extra)
    if world == 1 and not args.no_cpu_baseline:
        import oracle

        oracle.build()
        su, threads, sample, _ = cpu_reference_c2(20.0)
        line["cpu_baseline"] = {"value": su, "unit": "spin-updates/s", "cores": threads, "kind": "reference",
                                "sample": sample, "host": oracle.host_description()}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


# ------------------------------------------------------------------ TTS99

def measure_tts(s):
    """TTS99 on the N=2000 dense +-1 instance at the paper's K2000 settings
    (M=21500, A=0.2, dt=1.25, c=1/(2 sqrt N)), reference init
    (x ~ U(-1,1), y = 0) with batch_best_of's seeds derive_seed(1, {3, r}), r < 1000
    (bench.cpp:77-82) -- the SAME 1000 trials the reference ran for the fixture
    tests/golden/tts_ref_gbsb.npz (oracle/_ref run(), make_tts_ref.py). Target = the
    reference's best energy over those trials (north star: "the best cut found by the
    reference over long runs"). P_S, TTS via success_probability / time_to_solution
    (bench.cpp:15-68); T_com of a GPU run = the wall time of its 1000-run batch."""
    from paper_2508_17655_b200 import (InitMode, SolverConfig, TuningResult, Variant, success_probability,
                                       time_to_solution)

    out = {}
    if not os.path.exists(TTS_REF):
        return {"tts99": {"unavailable": f"missing {os.path.relpath(TTS_REF, ROOT)}"}}
    ref = np.load(TTS_REF)
    e_ref = ref["energies"]
    e_ref = e_ref[~np.isnan(e_ref)]
    target = float(e_ref.min())
    n_trials = int(e_ref.size)
    c = 1.0 / (2.0 * math.sqrt(N_SPINS))
    tun = TuningResult(c=c, dt=DT)
    for v in ("gbsb", "gdsb"):
        cfg = SolverConfig(variant=Variant[v], steps=TTS_M, dt=DT, c=c, a=A_CTRL, init_mode=InitMode.uniform_random)
        # warm-up at the batch's own replica count: the first run at a new R pays one-off costs (state
        # reallocation, first use of the kernels that geometry selects) that are not T_com
        s.run_batch(cfg, tun, n_trials, master_seed=7, want_spins=False)
        t0 = time.perf_counter()
        b = s.run_batch(cfg, tun, n_trials, master_seed=1, want_spins=False)  # derive_seed(1, {3, r})
        t_batch = time.perf_counter() - t0
        st = success_probability(b.energies, target)
        r = {"variant": v, "M": TTS_M, "A": A_CTRL, "runs": n_trials, "target_energy": target,
             "target": f"reference best energy over its {n_trials} run() trials (oracle/_ref, same seeds; "
                       "tests/golden/tts_ref_gbsb.npz)",
             "p_s": st.p_s, "delta_p_s": st.delta_p_s, "hits": int((b.energies <= target).sum()),
             "best_energy": float(b.energies.min()), "t_batch_s": t_batch,
             "device_ms_batch": b.timing["total_ms"]}
        if st.p_s > 0:
            run = time_to_solution(t_batch, st)
            amort = time_to_solution(t_batch / n_trials, st)
            r.update({"tts99_run_ms": run.tts_s * 1e3, "delta_tts99_run_ms": run.delta_tts_s * 1e3,
                      "tts99_amortised_ms": amort.tts_s * 1e3,
                      "note": "tts99_run: T_com = one run's wall time (the whole 1000-run batch); amortised: "
                              "T_com = batch time / 1000 (throughput-equivalent)"})
        else:
            r["tts99_run_ms"] = None
        out["tts99" if v == "gbsb" else "tts99_gdsb"] = r
    # the reference (CPU) on the same trials: P_S from the fixture, T_com of one run() timed here
    out["tts99"]["cpu_reference"] = cpu_tts(ref, target)
    return out


def cpu_tts(ref, target):
    import oracle

    from paper_2508_17655_b200 import success_probability, time_to_solution

    e = ref["energies"]
    e = e[~np.isnan(e)]
    st = success_probability(e, target)
    R = oracle.ref("timing")
    orc = oracle.orc()
    J64 = orc.gen_dense_i8(N_SPINS, INSTANCE_SEED).astype(np.float64)
    c = 1.0 / (2.0 * math.sqrt(N_SPINS))
    m_s = 1000
    t0 = time.perf_counter()
    R.run(2, J64, m_s, DT, c, A_CTRL, int(ref["seeds"][0]))
    t_run = (time.perf_counter() - t0) * TTS_M / m_s
    out = {"p_s": st.p_s, "delta_p_s": st.delta_p_s, "hits": int((e <= target).sum()), "runs": int(e.size),
           "t_com_s": t_run, "cores_per_run": 1,
           "t_com_source": f"one reference run() of {m_s} steps timed on this host (1 thread, "
                           f"{os.path.basename(R.path)}) x {TTS_M}/{m_s}",
           "p_s_source": "tests/golden/tts_ref_gbsb.npz (1000 reference run() trials, M=21500)"}
    if st.p_s > 0:
        tts = time_to_solution(t_run, st)
        out.update({"tts99_run_ms": tts.tts_s * 1e3, "delta_tts99_run_ms": tts.delta_tts_s * 1e3,
                    "tts99_all_cores_ms": tts.tts_s * 1e3 / max(1, R.effective_workers(0))})
    return out


# ------------------------------------------------------------------ the other BASELINE configs

def _tensor_roofline(name, fmt, ops_alg, ops_exec, us, passes):
    peak, src = tensor_peak(fmt)
    a = ops_alg / (us * 1e-6) / 1e12
    e = ops_exec / (us * 1e-6) / 1e12
    return {"bound": "tensor", "unit": "TFLOP/s", "peak": peak, "peak_source": src,
            "achieved": a, "frac": a / peak, "op_type": f"algorithmic 2N ops per spin-update ({fmt} pipe)",
            "executed_achieved": e, "executed_frac": e / peak,
            "executed_op_type": f"{passes} operand plane product(s) per algorithmic MAC ({name})"}


def measure_configs(args, device: int):
    """C1, C3, C4, C5-single-GPU of BASELINE.json on this GPU: K = --steps timed steps in one
    launch after a warm-up launch, the same timing as the headline; plus a CPU baseline each."""
    import oracle

    from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant

    orc = oracle.orc()
    hbm, hbm_src = peaks()
    K, W = args.steps, 3
    out = {}

    def timed(s, variant, n, R, c):
        cfg = SolverConfig(variant=variant, steps=M_SCHED + K + W, dt=DT, c=c, a=A_CTRL)
        s.init_state(R, InitMode.small_uniform, 1, 7)
        ms = timed_advance(s, cfg, W, K)
        return ms / K * 1e3

    def cpu_leg(variant, J64, R_s, c, budget, label, m_max=M_SCHED):
        x0, y0, _ = orc.init_small_uniform(J64.shape[0], R_s, master=1, tag=7)
        su, threads, m_s, wall, lib = cpu_fanout_sample(variant, J64, x0, y0, c, budget, m_max)
        return {"value": su, "unit": "spin-updates/s", "cores": threads, "kind": "reference",
                "sample": f"{R_s} replicas x {m_s} steps of the reference {label} step(), all host threads, {lib}"}

    # C1: N=2000 dense +-1, GbSB, R=1000 (4 signed-digit planes of x through kind::i8)
    with Solver(device) as s:
        n, R = 2000, 1000
        s.gen_random_dense(n, 1)
        c = 1.0 / (2.0 * math.sqrt(n))
        us = timed(s, Variant.gbsb, n, R, c)
        d = {"workload": "C1 (BASELINE configs[0]): N=2000 dense +-1, GbSB, R=1000", "us_per_step": us,
             "su_per_s": n * R / (us * 1e-6), "steps": K,
             "roofline": _tensor_roofline("q = rint(x 2^30) as 4 signed base-256 digits", "int8", 2.0 * n * n * R,
                                          4 * 2.0 * n * n * R, us, 4),
             "kernel": "gsb_multistep_pair_kernel<4,64,4,2> (fixed-point planes, CTA pairs)"}
        d["roofline"]["traffic"] = traffic_for("c1_planes", K)
        if not args.no_cpu_baseline:
            d["cpu_baseline"] = cpu_leg(2, orc.gen_dense_i8(n, 1).astype(np.float64), 32, c, 6.0, "gbsb")
        out["C1"] = d

    # C3: N=20000 Erdos-Renyi d=10 (m=100000 edges, w in +-1), CSR, GbSB, R=512
    with Solver(device) as s:
        n, m, R = 20000, 100000, 512
        (ei, ej, w), csr = orc.gen_er_csr(n, m, 1)
        s.set_instance_csr(n, *csr)
        c = 1.0 / (2.0 * math.sqrt(n) * math.sqrt(2.0 * m / (n * (n - 1.0))))  # Wigner on the dense view
        us = timed(s, Variant.gbsb, n, R, c)
        bps = 24.0 + (4.0 * (n + 1) + 5.0 * 2 * m) / (n * R)  # state + CSR once per step
        gbs = bps * n * R / (us * 1e-6) / 1e9
        d = {"workload": "C3 (BASELINE configs[2]): ER N=20000 d=10, CSR int8, GbSB, R=512", "us_per_step": us,
             "su_per_s": n * R / (us * 1e-6), "steps": K,
             "roofline": {"bound": "hbm", "unit": "GB/s", "achieved": gbs, "peak": hbm, "peak_source": hbm_src,
                          "frac": gbs / hbm, "bytes_per_su": bps,
                          "traffic": traffic_for("c3_csr", K)},
             "kernel": "csr_step_sm_kernel (warp per (row, 128 replicas), exact int64 row sums)"}
        if not args.no_cpu_baseline:
            # the reference has no CSR path: its dense fp64 J (3.2 GB) on a small sample, and
            # our CSR restatement (the oracle's fp32 mirror, one thread), both labelled
            dense = np.zeros((n, n), np.float64)
            dense[ei, ej] = -w
            dense[ej, ei] = -w
            cb = cpu_leg(2, dense, 16, c, 6.0, "gbsb (dense fp64 J: the reference has no CSR path)", m_max=50)
            del dense
            x0, y0, p0 = orc.init_small_uniform(n, 8, master=1, tag=7)
            t0 = time.perf_counter()
            orc.step_f32_csr(2, n, csr, x0, y0, p0, 0, M_SCHED, np.float32(DT), np.float32(c), np.float32(A_CTRL), 20)
            wall = time.perf_counter() - t0
            cb["restatement"] = {"value": n * 8 * 20 / wall, "unit": "spin-updates/s", "cores": 1, "kind": "port",
                                 "sample": "8 replicas x 20 steps of the oracle's CSR step (orc_step_f32_csr), "
                                           "1 thread"}
            d["cpu_baseline"] = cb
        out["C3"] = d

    # C4: SK N=4096, J ~ N(0, 1/N) fp32, GbSB, R=2048 (24-bit fixed-point J: 3 planes x 4 digit planes,
    # nine products formed)
    with Solver(device) as s:
        n, R = 4096, 2048
        J = orc.gen_sk_f32(n, 1)
        s.set_instance(J)
        c = 0.5  # Wigner for sigma = 1/sqrt(N): 1 / (2 sqrt(N) sigma)
        us = timed(s, Variant.gbsb, n, R, c)
        d = {"workload": "C4 (BASELINE configs[3]): SK N=4096 fp32 J, GbSB, R=2048", "us_per_step": us,
             "su_per_s": n * R / (us * 1e-6), "steps": K,
             "roofline": _tensor_roofline("3 J byte planes x 4 x digit planes, the 9 of weight >= 2^16, exact int "
                                          "products", "int8", 2.0 * n * n * R, 9 * 2.0 * n * n * R, us, 9),
             "kernel": "gsb_multistep_pair_kernel<4,128,2,2,16,false,3> (fixed-point real J on CTA pairs)"}
        d["roofline"]["traffic"] = traffic_for("c4_sk", K)
        if not args.no_cpu_baseline:
            d["cpu_baseline"] = cpu_leg(2, J.astype(np.float64), 32, c, 6.0, "gbsb (fp64 J)")
        out["C4"] = d

    # C5 on one GPU: N=100000 dense +-1 (gen_random_dense(100000, 1), 10 GB int8 + 5 GB e2m1), GdSB, R=256
    with Solver(device) as s:
        n, R = 100000, 256
        s.gen_random_dense(n, 1)
        c = 1.0 / (2.0 * math.sqrt(n))
        us = timed(s, Variant.gdsb, n, R, c)
        fmt = s.operand_format
        jb = float(n) * n / (2.0 if fmt == "e2m1" else 1.0)
        byts = jb + 24.0 * n * R
        gbs = byts / (us * 1e-6) / 1e9
        tpk, tsrc = tensor_peak(fmt)
        tops = 2.0 * n * n * R / (us * 1e-6) / 1e12
        d = {"workload": "C5 on ONE GPU (BASELINE configs[4] unsharded): N=100000 dense +-1, GdSB, R=256",
             "us_per_step": us, "su_per_s": n * R / (us * 1e-6), "steps": K, "operands": fmt,
             "roofline": {"bound": "hbm", "unit": "GB/s", "achieved": gbs, "peak": hbm, "peak_source": hbm_src,
                          "frac": gbs / hbm, "bytes_per_step": byts,
                          "tensor": {"achieved": tops, "peak": tpk, "peak_source": tsrc, "frac": tops / tpk,
                                     "unit": "TFLOP/s"},
                          "traffic": traffic_for("c5_single", K)},
             "kernel": "gsb_multistep_pair_kernel<1,256,5,2,16,true> (e2m1 J streamed, CTA pairs)"}
        if not args.no_cpu_baseline:
            # the reference's dense fp64 J would need 80 GB: an int8-J restatement (the oracle's fp32
            # mirror of the step) at N=4096, scaled by (N/4096)^2 (the step is the J.sign(x) product)
            nn = 4096
            Jq = orc.gen_dense_i8(nn, 1)
            x0, y0, p0 = orc.init_small_uniform(nn, 4, master=1, tag=7)
            t0 = time.perf_counter()
            orc.step_f32(3, Jq, x0, y0, p0, 0, M_SCHED, np.float32(DT), np.float32(1 / (2 * math.sqrt(nn))),
                         np.float32(A_CTRL), 5)
            wall = (time.perf_counter() - t0) * (n / nn) ** 2
            d["cpu_baseline"] = {"value": n * 4 * 5 / wall, "unit": "spin-updates/s", "cores": 1, "kind": "port",
                                 "sample": "4 replicas x 5 GdSB steps of the oracle's int8-J fp32 step "
                                           "(orc_step_f32) at N=4096, 1 thread, scaled by (100000/4096)^2"}
        out["C5_single_gpu"] = d

    # C5 row-sharded, emulated on this GPU: G rank groups of CTA pairs in ONE cooperative launch
    # (sbg_shard_advance_fused), the multi-step cross-rank waits and slab pushes of the sharded
    # protocol running for K steps; the energies are checked bitwise against the unsharded run.
    try:
        from paper_2508_17655_b200.distributed import advance_row_shards_fused, connect_row_shards_local

        n, R = 100000, 256
        cfg = SolverConfig(variant=Variant.gdsb, steps=M_SCHED + K + W, dt=DT, c=1.0 / (2.0 * math.sqrt(n)),
                           a=A_CTRL)
        with Solver(device) as u:
            u.gen_random_dense(n, 1)
            u.init_state(R, InitMode.small_uniform, 1, 7)
            u.advance(cfg, 0, W + K)
            _, e_ref, _, _ = u.readout()
        emu = {"workload": "C5 row shards emulated on ONE GPU: N=100000 dense +-1, GdSB, R=256, G rank groups of "
                           "2*floor(74/G) CTAs in one cooperative launch (multi-step cross-rank waits and epilogue "
                           "slab pushes as over NVLink; the GPU's SMs are divided between the ranks)",
               "unsharded_us_per_step": us, "steps": K}
        from paper_2508_17655_b200.distributed import row_sharded_energies
        for G in (2, 4, 8):
            shards = [Solver(device) for _ in range(G)]
            try:
                for k, sh in enumerate(shards):
                    sh.gen_random_dense(n, 1, G, k, shard=True)
                    sh.init_state(R, InitMode.small_uniform, 1, 7)
                connect_row_shards_local(shards)
                for sh in shards:
                    sh.shard_prepare(Variant.gdsb)
                for sh in shards:
                    sh.shard_push_slab()
                advance_row_shards_fused(shards, cfg, 0, W)
                ms = advance_row_shards_fused(shards, cfg, W, W + K)
                e = row_sharded_energies([sh.readout_partial() for sh in shards])
                emu[f"G{G}"] = {"us_per_step": ms * 1e3 / K, "pairs_per_rank": (148 // 2) // G,
                                "energies_equal_unsharded": bool((e == e_ref).all())}
            finally:
                for sh in shards:
                    sh.close()
        out["C5_row_shards_emulated"] = emu
    except Exception as ex:  # noqa: BLE001 -- evidence leg: never takes the bench line down
        out["C5_row_shards_emulated"] = {"error": str(ex)[:300]}
    return out


# ------------------------------------------------------------------ C5 row shards (N > 1)

def c5_leg_in_children(args, rank: int, world: int):
    """Run the C5 row-shard leg in one child process per rank (own process group on a fresh
    port, own CUDA context) under a timeout, so a failure there -- a CUDA fault, a hung peer --
    cannot take the headline measurement of this process down with it."""
    import tempfile

    import torch
    import torch.distributed as dist

    port = torch.tensor([free_port() if rank == 0 else 0], device="cuda", dtype=torch.int64)
    dist.broadcast(port, src=0)
    env = dict(os.environ, MASTER_PORT=str(int(port.item())), MASTER_ADDR="127.0.0.1")
    out = os.path.join(tempfile.gettempdir(), f"sbg_c5leg_{os.getpid()}_{rank}.json")
    cmd = [sys.executable, os.path.abspath(__file__), "--c5-child", out, "--gpus", str(world), "--steps",
           str(args.steps), "--warmup", str(args.warmup)]
    res = {"error": "child did not report"}
    try:
        rc = subprocess.run(cmd, env=env, timeout=900).returncode
        if os.path.exists(out):
            with open(out) as f:
                res = json.load(f)
        elif rc != 0:
            res = {"error": f"child exited with {rc}"}
    except subprocess.TimeoutExpired:
        res = {"error": "child timed out (900 s)"}
    finally:
        if os.path.exists(out):
            os.remove(out)
    return res


def c5_child_main(args):
    rank, world, local = dist_env()
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    res = c5_row_shard_leg(args, rank, world, local)
    with open(args.c5_child, "w") as f:
        json.dump(res, f)
    dist.destroy_process_group()


def c5_row_shard_leg(args, rank: int, world: int, local: int):
    """BASELINE configs[4]: N=100000 dense +-1 (gen_random_dense(100000, 1), each rank
    generating its own rows on the device), GdSB, R=256, row-sharded over the ranks. The
    ranks' G buffers and done counters are wired with CUDA IPC; each step's epilogue pushes
    this rank's slab of G_{t+1} to every peer over NVLink and releases their counters, so one
    persistent launch runs all K steps with no host round trip and no separate collective.
    Peer waits time out on the device after 4 s (the leg then reports the failure instead of
    hanging). Per-rank device time, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant
    from paper_2508_17655_b200.distributed import connect_row_shards_ipc

    n, R = 100000, 256
    cfg = SolverConfig(variant=Variant.gdsb, steps=5000, dt=DT, c=1 / (2 * math.sqrt(n)), a=A_CTRL)

    def all_ok(ok: bool) -> bool:
        t = torch.tensor([1 if ok else 0], device="cuda", dtype=torch.int32)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item())

    err = None
    s = None
    try:
        s = Solver(local)
        s.gen_random_dense(n, 1, world, rank, shard=True)
        s.init_state(R, InitMode.small_uniform, 1, 7)
        ok = True
    except Exception as e:  # noqa: BLE001
        ok, err = False, f"setup: {e}"
    if not all_ok(ok):
        return {"error": err or "setup failed on another rank"}
    try:
        connect_row_shards_ipc(s)
        ok = True
    except Exception as e:  # noqa: BLE001
        ok, err = False, f"ipc wiring: {e}"
    if not all_ok(ok):
        return {"error": err or "ipc wiring failed on another rank"}
    try:
        dist.barrier()
        s.shard_prepare(Variant.gdsb)
        dist.barrier()
        s.shard_push_slab()
        dist.barrier()
        s.advance(cfg, 0, 2)  # warm-up launch
        s.synchronize()
        dist.barrier()
        s.advance(cfg, 2, 2 + args.steps)
        s.synchronize()
        ms = s.last_advance_ms()
        ok = True
    except Exception as e:  # noqa: BLE001
        ok, err, ms = False, f"steps: {e}", float("nan")
    info = s.shard_info() if ok else {}
    fmt = s.operand_format
    part = None
    if ok:
        try:
            part = s.readout_partial()  # this rank's E2 share after all 2 + K steps
        except Exception as e:  # noqa: BLE001
            ok, err = False, f"readout: {e}"
    s.close()
    if not all_ok(ok):
        return {"error": err or "a rank failed (peer wait timeout or CUDA error)"}
    # correctness of the cross-GPU run: the ranks' E2 shares must sum to the energies of the same
    # 2 + K steps run unsharded on rank 0 (the whole J fits one B200), bitwise
    from paper_2508_17655_b200.distributed import row_sharded_energies

    t = torch.as_tensor(part, device="cuda")
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    check = None
    if rank == 0:
        e_sh = row_sharded_energies([q.cpu().numpy() for q in parts])
        with Solver(local) as u:
            u.gen_random_dense(n, 1)
            u.init_state(R, InitMode.small_uniform, 1, 7)
            u.advance(cfg, 0, 2)
            u.advance(cfg, 2, 2 + args.steps)
            _, e_un, _, _ = u.readout()
        check = bool((e_sh == e_un).all())
    t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    us = ms / args.steps * 1e3
    hbm, src = peaks()
    jb = info["rows_padded"] * info["kpad"] / (2.0 if fmt == "e2m1" else 1.0)
    byts = jb + 24.0 * (n / world) * R
    return {"workload": "C5 (BASELINE configs[4]): N=100000 dense +-1, GdSB, R=256, row-sharded", "ranks": world,
            "us_per_step_per_rank": us, "su_per_s_boxwide": n * R / (us * 1e-6), "steps": args.steps,
            "operands": fmt, "rows_per_rank": info["rows_padded"],
            "energies_bitwise_equal_unsharded": check,
            "hbm_gbs_per_rank": byts / (us * 1e-6) / 1e9, "hbm_frac": byts / (us * 1e-6) / 1e9 / hbm,
            "hbm_peak_source": src,
            "timed": "one persistent launch of K steps per rank, CUDA events, max over ranks"}


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
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--c5-child", default=None, help=argparse.SUPPRESS)  # internal: the N>1 C5 leg
    args = ap.parse_args()
    if args.c5_child:
        return c5_child_main(args)
    if args.warmup < 3:
        args.warmup = 3
    _, world, _ = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch_under_torchrun(args)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} rank(s)")
    global M_SCHED
    M_SCHED = max(M_SCHED, args.warmup + args.steps)  # per-step cost does not depend on M
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
