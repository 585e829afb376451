"""C5 row shards on ONE GPU: the per-rank step of an N = 100000 dense +-1 GdSB run (R = 256)
row-sharded over G ranks, measured in lockstep (all G shards live on this GPU; every launch
runs one step, so no kernel waits on another -- the cross-GPU waits need one GPU per rank).

Each shard owns kpad/G rows of J (gen_random_dense(100000, 1)'s exact draw order, generated
per shard on the device) and pushes its slab of G_{t+1} into the G buffers of the other G-1
shards from the step epilogue (the fused all-gather; here the peers are on the same GPU, so
the pushes go to local HBM instead of NVLink). Reported per rank: device time of one step
launch (CUDA events, median over ranks and steps), the J bytes it streams, HBM fraction.
"""
import argparse
import json
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant  # noqa: E402
from paper_2508_17655_b200.distributed import connect_row_shards_local  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100000)
ap.add_argument("--R", type=int, default=256)
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--steps", type=int, default=6)
args = ap.parse_args()
n, R, G = args.n, args.R, args.world
HBM = 6553.0
cfg = SolverConfig(variant=Variant.gdsb, steps=5000, dt=1.25, c=1 / (2 * math.sqrt(n)), a=0.2)
shards = [Solver(0) for _ in range(G)]
try:
    for k, s in enumerate(shards):
        s.gen_random_dense(n, 1, G, k)
        s.init_state(R, InitMode.small_uniform, 1, 7)
    connect_row_shards_local(shards)
    for s in shards:
        s.shard_prepare(Variant.gdsb)
    for s in shards:
        s.shard_push_slab()
    times = []
    for m in range(args.steps + 1):
        for s in shards:
            s.advance(cfg, m, m + 1)
            s.synchronize()
            if m > 0:  # step 0 is the warm-up
                times.append(s.last_advance_ms() * 1e3)
    info = shards[0].shard_info()
    fmt = shards[0].operand_format
    rows, kpad = info["rows_padded"], info["kpad"]
    us = statistics.median(times)
    jb = rows * kpad / (2.0 if fmt == "e2m1" else 1.0)
    state = 24.0 * (n / G) * R
    out = {
        "n": n, "R": R, "world": G, "operands": fmt, "rows_per_rank": rows, "kpad": kpad,
        "us_per_step_per_rank": us, "us_min": min(times), "us_max": max(times),
        "su_per_s_per_rank": (n / G) * R / (us * 1e-6),
        "su_per_s_boxwide_if_overlapped": n * R / (us * 1e-6),
        "J_bytes_per_step_per_rank": jb, "algorithmic_gbs": (jb + state) / (us * 1e-6) / 1e9,
        "hbm_frac": (jb + state) / (us * 1e-6) / 1e9 / HBM,
        "how": "lockstep on one GPU: one step per launch per shard, device events; peers' G pushes land in "
               "local HBM (NVLink on a real G-GPU box)",
    }
    print(json.dumps(out, indent=1))
finally:
    for s in shards:
        s.close()
