"""C5 row shards, multi-step, on ONE GPU: N = 100000 dense +-1 GdSB R=256 split into G row shards
that run as G rank groups of CTA pairs inside ONE cooperative launch (sbg_shard_advance_fused),
so the system-scope cross-rank waits and epilogue slab pushes of K7 execute step after step as
over NVLink, with the GPU's 148 SMs divided between the ranks. Compared with the unsharded
single-GPU run of the same steps (all SMs on one J): the difference is the cost of the sharded
protocol (dependency counting over G ranks, slab pushes) at equal hardware."""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant  # noqa: E402
from paper_2508_17655_b200.distributed import advance_row_shards_fused, connect_row_shards_local  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100000)
ap.add_argument("--R", type=int, default=256)
ap.add_argument("--worlds", default="2,4,8")
ap.add_argument("--steps", type=int, default=10)
args = ap.parse_args()
n, R, K = args.n, args.R, args.steps
cfg = SolverConfig(variant=Variant.gdsb, steps=5000, dt=1.25, c=1 / (2 * math.sqrt(n)), a=0.2)
out = {"n": n, "R": R, "steps": K}
with Solver(0) as s:
    s.gen_random_dense(n, 1)
    s.init_state(R, InitMode.small_uniform, 1, 7)
    s.advance(cfg, 0, 2)
    s.synchronize()
    s.advance(cfg, 2, 2 + K)
    out["unsharded_us_per_step"] = s.last_advance_ms() * 1e3 / K
for G in [int(g) for g in args.worlds.split(",")]:
    shards = [Solver(0) for _ in range(G)]
    try:
        for k, sh in enumerate(shards):
            sh.gen_random_dense(n, 1, G, k, shard=True)
            sh.init_state(R, InitMode.small_uniform, 1, 7)
        connect_row_shards_local(shards)
        for sh in shards:
            sh.shard_prepare(Variant.gdsb)
        for sh in shards:
            sh.shard_push_slab()
        advance_row_shards_fused(shards, cfg, 0, 2)
        ms = advance_row_shards_fused(shards, cfg, 2, 2 + K)
        out[f"G{G}_fused_us_per_step"] = ms * 1e3 / K
        out[f"G{G}_pairs_per_rank"] = (148 // 2) // G
    finally:
        for sh in shards:
            sh.close()
print(json.dumps(out, indent=1))
