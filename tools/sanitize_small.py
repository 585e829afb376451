"""Small end-to-end exercise of every kernel family for compute-sanitizer runs."""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, TuningResult, Variant  # noqa: E402

orc = oracle.orc()
n, R = 300, 70
J = orc.gen_dense_i8(n, 1)
with Solver(0) as s:
    s.set_instance(J)
    for v in (Variant.gdsb, Variant.gbsb, Variant.dsb, Variant.bsb):
        cfg = SolverConfig(variant=v, steps=20, dt=1.25, c=1 / (2 * math.sqrt(n)), a=0.2)
        s.init_state(R, InitMode.small_uniform, 1, 7)
        s.advance(cfg, 0, 20)
        s.readout()
        s.readout_best()
    S = np.where(np.random.default_rng(0).random((R, n)) < 0.5, -1, 1).astype(np.int8)
    s.fields_sign(S)
    s.fields_fixed(np.random.default_rng(1).uniform(-1, 1, (R, n)).astype(np.float32))
    (ei, ej, w), csr = orc.gen_er_csr(500, 2000, 3)
    s.set_instance_csr(500, *csr)
    for v in (Variant.gdsb, Variant.gbsb):
        s.run_batch(SolverConfig(variant=v, steps=10, dt=1.25, c=0.2, a=0.2), TuningResult(c=0.2, dt=1.25), 33,
                    master_seed=2)
    s.set_instance(orc.gen_sk_f32(200, 2))
    for v in (Variant.gdsb, Variant.gbsb):
        s.run_batch(SolverConfig(variant=v, steps=10, dt=1.25, c=0.5, a=0.2), TuningResult(c=0.5, dt=1.25), 40,
                    master_seed=2)
    # resident parts kernel over several replica groups (helper-warp G_0 of later groups),
    # sbg_run_best with pipelined host copies
    s.gen_random_dense(300, 4)
    cfg = SolverConfig(variant=Variant.gdsb, steps=6, dt=1.25, c=1 / (2 * math.sqrt(300)), a=0.2)
    s.init_state(6200, InitMode.small_uniform, 1, 7)
    s.advance(cfg, 0, 3)
    s.readout_best()
    x0, y0, _ = orc.init_small_uniform(300, 6200, master=3)
    s.run_best(cfg, TuningResult(c=cfg.c, dt=1.25), x0, y0)
# row shards in lockstep (2 shards on this GPU, one step per launch)
from paper_2508_17655_b200.distributed import connect_row_shards_local  # noqa: E402

shards = [Solver(0) for _ in range(2)]
try:
    for k, sh in enumerate(shards):
        sh.gen_random_dense(700, 5, 2, k)
        sh.init_state(40, InitMode.small_uniform, 1, 7)
    connect_row_shards_local(shards)
    for sh in shards:
        sh.shard_prepare(Variant.gdsb)
    for sh in shards:
        sh.shard_push_slab()
    cfg = SolverConfig(variant=Variant.gdsb, steps=10, dt=1.25, c=0.02, a=0.2)
    for m in range(3):
        for sh in shards:
            sh.advance(cfg, m, m + 1)
        for sh in shards:
            sh.synchronize()
    for sh in shards:
        sh.readout_partial()
finally:
    for sh in shards:
        sh.close()
print("sanitize run ok")
