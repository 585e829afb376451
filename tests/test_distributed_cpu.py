"""World-size-2 gloo tests of the replica-sharding host logic (no GPU).

The per-rank work is the oracle's fp32 mirror standing in for the device (the
product path runs paper_2508_17655_b200.Solver per GPU); what is under test is
the partition (global replica indices/seeds), the global winner rule with ties
to the lowest global index, and the winner-spin broadcast.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2508_17655_b200.distributed import ReplicaShard, shard_replicas, winner_from_gathered


def test_shards_cover_replicas_exactly():
    for total in (1, 7, 8192, 1000):
        for world in (1, 2, 3, 8):
            if total < world:
                continue
            shards = [shard_replicas(total, world, k) for k in range(world)]
            assert shards[0].offset == 0
            for a, b in zip(shards, shards[1:]):
                assert a.offset + a.count == b.offset
            assert shards[-1].offset + shards[-1].count == total
            assert max(s.count for s in shards) - min(s.count for s in shards) <= 1


def test_winner_rule_ties_to_lowest_global_index():
    assert winner_from_gathered([(-5.0, 3), (-5.0, 0)], [0, 10]) == (3, -5.0)
    assert winner_from_gathered([(-4.0, 3), (-5.0, 1)], [0, 10]) == (11, -5.0)
    assert winner_from_gathered([(-5.0, 2), (-5.0, 2)], [10, 0]) == (2, -5.0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, R, out):
    import torch.distributed as dist

    import oracle
    from paper_2508_17655_b200.distributed import global_best_of, shard_replicas

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = oracle.orc()
    J = orc.gen_dense_i8(n, 3)
    sh = shard_replicas(R, world, rank)
    x, y, p = orc.init_small_uniform(n, sh.count, master=5, tag=7, r0=sh.offset)
    x, y, p = orc.step_f32(3, J, x, y, p, 0, 60, np.float32(1.25), np.float32(1 / (2 * np.sqrt(n))),
                           np.float32(0.2), 60)
    e = -0.5 * orc.energy2_i8(J, x)
    li = int(np.flatnonzero(e == e.min())[0])
    spins = np.where(x[li] >= 0, 1, -1).astype(np.int8)
    gi, ge, ws = global_best_of(e, sh, spins)
    out[rank] = (gi, ge, ws.tolist(), e.tolist(), sh.offset)
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_batch_best_of_equals_single_process(orc):
    n, R, world = 48, 9, 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, R, out), nprocs=world, join=True)
    # single-process reference of the same R replicas
    J = orc.gen_dense_i8(n, 3)
    x, y, p = orc.init_small_uniform(n, R, master=5, tag=7)
    x, y, p = orc.step_f32(3, J, x, y, p, 0, 60, np.float32(1.25), np.float32(1 / (2 * np.sqrt(n))),
                           np.float32(0.2), 60)
    e = -0.5 * orc.energy2_i8(J, x)
    best = int(np.flatnonzero(e == e.min())[0])
    for rank in range(world):
        gi, ge, ws, _, _ = out[rank]
        assert gi == best and ge == e[best]
        assert ws == np.where(x[best] >= 0, 1, -1).tolist()
    joined = sum((out[k][3] for k in sorted(out.keys(), key=lambda k: out[k][4])), [])
    assert joined == e.tolist()  # sharded results are bitwise the unsharded ones


def _rowshard_worker(rank, world, port, n, R, steps, out):
    """One rank of the row-sharded protocol on CPU: its rows of J,
    its slice of x/y/p, an all_gather of the sign slabs every step (the exchange the
    GPU kernel does with NVLink peer stores), exact integer fields of its rows."""
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2508_17655_b200.distributed import row_shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = oracle.orc()
    J = orc.gen_dense_i8(n, 5)
    row0, valid, rows = row_shard(n, world, rank)
    Jr = J[row0:row0 + valid].astype(np.int64)
    xf, yf, pf = orc.init_small_uniform(n, R, master=2)
    x = np.ascontiguousarray(xf[:, row0:row0 + valid])
    y = np.ascontiguousarray(yf[:, row0:row0 + valid])
    p = np.ascontiguousarray(pf[:, row0:row0 + valid])
    c, dt, a = np.float32(1 / (2 * np.sqrt(n))), np.float32(1.25), np.float32(0.2)
    kpad = rows * world
    for m in range(steps):
        slab = np.zeros((R, rows), np.int8)
        slab[:, :valid] = np.where(x >= 0, 1, -1)
        gathered = [torch.zeros((R, rows), dtype=torch.int8) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(slab))
        S = torch.cat(gathered, dim=1).numpy()[:, :n].astype(np.int64)  # all spins, global order
        assert S.shape[1] <= kpad
        F = (S @ Jr.T).astype(np.float32)  # exact integers, local rows
        orc.phase_batch(F, x, y, p, a, c, dt, m, 200)
    out[rank] = (x.tolist(), y.tolist(), p.tolist(), row0, valid)
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_row_sharded_gdsb_equals_unsharded(orc):
    n, R, steps, world = 300, 6, 12, 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rowshard_worker, args=(world, _free_port(), n, R, steps, out), nprocs=world, join=True)
    J = orc.gen_dense_i8(n, 5)
    x, y, p = orc.init_small_uniform(n, R, master=2)
    x, y, p = orc.step_f32(3, J, x, y, p, 0, 200, np.float32(1.25), np.float32(1 / (2 * np.sqrt(n))),
                           np.float32(0.2), steps)
    for k in range(world):
        xs, ys, ps, row0, valid = out[k]
        assert (np.array(xs, np.float32) == x[:, row0:row0 + valid]).all()
        assert (np.array(ys, np.float32) == y[:, row0:row0 + valid]).all()
        assert (np.array(ps, np.float32) == p[:, row0:row0 + valid]).all()
