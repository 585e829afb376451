"""Multi-GPU host logic: replica sharding.

Replicas are independent (the reference already fans them out,
bench.cpp:78), so R replicas are split into contiguous shards, one per rank,
with NO per-step collective. Replica r keeps its global index, hence its seed
derive_seed(master, {tag, r}), so every result is bitwise independent of the
number of ranks. The only exchange is the final winner selection of
batch_best_of (bench.cpp:84-87: min energy, ties to the lowest GLOBAL index):
one all_gather of (energy, index) per rank and a broadcast of the winner's spins.
torch.distributed is plumbing only (NCCL on GPUs, gloo on CPU for tests).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np


@dataclasses.dataclass(frozen=True)
class ReplicaShard:
    offset: int  # first global replica index of this rank
    count: int  # replicas on this rank
    total: int


def shard_replicas(total: int, world: int, rank: int) -> ReplicaShard:
    """Contiguous balanced split, same rule as ThreadPool::chunk_bounds (parallel.cpp:13-19)."""
    if total < 1 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard request")
    q, r = divmod(total, world)
    begin = rank * q + min(rank, r)
    return ReplicaShard(begin, q + (1 if rank < r else 0), total)


def winner_from_gathered(energies_by_rank: list, offsets: list) -> tuple[int, float]:
    """Global batch_best_of winner from per-rank (local best energy, local best index) pairs."""
    best_e, best_i = None, None
    for (e, i), off in zip(energies_by_rank, offsets):
        gi = off + int(i)
        if best_e is None or e < best_e or (e == best_e and gi < best_i):
            best_e, best_i = float(e), gi
    return best_i, best_e


def global_best_of(local_energies: np.ndarray, shard: ReplicaShard, local_spins: Optional[np.ndarray] = None,
                   group=None, device=None):
    """Combine per-rank results into the batch_best_of winner (all ranks return it).

    local_energies: this rank's R_local energies (replica order). local_spins: the
    local winner's spins (n int8) or None. Returns (global_index, energy, spins|None).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    li = int(np.flatnonzero(local_energies == local_energies.min())[0])
    mine = torch.tensor([float(local_energies[li]), float(li), float(shard.offset)], dtype=torch.float64,
                        device=device)
    allv = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allv, mine, group=group)
    allv = [v.cpu().numpy() for v in allv]
    gi, ge = winner_from_gathered([(v[0], v[1]) for v in allv], [int(v[2]) for v in allv])
    spins = None
    if local_spins is not None:
        owner = next(k for k, v in enumerate(allv) if int(v[2]) <= gi < int(v[2]) + (
            shard_replicas(shard.total, world, k).count))
        t = torch.as_tensor(np.ascontiguousarray(local_spins, np.int8) if rank == owner else
                            np.zeros_like(local_spins, np.int8))
        if device is not None:
            t = t.to(device)
        dist.broadcast(t, src=owner, group=group)
        spins = t.cpu().numpy()
    return gi, ge, spins


def distributed_batch_best_of(solver, cfg, tuning, n_batch: int, master_seed: int, group=None, device=None):
    """batch_best_of (bench.cpp:70-92) over all ranks: each rank runs its replica
    shard on its own GPU, then the global winner is agreed on."""
    import torch.distributed as dist

    from .solver import SEED_STREAM_BATCH, RunResult, _derive_seed

    shard = shard_replicas(n_batch, dist.get_world_size(group), dist.get_rank(group))
    b = solver.run_batch(cfg, tuning, shard.count, master_seed=master_seed, tag=SEED_STREAM_BATCH,
                         replica_offset=shard.offset, want_spins=False)
    spins, _, li, _ = solver.readout_best()
    gi, ge, wspins = global_best_of(b.energies, shard, spins, group=group, device=device)
    echo = dataclasses.replace(b.config, seed=_derive_seed(master_seed, [SEED_STREAM_BATCH, gi]))
    return RunResult(final_spins=wspins, energy=ge, cut=None, wall_time_s=b.timing["total_ms"] / 1e3,
                     config_echo=echo, tuning_echo=tuning)


# ----------------------------------------------------------------- row sharding (C5)

def row_shard(n_global: int, world: int, rank: int) -> tuple[int, int, int]:
    """(row0, rows_valid, rows_padded): the split sbg_set_couplings_rows_i8 applies
    (kpad = n rounded up to 256*world, equal 256-multiple slabs: whole CTA pairs)."""
    kpad = -(-n_global // (256 * world)) * 256 * world
    rows = kpad // world
    row0 = rank * rows
    return row0, max(0, min(rows, n_global - row0)), rows


def connect_row_shards_local(solvers) -> None:
    """Peer wiring for shards that live in ONE process (device pointers of each other,
    e.g. several GPUs driven by one host thread, or the single-GPU lockstep emulation
    used by the tests, where every launch runs one step so no kernel waits on another)."""
    bufs = [s.shard_buffers() for s in solvers]
    for k, s in enumerate(solvers):
        s.shard_set_peers([b for j, b in enumerate(bufs) if j != k])


def advance_row_shards_fused(solvers, cfg, m_begin: int, m_end: int) -> float:
    """Test-only: advance row shards that ALL live on one GPU (wired with
    connect_row_shards_local, prepared with shard_prepare / shard_push_slab) from m_begin to
    m_end in ONE cooperative launch, each rank on its own group of CTA pairs, so the multi-step
    cross-rank waits run as they would over NVLink (sbg_shard_advance_fused). Returns the
    device milliseconds of the launch."""
    import ctypes as C

    lib = solvers[0]._L
    hs = (C.c_void_p * len(solvers))(*[s._h for s in solvers])
    prm = solvers[0].params(cfg)
    solvers[0]._check(lib.sbg_shard_advance_fused(hs, len(solvers), C.byref(prm), m_begin, m_end))
    return solvers[0].last_advance_ms()


def connect_row_shards_ipc(solver, group=None) -> None:
    """Peer wiring across processes (one rank per GPU): CUDA IPC handles of every rank's
    (G0, G1, done) are all-gathered over torch.distributed and opened locally."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = solver.shard_ipc_export()
    handles = [None] * world
    dist.all_gather_object(handles, mine, group=group)
    solver.shard_set_peers([solver.shard_ipc_open(h) for k, h in enumerate(handles) if k != rank])


def row_sharded_energies(partials_by_rank) -> np.ndarray:
    """ising_energy per replica from the ranks' E2 shares (model.cpp:112-123)."""
    return -0.5 * np.sum(np.stack(partials_by_rank), axis=0).astype(np.float64)
