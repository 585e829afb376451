"""Row sharding (C5) across PROCESSES: the CUDA-IPC wiring a multi-GPU run uses
(`connect_row_shards_ipc`: every rank exports its G buffers and done counters, the
handles are all-gathered over torch.distributed and opened by the peers), exercised on
one GPU with two processes.

Each process owns one row shard (`sbg_set_couplings_rows_i8`) on cuda:0. The ranks step
in LOCKSTEP: one step per launch, then a device synchronize and a host barrier, so no
kernel ever waits on a kernel of the other process (B200_PROFILING.md: kernels that wait
on one another must not share a GPU). Each step's epilogue pushes this rank's slab of
G_{t+1} into the peer's buffer through the IPC mapping and releases the peer's counter.

Checked bitwise against the unsharded run: x, y, p of every rank's rows after all steps,
and a mid-run `readout_partial` (E2 shares summing to the unsharded energies) between
two steps. Reference pieces: the row-chunk split of coupling_matvec
(proj/core/src/kernels.hpp:36-45) and ising_energy (proj/core/src/model.cpp:112-123).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, R, STEPS, MID, WORLD, M = 700, 100, 12, 5, 2, 200


def _instance():
    import oracle

    return oracle.orc().gen_dense_i8(N, 31)


def _cfg():
    from paper_2508_17655_b200 import SolverConfig, Variant

    return SolverConfig(variant=Variant.gdsb, steps=M, dt=1.25, c=1 / (2 * np.sqrt(N)), a=0.2)


def _rank_main(rank, port, out_dir):
    import torch.distributed as dist

    from paper_2508_17655_b200 import InitMode, Solver, Variant
    from paper_2508_17655_b200.distributed import connect_row_shards_ipc, row_shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    J = _instance()
    cfg = _cfg()
    row0, valid, _ = row_shard(N, WORLD, rank)
    with Solver(0) as s:
        s.set_instance_rows(J[row0:row0 + valid], N, WORLD, rank)
        s.init_state(R, InitMode.small_uniform, 3, 7)
        connect_row_shards_ipc(s)
        dist.barrier()  # every rank wired (and its counters zeroed) before any push
        s.shard_prepare(Variant.gdsb)
        dist.barrier()
        s.shard_push_slab()
        dist.barrier()
        mid = None
        for m in range(STEPS):
            s.advance(cfg, m, m + 1)
            s.synchronize()
            dist.barrier()
            if m + 1 == MID:
                mid = s.readout_partial()
                dist.barrier()
        x, y, p = s.get_state()
        fin = s.readout_partial()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), x=x, y=y, p=p, mid=mid, fin=fin, row0=row0, valid=valid)
        dist.barrier()
    dist.destroy_process_group()


def test_two_process_ipc_lockstep_equals_unsharded(tmp_path):
    import socket

    import torch.multiprocessing as mp

    from paper_2508_17655_b200 import InitMode, Solver
    from paper_2508_17655_b200.distributed import row_sharded_energies

    J = _instance()
    cfg = _cfg()
    with Solver(0) as full:
        full.set_instance(J)
        full.init_state(R, InitMode.small_uniform, 3, 7)
        full.advance(cfg, 0, MID)
        _, e_mid, _, _ = full.readout()
        full.advance(cfg, MID, STEPS)
        fx, fy, fp = full.get_state()
        _, e_fin, _, _ = full.readout()

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mp.start_processes(_rank_main, args=(port, str(tmp_path)), nprocs=WORLD, join=True, start_method="spawn")

    mids, fins = [], []
    for k in range(WORLD):
        d = np.load(tmp_path / f"rank{k}.npz")
        r0, v = int(d["row0"]), int(d["valid"])
        for name, ref in (("x", fx), ("y", fy), ("p", fp)):
            assert (d[name].view(np.uint32) == ref[:, r0:r0 + v].view(np.uint32)).all(), (k, name)
        mids.append(d["mid"])
        fins.append(d["fin"])
    assert (row_sharded_energies(mids) == e_mid).all()
    assert (row_sharded_energies(fins) == e_fin).all()
