"""Row sharding (C5) on one GPU: two shards driven in LOCKSTEP (one step per launch,
so no kernel ever waits on another; the multi-step cross-rank waits need one GPU per
rank) must reproduce the unsharded GdSB trajectory bit for bit, and their E2 shares
must sum to the unsharded energies."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# default: CTA-pair kernel on packed e2m1 J/G; SBG_Q4=0: CTA-pair kernel on int8 operands;
# + SBG_STEP_CFG=-1: the single-CTA int8 kernel
SHARD_KERNELS = [{}, {"SBG_Q4_NPAIR": "128"}, {"SBG_Q4": "0"}, {"SBG_Q4": "0", "SBG_STEP_CFG": "-1"}]


@pytest.fixture(params=SHARD_KERNELS, ids=["e2m1_pair", "e2m1_pair128", "int8_pair", "int8_single"])
def shard_kernel(request, monkeypatch):
    for k in ("SBG_Q4", "SBG_STEP_CFG", "SBG_Q4_NPAIR"):
        monkeypatch.delenv(k, raising=False)
    for k, v in request.param.items():
        monkeypatch.setenv(k, v)
    return request.param


@pytest.mark.parametrize("n,R,steps,world", [(700, 100, 25, 2), (3000, 300, 8, 4)])
def test_two_shards_lockstep_equal_unsharded(orc, shard_kernel, n, R, steps, world):
    from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant
    from paper_2508_17655_b200.distributed import connect_row_shards_local, row_shard, row_sharded_energies

    M = 200
    J = orc.gen_dense_i8(n, 31)
    cfg = SolverConfig(variant=Variant.gdsb, steps=M, dt=1.25, c=1 / (2 * np.sqrt(n)), a=0.2)
    with Solver(0) as full:
        full.set_instance(J)
        full.init_state(R, InitMode.small_uniform, 3, 7)
        mid = steps // 2
        full.advance(cfg, 0, mid)
        _, fe_mid, _, _ = full.readout()
        full.advance(cfg, mid, steps)
        fx, fy, fp = full.get_state()
        _, fe, _, _ = full.readout()
    shards = [Solver(0) for _ in range(world)]
    try:
        for k, s in enumerate(shards):
            row0, valid, _ = row_shard(n, world, k)
            s.set_instance_rows(J[row0:row0 + valid], n, world, k)
            assert s.operand_format == ("int8" if "SBG_Q4" in shard_kernel else "e2m1")
            s.init_state(R, InitMode.small_uniform, 3, 7)
            x0, _, _ = s.get_state()
            ex, _, _ = orc.init_small_uniform(n, R, master=3, tag=7)
            assert (x0 == ex[:, row0:row0 + valid]).all()
        connect_row_shards_local(shards)
        for s in shards:
            s.shard_prepare(Variant.gdsb)
        for s in shards:
            s.shard_push_slab()
        for m in range(steps):
            for s in shards:
                s.advance(cfg, m, m + 1)
            for s in shards:
                s.synchronize()
            if m + 1 == mid:  # mid-run readout between two steps (private unpack buffer)
                assert (row_sharded_energies([s.readout_partial() for s in shards]) == fe_mid).all()
        parts = []
        for k, s in enumerate(shards):
            row0, valid, _ = row_shard(n, world, k)
            x, y, p = s.get_state()
            assert (x == fx[:, row0:row0 + valid]).all(), k
            assert (y == fy[:, row0:row0 + valid]).all(), k
            assert (p == fp[:, row0:row0 + valid]).all(), k
            parts.append(s.readout_partial())
        assert (row_sharded_energies(parts) == fe).all()
    finally:
        for s in shards:
            s.close()


def test_hash_couplings_match_oracle_and_shards(orc, shard_kernel):
    """Device +-1 generator (large-N instances) == its oracle restatement; row shards of it
    reproduce the unsharded GdSB run bitwise (lockstep emulation)."""
    from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant
    from paper_2508_17655_b200.distributed import connect_row_shards_local, row_shard

    n, R, seed, world, steps = 900, 64, 77, 2, 12
    J = orc.gen_hash_pm1_rows(n, seed, 0, n)
    assert (J == J.T).all() and (np.diag(J) == 0).all()
    rng = np.random.default_rng(0)
    S = np.where(rng.random((R, n)) < 0.5, -1, 1).astype(np.int8)
    cfg = SolverConfig(variant=Variant.dsb, steps=100, dt=1.25, c=1 / (2 * np.sqrt(n)), a=0.0)
    with Solver(0) as full:
        full.gen_hash_pm1(n, seed)
        assert (full.fields_sign(S) == orc.fields_i8(J, S)).all()
        full.init_state(R, InitMode.small_uniform, 9, 7)
        full.advance(cfg, 0, steps)
        fx, _, _ = full.get_state()
    shards = [Solver(0) for _ in range(world)]
    try:
        for k, s in enumerate(shards):
            s.gen_hash_pm1(n, seed, world, k)
            s.init_state(R, InitMode.small_uniform, 9, 7)
        connect_row_shards_local(shards)
        for s in shards:
            s.shard_prepare(Variant.dsb)
        for s in shards:
            s.shard_push_slab()
        for m in range(steps):
            for s in shards:
                s.advance(cfg, m, m + 1)
            for s in shards:
                s.synchronize()
        for k, s in enumerate(shards):
            row0, valid, _ = row_shard(n, world, k)
            x, _, _ = s.get_state()
            assert (x == fx[:, row0:row0 + valid]).all()
    finally:
        for s in shards:
            s.close()


@pytest.mark.parametrize("n,R,world,chunks", [(3000, 300, 2, (0, 5, 13)), (6000, 256, 4, (0, 1, 9, 12)),
                                              (8000, 100, 8, (0, 7))])
def test_fused_multistep_row_shards_equal_unsharded(orc, n, R, world, chunks):
    """The K7 protocol MULTI-STEP: `world` e2m1 row shards on this GPU advanced in one
    cooperative launch per chunk (sbg_shard_advance_fused: each rank on its own CTA pairs, the
    same system-scope waits on peer counters and epilogue slab pushes as across GPUs), chunks
    of several steps back to back with no host barrier between the ranks' steps, a mid-run
    readout_partial between two chunks -- bitwise equal to the unsharded run."""
    from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant
    from paper_2508_17655_b200.distributed import (advance_row_shards_fused, connect_row_shards_local, row_shard,
                                                   row_sharded_energies)

    M = 200
    J = orc.gen_dense_i8(n, 29)
    cfg = SolverConfig(variant=Variant.gdsb, steps=M, dt=1.25, c=1 / (2 * np.sqrt(n)), a=0.2)
    mid = chunks[len(chunks) // 2]
    with Solver(0) as full:
        full.set_instance(J)
        full.init_state(R, InitMode.small_uniform, 5, 7)
        full.advance(cfg, 0, mid)
        _, fe_mid, _, _ = full.readout()
        full.advance(cfg, mid, chunks[-1])
        fx, fy, fp = full.get_state()
        _, fe, _, _ = full.readout()
    shards = [Solver(0) for _ in range(world)]
    try:
        for k, s in enumerate(shards):
            row0, valid, _ = row_shard(n, world, k)
            s.set_instance_rows(J[row0:row0 + valid], n, world, k)
            assert s.operand_format == "e2m1"
            s.init_state(R, InitMode.small_uniform, 5, 7)
        connect_row_shards_local(shards)
        for s in shards:
            s.shard_prepare(Variant.gdsb)
        for s in shards:
            s.shard_push_slab()
        for m0, m1 in zip(chunks[:-1], chunks[1:]):
            assert advance_row_shards_fused(shards, cfg, m0, m1) > 0
            if m1 == mid:
                assert (row_sharded_energies([s.readout_partial() for s in shards]) == fe_mid).all()
        parts = []
        for k, s in enumerate(shards):
            row0, valid, _ = row_shard(n, world, k)
            x, y, p = s.get_state()
            assert (x == fx[:, row0:row0 + valid]).all(), k
            assert (y == fy[:, row0:row0 + valid]).all(), k
            assert (p == fp[:, row0:row0 + valid]).all(), k
            parts.append(s.readout_partial())
        assert (row_sharded_energies(parts) == fe).all()
    finally:
        for s in shards:
            s.close()
