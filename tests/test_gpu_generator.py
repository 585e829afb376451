"""Device gen_random_dense (gen_dense.cuh) against the oracle's serial walk of the
reference's draw order (model.cpp:144-159; the oracle is pinned to the reference's
own J matrices in test_oracle.py): bit-identical for whole matrices, row shards,
tiny jump segments (every row crosses segment boundaries), and sampled rows of
C5's n = 100000 instance."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def solver():
    from paper_2508_17655_b200 import Solver

    s = Solver(0)
    yield s
    s.close()


@pytest.mark.parametrize("n,seed", [(2, 1), (3, 9), (37, 5), (300, 1), (2000, 1), (4099, 77)])
def test_whole_matrix_bitwise(solver, orc, n, seed):
    solver.gen_random_dense(n, seed)
    assert (solver.get_couplings() == orc.gen_dense_i8(n, seed)).all()


@pytest.mark.parametrize("seg", ["8", "24"])
def test_small_segments(solver, orc, seg, monkeypatch):
    monkeypatch.setenv("SBG_GEN_SEG", seg)
    for n, world in ((261, 1), (261, 2), (700, 3)):
        for rank in range(world):
            solver.gen_random_dense(n, 3, world, rank)
            info = solver.shard_info() if world > 1 else {"row0": 0, "rows_valid": n}
            want = orc.gen_dense_i8_rows(n, 3, info["row0"], info["rows_valid"])
            assert (solver.get_couplings() == want).all(), (n, world, rank)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_row_shards_bitwise(solver, orc, world):
    from paper_2508_17655_b200.distributed import row_shard

    n = 3001
    full = orc.gen_dense_i8(n, 11)
    for rank in range(world):
        row0, valid, _ = row_shard(n, world, rank)
        if valid == 0:
            continue
        solver.gen_random_dense(n, 11, world, rank)
        assert solver.shard_info()["row0"] == row0
        assert (solver.get_couplings() == full[row0:row0 + valid]).all(), rank


def test_c5_instance_rows(solver, orc):
    """n = 100000 (10 GB int8): the first 64 rows and 64 rows of rank 1 of an 8-way
    row split, against the oracle's serial walk (which stops at the last needed row)."""
    n = 100_000
    solver.gen_random_dense(n, 1)
    head = solver.get_couplings(0, 64)
    assert (head == orc.gen_dense_i8_rows(n, 1, 0, 64)).all()
    assert (solver.get_couplings(12544, 64) == orc.gen_dense_i8_rows(n, 1, 12544, 64)).all()
    # the far corner (mirror of the last tiles) and the value law of the last rows
    tail = solver.get_couplings(n - 64, 64)
    assert (tail[:, :64] == head[:, n - 64:].T).all()
    assert (np.diagonal(tail[:, n - 64:]) == 0).all()
    off = tail[:, : n - 64]
    assert set(np.unique(off)) == {-1, 1} and abs(off.mean()) < 0.01
    solver.gen_random_dense(n, 1, 8, 1)
    assert (solver.get_couplings(0, 64) == orc.gen_dense_i8_rows(n, 1, 12544, 64)).all()
