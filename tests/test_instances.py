"""Instance ingestion host logic (instances.py) against the reference's own parse_gset /
cut_value / instance_from_json / instance_to_json (model.cpp:125-348, compiled in
oracle/_ref): same accepted graphs, same ParseError messages (test_model.cpp:240-300
cases and more), same JSON documents. CPU only."""
import numpy as np
import pytest

import oracle
from paper_2508_17655_b200.instances import (CouplingEntries, CutGraph, ParseError, cut_value, entries_from_dense,
                                             instance_from_json, instance_to_json, parse_gset, serialize_gset)

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="needs oracle/_ref (the compiled reference)")

GOOD = [
    "3 2\n1 2 1\n2 3 -1\n",
    "2 1\n1 2\n",
    "  3   2 \n\n  1\t2   1\n 2  3\t-1 \n",
    "4 0\n",
    "4 3\r\n1 2 +3\r\n3 4 -7\r\n\r\n2 4\r\n",
    "5 2\n1 5 +-2\n2 3 9223372036854775807\n",
    "3 1\n3 1 4",
]
BAD = [
    "2 1\n1 3 1\n", "2 1\n1 1 1\n", "3 2\n1 2 1\n2 1 1\n", "3 1\n1 x 1\n", "3 2\n1 2 1\n", "3 1\n1 2 1\n2 3 1\n",
    "", "3\n", "\n\n", "0 0\n", "3 -1\n", "3 1\n1 2 1 4\n", "3 1\n1\n", "3 1\n1 2 1.5\n", "3 1\n1 2 ++1\n",
    "3 1\n0 2\n", "x 1\n", "3 1\n1 2 99999999999999999999\n", "3 1\n 1 2 - \n", "3 2\n1 2\n\n2 1\n",
]


@pytest.mark.parametrize("text", GOOD)
def test_parse_gset_accepts_like_reference(text):
    n, ei, ej, w = oracle.ref().parse_gset(text)
    g = parse_gset(text)
    assert g.n == n and (g.i == ei).all() and (g.j == ej).all() and (g.w == w).all()
    assert parse_gset(serialize_gset(g)) == g


@pytest.mark.parametrize("text", BAD)
def test_parse_gset_errors_like_reference(text):
    with pytest.raises(ValueError) as want:
        oracle.ref().parse_gset(text)
    with pytest.raises(ParseError) as got:
        parse_gset(text)
    assert str(got.value) == str(want.value)


def test_cut_value_and_bridge(orc):
    (ei, ej, w), _ = orc.gen_er_csr(200, 700, 3)
    g = CutGraph(200, ei, ej, -w.astype(np.int64))
    rng = np.random.default_rng(0)
    for _ in range(5):
        s = np.where(rng.random(200) < 0.5, 1, -1).astype(np.int8)
        assert cut_value(g, s) == oracle.ref().cut_value(200, g.i, g.j, g.w, s)


def test_cutgraph_ctor_checks():
    for args, msg in [((3, [0], [0], [1]), "self-loops"), ((3, [0], [3], [1]), "out of range"),
                      ((3, [0, 1], [1, 0], [1, 2]), "duplicate edge \\(1, 0\\)")]:
        with pytest.raises(ValueError, match=msg):
            CutGraph(*args)


def test_json_round_trip_matches_reference(orc):
    J = orc.gen_dense_i8(12, 5).astype(np.float64)
    J[0, 3] = J[3, 0] = 0.0
    J[2, 7] = J[7, 2] = 0.5
    J[4, 9] = J[9, 4] = -1e-05
    doc = oracle.ref().instance_to_json(J)
    assert instance_to_json(entries_from_dense(J)) == doc
    e = instance_from_json(doc)
    dense = np.zeros((e.n, e.n))
    dense[e.i, e.j] = e.value
    dense[e.j, e.i] = e.value
    assert (dense == oracle.ref().instance_from_json(doc)).all() and (dense == J).all()


@pytest.mark.parametrize("doc", ['not json', '{"n": 3}', '{"n": 2, "edges": [[0, 0, 1.0]]}',
                                 '{"n": 2, "edges": [[0, 2, 1.0]]}', '{"n": 3, "edges": [[0, 1, 1], [1, 0, 2]]}',
                                 '{"n": 3, "edges": [[0, 1]]}', '[1, 2]'])
def test_json_errors_like_reference(doc):
    with pytest.raises(ValueError) as want:
        oracle.ref().instance_from_json(doc)
    with pytest.raises(ParseError) as got:
        instance_from_json(doc)
    if "invalid JSON" not in str(want.value):
        assert str(got.value) == str(want.value)
    assert str(got.value).startswith("line 1: ")


def test_entries_dataclass_shape():
    e = CouplingEntries(3, np.array([0]), np.array([2]), np.array([1.0]))
    assert instance_to_json(e) == '{"edges":[[0,2,1.0]],"label":"","n":3}'
