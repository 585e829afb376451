"""Instance ingestion without dense fp64: G-set MAX-CUT graphs and
JSON instance documents go straight to the device as CSR int8 (or the dense int8 /
real-J images), instead of the reference's maxcut_to_ising / instance_from_json,
which materialise an n x n fp64 matrix (3.2 GB at n = 20000, 80 GB at n = 1e5).

Host-side text formats follow the reference exactly (model.cpp:204-348): same
tokenisation, same validation order and the same ParseError messages ("line L: ...").
"""
from __future__ import annotations

import dataclasses
import json
import re

import numpy as np

_WS = re.compile(r"[ \t\n\v\f\r]+")  # std::istream >> std::string separators
_INT = re.compile(r"-?[0-9]+\Z")


class ParseError(ValueError):
    """errors.hpp:10-19: message prefixed with the offending line number."""

    def __init__(self, line: int, message: str):
        super().__init__(f"line {line}: {message}")
        self.line = line


@dataclasses.dataclass
class CutGraph:  # model.hpp:72-95 (0-based endpoints)
    n: int
    i: np.ndarray
    j: np.ndarray
    w: np.ndarray

    def __post_init__(self):
        self.i = np.ascontiguousarray(self.i, np.int64)
        self.j = np.ascontiguousarray(self.j, np.int64)
        self.w = np.ascontiguousarray(self.w, np.int64)
        # CutGraph ctor checks (model.cpp:91-103), in input order
        seen = set()
        for a, b in zip(self.i.tolist(), self.j.tolist()):
            if not (0 <= a < self.n and 0 <= b < self.n):
                raise ValueError("edge endpoint out of range")
            if a == b:
                raise ValueError("self-loops are not allowed")
            key = (min(a, b), max(a, b))
            if key in seen:
                raise ValueError(f"duplicate edge ({a}, {b})")
            seen.add(key)

    @property
    def m(self) -> int:
        return len(self.i)

    def total_weight(self) -> int:  # model.cpp:105-109
        return int(self.w.sum())

    def __eq__(self, other) -> bool:
        return (isinstance(other, CutGraph) and self.n == other.n and np.array_equal(self.i, other.i)
                and np.array_equal(self.j, other.j) and np.array_equal(self.w, other.w))


def _parse_integer(tok: str, line_no: int, what: str) -> int:  # model.cpp:207-220 (std::from_chars)
    body = tok[1:] if tok.startswith("+") else tok
    if not _INT.match(body) or not -(1 << 63) <= int(body) < (1 << 63):
        raise ParseError(line_no, f"expected integer {what}, got '{tok}'")
    return int(body)


def parse_gset(text: str) -> CutGraph:
    """parse_gset (model.cpp:225-282): "n m" header, then m lines "i j [w]" (1-based,
    default weight 1); blank lines ignored."""
    lines = text.split("\n")
    if text.endswith("\n"):
        lines.pop()
    if text == "":
        lines = []
    n, m = 0, -1
    ei, ej, ew = [], [], []
    seen = set()
    line_no = 0
    for line in lines:
        line_no += 1
        tokens = [t for t in _WS.split(line) if t]
        if not tokens:
            continue
        if m < 0:
            if len(tokens) != 2:
                raise ParseError(line_no, "expected header 'n m'")
            header_n = _parse_integer(tokens[0], line_no, "vertex count")
            m = _parse_integer(tokens[1], line_no, "edge count")
            if header_n < 1:
                raise ParseError(line_no, "vertex count must be >= 1")
            if m < 0:
                raise ParseError(line_no, "edge count must be >= 0")
            n = header_n
            continue
        if len(ei) == m:
            raise ParseError(line_no, f"unexpected line after {m} edges")
        if len(tokens) not in (2, 3):
            raise ParseError(line_no, "expected edge 'i j [w]'")
        i1 = _parse_integer(tokens[0], line_no, "endpoint")
        j1 = _parse_integer(tokens[1], line_no, "endpoint")
        w = _parse_integer(tokens[2], line_no, "weight") if len(tokens) == 3 else 1
        if i1 < 1 or j1 < 1 or i1 > n or j1 > n:
            raise ParseError(line_no, f"vertex index out of range [1, {n}]")
        if i1 == j1:
            raise ParseError(line_no, f"self-loop on vertex {i1}")
        key = (min(i1, j1), max(i1, j1))
        if key in seen:
            raise ParseError(line_no, f"duplicate edge ({tokens[0]}, {tokens[1]})")
        seen.add(key)
        ei.append(i1 - 1)
        ej.append(j1 - 1)
        ew.append(w)
    if m < 0:
        raise ParseError(line_no or 1, "missing header 'n m'")
    if len(ei) != m:
        raise ParseError(line_no or 1, f"expected {m} edges, got {len(ei)}")
    return CutGraph(n, np.array(ei, np.int64), np.array(ej, np.int64), np.array(ew, np.int64))


def load_gset(path: str) -> CutGraph:
    with open(path, "r") as f:
        return parse_gset(f.read())


def serialize_gset(graph: CutGraph) -> str:  # model.cpp:289-295
    out = [f"{graph.n} {graph.m}\n"]
    out += [f"{a + 1} {b + 1} {w}\n" for a, b, w in zip(graph.i.tolist(), graph.j.tolist(), graph.w.tolist())]
    return "".join(out)


@dataclasses.dataclass
class CouplingEntries:
    """An IsingInstance as its strict-upper-triangle entries (IsingInstance::from_entries,
    model.cpp:70-86), never densified on the host."""
    n: int
    i: np.ndarray
    j: np.ndarray
    value: np.ndarray
    label: str = ""


def instance_from_json(text: str) -> CouplingEntries:
    """instance_from_json (model.cpp:318-348): {"n", "label", "edges": [[i, j, J_ij], ...]}."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise ParseError(1, f"invalid JSON: {e}") from None
    if not isinstance(doc, dict) or "n" not in doc or "edges" not in doc:
        raise ParseError(1, "instance document needs fields 'n' and 'edges'")
    n = int(doc["n"])
    label = doc.get("label", "")
    ei, ej, ev = [], [], []
    for e in doc["edges"]:
        if not isinstance(e, list) or len(e) != 3:
            raise ParseError(1, "each edge must be a [i, j, value] triple")
        ei.append(int(e[0]))
        ej.append(int(e[1]))
        ev.append(float(e[2]))
    if n < 1:
        raise ParseError(1, "instance size must be >= 1")
    seen = set()
    for a, b in zip(ei, ej):  # from_entries checks, rethrown as ParseError(1, ...)
        if a >= n or b >= n or a < 0 or b < 0:
            raise ParseError(1, "coupling index out of range")
        if a == b:
            raise ParseError(1, "diagonal couplings are not allowed")
        key = (min(a, b), max(a, b))
        if key in seen:
            raise ParseError(1, f"duplicate coupling entry ({a}, {b})")
        seen.add(key)
    return CouplingEntries(n, np.array(ei, np.int64), np.array(ej, np.int64), np.array(ev, np.float64), label)


def instance_to_json(entries: CouplingEntries) -> str:
    """instance_to_json (model.cpp:296-316): nonzero strict-upper entries in row-major
    order, keys sorted, compact separators (nlohmann's dump())."""
    a = np.minimum(entries.i, entries.j)
    b = np.maximum(entries.i, entries.j)
    keep = entries.value != 0.0
    order = np.lexsort((b[keep], a[keep]))
    edges = [[int(x), int(y), float(v)] for x, y, v in zip(a[keep][order], b[keep][order], entries.value[keep][order])]
    return json.dumps({"edges": edges, "label": entries.label, "n": entries.n}, separators=(",", ":"))


def entries_from_dense(J: np.ndarray, label: str = "") -> CouplingEntries:
    iu, ju = np.nonzero(np.triu(J, 1))
    return CouplingEntries(J.shape[0], iu.astype(np.int64), ju.astype(np.int64), J[iu, ju].astype(np.float64), label)


def cut_value(graph: CutGraph, spins: np.ndarray) -> int:  # model.cpp:125-132 (host check)
    s = np.asarray(spins, np.int64)
    return int(graph.w[s[graph.i] != s[graph.j]].sum())


__all__ = ["ParseError", "CutGraph", "parse_gset", "load_gset", "serialize_gset", "CouplingEntries",
           "instance_from_json", "instance_to_json", "entries_from_dense", "cut_value"]
