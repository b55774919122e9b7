"""MULTICUT text format: the native parser/serializer
(rama_parse_multicut / rama_serialize_multicut, host C++, no GPU needed)
against the reference's own parse_instance / serialize_instance outputs
(tests/golden/io_cases.json, made by tests/golden/make_golden_io.py):
identical graphs (canonicalised by the oracle here), identical ParseError
messages, byte-identical serialized text."""

import json
import os

import numpy as np
import pytest

import oracle as O
import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import graph as G

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def cases():
    with open(os.path.join(HERE, "golden", "io_cases.json")) as fh:
        return json.load(fh)


def _canonical(n, u, v, c):
    g = O.Graph(n, u, v, c)
    return g.num_nodes, g.edges_u.tolist(), g.edges_v.tolist(), [repr(float(x)) for x in g.costs]


@pytest.mark.parametrize("threads", [1, 4])
def test_parse_matches_reference(cases, threads):
    for case in cases["parse"]:
        text = case["text"]
        if "error" in case:
            with pytest.raises(P.ParseError) as exc:
                G._parse_native(text=text, threads=threads)
            assert str(exc.value) == case["error"], text
        else:
            n, u, v, c = G._parse_native(text=text, threads=threads)
            ref = case["graph"]
            assert _canonical(n, u, v, c) == (ref["n"], ref["u"], ref["v"], ref["c"]), text


def test_serialize_matches_reference(cases):
    for case in cases["serialize"]:
        gd = case["graph"]
        g = P.WeightedGraph._from_canonical(gd["n"], np.array(gd["u"], np.int64), np.array(gd["v"], np.int64),
                                            np.array([float(x) for x in gd["c"]]))
        assert P.serialize_instance(g) == case["text"]


def test_large_file_round_trip(tmp_path):
    """A 1.2M-edge instance through a file (mmap) with many threads: the
    parallel chunking must give the same edges, in file order."""
    rng = np.random.default_rng(3)
    n, m = 200_000, 1_200_000
    u = rng.integers(0, n, m)
    v = (u + 1 + rng.integers(0, n - 1, m)) % n
    c = rng.standard_normal(m)
    g = P.WeightedGraph._from_canonical(n, u, v, c)
    text = P.serialize_instance(g, threads=8)
    assert text.count("\n") == m + 2
    path = tmp_path / "big.txt"
    path.write_text(text)
    for threads in (1, 8):
        nn, pu, pv, pc = G._parse_native(path=str(path), threads=threads)
        assert nn == n and np.array_equal(pu, u) and np.array_equal(pv, v) and np.array_equal(pc, c)
    # one bad line deep inside: the reference's line-by-line message
    lines = text.split("\n")
    lines[700_003] = "5 5 1.0"
    (tmp_path / "bad.txt").write_text("\n".join(lines))
    with pytest.raises(P.ParseError, match="line 700004: self-loop edge"):
        G._parse_native(path=str(tmp_path / "bad.txt"), threads=8)
