"""Parity of the C4 (power-law, scaled) and C5 (64-instance batch) configs
against the REFERENCE's own solves.

Fixtures: tests/golden/c4_reference.json and c5_reference.json, written by
tests/golden/make_golden_c4c5.py, which runs ``parcut.solve`` itself in the
build container (objectives + per-round (n, m, T, |S|) traces).

* C4 scaled (Chung-Lu alpha 2.1, n = 10k / 20k / 50k):
  - mode P has no separation, so it is exact: every round and the primal
    equal the reference's;
  - mode PD reproduces every round of the reference and its LB (the hub
    5-cycle searches are exact); the primal is within the north-star 0.5 %
    (the cleanup is deviation D1).
* C5: every one of the 64 instances, solved as one batch, has the
  reference's LB and all its rounds, and a primal within 0.5 % (the cleanup
  is deviation D1).
"""

import json
import os

import numpy as np
import pytest

import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import instances
from tests._golden import DIR

pytestmark = pytest.mark.gpu

GAP = 0.005


def rel_gap(a, b):
    return abs(a - b) / max(abs(b), 1e-12)


def _load(name):
    with open(os.path.join(DIR, name)) as fh:
        return json.load(fh)


def _c4_graph(n):
    return P.WeightedGraph(*instances.chung_lu_coo(n, 2.1, 26 * n, seed=0))


def _rounds(sol):
    return [[r.nodes, r.edges, r.triplets, r.contracted] for r in sol.trace if r.phase in ("primal-dual", "contract")]


C4_RUNS = [(r["arg"], r["mode"]) for r in _load("c4_reference.json")["runs"]]


@pytest.mark.parametrize("n,mode", sorted(C4_RUNS))
def test_c4_scaled_matches_reference(n, mode):
    ref = next(r for r in _load("c4_reference.json")["runs"] if r["arg"] == n and r["mode"] == mode)
    g = _c4_graph(n)
    assert g.num_edges == ref["edges"]
    sol = P.solve(g, P.SolverConfig(mode=mode))
    assert sol.primal_cost == pytest.approx(P.clustering_cost(g, sol.labeling), rel=1e-12)
    if mode == "P":
        assert _rounds(sol) == ref["rounds"]
        assert sol.primal_cost == pytest.approx(ref["primal"], rel=1e-12)
        assert sol.lower_bound == float("-inf")
        return
    assert _rounds(sol) == ref["rounds"]
    assert sol.lower_bound == pytest.approx(ref["lower_bound"], rel=1e-11)
    assert rel_gap(sol.primal_cost, ref["primal"]) <= GAP, (sol.primal_cost, ref["primal"])
    assert sol.lower_bound <= sol.primal_cost


def test_c5_batch_all_64_match_reference():
    ref = _load("c5_reference.json")["runs"]
    assert [r["arg"] for r in ref] == list(range(64))
    graphs = [P.WeightedGraph(*instances.grid_coo(512, 512, 0, seed=s)) for s in range(64)]
    sols = P.solve_batch(graphs, P.SolverConfig(mode="PD"))
    gaps = []
    for s, (sol, r) in enumerate(zip(sols, ref)):
        assert graphs[s].num_edges == r["edges"]
        assert sol.lower_bound == pytest.approx(r["lower_bound"], rel=1e-11), s
        gaps.append(rel_gap(sol.primal_cost, r["primal"]))
        assert sol.primal_cost == pytest.approx(P.clustering_cost(graphs[s], sol.labeling), rel=1e-12), s
    assert max(gaps) <= GAP, max(gaps)
    # the batch equals single solves (same instance, same labels)
    for s in (0, 37, 63):
        one = P.solve(graphs[s], P.SolverConfig(mode="PD"))
        assert np.array_equal(one.labeling, sols[s].labeling), s
        assert _rounds(one) == ref[s]["rounds"], s
