"""Pin the CPU oracle (oracle/rama_oracle.c) to the reference.

1. Known-answer vectors from the reference's own tests (cited per test).
2. Golden fixtures produced by running the reference itself
   (tests/golden/make_golden.py): every operator and every solver mode on 60
   random graphs, C1 grids (mode P, seeds 0-9) and PD grids -- bit-exact.
3. numpy summation-order restatements vs numpy.
"""

import json
import os

import numpy as np
import pytest

import oracle as O
from tests._golden import load


def tri():
    return O.Graph(3, [0, 1, 0], [1, 2, 2], [1.0, 1.0, -2.0])


# ------------------------------------------------------------ sum orders

@pytest.mark.parametrize("n", [0, 1, 2, 7, 8, 9, 15, 16, 100, 128, 129, 1000, 4097, 100003])
def test_np_sum_matches_numpy(n):
    x = np.random.default_rng(n).standard_normal(n)
    assert O.np_sum(x) == float(x.sum())


def test_seg_sum_matches_reduceat():
    rng = np.random.default_rng(5)
    for _ in range(300):
        x = rng.standard_normal(int(rng.integers(1, 700)))
        assert O.seg_sum(x) == float(np.add.reduceat(x, [0])[0])
    # signed zeros: numpy keeps -0.0 (short sums start at -0.0)
    for x in ([-0.0], [-0.0, -0.0], [-0.0, 0.0], [0.0, -0.0], [-0.0] * 9, [1.0, -1.0], [-1.0, 1.0, -0.0]):
        x = np.array(x)
        assert np.signbit(O.seg_sum(x)) == np.signbit(np.add.reduceat(x, [0])[0]), x


# -------------------------------------------------- known-answer vectors

def test_canonical_ctor():  # graph.py:29-57, test_graph.py:115-141
    g = O.Graph(3, [1, 0, 2, 1], [0, 1, 1, 2], [1.0, 0.5, 2.0, -1.0])
    assert g.edges_u.tolist() == [0, 1] and g.edges_v.tolist() == [1, 2]
    assert g.costs.tolist() == [1.5, 1.0]
    with pytest.raises(ValueError):
        O.Graph(2, [0], [0], [1.0])
    with pytest.raises(ValueError):
        O.Graph(2, [0], [2], [1.0])


def test_components_known():  # test_contraction.py:43-57
    m, k = O.connected_components(5, [(0, 1), (1, 2)])
    assert m.tolist() == [0, 0, 0, 1, 2] and k == 3
    m, k = O.connected_components(4, [(2, 3), (0, 3)])
    assert m.tolist() == [0, 1, 0, 0] and k == 2


def test_contract_known():  # test_contraction.py:97-109
    g = O.Graph(3, [0, 1, 0], [1, 2, 2], [2.0, 3.0, -1.0])
    f, k = O.connected_components(3, [(1, 2)])
    gq, joined = O.contract_graph(g, f, k)
    assert gq.edges_u.tolist() == [0] and gq.edges_v.tolist() == [1] and gq.costs.tolist() == [1.0]
    assert joined == 3.0


def test_strategies_known():  # test_contraction.py:177-219
    g = O.Graph(3, [0, 1], [1, 2], [5.0, 3.0])
    assert O.select_matching(g).tolist() == [[0, 1]]
    sq = O.Graph(4, [0, 1, 2, 0], [1, 2, 3, 3], [1.0] * 4)
    assert O.select_matching(sq).tolist() == [[0, 1], [2, 3]]
    assert O.select_spanning_forest_no_conflicts(tri()).tolist() == [[1, 2]]
    star = O.Graph(3, [0, 0], [1, 2], [2.0, 3.0])
    assert O.select_spanning_forest_no_conflicts(star).tolist() == [[0, 1], [0, 2]]
    g2, f, nt, joined, _ = O.contraction_step(tri(), "forest")
    assert f.tolist() == [0, 1, 1] and g2.costs.tolist() == [-1.0] and joined == 1.0


def test_auto_switch_star():  # test_contraction.py:264-272
    g = O.Graph(21, [0] * 20, list(range(1, 21)), [float(i) for i in range(1, 21)])
    assert len(O.select_matching(g)) == 1
    _, _, nt, joined, _ = O.contraction_step(g, "auto")
    assert nt == 1 and joined == sum(range(1, 21))


def test_separation_known():  # test_dual.py:61-82
    lengths, nodes = O.separate(tri(), 3)
    assert lengths.tolist() == [3] and nodes[0].tolist() == [0, 1, 2]
    sq = O.Graph(4, [0, 1, 2, 0], [1, 2, 3, 3], [1.0, 1.0, 1.0, -1.0])
    assert O.separate(sq, 3)[0].tolist() == [0]
    lengths, nodes = O.separate(sq, 4)
    assert lengths.tolist() == [4] and nodes[0].tolist() == [0, 1, 2, 3]
    tie = O.Graph(4, [0, 0, 1, 2, 0], [1, 2, 3, 3, 3], [1.0, 1.0, 1.0, 1.0, -1.0])
    lengths, nodes = O.separate(tie, 5)
    assert nodes[0, :3].tolist() == [0, 1, 3]


def test_triangulation_square_fan():  # test_dual.py:121-134
    sq = O.Graph(4, [0, 1, 2, 0], [1, 2, 3, 3], [1.0, 1.0, 1.0, -1.0])
    st = O.triangulate(sq, *O.separate(sq, 4))
    assert st.tri_nodes.tolist() == [[0, 1, 2], [0, 2, 3]]
    assert st.num_edges == 5 and (st.edges_u[4], st.edges_v[4]) == (0, 2)
    assert st.coverage[4] == 2


def test_mp_known():  # test_dual.py:204-257
    g = O.Graph(4, [0, 0, 0, 1, 1, 2], [1, 2, 3, 2, 3, 3], [4.0, -2.0, 1.0, 1.0, 1.0, 7.0])
    st = O.DualState(4, 6, g.edges_u, g.edges_v, g.costs, np.array([[0, 1, 2], [0, 1, 3]]),
                     np.array([[0, 1, 3], [0, 2, 4]]), np.array([2, 1, 1, 1, 1, 0]), np.zeros((2, 3)))
    cl = O.reparametrized_edge_costs(st)
    assert cl.tolist() == g.costs.tolist()
    t = tri()
    st = O.triangulate(t, *O.separate(t, 3))
    O.message_passing(st, 1)
    assert np.allclose(O.reparametrized_edge_costs(st), [0.0, -1.0, 0.0], atol=1e-12)
    assert O.lower_bound(st) == pytest.approx(-1.0, abs=1e-12)


def test_solver_known():  # test_solver.py:53-92
    for mode in ("P", "PD", "PD+", "GAEC"):
        assert O.solve(tri(), mode=mode).primal_cost == -1.0
    assert O.solve(tri(), mode="D", mp_iterations=1).lower_bound == pytest.approx(-1.0, abs=1e-9)
    assert O.solve(tri(), mode="GAEC").labeling.tolist() == [0, 0, 1]
    neg = O.Graph(4, [0, 1, 2], [1, 2, 3], [-1.0, -0.5, -2.0])
    for mode in ("P", "PD", "GAEC"):
        assert O.solve(neg, mode=mode).labeling.tolist() == [0, 1, 2, 3]


# ------------------------------------------------------- golden fixtures

def _graph(fx, i):
    n, u, v, c = fx.graph_arrays(i)
    return O.Graph(n, u, v, c, canonical=True)


def test_golden_ops():
    fx = load("ops_small.npz")
    for i in range(fx.count("edges")):
        g = _graph(fx, i)
        assert np.array_equal(O.select_matching(g).reshape(-1), fx.vec("matching", i))
        assert np.array_equal(O.select_spanning_forest_no_conflicts(g).reshape(-1), fx.vec("forest", i))
        assert np.array_equal(O.select_max_edge(g).reshape(-1), fx.vec("max_edge", i))
        S = fx.get("S", i).reshape(-1, 2)
        fmap, nt = O.connected_components(g.num_nodes, S)
        assert np.array_equal(fmap, fx.vec("cc_map", i))
        gq, joined = O.contract_graph(g, fmap, nt)
        assert np.array_equal(np.stack([gq.edges_u, gq.edges_v], 1).reshape(-1), fx.vec("contract_edges", i))
        assert np.array_equal(gq.costs, fx.vec("contract_costs", i))  # bit-exact
        assert joined == fx.scalar("contract_joined", i)
        for L in (3, 4, 5):
            lengths, nodes = O.separate(g, L)
            assert np.array_equal(lengths, fx.vec("sep%d_len" % L, i))
            assert np.array_equal(nodes.reshape(-1), fx.vec("sep%d_nodes" % L, i))
        st = O.triangulate(g, *O.separate(g, 5))
        assert np.array_equal(np.stack([st.edges_u, st.edges_v], 1).reshape(-1), fx.vec("tri_aug", i))
        assert np.array_equal(st.base_costs, fx.vec("tri_base", i))
        assert np.array_equal(st.tri_nodes.reshape(-1), fx.vec("tri_nodes", i))
        assert np.array_equal(st.tri_edges.reshape(-1), fx.vec("tri_edges", i))
        assert np.array_equal(st.coverage, fx.vec("tri_cov", i))
        assert O.lower_bound(st) == fx.scalar("lb0", i)
        O.message_passing(st, 5)
        assert np.array_equal(st.lam.reshape(-1), fx.vec("lam5", i))
        assert np.array_equal(O.reparametrized_edge_costs(st), fx.vec("cl5", i))
        assert O.lower_bound(st) == fx.scalar("lb5", i)
        gm, _, _ = O.gaec_exhaustive(g)
        assert np.array_equal(gm, fx.vec("gaec_map", i))


def test_golden_solve_all_modes():
    fx = load("solve_small.npz")
    for i in range(fx.count("edges")):
        g = _graph(fx, i)
        for mode in ("P", "PD", "PD+", "D", "GAEC"):
            sol = O.solve(g, mode=mode)
            assert np.array_equal(sol.labeling, fx.vec("labels_" + mode, i)), (i, mode)
            assert sol.primal_cost == fx.scalar("primal_" + mode, i)
            assert sol.lower_bound == fx.scalar("lb_" + mode, i)
            tr = np.array([[r.nodes, r.edges, r.triplets, r.contracted] for r in sol.trace]).reshape(-1)
            assert np.array_equal(tr, fx.vec("trace_" + mode, i))


def test_golden_grids():
    fx = load("grids.npz")
    for s in range(10):
        g = O.grid_graph(64, 64, 0, s)
        sol = O.solve(g, mode="P")
        assert np.array_equal(sol.labeling, fx.vec("c1_labels", s))
        assert sol.primal_cost == fx.scalar("c1_primal", s)
    for s in range(2):
        sol = O.solve(O.grid_graph(64, 64, 0, s), mode="PD")
        assert np.array_equal(sol.labeling, fx.vec("c1pd_labels", s))
        assert sol.primal_cost == fx.scalar("c1pd_primal", s)
        assert sol.lower_bound == fx.scalar("c1pd_lb", s)
    sol = O.solve(O.grid_graph(48, 64, 3, 7), mode="PD")
    assert np.array_equal(sol.labeling, fx.vec("s3_labels", 0))
    assert sol.primal_cost == fx.scalar("s3_primal", 0)
    assert sol.lower_bound == fx.scalar("s3_lb", 0)


def test_handshake_cleanup_equals_contraction_rounds():
    """D1: the oracle's in-place handshake cleanup equals the
    plain definition -- one select_matching round, connected_components,
    contract_graph, repeat -- on seeded random graphs and grids."""
    from paper_2109_01838_b200 import instances

    def by_contraction(g):
        fmap = np.arange(g.num_nodes, dtype=np.int64)
        cur = g
        while True:
            S = O.select_matching(cur, rounds=1)
            if S.shape[0] == 0:
                return fmap, cur.num_nodes
            f, nt = O.connected_components(cur.num_nodes, S)
            cur, _ = O.contract_graph(cur, f, nt)
            fmap = f[fmap]

    graphs = [O.Graph(*instances.random_coo(8 + s % 40, 0.3, seed=s)) for s in range(60)]
    graphs += [O.grid_graph(64, 64, 0, 0), O.grid_graph(48, 64, 3, 7)]
    for g in graphs:
        a, na = by_contraction(g)
        b, nb = O.handshake_cleanup(g)
        assert na == nb and np.array_equal(a, b)


def test_extend_separation_matches_reference_mode_d_rounds():
    """Mode D with separation_rounds 2-4 (extend_separation, dual.py:414-474)
    against the reference's own results (tests/golden/dual_rounds.npz)."""
    d = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "dual_rounds.npz"))
    for i in range(int(d["count"][0])):
        g = O.Graph(int(d["g%d_n" % i][0]), d["g%d_u" % i], d["g%d_v" % i], d["g%d_c" % i], canonical=True)
        for r in (2, 3, 4):
            sol = O.solve(g, mode="D", separation_rounds=r)
            tr = np.array([[t.edges, t.triplets] for t in sol.trace], dtype=np.int64)
            assert np.array_equal(tr, d["g%d_r%d_trace" % (i, r)]), (i, r)
            assert sol.lower_bound == pytest.approx(float(d["g%d_r%d_lb" % (i, r)][0]), rel=1e-12, abs=1e-12)


def _agreement_cases():
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "agreement.json")) as fh:
        return json.load(fh)


def test_agreement_matches_reference():
    """check_edge_triangle_agreement (dual.py:477-531) on states after 0-200
    MP iterations, against the reference's verdicts (golden/agreement.json)."""
    for case in _agreement_cases():
        g = O.Graph(case["n"], case["u"], case["v"], [float(x) for x in case["c"]], canonical=True)
        lengths, nodes = O.separate(g, 5)
        st = O.triangulate(g, lengths, nodes)
        O.message_passing(st, case["iters"])
        assert O.check_edge_triangle_agreement(st, case["eps"]) == case["agree"], case["iters"]
