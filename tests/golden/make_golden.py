"""Generate golden fixtures by running the REFERENCE parcut package.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/*.npz.  The GPU box has no /root/reference, so the
tests read only these committed fixtures.  Every array below is produced by
a reference call named in the key.
"""

import os
import sys

import numpy as np

import parcut
from parcut import dual as D

OUT = os.path.dirname(os.path.abspath(__file__))


class Pack:
    """Ragged arrays -> flat npz entries (key, key__off)."""

    def __init__(self):
        self.d = {}

    def add(self, key, arr):
        self.d.setdefault(key, []).append(np.asarray(arr))

    def scalar(self, key, x):
        self.d.setdefault(key, []).append(np.asarray([x], dtype=np.float64))

    def save(self, name):
        out = {}
        for k, parts in self.d.items():
            flat = [p.reshape(p.shape[0], int(np.prod(p.shape[1:]))) if p.ndim > 1 else p.reshape(-1, 1)
                    for p in parts]
            width = max(f.shape[1] for f in flat) if flat else 1
            rows = [np.pad(f, ((0, 0), (0, width - f.shape[1]))) for f in flat]
            out[k] = np.concatenate(rows) if rows else np.zeros((0, width))
            off = np.zeros(len(parts) + 1, np.int64)
            off[1:] = np.cumsum([f.shape[0] for f in flat])
            out[k + "__off"] = off
        np.savez_compressed(os.path.join(OUT, name), **out)
        print("wrote", name, sum(v.nbytes for v in out.values()), "bytes")


def graph_arrays(g):
    return np.stack([g.edges_u, g.edges_v], axis=1), g.costs


def small_graphs(count):
    for seed in range(count):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(4, 32))
        p = float(rng.uniform(0.15, 0.7))
        yield seed, n, p, parcut.random_graph(n, p, seed)


def solve_small():
    P = Pack()
    for seed, n, p, g in small_graphs(60):
        e, c = graph_arrays(g)
        P.add("edges", e)
        P.add("costs", c)
        P.scalar("n", n)
        for mode in ("P", "PD", "PD+", "D", "GAEC"):
            sol = parcut.solve(g, parcut.SolverConfig(mode=mode))
            P.add("labels_" + mode, sol.labeling)
            P.scalar("primal_" + mode, sol.primal_cost)
            P.scalar("lb_" + mode, sol.lower_bound)
            P.add("trace_" + mode, np.array([[r.nodes, r.edges, r.triplets, r.contracted] for r in sol.trace]))
    P.save("solve_small.npz")


def ops_small():
    P = Pack()
    for seed, n, p, g in small_graphs(60):
        rng = np.random.default_rng(1000 + seed)
        e, c = graph_arrays(g)
        P.add("edges", e)
        P.add("costs", c)
        P.scalar("n", n)
        # contraction-set strategies (contraction.py:179, 287, 166)
        P.add("matching", parcut.select_matching(g).reshape(-1, 2))
        P.add("forest", parcut.select_spanning_forest_no_conflicts(g).reshape(-1, 2))
        P.add("max_edge", parcut.select_max_edge(g).reshape(-1, 2))
        # components + contraction on a random subset S (contraction.py:101, 142)
        m = g.num_edges
        k = int(rng.integers(0, m + 1)) if m else 0
        idx = rng.choice(m, size=k, replace=False) if k else np.empty(0, np.int64)
        S = np.stack([g.edges_u[idx], g.edges_v[idx]], axis=1)
        f = parcut.connected_components(n, S)
        P.add("S", S.reshape(-1, 2))
        P.add("cc_map", f.map)
        gq, joined = parcut.contract_graph(g, f)
        eq, cq = graph_arrays(gq)
        P.add("contract_edges", eq.reshape(-1, 2))
        P.add("contract_costs", cq)
        P.scalar("contract_joined", joined)
        # separation for L = 3, 4, 5 (dual.py:169)
        for L in (3, 4, 5):
            lengths, mat = D._separate_arrays(g, L)
            P.add("sep%d_len" % L, lengths)
            P.add("sep%d_nodes" % L, mat.reshape(-1, L))
        # triangulation + 5 MP iterations + LB (dual.py:255, 389, 395)
        lengths, mat = D._separate_arrays(g, 5)
        st = D._triangulate_arrays(g, lengths, mat)
        P.add("tri_aug", np.stack([st.edges_u, st.edges_v], axis=1))
        P.add("tri_base", st.base_costs)
        P.add("tri_nodes", st.tri_nodes.reshape(-1, 3))
        P.add("tri_edges", st.tri_edges.reshape(-1, 3))
        P.add("tri_cov", st.coverage)
        P.scalar("lb0", D.lower_bound(st))
        for it in range(5):
            D.message_passing_iteration(st)
        P.add("lam5", st.lam.reshape(-1, 3))
        P.add("cl5", D.reparametrized_edge_costs(st))
        P.scalar("lb5", D.lower_bound(st))
        gm, _ = parcut.gaec_exhaustive(g)
        P.add("gaec_map", gm.map)
    P.save("ops_small.npz")


def grids():
    P = Pack()
    for seed in range(10):
        g = parcut.grid_graph(64, 64, 0, seed)
        sol = parcut.solve(g, parcut.SolverConfig(mode="P"))
        P.add("c1_labels", sol.labeling.astype(np.int32))
        P.scalar("c1_primal", sol.primal_cost)
    for seed in range(2):
        g = parcut.grid_graph(64, 64, 0, seed)
        sol = parcut.solve(g, parcut.SolverConfig(mode="PD"))
        P.add("c1pd_labels", sol.labeling.astype(np.int32))
        P.scalar("c1pd_primal", sol.primal_cost)
        P.scalar("c1pd_lb", sol.lower_bound)
        P.add("c1pd_trace", np.array([[r.nodes, r.edges, r.triplets, r.contracted] for r in sol.trace]))
    # stride-3 grid (long-range edges -> 3/4/5-cycles), PD
    g = parcut.grid_graph(48, 64, 3, 7)
    sol = parcut.solve(g, parcut.SolverConfig(mode="PD"))
    P.add("s3_labels", sol.labeling.astype(np.int32))
    P.scalar("s3_primal", sol.primal_cost)
    P.scalar("s3_lb", sol.lower_bound)
    P.add("s3_trace", np.array([[r.nodes, r.edges, r.triplets, r.contracted] for r in sol.trace]))
    P.save("grids.npz")


if __name__ == "__main__":
    which = sys.argv[1:] or ["solve_small", "ops_small", "grids"]
    for w in which:
        globals()[w]()
