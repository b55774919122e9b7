"""Edge contraction -- drop-in for ``parcut.contraction``.

Every operator runs on the GPU through the C ABI (include/rama_b200.h):
components (lock-free union-find, canonical ids), contraction (bucket sort +
numpy-order segmented reduce, bit-identical costs), handshake matching
(atomic max/min votes), and the exact conflict-free maximum spanning forest
(Boruvka + Euler tour + binary-lifting resolution of the reference's
sequential conflict pass).  ``ContractionMapping`` stays a host container
like the reference's (contraction.py:18-58).
"""

from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .graph import SparseAdjacency, WeightedGraph, build_adjacency, graph_from_device

POLICIES = {"gaec": 0, "matching": 1, "forest": 2, "auto": 3}


class ContractionMapping:
    """Surjective relabeling onto 0..num_targets-1 in canonical order (contraction.py:18-58)."""

    __slots__ = ("map", "num_targets")

    def __init__(self, map_array, num_targets):
        self.map = np.asarray(map_array, dtype=np.int64)
        self.num_targets = int(num_targets)

    @classmethod
    def identity(cls, num_nodes):
        return cls(np.arange(num_nodes, dtype=np.int64), num_nodes)

    @property
    def num_sources(self):
        return int(self.map.size)

    @property
    def is_identity(self):
        return self.num_targets == self.map.size

    def then(self, other):
        if other.map.size != self.num_targets:
            raise ValueError("cannot compose: %d targets vs %d sources" % (self.num_targets, other.map.size))
        return ContractionMapping(other.map[self.map], other.num_targets)

    def __call__(self, nodes):
        return self.map[np.asarray(nodes, dtype=np.int64)]

    def __repr__(self):
        return "ContractionMapping(%d -> %d)" % (self.map.size, self.num_targets)


@dataclass
class ContractionResult:
    contracted: SparseAdjacency
    mapping: ContractionMapping
    joined_cost: float


def _edge_array(S):
    arr = np.asarray(S, dtype=np.int64)
    if arr.size == 0:
        return arr.reshape(0, 2)
    if arr.ndim != 2 or arr.shape[1] != 2:
        raise ValueError("edge set must be an array of (u, v) pairs")
    return arr


def connected_components(num_nodes, S):
    """Mapping whose fibers are the components of (V, S) (contraction.py:101-111)."""
    S = _edge_array(S)
    if S.size and (S.min() < 0 or S.max() >= num_nodes):
        raise ValueError("contraction edge endpoint out of range")
    n = int(num_nodes)
    if n == 0:
        return ContractionMapping(np.zeros(0, np.int64), 0)
    su, sv = L.i32(S[:, 0]), L.i32(S[:, 1])
    out = L.empty_i32(n)
    nt = L.ctypes.c_int64()
    L.call("rama_components", n, L.ptr(su), L.ptr(sv), S.shape[0], L.ptr(out), L.ctypes.byref(nt), L.stream())
    return ContractionMapping(L.host_i64(out, n), nt.value)


def contract_graph(g, f):
    """Contract a WeightedGraph along a mapping -> (graph, joined) (contraction.py:142-163)."""
    if f.map.size != g.num_nodes:
        raise ValueError("mapping length does not match graph size")
    m = g.num_edges
    if m == 0:
        return WeightedGraph._from_canonical(f.num_targets, np.zeros(0, np.int64), np.zeros(0, np.int64),
                                             np.zeros(0)), 0.0
    du, dv, dc = g.device()
    dmap = L.i32(f.map)
    ou, ov, oc = L.empty_i32(m), L.empty_i32(m), L.empty_f64(m)
    mo = L.ctypes.c_int64()
    joined = L.ctypes.c_double()
    L.call("rama_contract", g.num_nodes, L.ptr(du), L.ptr(dv), L.ptr(dc), m, L.ptr(dmap), f.num_targets, L.ptr(ou),
           L.ptr(ov), L.ptr(oc), L.ctypes.byref(mo), L.ctypes.byref(joined), L.stream())
    return graph_from_device(f.num_targets, ou, ov, oc, mo.value), float(joined.value)


def contract(adj, f):
    """Contract a symmetric adjacency (contraction.py:114-139; Alg. 5).

    The symmetric form is folded to its upper triangle, contracted on the
    GPU with contract_graph, and mirrored back.
    """
    if f.map.size != adj.num_nodes:
        raise ValueError("mapping length does not match adjacency size")
    upper = adj.rows < adj.cols
    g = WeightedGraph._from_canonical(adj.num_nodes, adj.rows[upper], adj.cols[upper], adj.vals[upper])
    gq, joined = contract_graph(g, f)
    return ContractionResult(build_adjacency(gq), f, joined)


def _select(name, g, cap, *extra):
    n, m = g.num_nodes, g.num_edges
    if m == 0 or n == 0:
        return np.empty((0, 2), dtype=np.int64)
    du, dv, dc = g.device()
    su, sv = L.empty_i32(cap), L.empty_i32(cap)
    k = L.ctypes.c_int64()
    L.call(name, n, L.ptr(du), L.ptr(dv), L.ptr(dc), m, *extra, L.ptr(su), L.ptr(sv), L.ctypes.byref(k), L.stream())
    k = k.value
    return np.stack([L.host_i64(su, k), L.host_i64(sv, k)], axis=1)


def select_max_edge(g):
    """Largest strictly-positive edge, ties lexicographic (contraction.py:166-176)."""
    if g.num_edges == 0:
        return np.empty((0, 2), dtype=np.int64)
    du, dv, dc = g.device()
    e = L.ctypes.c_int64()
    L.call("rama_select_max_edge", g.num_nodes, L.ptr(du), L.ptr(dv), L.ptr(dc), g.num_edges, L.ctypes.byref(e),
           L.stream())
    if e.value < 0:
        return np.empty((0, 2), dtype=np.int64)
    return np.array([[g.edges_u[e.value], g.edges_v[e.value]]], dtype=np.int64)


def select_matching(g, seed=0, rounds=5):
    """Handshake matching of positive edges (contraction.py:179-228); seed unused as in the reference."""
    del seed
    return _select("rama_select_matching", g, g.num_nodes // 2 + 1, L.ctypes.c_int32(rounds))


def select_spanning_forest_no_conflicts(g):
    """Conflict-free maximum spanning forest (contraction.py:287-366)."""
    return _select("rama_select_forest", g, g.num_nodes + 1)


def contraction_step(g, policy, seed=0, switch_fraction=0.1):
    """One contraction round (contraction.py:369-394) -> (graph, mapping, joined)."""
    if policy not in POLICIES:
        raise ValueError("unknown contraction policy %r" % (policy,))
    del seed
    n, m = g.num_nodes, g.num_edges
    if m == 0:
        return g, ContractionMapping.identity(n), 0.0
    du, dv, dc = g.device()
    dmap = L.empty_i32(n)
    ou, ov, oc = L.empty_i32(m), L.empty_i32(m), L.empty_f64(m)
    info = (L.ctypes.c_int64 * 4)()
    joined = L.ctypes.c_double()
    L.call("rama_contraction_step", n, L.ptr(du), L.ptr(dv), L.ptr(dc), m, POLICIES[policy], float(switch_fraction),
           L.ptr(dmap), L.ptr(ou), L.ptr(ov), L.ptr(oc), info, L.ctypes.byref(joined), L.stream())
    nt, k, mo = info[0], info[1], info[2]
    if k == 0:
        return g, ContractionMapping.identity(n), 0.0
    g2 = graph_from_device(nt, ou, ov, oc, mo)
    return g2, ContractionMapping(L.host_i64(dmap, n), nt), float(joined.value)


def gaec_exhaustive(g):
    """Greedy additive edge contraction to exhaustion (contraction.py:397-452).

    Runs on the GPU as the reference's one-join-per-round form (max positive
    edge, ties lexicographic in canonical cluster ids, then contract) via the
    solver's GAEC mode; returns (ContractionMapping, joined_cost).
    """
    from .solver import SolverConfig, solve

    sol = solve(g, SolverConfig(mode="GAEC"))
    f = ContractionMapping(sol.labeling, int(sol.labeling.max()) + 1 if sol.labeling.size else 0)
    total = float(g.costs.sum()) if g.num_edges else 0.0
    return f, total - sol.primal_cost
