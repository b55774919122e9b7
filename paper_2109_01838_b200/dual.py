"""Dual machinery -- drop-in for ``parcut.dual``.

Separation, triangulation, message passing, the lower bound and the
reparametrized graph run on the GPU (dual.cu).  ``DualState`` keeps the
reference's public numpy fields (dual.py:48-106) so callers can read and set
``lam`` directly; each operator uploads the state, runs its kernels and
writes ``lam`` back.  The fused solve (solver.py) never leaves the device.
"""

from typing import NamedTuple

import numpy as np

from . import _lib as L
from .graph import WeightedGraph, graph_from_device

MC_TRIANGLE = ((0, 0, 0), (1, 1, 0), (1, 0, 1), (0, 1, 1), (1, 1, 1))


class ConflictedCycle(NamedTuple):
    """Attractive path closed by one repulsive edge (nodes[0] < nodes[-1]) (dual.py:21-36)."""

    nodes: tuple

    @property
    def repulsive_edge(self):
        return (self.nodes[0], self.nodes[-1])

    @property
    def length(self):
        return len(self.nodes)


class Triplet(NamedTuple):
    i: int
    j: int
    k: int
    e_ij: int
    e_ik: int
    e_jk: int


class DualState:
    """Edges (originals then zero-cost chords), triplets, multipliers (dual.py:48-106)."""

    __slots__ = ("graph", "num_nodes", "num_original_edges", "edges_u", "edges_v", "base_costs", "tri_nodes",
                 "tri_edges", "lam", "coverage")

    def __init__(self, graph, edges_u, edges_v, base_costs, num_original_edges, tri_nodes, tri_edges):
        self.graph = graph
        self.num_nodes = graph.num_nodes
        self.num_original_edges = int(num_original_edges)
        self.edges_u = np.asarray(edges_u, dtype=np.int64)
        self.edges_v = np.asarray(edges_v, dtype=np.int64)
        self.base_costs = np.asarray(base_costs, dtype=np.float64)
        self.tri_nodes = np.asarray(tri_nodes, dtype=np.int64).reshape(-1, 3)
        self.tri_edges = np.asarray(tri_edges, dtype=np.int64).reshape(-1, 3)
        self.lam = np.zeros((self.tri_nodes.shape[0], 3))
        self.coverage = np.bincount(self.tri_edges.ravel(), minlength=self.edges_u.size).astype(np.int64)

    @property
    def num_edges(self):
        return int(self.edges_u.size)

    @property
    def num_triplets(self):
        return int(self.tri_nodes.shape[0])

    def triplet(self, t):
        i, j, k = self.tri_nodes[t].tolist()
        a, b, c = self.tri_edges[t].tolist()
        return Triplet(i, j, k, a, b, c)

    def __repr__(self):
        return "DualState(nodes=%d, edges=%d, triplets=%d)" % (self.num_nodes, self.num_edges, self.num_triplets)

    # device views of the current state
    def _dev(self):
        return (L.f64(self.base_costs), L.i32(self.tri_edges.ravel()),
                L.f64(np.ascontiguousarray(self.lam, dtype=np.float64).ravel()))


def _separate(g, max_len):
    m = g.num_edges
    if m == 0:
        return np.zeros(0, np.int64), np.zeros((0, max(max_len, 1)), np.int64)
    du, dv, dc = g.device()
    olen, onodes = L.empty_i32(m), L.empty_i32(m * max_len)
    rows = L.ctypes.c_int64()
    L.call("rama_separate", g.num_nodes, L.ptr(du), L.ptr(dv), L.ptr(dc), m, int(max_len), L.ptr(olen), L.ptr(onodes),
           L.ctypes.byref(rows), L.stream())
    r = rows.value
    return L.host_i64(olen, r), L.host_i64(onodes, r * max_len).reshape(r, max_len)


def separate_conflicted_cycles(g, max_len):
    """One hop-shortest conflicted cycle per repulsive edge (dual.py:200-213)."""
    if max_len < 3:
        raise ValueError("max_len must be at least 3")
    lengths, mat = _separate(g, max_len)
    return [ConflictedCycle(tuple(mat[i, : lengths[i]].tolist())) for i in np.flatnonzero(lengths)]


def _triangulate_arrays(g, lengths, mat):
    lengths = np.asarray(lengths, dtype=np.int64)
    rows = lengths.size
    L_ = int(mat.shape[1]) if rows else 3
    n, m = g.num_nodes, g.num_edges
    if g.num_edges:
        du, dv, dc = g.device()
    else:
        du = dv = L.empty_i32(1)
        dc = L.empty_f64(1)
    dl = L.i32(lengths) if rows else L.empty_i32(1)
    dn = L.i32(np.asarray(mat).ravel()) if rows else L.empty_i32(1)
    ntri = int(np.maximum(lengths - 2, 0).sum()) if rows else 0
    nch = int(np.maximum(lengths - 3, 0).sum()) if rows else 0
    au, av, ab, cov = L.empty_i32(m + nch), L.empty_i32(m + nch), L.empty_f64(m + nch), L.empty_i32(m + nch)
    tn, te = L.empty_i32(3 * ntri), L.empty_i32(3 * ntri)
    ma, T = L.ctypes.c_int64(), L.ctypes.c_int64()
    L.call("rama_triangulate", n, L.ptr(du), L.ptr(dv), L.ptr(dc), m, L.ptr(dl), L.ptr(dn), rows, L_, L.ptr(au),
           L.ptr(av), L.ptr(ab), L.ctypes.byref(ma), L.ptr(tn), L.ptr(te), L.ctypes.byref(T), L.ptr(cov), L.stream())
    k, t = ma.value, T.value
    st = object.__new__(DualState)
    st.graph = g
    st.num_nodes = n
    st.num_original_edges = m
    st.edges_u = L.host_i64(au, k)
    st.edges_v = L.host_i64(av, k)
    st.base_costs = L.host_f64(ab, k)
    st.tri_nodes = L.host_i64(tn, 3 * t).reshape(t, 3)
    st.tri_edges = L.host_i64(te, 3 * t).reshape(t, 3)
    st.lam = np.zeros((t, 3))
    st.coverage = L.host_i64(cov, k)
    return st


def triangulate(cycles, g):
    """Fan triangulation into a DualState (dual.py:293-306)."""
    lengths = np.array([c.length for c in cycles], dtype=np.int64)
    width = int(lengths.max()) if lengths.size else 3
    mat = np.zeros((len(cycles), max(width, 3)), dtype=np.int64)
    for r, cyc in enumerate(cycles):
        mat[r, : lengths[r]] = cyc.nodes
    return _triangulate_arrays(g, lengths, mat)


def reparametrized_edge_costs(state):
    """c^lambda = base + per-edge sum of covering multipliers (dual.py:309-316)."""
    if state.num_edges == 0:
        return np.zeros(0)
    base, te, lam = state._dev()
    cl = L.empty_f64(state.num_edges)
    L.call("rama_reparam_costs", state.num_edges, L.ptr(base), state.num_triplets, L.ptr(te), L.ptr(lam), L.ptr(cl),
           L.stream())
    return L.host_f64(cl, state.num_edges)


def _mp(state, iters, phases):
    if state.num_triplets == 0:
        return
    base, te, lam = state._dev()
    L.call("rama_message_passing", state.num_edges, L.ptr(base), state.num_triplets, L.ptr(te), L.ptr(lam), iters,
           phases, L.stream())
    state.lam = L.host_f64(lam, 3 * state.num_triplets).reshape(-1, 3)


def mp_edge_to_triplets(state):
    """Edge phase of Alg. 2 (dual.py:358-368)."""
    _mp(state, 1, 1)


def mp_triplets_to_edges(state):
    """Damped six-step triplet phase (dual.py:374-386)."""
    _mp(state, 1, 2)


def message_passing_iteration(state):
    """One edge phase + triplet phase (dual.py:389-392)."""
    _mp(state, 1, 3)


def message_passing(state, iterations):
    """``iterations`` consecutive message_passing_iteration calls on the device."""
    _mp(state, int(iterations), 3)


def lower_bound(state):
    """LB(lambda) of Eq. 5 (dual.py:395-405)."""
    if state.num_edges == 0 and state.num_triplets == 0:
        return 0.0
    base, te, lam = state._dev() if state.num_edges else (L.empty_f64(1), L.empty_i32(1), L.empty_f64(1))
    out = L.ctypes.c_double()
    L.call("rama_lower_bound", state.num_edges, L.ptr(base), state.num_triplets, L.ptr(te), L.ptr(lam),
           L.ctypes.byref(out), L.stream())
    return float(out.value)


def reparametrized_graph(state):
    """WeightedGraph over augmented edges with c^lambda (dual.py:408-411)."""
    cl = reparametrized_edge_costs(state)
    return WeightedGraph(state.num_nodes, state.edges_u, state.edges_v, cl)


def triangle_min_marginal(state, t, e):
    """Min-marginal of edge e in triplet t by enumerating MC_TRIANGLE (dual.py:339-355).

    A scalar API helper (host arithmetic on three numbers), not a hot path.
    """
    slots = state.tri_edges[t]
    hit = np.flatnonzero(slots == e)
    if hit.size == 0:
        raise ValueError("edge %d is not part of triplet %d" % (e, t))
    s = int(hit[0])
    lam = state.lam[t]
    on, off = np.inf, np.inf
    for y in MC_TRIANGLE:
        cost = -(lam[0] * y[0] + lam[1] * y[1] + lam[2] * y[2])
        if y[s]:
            on = min(on, cost)
        else:
            off = min(off, cost)
    return float(on - off)


def extend_separation(state, max_len):
    """Separate on the current reparametrized costs and add new triplets
    (dual.py:414-474): new chords join at base cost 0, new triplets start
    with zero multipliers.  Returns the number of triplets added."""
    if max_len < 3:
        raise ValueError("max_len must be at least 3")
    m, T, n = state.num_edges, state.num_triplets, state.num_nodes
    if m == 0:
        return 0
    extra = m * max(max_len - 2, 1)
    eu, ev, base = L.i32(state.edges_u), L.i32(state.edges_v), L.f64(state.base_costs)
    tn = L.i32(state.tri_nodes.ravel()) if T else L.empty_i32(1)
    te = L.i32(state.tri_edges.ravel()) if T else L.empty_i32(1)
    lam = L.f64(np.ascontiguousarray(state.lam).ravel()) if T else L.empty_f64(1)
    oeu, oev, obase, ocov = L.empty_i32(m + extra), L.empty_i32(m + extra), L.empty_f64(m + extra), \
        L.empty_i32(m + extra)
    otn, ote, olam = L.empty_i32(3 * (T + extra)), L.empty_i32(3 * (T + extra)), L.empty_f64(3 * (T + extra))
    om, oT, added = L.ctypes.c_int64(), L.ctypes.c_int64(), L.ctypes.c_int64()
    L.call("rama_extend_separation", n, m, L.ptr(eu), L.ptr(ev), L.ptr(base), T, L.ptr(tn), L.ptr(te), L.ptr(lam),
           int(max_len), m + extra, T + extra, L.ptr(oeu), L.ptr(oev), L.ptr(obase), L.ctypes.byref(om),
           L.ptr(otn), L.ptr(ote), L.ptr(olam), L.ctypes.byref(oT), L.ptr(ocov), L.ctypes.byref(added),
           L.stream())
    k, t = om.value, oT.value
    state.edges_u = L.host_i64(oeu, k)
    state.edges_v = L.host_i64(oev, k)
    state.base_costs = L.host_f64(obase, k)
    state.tri_nodes = L.host_i64(otn, 3 * t).reshape(t, 3)
    state.tri_edges = L.host_i64(ote, 3 * t).reshape(t, 3)
    state.lam = L.host_f64(olam, 3 * t).reshape(t, 3)
    state.coverage = L.host_i64(ocov, k)
    return int(added.value)


def check_edge_triangle_agreement(state, eps):
    """Arc consistency of the eps-optimal edge and triplet label sets
    (dual.py:477-531): True iff every set stays non-empty.  On the device
    (rama_check_agreement: Jacobi sweeps until no bit changes)."""
    if eps < 0:
        raise ValueError("eps must be non-negative")
    if state.num_edges == 0:
        return True
    base, te, lam = state._dev()
    if state.num_triplets == 0:
        te, lam = L.empty_i32(1), L.empty_f64(1)
    out = L.ctypes.c_int32()
    L.call("rama_check_agreement", state.num_edges, L.ptr(base), state.num_triplets, L.ptr(te), L.ptr(lam),
           float(eps), L.ctypes.byref(out), L.stream())
    return bool(out.value)
