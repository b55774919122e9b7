"""CPU oracle for the RAMA primal-dual hot path -- TEST INFRASTRUCTURE.

A plain-C restatement (``rama_oracle.c``) of the reference ``parcut``
solver (``/root/reference/pkg/src/parcut``), driven from Python the way
``parcut.solver`` drives its kernels.  It is the checker for the B200
kernels and the CPU baseline timed by ``bench.py``; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` may import it.  The product
package (``paper_2109_01838_b200``) never imports this module.

Parity pinning: ``tests/test_oracle.py`` checks every function here
against the reference's own known-answer tests (pkg/tests/*.py) and
against golden fixtures generated from the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``).

Build: ``python -m oracle.build`` (gcc -O2, output under
``oracle/_build/``); ``__graft_entry__.build()`` runs it too.
"""

import ctypes
import os
import time
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "librama_oracle.so")
_lib = None

_I64P = ctypes.POINTER(ctypes.c_int64)
_F64P = ctypes.POINTER(ctypes.c_double)


def build(force=False):
    """Compile rama_oracle.c with gcc into oracle/_build/."""
    src = os.path.join(_HERE, "rama_oracle.c")
    if not force and os.path.exists(_SO) and os.path.getmtime(_SO) >= os.path.getmtime(src):
        return _SO
    os.makedirs(os.path.dirname(_SO), exist_ok=True)
    tmp = _SO + ".tmp%d" % os.getpid()
    cmd = "gcc -O2 -fno-fast-math -ffp-contract=off -fPIC -shared -o %s %s" % (tmp, src)
    if os.system(cmd) != 0:
        raise RuntimeError("oracle build failed: " + cmd)
    os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        _lib = ctypes.CDLL(_SO)
        _lib.orc_np_sum.restype = ctypes.c_double
        _lib.orc_seg_sum.restype = ctypes.c_double
        _lib.orc_clustering_cost.restype = ctypes.c_double
        _lib.orc_lower_bound.restype = ctypes.c_double
    return _lib


def _p64(a):
    return a.ctypes.data_as(_I64P)


def _pf(a):
    return a.ctypes.data_as(_F64P)


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64).ravel())


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).ravel())


def _check(rc):
    if rc == -1:
        raise ValueError("self-loops are not allowed")
    if rc == -2:
        raise ValueError("edge endpoint out of range")
    if rc == -3:
        raise ValueError("invalid argument")
    if rc != 0:
        raise RuntimeError("oracle error %d" % rc)


# ------------------------------------------------------------------ graphs

class Graph:
    """Canonical COO (u < v, sorted, unique), like parcut.WeightedGraph."""

    __slots__ = ("num_nodes", "edges_u", "edges_v", "costs")

    def __init__(self, num_nodes, edges_u=(), edges_v=(), costs=(), canonical=False):
        u, v, c = _i64(edges_u), _i64(edges_v), _f64(costs)
        if not (u.shape == v.shape == c.shape):
            raise ValueError("edge arrays must have equal length")
        if num_nodes < 0:
            raise ValueError("num_nodes must be non-negative")
        self.num_nodes = int(num_nodes)
        if canonical:
            self.edges_u, self.edges_v, self.costs = u, v, c
            return
        m = u.size
        ou, ov, oc = np.empty(m, np.int64), np.empty(m, np.int64), np.empty(m)
        mo = ctypes.c_int64()
        _check(lib().orc_canonicalize(ctypes.c_int64(self.num_nodes), ctypes.c_int64(m),
                                      _p64(u), _p64(v), _pf(c), _p64(ou), _p64(ov), _pf(oc),
                                      ctypes.byref(mo)))
        k = mo.value
        self.edges_u, self.edges_v, self.costs = ou[:k].copy(), ov[:k].copy(), oc[:k].copy()

    @property
    def num_edges(self):
        return int(self.edges_u.size)


def np_sum(a):
    a = _f64(a)
    return lib().orc_np_sum(_pf(a), ctypes.c_int64(a.size))


def seg_sum(a):
    a = _f64(a)
    return lib().orc_seg_sum(_pf(a), ctypes.c_int64(a.size))


def clustering_cost(g, labels):
    lab = _i64(labels)
    if lab.shape != (g.num_nodes,):
        raise ValueError("labeling length mismatch")
    return lib().orc_clustering_cost(ctypes.c_int64(g.num_edges), _p64(g.edges_u),
                                     _p64(g.edges_v), _pf(g.costs), _p64(lab))


# ------------------------------------------------------------- contraction

def connected_components(n, S):
    """-> (map int64[n], num_targets); contraction.py:101-111."""
    S = np.asarray(S, dtype=np.int64).reshape(-1, 2)
    su, sv = _i64(S[:, 0]), _i64(S[:, 1])
    out = np.empty(n, np.int64)
    nt = ctypes.c_int64()
    _check(lib().orc_components(ctypes.c_int64(n), ctypes.c_int64(su.size), _p64(su), _p64(sv),
                                _p64(out), ctypes.byref(nt)))
    return out, nt.value


def contract_graph(g, fmap, n_targets):
    """-> (Graph, joined); contraction.py:142-163."""
    fmap = _i64(fmap)
    m = g.num_edges
    ou, ov, oc = np.empty(m, np.int64), np.empty(m, np.int64), np.empty(m)
    mo = ctypes.c_int64()
    joined = ctypes.c_double()
    _check(lib().orc_contract(ctypes.c_int64(g.num_nodes), ctypes.c_int64(m), _p64(g.edges_u),
                              _p64(g.edges_v), _pf(g.costs), _p64(fmap), ctypes.c_int64(n_targets),
                              _p64(ou), _p64(ov), _pf(oc), ctypes.byref(mo), ctypes.byref(joined)))
    k = mo.value
    return Graph(n_targets, ou[:k].copy(), ov[:k].copy(), oc[:k].copy(), canonical=True), joined.value


def select_max_edge(g):
    idx = ctypes.c_int64()
    lib().orc_max_edge(ctypes.c_int64(g.num_edges), _pf(g.costs), ctypes.byref(idx))
    if idx.value < 0:
        return np.empty((0, 2), np.int64)
    return np.array([[g.edges_u[idx.value], g.edges_v[idx.value]]], np.int64)


def select_matching(g, rounds=5):
    """contraction.py:179-228."""
    n, m = g.num_nodes, g.num_edges
    ou, ov = np.empty(max(n // 2, 1), np.int64), np.empty(max(n // 2, 1), np.int64)
    k = ctypes.c_int64()
    lib().orc_matching(ctypes.c_int64(n), ctypes.c_int64(m), _p64(g.edges_u), _p64(g.edges_v),
                       _pf(g.costs), ctypes.c_int(rounds), _p64(ou), _p64(ov), ctypes.byref(k))
    return np.stack([ou[:k.value], ov[:k.value]], axis=1)


def select_spanning_forest_no_conflicts(g):
    """contraction.py:287-366."""
    n, m = g.num_nodes, g.num_edges
    cap = max(n, 1)
    ou, ov = np.empty(cap, np.int64), np.empty(cap, np.int64)
    k = ctypes.c_int64()
    lib().orc_forest(ctypes.c_int64(n), ctypes.c_int64(m), _p64(g.edges_u), _p64(g.edges_v),
                     _pf(g.costs), _p64(ou), _p64(ov), ctypes.byref(k))
    return np.stack([ou[:k.value], ov[:k.value]], axis=1)


def contraction_step(g, policy="auto", switch_fraction=0.1):
    """contraction.py:369-394 -> (graph', map, num_targets, joined, |S|)."""
    if policy == "gaec":
        S = select_max_edge(g)
    elif policy == "matching":
        S = select_matching(g)
    elif policy == "forest":
        S = select_spanning_forest_no_conflicts(g)
    elif policy == "auto":
        S = select_matching(g)
        if S.shape[0] < switch_fraction * g.num_nodes:
            S = select_spanning_forest_no_conflicts(g)
    else:
        raise ValueError("unknown contraction policy %r" % (policy,))
    if S.shape[0] == 0:
        return g, np.arange(g.num_nodes, dtype=np.int64), g.num_nodes, 0.0, 0
    fmap, nt = connected_components(g.num_nodes, S)
    g2, joined = contract_graph(g, fmap, nt)
    return g2, fmap, nt, joined, int(S.shape[0])


def gaec_exhaustive(g):
    """contraction.py:397-452 -> (map, num_targets, joined)."""
    out = np.empty(g.num_nodes, np.int64)
    nt = ctypes.c_int64()
    joined = ctypes.c_double()
    lib().orc_gaec(ctypes.c_int64(g.num_nodes), ctypes.c_int64(g.num_edges), _p64(g.edges_u),
                   _p64(g.edges_v), _pf(g.costs), _p64(out), ctypes.byref(nt), ctypes.byref(joined))
    return out, nt.value, joined.value


def handshake_cleanup(g, with_rounds=False):
    """The B200 build's parallel cleanup (deviation D1): repeated
    handshake rounds on the quotient under its own costs, merged pairs keep
    the smaller id, parallel edges fold into the smallest edge slot with a
    sequential sum (rama_oracle.c orc_cleanup_handshake)."""
    out = np.empty(g.num_nodes, np.int64)
    nt = ctypes.c_int64()
    rounds = ctypes.c_int64()
    lib().orc_cleanup_handshake(ctypes.c_int64(g.num_nodes), ctypes.c_int64(g.num_edges), _p64(g.edges_u),
                                _p64(g.edges_v), _pf(g.costs), _p64(out), ctypes.byref(nt), ctypes.byref(rounds))
    if with_rounds:
        return out, nt.value, rounds.value
    return out, nt.value


# -------------------------------------------------------------------- dual

def separate(g, L):
    """_separate_arrays (dual.py:169-197) -> (lengths, nodes[rows, L])."""
    if L < 3:
        raise ValueError("max_len must be at least 3")
    m = g.num_edges
    nneg = int(np.count_nonzero(g.costs < 0.0))
    out_len = np.zeros(max(nneg, 1), np.int64)
    out_nodes = np.zeros((max(nneg, 1), L), np.int64)
    nn = ctypes.c_int64()
    _check(lib().orc_separate(ctypes.c_int64(g.num_nodes), ctypes.c_int64(m), _p64(g.edges_u),
                              _p64(g.edges_v), _pf(g.costs), ctypes.c_int(L), _p64(out_len),
                              _p64(out_nodes), ctypes.byref(nn)))
    return out_len[:nneg].copy(), out_nodes[:nneg].copy()


@dataclass
class DualState:
    num_nodes: int
    num_original_edges: int
    edges_u: np.ndarray
    edges_v: np.ndarray
    base_costs: np.ndarray
    tri_nodes: np.ndarray
    tri_edges: np.ndarray
    coverage: np.ndarray
    lam: np.ndarray

    @property
    def num_edges(self):
        return int(self.edges_u.size)

    @property
    def num_triplets(self):
        return int(self.tri_nodes.shape[0])


def triangulate(g, lengths, nodes):
    """_triangulate_arrays (dual.py:255-290)."""
    lengths = _i64(lengths)
    rows = lengths.size
    L = int(nodes.shape[1]) if rows else 3
    nodes = _i64(nodes) if rows else np.zeros(3, np.int64)
    ntri = int(np.sum(np.maximum(lengths - 2, 0))) if rows else 0
    nch = int(np.sum(np.maximum(lengths - 3, 0))) if rows else 0
    m = g.num_edges
    aug_u = np.empty(m + nch, np.int64)
    aug_v = np.empty(m + nch, np.int64)
    base = np.empty(m + nch)
    cov = np.empty(m + nch, np.int64)
    tri_nodes = np.empty((max(ntri, 1), 3), np.int64)
    tri_edges = np.empty((max(ntri, 1), 3), np.int64)
    ma, T = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().orc_triangulate(ctypes.c_int64(g.num_nodes), ctypes.c_int64(m), _p64(g.edges_u),
                                 _p64(g.edges_v), _pf(g.costs), ctypes.c_int64(rows), ctypes.c_int(L),
                                 _p64(lengths), _p64(nodes), _p64(aug_u), _p64(aug_v), _pf(base),
                                 ctypes.byref(ma), _p64(tri_nodes), _p64(tri_edges), ctypes.byref(T),
                                 _p64(cov)))
    k, t = ma.value, T.value
    return DualState(g.num_nodes, m, aug_u[:k].copy(), aug_v[:k].copy(), base[:k].copy(),
                     tri_nodes[:t].copy(), tri_edges[:t].copy(), cov[:k].copy(), np.zeros((t, 3)))


def reparametrized_edge_costs(st):
    cl = np.empty(st.num_edges)
    lam = np.ascontiguousarray(st.lam)
    te = np.ascontiguousarray(st.tri_edges)
    lib().orc_reparam(ctypes.c_int64(st.num_edges), _pf(st.base_costs), ctypes.c_int64(st.num_triplets),
                      _p64(te), _pf(lam), _pf(cl))
    return cl


def message_passing(st, iterations=1):
    """message_passing_iteration (dual.py:389-392), in place on st.lam."""
    if st.num_triplets == 0:
        return
    st.lam = np.ascontiguousarray(st.lam)
    te = np.ascontiguousarray(st.tri_edges)
    lib().orc_mp(ctypes.c_int64(st.num_edges), _pf(st.base_costs), _p64(st.coverage),
                 ctypes.c_int64(st.num_triplets), _p64(te), _pf(st.lam), ctypes.c_int(iterations))


def lower_bound(st):
    lam = np.ascontiguousarray(st.lam)
    te = np.ascontiguousarray(st.tri_edges)
    return lib().orc_lower_bound(ctypes.c_int64(st.num_edges), _pf(st.base_costs),
                                 ctypes.c_int64(st.num_triplets), _p64(te), _pf(lam))


def _dedupe_rows(arr):
    """dual.py:214-224: lexicographic sort, drop consecutive duplicates."""
    if arr.shape[0] == 0:
        return arr
    order = np.lexsort(tuple(arr[:, col] for col in range(arr.shape[1] - 1, -1, -1)))
    arr = arr[order]
    keep = np.empty(arr.shape[0], dtype=bool)
    keep[0] = True
    keep[1:] = np.any(arr[1:] != arr[:-1], axis=1)
    return arr[keep]


def _fan_arrays(lengths, mat):
    """dual.py:228-252: fan triplets (sorted rows, deduped) and chords."""
    tri, chords = [], []
    max_l = int(lengths.max()) if lengths.size else 0
    for ln in range(3, max_l + 1):
        rows = np.flatnonzero(lengths == ln)
        if rows.size == 0:
            continue
        v0 = mat[rows, 0]
        for k in range(1, ln - 1):
            tri.append(np.stack([v0, mat[rows, k], mat[rows, k + 1]], axis=1))
        for k in range(2, ln - 1):
            b = mat[rows, k]
            chords.append(np.stack([np.minimum(v0, b), np.maximum(v0, b)], axis=1))
    tri_nodes = np.concatenate(tri, axis=0) if tri else np.zeros((0, 3), np.int64)
    tri_nodes = _dedupe_rows(np.sort(tri_nodes, axis=1))
    chord_pairs = np.concatenate(chords, axis=0) if chords else np.zeros((0, 2), np.int64)
    return tri_nodes, _dedupe_rows(chord_pairs)


def extend_separation(st, L):
    """dual.py:414-474 (numpy restatement): separate on the reparametrized
    costs, append new chords (base 0) and new triplets (zero multipliers).
    Returns the number of triplets added."""
    g_rep = Graph(st.num_nodes, st.edges_u.copy(), st.edges_v.copy(), reparametrized_edge_costs(st))
    lengths, mat = separate(g_rep, L)
    keep = lengths >= 3
    tri_nodes, chord_pairs = _fan_arrays(lengths[keep], mat[keep])
    if tri_nodes.shape[0] == 0:
        return 0
    n = st.num_nodes
    keys = st.edges_u * n + st.edges_v
    if chord_pairs.shape[0]:
        order = np.argsort(keys, kind="stable")
        ckeys = chord_pairs[:, 0] * n + chord_pairs[:, 1]
        pos = np.searchsorted(keys[order], ckeys)
        pos_c = np.minimum(pos, max(keys.size - 1, 0))
        hit = (pos < keys.size) & (keys[order][pos_c] == ckeys)
        chord_pairs = chord_pairs[~hit]
    st.edges_u = np.concatenate([st.edges_u, chord_pairs[:, 0]])
    st.edges_v = np.concatenate([st.edges_v, chord_pairs[:, 1]])
    st.base_costs = np.concatenate([st.base_costs, np.zeros(chord_pairs.shape[0])])
    if st.tri_nodes.shape[0]:
        both = np.concatenate([st.tri_nodes, tri_nodes])
        flags = np.concatenate([np.zeros(st.tri_nodes.shape[0], bool), np.ones(tri_nodes.shape[0], bool)])
        order = np.lexsort((both[:, 2], both[:, 1], both[:, 0]))
        both, flags = both[order], flags[order]
        dup = np.zeros(both.shape[0], dtype=bool)
        dup[1:] = np.all(both[1:] == both[:-1], axis=1)
        tri_nodes = _dedupe_rows(both[flags & ~dup])
    if tri_nodes.shape[0] == 0:
        st.coverage = np.bincount(st.tri_edges.ravel(), minlength=st.edges_u.size).astype(np.int64)
        return 0
    keys = st.edges_u * n + st.edges_v
    order = np.argsort(keys, kind="stable")
    sorted_keys = keys[order]

    def handles(a, b):
        return order[np.searchsorted(sorted_keys, a * n + b)]

    i, j, k = tri_nodes[:, 0], tri_nodes[:, 1], tri_nodes[:, 2]
    new_edges = np.stack([handles(i, j), handles(i, k), handles(j, k)], axis=1)
    added = tri_nodes.shape[0]
    st.tri_nodes = np.concatenate([st.tri_nodes, tri_nodes])
    st.tri_edges = np.concatenate([st.tri_edges, new_edges])
    st.lam = np.concatenate([st.lam, np.zeros((added, 3))])
    st.coverage = np.bincount(st.tri_edges.ravel(), minlength=st.edges_u.size).astype(np.int64)
    return added


_MC = np.array([(0, 0, 0), (1, 1, 0), (1, 0, 1), (0, 1, 1), (1, 1, 1)], dtype=np.int8)  # dual.py:17-18


def check_edge_triangle_agreement(st, eps):
    """dual.py:477-531 (numpy restatement): arc-consistent kernel of the
    eps-optimal edge / triplet label sets is non-empty."""
    if eps < 0:
        raise ValueError("eps must be non-negative")
    cl = reparametrized_edge_costs(st)
    best = np.minimum(cl, 0.0)
    em = np.zeros(cl.size, dtype=np.uint8)
    em[0.0 <= best + eps] |= 1
    em[cl <= best + eps] |= 2
    T = st.num_triplets
    if T == 0:
        return bool(np.all(em != 0))
    lam = np.asarray(st.lam).reshape(-1, 3)
    l0, l1, l2 = lam[:, 0], lam[:, 1], lam[:, 2]
    pc = np.stack([np.zeros(T), -(l0 + l1), -(l0 + l2), -(l1 + l2), -((l0 + l1) + l2)], axis=1)
    tb = pc.min(axis=1)
    tm = np.zeros(T, dtype=np.uint8)
    for p in range(5):
        tm[pc[:, p] <= tb + eps] |= np.uint8(1 << p)
    e = np.asarray(st.tri_edges).reshape(-1, 3)
    zero_bits = [sum(1 << p for p in range(5) if _MC[p, s] == 0) for s in range(3)]
    one_bits = [sum(1 << p for p in range(5) if _MC[p, s] == 1) for s in range(3)]
    while True:
        oe, ot = em.copy(), tm.copy()
        for p in range(5):
            ok = np.ones(T, dtype=bool)
            for s in range(3):
                ok &= (em[e[:, s]] & np.uint8(1 << _MC[p, s])) != 0
            tm[~ok] &= np.uint8(~np.uint8(1 << p))
        for s in range(3):
            em[e[(tm & zero_bits[s]) == 0, s]] &= np.uint8(~np.uint8(1))
            em[e[(tm & one_bits[s]) == 0, s]] &= np.uint8(~np.uint8(2))
        if np.array_equal(em, oe) and np.array_equal(tm, ot):
            break
    return bool(np.all(em != 0) and np.all(tm != 0))


def reparametrized_graph(st):
    """dual.py:408-411 (re-canonicalised)."""
    return Graph(st.num_nodes, st.edges_u, st.edges_v, reparametrized_edge_costs(st))


# ------------------------------------------------------------------ solver

@dataclass
class Round:
    round_index: int
    phase: str
    nodes: int
    edges: int
    triplets: int
    lb: float
    lb_valid: bool
    contracted: int
    time_ms: float


@dataclass
class Result:
    labeling: np.ndarray
    primal_cost: float
    lower_bound: float
    trace: list = field(default_factory=list)


_LDEF = {"P": 5, "PD": 5, "PD+": 7, "D": 5, "GAEC": 5}


def solve(g, mode="PD", mp_iterations=5, max_cycle_length=None, matching_switch_fraction=0.1,
          max_rounds=100, cleanup="gaec", separation_rounds=1):
    """solver.py:113-240.  cleanup='gaec' follows the reference exactly
    (solver.py:187-207); cleanup='handshake' follows the B200 build."""
    L = _LDEF.get(mode, 5) if max_cycle_length is None else int(max_cycle_length)
    n0 = g.num_nodes
    if mode == "GAEC":
        t0 = time.perf_counter()
        fmap, nt, _ = gaec_exhaustive(g)
        rec = Round(1, "gaec", n0, g.num_edges, 0, None, False, n0 - nt,
                    (time.perf_counter() - t0) * 1e3)
        return Result(fmap, clustering_cost(g, fmap), float("-inf"), [rec])
    if mode == "D":  # solver.py:211-240
        st, lb, trace = None, None, []
        for rnd in range(1, separation_rounds + 1):
            t0 = time.perf_counter()
            if st is None:
                lengths, nodes = separate(g, L)
                st = triangulate(g, lengths, nodes)
            else:
                extend_separation(st, L)
            message_passing(st, mp_iterations)
            lb = lower_bound(st)
            trace.append(Round(rnd, "dual", n0, st.num_edges, st.num_triplets, lb, True, 0,
                               (time.perf_counter() - t0) * 1e3))
        lab = np.arange(n0, dtype=np.int64)
        return Result(lab, clustering_cost(g, lab), lb, trace)
    f_total = np.arange(n0, dtype=np.int64)
    cur = g
    lb = None
    trace = []
    dual = mode in ("PD", "PD+")
    for rnd in range(1, max_rounds + 1):
        t0 = time.perf_counter()
        nb, eb = cur.num_nodes, cur.num_edges
        T = 0
        lb_r = None
        if dual:
            lengths, nodes = separate(cur, L)
            st = triangulate(cur, lengths, nodes)
            message_passing(st, mp_iterations)
            lb_r = lower_bound(st)
            T = st.num_triplets
            if rnd == 1:
                lb = lb_r
            work = reparametrized_graph(st)
        else:
            work = cur
        nxt, f, nt, _, k = contraction_step(work, "auto", matching_switch_fraction)
        trace.append(Round(rnd, "primal-dual" if dual else "contract", nb, eb, T, lb_r,
                           dual and rnd == 1, nb - nt, (time.perf_counter() - t0) * 1e3))
        if nt == cur.num_nodes:
            break
        f_total = f[f_total]
        cur = nxt
        if cur.num_nodes <= 1:
            break
    if not dual:
        return Result(f_total, clustering_cost(g, f_total), float("-inf"), trace)
    t0 = time.perf_counter()
    ntq = int(f_total.max()) + 1 if n0 else 0
    quotient, _ = contract_graph(g, f_total, ntq)
    if cleanup == "gaec":
        fc, ntc, _ = gaec_exhaustive(quotient)
    else:
        fc, ntc = handshake_cleanup(quotient)
    trace.append(Round(len(trace) + 1, "cleanup", quotient.num_nodes, quotient.num_edges, 0, None,
                       False, quotient.num_nodes - ntc, (time.perf_counter() - t0) * 1e3))
    lab = fc[f_total]
    return Result(lab, clustering_cost(g, lab), lb, trace)


# -------------------------------------------------------------- generators

def grid_graph(height, width, stride=0, seed=0):
    """Same instance as parcut.grid_graph (generate.py:28-62): row-major
    4-connected grid, optional coarse lattice (right then down), costs from
    one default_rng(seed).standard_normal draw in that block order."""
    ids = np.arange(height * width, dtype=np.int64).reshape(height, width)
    us = [ids[:, :-1].ravel(), ids[:-1, :].ravel()]
    vs = [ids[:, 1:].ravel(), ids[1:, :].ravel()]
    if stride >= 2:
        r, c = np.meshgrid(np.arange(0, height, stride), np.arange(0, width, stride), indexing="ij")
        ok = c + stride < width
        us.append(ids[r[ok], c[ok]])
        vs.append(ids[r[ok], c[ok] + stride])
        ok = r + stride < height
        us.append(ids[r[ok], c[ok]])
        vs.append(ids[r[ok] + stride, c[ok]])
    u, v = np.concatenate(us), np.concatenate(vs)
    cost = np.random.default_rng(seed).standard_normal(u.size)
    return Graph(height * width, u, v, cost)


def random_graph(num_nodes, p, seed=0):
    """Same instance as parcut.random_graph (generate.py:8-25)."""
    rng = np.random.default_rng(seed)
    iu, iv = np.triu_indices(num_nodes, k=1)
    keep = rng.random(iu.size) < p
    u, v = iu[keep].astype(np.int64), iv[keep].astype(np.int64)
    return Graph(num_nodes, u, v, rng.standard_normal(u.size))
