"""Instance types and the objective -- drop-in for ``parcut.graph``.

``WeightedGraph`` keeps the reference's public layout (numpy int64
``edges_u``/``edges_v`` with u < v sorted unique, float64 ``costs``;
graph.py:17-57) but canonicalises on the GPU (``rama_canonicalize``: bucket
sort + numpy-order segmented sums) and caches its device copy, so solves and
operator calls on the same instance upload it once.
"""

import numpy as np

from . import _lib as L


class ParseError(ValueError):
    """Raised when instance text does not follow the MULTICUT format (graph.py:13)."""


class WeightedGraph:
    """Undirected graph with fp64 edge costs and dense 0-based node ids.

    Canonical form (graph.py:17-28): u < v, sorted by (u, v), one entry per
    pair; parallel input edges are summed.  Immutable after construction.
    """

    __slots__ = ("num_nodes", "edges_u", "edges_v", "costs", "_dev")

    def __init__(self, num_nodes, edges_u=(), edges_v=(), costs=()):
        num_nodes = int(num_nodes)
        if num_nodes < 0:
            raise ValueError("num_nodes must be non-negative")
        u = _as_i64(edges_u)
        v = _as_i64(edges_v)
        c = _as_f64(costs)
        if not (u.shape == v.shape == c.shape):
            raise ValueError("edge arrays must have equal length")
        self.num_nodes = num_nodes
        self._dev = None
        if u.size == 0:
            self.edges_u, self.edges_v, self.costs = u, v, c
            return
        # validation messages of graph.py:38-42 (checked on the host arrays
        # the caller handed in; the device kernel re-checks)
        if np.any(u == v):
            raise ValueError("self-loops are not allowed")
        if min(u.min(), v.min()) < 0 or max(u.max(), v.max()) >= num_nodes:
            raise ValueError("edge endpoint out of range")
        m = u.size
        du, dv, dc = L.i32(u), L.i32(v), L.f64(c)
        ou, ov, oc = L.empty_i32(m), L.empty_i32(m), L.empty_f64(m)
        mo = L.ctypes.c_int64()
        L.call("rama_canonicalize", num_nodes, L.ptr(du), L.ptr(dv), L.ptr(dc), m, L.ptr(ou), L.ptr(ov), L.ptr(oc),
               L.ctypes.byref(mo), L.stream())
        k = mo.value
        self._dev = (ou[:k], ov[:k], oc[:k])
        self.edges_u = L.host_i64(ou, k)
        self.edges_v = L.host_i64(ov, k)
        self.costs = L.host_f64(oc, k)

    @classmethod
    def from_edges(cls, num_nodes, triples):
        triples = list(triples)
        return cls(num_nodes, [t[0] for t in triples], [t[1] for t in triples], [t[2] for t in triples])

    @classmethod
    def _from_canonical(cls, num_nodes, edges_u, edges_v, costs, dev=None):
        g = object.__new__(cls)
        g.num_nodes = int(num_nodes)
        g.edges_u = edges_u
        g.edges_v = edges_v
        g.costs = costs
        g._dev = dev
        return g

    def device(self):
        """(u int32, v int32, c float64) CUDA tensors of the canonical edges."""
        if self._dev is None:
            self._dev = (L.i32(self.edges_u), L.i32(self.edges_v), L.f64(self.costs))
        return self._dev

    @property
    def num_edges(self):
        return int(self.edges_u.size)

    @property
    def edges(self):
        return list(zip(self.edges_u.tolist(), self.edges_v.tolist(), self.costs.tolist()))

    def __repr__(self):
        return "WeightedGraph(num_nodes=%d, num_edges=%d)" % (self.num_nodes, self.num_edges)


def _is_tensor(x):
    try:
        import torch

        return isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


def _as_i64(x):
    if _is_tensor(x):
        x = x.detach().cpu().numpy()
    return np.asarray(x, dtype=np.int64).ravel()


def _as_f64(x):
    if _is_tensor(x):
        x = x.detach().cpu().numpy()
    return np.asarray(x, dtype=np.float64).ravel()


def graph_from_device(num_nodes, du, dv, dc, k):
    """Wrap device outputs (already canonical) as a WeightedGraph."""
    u, v, c = du[:k], dv[:k], dc[:k]
    return WeightedGraph._from_canonical(num_nodes, L.host_i64(u, k), L.host_i64(v, k), L.host_f64(c, k),
                                         dev=(u, v, c))


class SparseAdjacency:
    """Symmetric sorted COO cost matrix (graph.py:98-122)."""

    __slots__ = ("rows", "cols", "vals", "num_nodes")

    def __init__(self, rows, cols, vals, num_nodes):
        self.rows = np.asarray(rows, dtype=np.int64)
        self.cols = np.asarray(cols, dtype=np.int64)
        self.vals = np.asarray(vals, dtype=np.float64)
        self.num_nodes = int(num_nodes)

    @property
    def nnz(self):
        return int(self.rows.size)

    def entries(self):
        return list(zip(self.rows.tolist(), self.cols.tolist(), self.vals.tolist()))

    def __repr__(self):
        return "SparseAdjacency(num_nodes=%d, nnz=%d)" % (self.num_nodes, self.nnz)


def build_adjacency(g):
    """Symmetric sorted COO of a canonical graph (graph.py:125-131).

    Format conversion for the SparseAdjacency API only (not on the solve
    path): both orientations of every edge, sorted by (row, col).
    """
    rows = np.concatenate([g.edges_u, g.edges_v])
    cols = np.concatenate([g.edges_v, g.edges_u])
    vals = np.concatenate([g.costs, g.costs])
    order = np.argsort(rows * max(g.num_nodes, 1) + cols, kind="stable")
    return SparseAdjacency(rows[order], cols[order], vals[order], g.num_nodes)


def clustering_cost(g, labels):
    """Total cost of edges whose endpoints carry different labels (graph.py:134-145)."""
    lab = np.asarray(labels)
    if lab.shape != (g.num_nodes,):
        raise ValueError("labeling has length %d, graph has %d nodes" % (lab.size, g.num_nodes))
    if g.num_edges == 0:
        return 0.0
    du, dv, dc = g.device()
    if not (lab.dtype.kind in "iu" and (lab.size == 0 or (lab.min() >= 0 and lab.max() < 2 ** 31))):
        # the kernel compares int32 labels: map arbitrary labels (any dtype,
        # negative or >= 2^31) to dense ids first, equality is preserved
        lab = np.unique(lab, return_inverse=True)[1].ravel()
    dl = L.i32(lab)
    out = L.ctypes.c_double()
    L.call("rama_clustering_cost", g.num_nodes, L.ptr(du), L.ptr(dv), L.ptr(dc), g.num_edges, L.ptr(dl),
           L.ctypes.byref(out), L.stream())
    return float(out.value)


def canonical_labels(labels):
    """Relabel to 0..k-1 in order of first occurrence (graph.py:148-157)."""
    labels = np.asarray(labels)
    if labels.size == 0:
        return np.zeros(0, dtype=np.int64)
    _, first, inv = np.unique(labels, return_index=True, return_inverse=True)
    rank = np.empty(first.size, dtype=np.int64)
    rank[np.argsort(first, kind="stable")] = np.arange(first.size)
    return rank[inv.ravel()]


# ------------------------------------------------------ MULTICUT text I/O
# Host file plumbing (NEXT); same grammar and errors
# as graph.py:160-313.

def _parse_native(text=None, path=None, threads=0):
    if path is not None:
        import os

        size = os.path.getsize(path)
        data, length, cpath = None, 0, os.fsencode(path)
    else:
        if isinstance(text, str):
            text = text.encode("utf-8")
        data, length, cpath = text, len(text), None
        size = length
    cap = size // 5 + 2  # an edge line takes at least 6 bytes
    while True:
        u = np.empty(cap, np.int64)
        v = np.empty(cap, np.int64)
        c = np.empty(cap, np.float64)
        n, m = L.ctypes.c_int64(), L.ctypes.c_int64()
        try:
            L.call_host("rama_parse_multicut", data, length, cpath, L.ctypes.byref(n), L.ctypes.byref(m),
                        u.ctypes.data, v.ctypes.data, c.ctypes.data, cap, int(threads))
        except ValueError as exc:
            raise ParseError(str(exc)) from None
        if m.value <= cap:
            return n.value, u[: m.value], v[: m.value], c[: m.value]
        cap = m.value


def parse_instance(text, threads=0):
    """Parse MULTICUT instance text into a WeightedGraph (graph.py:204-263).

    Native C++ parser (rama_parse_multicut: line-aligned chunks parsed by a
    thread pool with std::from_chars) with the reference's acceptance rules
    and ParseError messages; the COO is then canonicalised on the GPU.
    """
    n, u, v, c = _parse_native(text=text, threads=threads)
    return WeightedGraph(n, u, v, c)


def read_instance(path, threads=0):
    """parse_instance on a file, memory-mapped by the native parser."""
    n, u, v, c = _parse_native(path=path, threads=threads)
    return WeightedGraph(n, u, v, c)


def serialize_instance(g, threads=0):
    """MULTICUT text with a NODES line; costs as Python repr, so parsing the
    output reproduces them bit-exactly (graph.py:300-313).  Native
    (rama_serialize_multicut, Python float repr rules)."""
    u = np.ascontiguousarray(g.edges_u, dtype=np.int64)
    v = np.ascontiguousarray(g.edges_v, dtype=np.int64)
    c = np.ascontiguousarray(g.costs, dtype=np.float64)
    length = L.ctypes.c_int64()
    L.call_host("rama_serialize_multicut", int(g.num_nodes), u.ctypes.data, v.ctypes.data, c.ctypes.data, u.size,
                None, 0, L.ctypes.byref(length), int(threads))
    buf = L.ctypes.create_string_buffer(length.value + 1)
    L.call_host("rama_serialize_multicut", int(g.num_nodes), u.ctypes.data, v.ctypes.data, c.ctypes.data, u.size,
                buf, length.value + 1, L.ctypes.byref(length), int(threads))
    return buf.raw[: length.value].decode("ascii")