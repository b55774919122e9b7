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

def parse_instance(text):
    """Parse MULTICUT instance text into a WeightedGraph."""
    if isinstance(text, bytes):
        text = text.decode("utf-8")
    lines = text.splitlines()
    i = 0
    while i < len(lines) and (not lines[i].strip() or lines[i].strip().startswith("#")):
        i += 1
    if i == len(lines):
        raise ParseError("missing MULTICUT header")
    if lines[i] != "MULTICUT":
        raise ParseError("line %d: expected MULTICUT header, got %r" % (i + 1, lines[i]))
    i += 1
    declared = None
    j = i
    while j < len(lines) and (not lines[j].strip() or lines[j].strip().startswith("#")):
        j += 1
    if j < len(lines):
        tok = lines[j].split()
        if tok[0] == "NODES":
            if len(tok) != 2:
                raise ParseError("line %d: expected 'NODES <n>'" % (j + 1))
            try:
                declared = int(tok[1])
            except ValueError:
                raise ParseError("line %d: NODES count must be an integer" % (j + 1)) from None
            if declared < 0:
                raise ParseError("line %d: NODES count must be non-negative" % (j + 1))
            i = j + 1
    us, vs, cs = [], [], []
    for k in range(i, len(lines)):
        s = lines[k].strip()
        if not s or s.startswith("#"):
            continue
        tok = s.split()
        if len(tok) != 3:
            raise ParseError("line %d: expected '<u> <v> <cost>', got %r" % (k + 1, lines[k]))
        try:
            a, b = int(tok[0]), int(tok[1])
        except ValueError:
            raise ParseError("line %d: node ids must be decimal integers" % (k + 1)) from None
        try:
            w = float(tok[2])
        except ValueError:
            raise ParseError("line %d: malformed cost %r" % (k + 1, tok[2])) from None
        if not np.isfinite(w):
            raise ParseError("line %d: cost must be finite" % (k + 1))
        if a < 0 or b < 0:
            raise ParseError("line %d: negative node id" % (k + 1))
        if a == b:
            raise ParseError("line %d: self-loop edge (%d, %d)" % (k + 1, a, b))
        if declared is not None and (a >= declared or b >= declared):
            raise ParseError("line %d: node id exceeds declared NODES %d" % (k + 1, declared))
        us.append(a)
        vs.append(b)
        cs.append(w)
    if declared is not None:
        n = declared
    elif us:
        n = max(max(us), max(vs)) + 1
    else:
        n = 0
    return WeightedGraph(n, us, vs, cs)


def serialize_instance(g):
    """MULTICUT text with a NODES line; costs via repr (bit-exact round trip)."""
    out = ["MULTICUT", "NODES %d" % g.num_nodes]
    out.extend("%d %d %r" % e for e in g.edges)
    return "\n".join(out) + "\n"
