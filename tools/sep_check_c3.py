"""Separation parity at C3 round-2 scale: the oracle builds the round-2 graph
(exact pipeline), then GPU separation vs oracle separation on it."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import instances

n, u, v, c = instances.make("c3")
g = O.Graph(n, u, v, c)
t = time.time()
lengths, nodes = O.separate(g, 5)
st = O.triangulate(g, lengths, nodes)
O.message_passing(st, 5)
work = O.reparametrized_graph(st)
g2, f, nt, _, k = O.contraction_step(work, "auto", 0.1)
print("round-2 graph", g2.num_nodes, g2.num_edges, "%.1fs" % (time.time() - t), flush=True)
t = time.time()
L2, N2 = O.separate(g2, 5)
print("oracle separate %.1fs" % (time.time() - t), flush=True)
pg = P.WeightedGraph._from_canonical(g2.num_nodes, g2.edges_u, g2.edges_v, g2.costs)
gl, gn = P.dual._separate(pg, 5)
gl = np.asarray(gl); gn = np.asarray(gn)
bad = np.nonzero((gl != L2) | np.any(gn != N2, axis=1))[0]
print("rows", L2.size, "mismatches", bad.size, flush=True)
for r in bad[:10]:
    print(r, "gpu", gl[r], gn[r].tolist(), "oracle", L2[r], N2[r].tolist())

# diagnose: positive CSR of g2, levels of the first bad sources
pos = g2.costs > 0
pu, pv = g2.edges_u[pos], g2.edges_v[pos]
adj = [[] for _ in range(g2.num_nodes)]
for x, y in zip(pu.tolist(), pv.tolist()):
    adj[x].append(y); adj[y].append(x)
for r in bad[:8]:
    a = int(N2[r][0]) if L2[r] else int(gn[r][0])
    Na = sorted(adj[a])
    L2set = set()
    for x in Na:
        for y in adj[x]:
            if y != a and y not in Na:
                L2set.add(y)
    print("row", r, "a", a, "la", len(Na), "|L2|", len(L2set), "gpu y in L2:", int(gn[r][2]) in L2set)
