import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import instances
d, h, w = (int(x) for x in sys.argv[1:4])
n, u, v, c = instances.grid3d_coo(d, h, w, stride=2, seed=0)
g = P.WeightedGraph(n, u, v, c)
sol = P.solve(g, P.SolverConfig(mode="PD"))
ref = O.solve(O.Graph(n, u, v, c), mode="PD", cleanup="handshake")
a = [(r.nodes, r.edges, r.triplets, r.contracted) for r in sol.trace]
b = [(r.nodes, r.edges, r.triplets, r.contracted) for r in ref.trace]
print("same" if a == b else "DIFF", a[:4], b[:4], flush=True)
