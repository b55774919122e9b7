"""PD+ determinism on mid-size 3-D grids (hashed BFS + dense fallback)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import instances
dims = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (48, 96, 96)
n, u, v, c = instances.grid3d_coo(*dims, stride=2, seed=0)
g = P.WeightedGraph(n, u, v, c)
sols = [P.solve(g, P.SolverConfig(mode="PD+")) for _ in range(3)]
print(dims, [s.primal_cost for s in sols], [len(s.trace) for s in sols], flush=True)
for r in range(len(sols[0].trace)):
    rows = [(s.trace[r].nodes, s.trace[r].edges, s.trace[r].triplets, s.trace[r].contracted) if r < len(s.trace) else None for s in sols]
    if len(set(rows)) > 1:
        print("round", r + 1, "differs:", rows)
        break
