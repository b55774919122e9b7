"""Solve the same instance repeatedly in one process; report any drift."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import instances

shape = sys.argv[1] if len(sys.argv) > 1 else "small"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
if shape == "c2":
    n, u, v, c = instances.make("c2")
else:
    n, u, v, c = instances.grid8_coo(96, 128, strides=(2, 3), seed=0)
g = P.WeightedGraph(n, u, v, c)
base = None
for r in range(reps):
    sol = P.solve(g, P.SolverConfig(mode="PD"))
    tr = [(t.nodes, t.edges, t.triplets, t.contracted) for t in sol.trace]
    print(r, repr(sol.primal_cost), repr(sol.lower_bound), tr, flush=True)
    if base is None:
        base = (sol.labeling.copy(), tr)
    else:
        same = np.array_equal(base[0], sol.labeling)
        print("  same labels:", same, " same trace:", tr == base[1], flush=True)
