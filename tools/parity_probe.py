"""GPU vs oracle parity on a few larger shapes (PD with the handshake cleanup):
prints per-round (n, m, T, |S|) mismatches and the separation diff of the
first differing round.  python tools/parity_probe.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import instances

shapes = [("c3crop", lambda: instances.grid3d_coo(16, 64, 64, stride=2, seed=0)),
          ("c3crop2", lambda: instances.grid3d_coo(32, 96, 96, stride=2, seed=1)),
          ("c2crop", lambda: instances.grid8_coo(128, 256, strides=(2, 3), seed=3))]
for name, fn in shapes:
    n, u, v, c = fn()
    g = P.WeightedGraph(n, u, v, c)
    sol = P.solve(g, P.SolverConfig(mode="PD"))
    ref = O.solve(O.Graph(n, u, v, c), mode="PD", cleanup="handshake")
    a = [(r.nodes, r.edges, r.triplets, r.contracted) for r in sol.trace]
    b = [(r.nodes, r.edges, r.triplets, r.contracted) for r in ref.trace]
    same = a == b and np.array_equal(sol.labeling, ref.labeling)
    print(name, "same" if same else "DIFF", sol.primal_cost, ref.primal_cost, flush=True)
    if not same:
        for i, (x, y) in enumerate(zip(a, b)):
            if x != y:
                print("  round", i + 1, "gpu", x, "oracle", y)
                break
