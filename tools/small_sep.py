import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import instances
d, h, w = (int(x) for x in sys.argv[1:4])
n, u, v, c = instances.grid3d_coo(d, h, w, stride=2, seed=0)
g = P.WeightedGraph(n, u, v, c)
og = O.Graph(n, u, v, c)
for L in (4, 5):
    gl, gn = P.dual._separate(g, L)
    ol, on = O.separate(og, L)
    bad = np.nonzero((np.asarray(gl) != ol) | np.any(np.asarray(gn) != on, axis=1))[0]
    print("L", L, "rows", ol.size, "bad", bad.size, flush=True)
    for r in bad[:3]:
        print("  ", r, gl[r], gn[r].tolist(), ol[r], on[r].tolist())
