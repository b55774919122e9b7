import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import instances
L = int(sys.argv[1])
n, u, v, c = instances.random_coo(12, 0.5, seed=3)
g = P.WeightedGraph(n, u, v, c)
print("graph", g.num_edges, flush=True)
print(P.dual._separate(g, L), flush=True)
