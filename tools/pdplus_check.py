import sys, time; sys.path.insert(0, '/root/repo')
import numpy as np, oracle as O
import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import instances
for dims in ((8, 24, 24), (16, 32, 32), (24, 48, 48)):
    n, u, v, c = instances.grid3d_coo(*dims, stride=2, seed=1)
    g = P.WeightedGraph(n, u, v, c)
    sols = [P.solve(g, P.SolverConfig(mode="PD+")) for _ in range(3)]
    same = all(np.array_equal(sols[0].labeling, s.labeling) for s in sols)
    t = time.time()
    ref = O.solve(O.Graph(n, u, v, c), mode="PD+", cleanup="handshake")
    print(dims, "n", n, "deterministic", same, "== oracle", np.array_equal(sols[0].labeling, ref.labeling),
          sols[0].primal_cost, ref.primal_cost, "oracle %.1fs" % (time.time() - t), flush=True)
