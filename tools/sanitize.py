"""Small solves through every path, for compute-sanitizer runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import instances
for args in [(24, 32, 3, 1), (16, 16, 0, 2)]:
    g = P.grid_graph(*args)
    for mode in ("P", "PD", "PD+", "D", "GAEC"):
        s = P.solve(g, P.SolverConfig(mode=mode, separation_rounds=2 if mode == "D" else 1))
        print(mode, s.primal_cost, s.lower_bound, flush=True)
g = P.WeightedGraph(*instances.grid8_coo(20, 24, strides=(2, 3), seed=3))
print("8conn", P.solve(g, P.SolverConfig(mode="PD")).primal_cost)
g = P.WeightedGraph(*instances.chung_lu_coo(600, 2.1, 9000, seed=1))
print("chunglu", P.solve(g, P.SolverConfig(mode="PD")).primal_cost)
g = P.WeightedGraph(*instances.random_coo(160, 0.35, seed=4))  # dense: tier-2 separation tables
print("dense", P.solve(g, P.SolverConfig(mode="PD")).primal_cost)
g = P.WeightedGraph(*instances.grid3d_coo(8, 12, 12, stride=2, seed=2))
print("3d", P.solve(g, P.SolverConfig(mode="PD")).primal_cost)
gs = [P.WeightedGraph(*instances.grid_coo(16, 16, 0, seed=s)) for s in range(4)]
print("batch", [s.primal_cost for s in P.solve_batch(gs, P.SolverConfig(mode="PD"), workers=2)])
n, u, v, c = instances.random_coo(40, 0.3, seed=5)
g = P.WeightedGraph(n, u, v, c)
st = P.triangulate(P.separate_conflicted_cycles(g, 5), g)
P.message_passing(st, 20)
print("agree", P.check_edge_triangle_agreement(st, 1e-3), "ext", P.extend_separation(st, 5))
