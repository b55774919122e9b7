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
# round-2 paths: hub rows (device-wide radix sort of long rows, run-aggregated
# histograms, hub slot lists), exact 5-cycle searches, the union batch with
# empty / single-node / all-repulsive instances, caller workspace, staging
rng = np.random.default_rng(7)
nh = 6000
hu = np.concatenate([np.zeros(nh - 1, np.int64), rng.integers(1, nh, 8000)])
hv = np.concatenate([np.arange(1, nh), rng.integers(1, nh, 8000)])
keep = hu != hv
g = P.WeightedGraph(nh, hu[keep], hv[keep], rng.standard_normal(keep.sum()) + 0.3)
print("hub", P.solve(g, P.SolverConfig(mode="PD")).primal_cost)
n, u, v, c = instances.grid_coo(12, 14, 0, seed=3)
gs = [P.WeightedGraph(*instances.grid_coo(16, 16, 0, seed=s)) for s in range(2)]
gs += [P.WeightedGraph(5), P.WeightedGraph(1), P.WeightedGraph(n, u, v, -np.abs(c)),
       P.WeightedGraph(*instances.chung_lu_coo(400, 2.1, 5000, seed=2))]
for mode in ("PD", "P"):
    print("union", mode, [s.primal_cost for s in P.solve_batch(gs, P.SolverConfig(mode=mode), workers=1)])
g = P.WeightedGraph(*instances.grid8_coo(30, 40, strides=(2, 3), seed=6))
du, dv, dc = g.device()
print("ws", P.solve_device(g.num_nodes, du, dv, dc, g.num_edges, P.SolverConfig(mode="PD"), workspace="torch")[1])
n, u, v, c = instances.grid_coo(400, 900, 0, seed=1)  # ~720k edges: several 4 MiB staging chunks
g = P.WeightedGraph(n, u, v, c)
print("host", P.solve_host(n, np.ascontiguousarray(g.edges_u, np.int32), np.ascontiguousarray(g.edges_v, np.int32),
                           np.ascontiguousarray(g.costs), P.SolverConfig(mode="P"))[1])
# round-2 late: forests of small trees (per-tree conflict loop) and of larger trees
for shift in (1.0, 0.8):
    n, u, v, c = instances.grid_coo(60, 80, 2, seed=3)
    g = P.WeightedGraph(n, u, v, c - shift)
    print("forest", shift, len(P.select_spanning_forest_no_conflicts(g)))
