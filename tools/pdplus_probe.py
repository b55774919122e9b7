"""PD+ (L = 7, exact BFS separation) on C2 / C3-sized graphs: time and memory."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import instances
for name in sys.argv[1:] or ["c2"]:
    n, u, v, c = instances.make(name)
    g = P.WeightedGraph(n, u, v, c)
    du, dv, dc = g.device()
    for mode in ("PD", "PD+"):
        cfg = P.SolverConfig(mode=mode)
        for rep in range(2):
            torch.cuda.synchronize()
            t = time.perf_counter()
            lab, primal, lb, trace = P.solve_device(n, du, dv, dc, g.num_edges, cfg)
            torch.cuda.synchronize()
            print(name, mode, rep, "%.1f ms" % ((time.perf_counter() - t) * 1e3), primal, lb, len(trace), flush=True)
