"""Workspace high-water marks of rama_solve_ws per config (calibrates rama_ws_bytes)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import instances

for name in sys.argv[1:] or ["c1", "c5", "c2", "c3", "c4"]:
    n, u, v, c = instances.make(name)
    g = P.WeightedGraph(n, u, v, c)
    du, dv, dc = g.device()
    cfg = P.SolverConfig(mode=instances.CONFIGS[name]["mode"])
    P.solve_device(n, du, dv, dc, g.num_edges, cfg)
    torch.cuda.synchronize()
    t = time.perf_counter()
    P.solve_device(n, du, dv, dc, g.num_edges, cfg)
    torch.cuda.synchronize()
    t_pool = time.perf_counter() - t
    ws = torch.empty(P.workspace_bytes(n, g.num_edges, cfg), dtype=torch.uint8, device="cuda")
    P.solve_device(n, du, dv, dc, g.num_edges, cfg, workspace=ws)
    torch.cuda.synchronize()
    t = time.perf_counter()
    P.solve_device(n, du, dv, dc, g.num_edges, cfg, workspace=ws)
    torch.cuda.synchronize()
    t_ws = time.perf_counter() - t
    peak = P.solve_device.last_workspace_peak
    print("%s n %d m %d: peak %.1f MB = %.0f B/edge (estimate %.1f MB); solve %.2f ms pool / %.2f ms workspace"
          % (name, n, g.num_edges, peak / 1e6, peak / max(g.num_edges, 1), ws.numel() / 1e6, t_pool * 1e3,
             t_ws * 1e3), flush=True)
    del ws
