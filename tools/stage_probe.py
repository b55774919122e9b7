"""rama_solve_host (pageable numpy) vs rama_solve (device) on C2: staging overhead."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import instances
n, u, v, c = instances.make("c2")
g = P.WeightedGraph(n, u, v, c)
du, dv, dc = g.device()
cfg = P.SolverConfig(mode="PD")
hu, hv, hc = (np.ascontiguousarray(x) for x in (g.edges_u.astype(np.int32), g.edges_v.astype(np.int32), g.costs))
hl = np.empty(n, np.int32)
def t(f, k=5):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3
dev = t(lambda: P.solve_device(n, du, dv, dc, g.num_edges, cfg))
host = t(lambda: P.solve_host(n, hu, hv, hc, cfg, labels=hl))
print("chunk %s threads %s: device %.2f ms host %.2f ms overhead %.2f ms" % (os.environ.get("RAMA_STAGE_CHUNK_MB", "16"), os.environ.get("RAMA_STAGE_THREADS", "auto"), dev, host, host - dev), flush=True)
