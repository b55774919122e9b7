"""Solve one named config on cuda:0 a few times; print time, objective,
trace and kernel-family times.  python tools/probe_configs.py c3 [reps]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import _lib, instances

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kw = {}
for a in sys.argv[3:]:
    k, v = a.split("=")
    kw[k] = int(v)
t0 = time.time()
n, u, v, c = instances.make(name, **kw)
print("generated", n, u.size, "in %.1fs" % (time.time() - t0), flush=True)
g = P.WeightedGraph(n, u, v, c)
print("canonical edges", g.num_edges, flush=True)
du, dv, dc = g.device()
cfg = P.SolverConfig(mode=instances.CONFIGS[name]["mode"])
for r in range(reps):
    _lib.profile_enable(True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lab, primal, lb, trace = P.solve_device(n, du, dv, dc, g.num_edges, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    fam = _lib.profile_read()
    _lib.profile_enable(False)
    print(json.dumps({"rep": r, "ms": dt * 1e3, "primal": primal, "lb": lb, "rounds": len(trace),
                      "fam_ms": {k: round(v[0], 3) for k, v in fam.items() if v[2]}}), flush=True)
for t in trace:
    print("  ", t.round_index, t.phase, t.nodes, t.edges, t.triplets, t.contracted, "%.2f ms" % t.time_ms)
