"""Record the reference's own C2 result for the full-size
parity test.  Runs parcut (the REFERENCE, ~80 s) and the oracle with the
B200 handshake cleanup; writes tests/golden/c2_reference.json.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_c2_reference.py
"""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import parcut  # noqa: E402

import oracle  # noqa: E402
from paper_2109_01838_b200 import instances  # noqa: E402

n, u, v, c = instances.make("c2")
g = parcut.WeightedGraph(n, u, v, c)
parcut.solve(parcut.grid_graph(8, 8, 0, 0), parcut.SolverConfig(mode="PD"))  # numba warm-up
t0 = time.perf_counter()
sol = parcut.solve(g, parcut.SolverConfig(mode="PD"))
t_ref = time.perf_counter() - t0
hs = oracle.solve(oracle.Graph(n, u, v, c), mode="PD", cleanup="handshake")
out = {
    "config": "c2: 8-connected 1024x2048 + lattice strides 2,3, seed 0, mode PD",
    "nodes": n,
    "edges": int(g.num_edges),
    "primal": sol.primal_cost,
    "lower_bound": sol.lower_bound,
    "primal_handshake_oracle": hs.primal_cost,
    "rounds": [[r.nodes, r.edges, r.triplets, r.contracted] for r in sol.trace if r.phase == "primal-dual"],
    "reference_seconds": t_ref,
    "reference_host": os.uname().nodename,
}
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "c2_reference.json"), "w") as fh:
    json.dump(out, fh, indent=1)
print(json.dumps(out))
