"""Golden fixtures for mode D with separation_rounds > 1 (extend_separation,
dual.py:414-474; solver.py:211-240), produced by the REFERENCE parcut.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_dual_rounds.py

Writes tests/golden/dual_rounds.npz: per instance the canonical graph, and
for separation_rounds in (2, 3, 4) the lower bound and the per-round
(edges, triplets) trace.
"""

import os
import sys

import numpy as np

import parcut

OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
from paper_2109_01838_b200 import instances  # noqa: E402

graphs = []
for s in range(12):
    graphs.append(instances.random_coo(10 + 3 * s, 0.35, seed=100 + s))
graphs.append(instances.grid_coo(24, 32, 3, seed=4))
graphs.append(instances.grid8_coo(20, 24, strides=(2, 3), seed=5))
out = {}
for i, (n, u, v, c) in enumerate(graphs):
    g = parcut.WeightedGraph(n, u, v, c)
    out["g%d_n" % i] = np.array([n])
    out["g%d_u" % i] = g.edges_u
    out["g%d_v" % i] = g.edges_v
    out["g%d_c" % i] = g.costs
    for r in (2, 3, 4):
        sol = parcut.solve(g, parcut.SolverConfig(mode="D", separation_rounds=r))
        out["g%d_r%d_lb" % (i, r)] = np.array([sol.lower_bound])
        out["g%d_r%d_trace" % (i, r)] = np.array([[t.edges, t.triplets] for t in sol.trace], dtype=np.int64)
out["count"] = np.array([len(graphs)])
np.savez_compressed(os.path.join(OUT, "dual_rounds.npz"), **out)
print("wrote", len(graphs), "instances")
