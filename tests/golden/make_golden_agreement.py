"""Golden fixtures for check_edge_triangle_agreement (dual.py:477-531),
made by the REFERENCE parcut (acceptance 09 / test_dual.py:406-429 style).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_agreement.py
"""

import json
import os
import sys

import parcut
from parcut import dual as D

OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
from paper_2109_01838_b200 import instances  # noqa: E402

cases = []
for seed in range(40):
    n, u, v, c = instances.random_coo(5 + seed % 9, 0.6, seed=500 + seed)
    g = parcut.WeightedGraph(n, u, v, c)
    for iters in (0, 1, 3, 20, 200):
        st = parcut.triangulate(parcut.separate_conflicted_cycles(g, 5), g)
        for _ in range(iters):
            parcut.message_passing_iteration(st)
        for eps in (1e-6, 1e-2):
            cases.append({"n": n, "u": g.edges_u.tolist(), "v": g.edges_v.tolist(), "c": [repr(x) for x in g.costs.tolist()],
                          "iters": iters, "eps": eps, "agree": bool(D.check_edge_triangle_agreement(st, eps))})
with open(os.path.join(OUT, "agreement.json"), "w") as fh:
    json.dump(cases, fh)
print(len(cases), "cases,", sum(c["agree"] for c in cases), "agree")
