"""Golden fixtures for the MULTICUT text format (graph.py:160-313), made by
the REFERENCE parcut.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_io.py

Writes tests/golden/io_cases.json: for every text either the parsed graph
(num_nodes, canonical edges with costs as repr strings) or the ParseError
message, and serialize_instance outputs of a few graphs.
"""

import json
import os

import numpy as np

import parcut

CASES = [
    "MULTICUT\n0 1 2.5\n",
    "MULTICUT\n0 1 1.0\n1 0 0.5\n",
    "# generated\n\nMULTICUT\nNODES 5\n0 1 1.5\n\n2 3 -0.5\n",
    "MULTICUT\r\n0\t1\t2.5\r\n1\t2\t-1.0\r\n",
    "MULTICUT\nNODES 3\n",
    "0 1 2.5\n",
    "MULTICUT\n0 0 1.0\n",
    "MULTICUT\n0 1\n",
    "MULTICUT\n0 x 1.0\n",
    "MULTICUT\n0 1 1.0e\n",
    "MULTICUT\n-1 2 1.0\n",
    "MULTICUT\n0 1 nan\n",
    "MULTICUT\n0 1 inf\n",
    "MULTICUT\nNODES 2\n0 5 1.0\n",
    "",
    "\n\n# only comments\n",
    "MULTICUT \n0 1 1.0\n",
    "MULTICUT\nNODES\n0 1 1\n",
    "MULTICUT\nNODES x\n0 1 1\n",
    "MULTICUT\nNODES -3\n",
    "MULTICUT\nNODES 4 5\n",
    "MULTICUT\n0.0 1.0 2.0\n",
    "MULTICUT\n0 1 2 # inline comment\n2 3 -1\n",
    "MULTICUT\n0 1 2 # inline comment\n2 3 x\n",
    "MULTICUT\n1e1 2 3.25\n",
    "MULTICUT\n0 1 +1.5\n1 2 -.5\n2 3 1e-7\n3 4 1E+3\n",
    "MULTICUT\n0 1 1\n0 1 1\n1 0 -2\n",
    "MULTICUT\n0 1 1_0\n",
    "MULTICUT\n1_0 2 3.0\n",
    "MULTICUT\n0 1 1.5\r2 3 2.5\r",
    "MULTICUT\n0 1 0.1\n1 2 0.2\n0 2 0.30000000000000004\n",
    "MULTICUT\n\t 0   1   7.25  \n",
    "MULTICUT\n0 1 2 3\n",
    "MULTICUT\n0 1 'q'\n",
    "MULTICUT\n0 1 1.0\n5 5 2.0\n",
    "#c\nMULTICUT\n#c\nNODES 10\n#c\n0 9 1\n9 3 -1\n",
    "MULTICUT\nNODES 3\n0 1 1\n2 1 -1\n# tail\n",
    "MULTICUT\n0 1 1e400\n",
    "MULTICUT\n0 1 1e-400\n",
    "MULTICUT\n0 1 -0.0\n",
]


def graph_dict(g):
    return {"n": int(g.num_nodes), "u": g.edges_u.tolist(), "v": g.edges_v.tolist(),
            "c": [repr(float(x)) for x in g.costs.tolist()]}


out = {"parse": [], "serialize": []}
for text in CASES:
    try:
        out["parse"].append({"text": text, "graph": graph_dict(parcut.parse_instance(text))})
    except parcut.ParseError as exc:
        out["parse"].append({"text": text, "error": str(exc)})
rng = np.random.default_rng(0)
for seed in range(6):
    g = parcut.random_graph(int(rng.integers(2, 40)), 0.4, seed)
    out["serialize"].append({"graph": graph_dict(g), "text": parcut.serialize_instance(g)})
g = parcut.WeightedGraph.from_edges(4, [(0, 1, 1e16), (1, 2, 1e-5), (2, 3, -0.0), (0, 3, 123456789012345.6),
                                        (0, 2, 5e-324), (1, 3, 1.7976931348623157e308)])
out["serialize"].append({"graph": graph_dict(g), "text": parcut.serialize_instance(g)})
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "io_cases.json"), "w") as fh:
    json.dump(out, fh, indent=0)
print(len(out["parse"]), "parse cases,", len(out["serialize"]), "serialize cases")
