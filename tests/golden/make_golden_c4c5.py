"""Record the REFERENCE's own results on the C4-scaled and C5 parity sets
 for the -m gpu parity tests.

* C4 scaled: Chung-Lu alpha 2.1 (instances.chung_lu_coo, 26 n draws,
  seed 0) at n = 10k / 20k / 50k, modes P and PD (~15 min in total; the
  n = 50k PD solve alone is ~11 min).
* C5: parcut.grid_graph(512, 512, 0, seed=s), s = 0..63, mode PD.

Writes tests/golden/c4_reference.json and tests/golden/c5_reference.json
(objectives + per-round (n, m, T, contracted) traces).  Run here, in the
build container, where the reference imports:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_c4c5.py
"""

import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))


def _run(task):
    import parcut
    from paper_2109_01838_b200 import instances

    kind, arg, mode = task
    parcut.solve(parcut.grid_graph(8, 8, 0, 0), parcut.SolverConfig(mode=mode))  # numba warm-up
    if kind == "c4":
        n, u, v, c = instances.chung_lu_coo(arg, 2.1, 26 * arg, seed=0)
        g = parcut.WeightedGraph(n, u, v, c)
    else:
        g = parcut.grid_graph(512, 512, 0, seed=arg)
    t0 = time.perf_counter()
    sol = parcut.solve(g, parcut.SolverConfig(mode=mode))
    secs = time.perf_counter() - t0
    rounds = [[r.nodes, r.edges, r.triplets, r.contracted] for r in sol.trace if r.phase in ("primal-dual", "contract")]
    return {"kind": kind, "arg": arg, "mode": mode, "nodes": int(g.num_nodes), "edges": int(g.num_edges),
            "primal": float(sol.primal_cost), "lower_bound": float(sol.lower_bound), "rounds": rounds,
            "reference_seconds": secs}


def main():
    tasks = [("c4", 50000, "PD"), ("c4", 20000, "PD"), ("c4", 10000, "PD"),
             ("c4", 50000, "P"), ("c4", 20000, "P"), ("c4", 10000, "P")]
    tasks += [("c5", s, "PD") for s in range(64)]
    with mp.Pool(int(os.environ.get("WORKERS", "7"))) as pool:
        res = pool.map(_run, tasks, chunksize=1)
    c4 = [r for r in res if r["kind"] == "c4"]
    c5 = [r for r in res if r["kind"] == "c5"]
    meta = {"host": os.uname().nodename, "cpu_count": os.cpu_count(),
            "note": "reference parcut.solve, one process per instance (single-threaded each)"}
    with open(os.path.join(HERE, "c4_reference.json"), "w") as fh:
        json.dump({"meta": meta, "generator": "instances.chung_lu_coo(n, 2.1, 26*n, seed=0)", "runs": c4}, fh,
                  indent=1)
    with open(os.path.join(HERE, "c5_reference.json"), "w") as fh:
        json.dump({"meta": meta, "generator": "parcut.grid_graph(512, 512, 0, seed=s)", "runs": c5}, fh)
    for r in c4:
        print(r["arg"], r["mode"], r["edges"], r["primal"], r["lower_bound"], "%.1f s" % r["reference_seconds"])


if __name__ == "__main__":
    main()
