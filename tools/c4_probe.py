"""C4 probe: scaled C4 (10k/20k/50k) PD against the reference fixtures, and
the full C4 solve time.  python tools/c4_probe.py [full]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import instances

ref = {(r["arg"], r["mode"]): r for r in json.load(open("tests/golden/c4_reference.json"))["runs"]}
for n in (10000, 20000, 50000):
    g = P.WeightedGraph(*instances.chung_lu_coo(n, 2.1, 26 * n, seed=0))
    r = ref[(n, "PD")]
    for ex in (True,):
        t = time.perf_counter()
        s = P.solve(g, P.SolverConfig(mode="PD"))
        dt = time.perf_counter() - t
        rounds = [[x.nodes, x.edges, x.triplets, x.contracted] for x in s.trace if x.phase == "primal-dual"]
        print(json.dumps({"n": n, "exact": ex, "ms": round(dt * 1e3, 1), "primal": s.primal_cost,
                          "ref_primal": r["primal"], "gap_primal_pct": 100 * (s.primal_cost - r["primal"]) / abs(r["primal"]),
                          "lb": s.lower_bound, "ref_lb": r["lower_bound"],
                          "gap_lb_pct": 100 * (s.lower_bound - r["lower_bound"]) / abs(r["lower_bound"]),
                          "rounds_equal": rounds == r["rounds"], "n_rounds": len(rounds)}), flush=True)
if "full" in sys.argv:
    n, u, v, c = instances.make("c4")
    g = P.WeightedGraph(n, u, v, c)
    for ex in (True, True):
        torch.cuda.synchronize()
        t = time.perf_counter()
        s = P.solve(g, P.SolverConfig(mode="PD"))
        dt = time.perf_counter() - t
        print(json.dumps({"full_c4": True, "exact": ex, "ms": round(dt * 1e3, 1), "primal": s.primal_cost,
                          "lb": s.lower_bound, "rounds": len(s.trace)}), flush=True)
