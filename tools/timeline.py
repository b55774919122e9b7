"""Kernel timeline of one solve (CUPTI through torch.profiler): where the
device sits idle and which host call precedes each gap.
python tools/timeline.py c2 [out.json]"""
import json, os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import instances

name = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/timeline_%s.json" % name
n, u, v, c = instances.make(name)
g = P.WeightedGraph(n, u, v, c)
du, dv, dc = g.device()
cfg = P.SolverConfig(mode=instances.CONFIGS[name]["mode"])
for _ in range(3):
    P.solve_device(n, du, dv, dc, g.num_edges, cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    P.solve_device(n, du, dv, dc, g.num_edges, cfg)
    torch.cuda.synchronize()
ev = [e for e in prof.events()]
kern = sorted([e for e in ev if e.device_type == torch.autograd.DeviceType.CUDA],
              key=lambda e: e.time_range.start)
api = sorted([e for e in ev if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cuda")],
             key=lambda e: e.time_range.start)
t0, t1 = kern[0].time_range.start, kern[-1].time_range.end
busy = sum(e.time_range.end - e.time_range.start for e in kern)
gaps = []
for a, b in zip(kern, kern[1:]):
    gap = b.time_range.start - a.time_range.end
    if gap > 0:
        gaps.append((gap, a.name[:60], b.name[:60]))
by_prev = collections.Counter()
cnt_prev = collections.Counter()
for gap, a, b in gaps:
    by_prev[a] += gap
    cnt_prev[a] += 1
api_tot = collections.Counter()
api_cnt = collections.Counter()
for e in api:
    api_tot[e.name] += e.time_range.end - e.time_range.start
    api_cnt[e.name] += 1
res = {
    "span_us": t1 - t0, "kernel_busy_us": busy, "idle_us": (t1 - t0) - busy, "kernels": len(kern),
    "gaps_over_5us": sum(1 for g_ in gaps if g_[0] > 5),
    "idle_after_kernel_us": [(k, round(v, 1), cnt_prev[k]) for k, v in by_prev.most_common(40)],
    "api_us": [(k, round(v, 1), api_cnt[k]) for k, v in api_tot.most_common(20)],
    "largest_gaps": sorted(gaps, reverse=True)[:40],
}
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: res[k] for k in ("span_us", "kernel_busy_us", "idle_us", "kernels", "gaps_over_5us")}))
for k, v, c_ in res["idle_after_kernel_us"][:25]:
    print("  idle after %-60s %8.1f us  (%d)" % (k, v, c_))
for k, v, c_ in res["api_us"][:12]:
    print("  api %-40s %8.1f us  (%d)" % (k, v, c_))
