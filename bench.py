"""Benchmark: RAMA primal-dual multicut solve on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload c2|c3|c4|c5|c1]

One step = one full PD solve (separation, triangulation, 5 MP iterations,
contraction rounds, cleanup, objective) of one synthetic instance of the
named shape.  Default workload: C2 (8-connected 1024x2048 grid + lattice
strides 2, 3; 2,097,152 nodes / 9,892,581 edges), BASELINE.json configs[1].

* value : edges/s with the canonical COO resident in HBM (rama_solve on
          device buffers), CUDA events on the solving stream, L2 flushed
          (256 MiB write) between steps outside the events.
* e2e   : edges/s through the C ABI with HOST buffers (rama_solve_host:
          H2D of u, v, c + solve + D2H of labels inside the timed region).
* N > 1 : one process per GPU (bench.py re-execs itself under
          torch.distributed.run when WORLD_SIZE is unset), each rank solves its own
          independent instance (seed = rank) and the labels/objectives are
          gathered over NCCL every step -- weak scaling, no other exchange.
* --impl reference : the CPU oracle port of the reference solver
          (oracle/, single-threaded like the reference) on the full C2
          instance, one solve per step, steps spread over the host cores.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BATCH_INSTANCES = 64   # C5: 64 independent 512x512 grids per step
BATCH_WORKERS = int(os.environ.get("RAMA_BATCH_WORKERS", "1"))  # union groups (streams) per GPU for a batch


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5", "c5batch"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


WORKLOAD_DESC = {
    "c1": "C1: 4-connected 64x64 grid, N(0,1) costs",
    "c2": "C2: 8-connected 1024x2048 grid + lattice strides 2,3 (Cityscapes-like), N(0,1) costs",
    "c3": "C3: 6-connected 3D grid 128x256x256 + stride-2 lattice (connectomics-like), N(0,1) costs",
    "c4": "C4: Chung-Lu power-law graph, 1M nodes, alpha 2.1, mixed-sign costs",
    "c5": "C5: one 512x512 4-connected grid instance",
    "c5batch": "C5: batch of 64 independent 512x512 4-connected grids (seeds 0-63), sharded over the GPUs",
}


def mode_of(workload):
    return "P" if workload == "c1" else "PD"


# ------------------------------------------------------------ CPU oracle

def cpu_sample(workload):
    """The instance the CPU arms solve per step: the FULL workload where the
    single-threaded port finishes it in ~20 s (C1, C2, C5), a crop where it
    cannot (C3 ~2 min per solve; C4, whose reference run does not finish).
    Returns ((n, u, v, c), description, same_config)."""
    from paper_2109_01838_b200 import instances

    if workload == "c3":
        n, u, v, c = instances.grid3d_coo(16, 256, 256, stride=2, seed=0)
        return (n, u, v, c), "C3-shaped crop 16x256x256 (+stride 2), seed 0, %d raw edges, full PD solve" % u.size, False
    if workload == "c4":
        n, u, v, c = instances.chung_lu_coo(10_000, 2.1, 260_000, seed=0)
        return (n, u, v, c), "C4-shaped Chung-Lu n=10k (26 n draws), seed 0, full PD solve", False
    if workload == "c5batch":
        return instances.make("c5", seed=0), "one instance of the batch (512x512, seed 0), full PD solve", False
    return instances.make(workload), "the full %s instance (seed 0), full %s solve" % (workload, mode_of(workload)), True


def run_oracle(sample, mode):
    import oracle

    n, u, v, c = sample
    g = oracle.Graph(n, u, v, c)
    t0 = time.perf_counter()
    sol = oracle.solve(g, mode=mode)
    return time.perf_counter() - t0, g.num_edges, sol


def cpu_baseline(workload):
    """One single-threaded oracle solve of the sample, in-process."""
    sample, desc, same = cpu_sample(workload)
    secs, m, _ = run_oracle(sample, mode_of(workload))
    return {"value": m / secs, "unit": "edges/s", "cores": 1, "kind": "port", "same_config": same,
            "sample": desc + "; %.2f s on 1 host core (oracle/rama_oracle.c; the reference is single-threaded too)"
            % secs}


_POOL_SAMPLE = None  # set before the pool forks (shared copy-on-write)


def _pool_warm(mode):
    import oracle
    from paper_2109_01838_b200 import instances

    oracle.solve(oracle.Graph(*instances.grid_coo(64, 64, 0, seed=0)), mode=mode)
    return os.getpid()


def _pool_solve(mode):
    secs, m, _ = run_oracle(_POOL_SAMPLE, mode)
    return secs, m


def _host_mem_gb():
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) / 1e6
    except OSError:
        pass
    return 16.0


# --------------------------------------------------------------- clocks

class ClockSampler:
    def __init__(self, index):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                clk, mx, util = float(f[0]), float(f[1]), float(f[7])
            except ValueError:
                continue
            smax = mx
            sm.append(clk)  # every sample falls inside the timed region
            for nm, val in zip(names, f[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "interval_ms": 20}


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_from_profiles(kernel, workload):
    """dram read+write bytes of one launch of `kernel` from the committed ncu
    --set full summary (profiles/ncu_summary.json: launches of a C2 solve,
    so only C2 lines carry it)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if workload != "c2" or not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    return d.get("traffic_bytes_per_launch", {}).get(kernel)


# ---------------------------------------------------------------- arms

def reference_arm(args):
    """The reference's CPU algorithm (the oracle port: the reference itself is
    Python+numba and single-threaded) on the box's host cores: every step is
    one full solve of the sample, the steps run concurrently in a process
    pool with one single-threaded solver per core, value = edges of all steps
    / wall time of the timed steps."""
    global _POOL_SAMPLE
    import multiprocessing as mp

    rank, _, world = dist_env()
    if rank != 0:
        return
    mode = mode_of(args.workload)
    _POOL_SAMPLE, desc, same = cpu_sample(args.workload)
    cpus = os.cpu_count() or 1
    per_solve_gb = 3.0 * max(1.0, _POOL_SAMPLE[1].size / 10e6)  # ~1.5 GB RSS per 10 M-edge solve, 2x margin
    workers = max(1, min(args.steps, cpus, int(_host_mem_gb() / per_solve_gb)))
    ctx = mp.get_context("fork")
    with ctx.Pool(workers) as pool:
        pool.map(_pool_warm, [mode] * max(workers, args.warmup))  # page in the library in every worker
        t0 = time.perf_counter()
        res = pool.map(_pool_solve, [mode] * args.steps, chunksize=1)
        wall = time.perf_counter() - t0
    m = res[0][1]
    value = m * args.steps / wall
    lat = [r[0] for r in res]
    sample = "%s; %d steps over %d worker processes (1 thread each, %d host cores), solve latency %.2f s mean" % (
        desc, args.steps, workers, cpus, statistics.mean(lat))
    line = {
        "impl": "reference", "metric": "multicut solve throughput (edges/s)", "value": value, "unit": "edges/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD_DESC[args.workload], "edges": int(m), "mode": mode, "sample": desc,
                   "same_config": same},
        "solve_latency_s": statistics.mean(lat),
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": workers, "kind": "port", "sample": sample,
                         "same_config": same},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def b200_arm(args):
    import torch

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2109_01838_b200 as P
    from paper_2109_01838_b200 import _lib, instances

    mode = mode_of(args.workload)
    cfg = P.SolverConfig(mode=mode)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    if args.workload == "c5batch":
        # 64 independent 512x512 instances sharded over the
        # ranks, solved concurrently per GPU, one NCCL gather at the end
        from paper_2109_01838_b200 import batch as B

        count = BATCH_INSTANCES
        lo, hi = B.shard_range(count, rank, world)
        graphs = [P.WeightedGraph(*instances.make("c5", seed=s)) for s in range(lo, hi)]
        n = graphs[0].num_nodes
        m_inst = graphs[0].num_edges
        node_off = np.arange(hi - lo + 1, dtype=np.int64) * n
        edge_off = np.concatenate([[0], np.cumsum([gg.num_edges for gg in graphs])]).astype(np.int64)
        du = torch.cat([gg.device()[0] for gg in graphs])
        dv = torch.cat([gg.device()[1] for gg in graphs])
        dc = torch.cat([gg.device()[2] for gg in graphs])
        labels = torch.empty(int(node_off[-1]), dtype=torch.int32, device="cuda")
        m = int(edge_off[-1])  # this rank's edges per step
        m_step = count * m_inst
        g = None

        def step():
            _, out = P.solve_batch_device(node_off, edge_off, du, dv, dc, cfg, BATCH_WORKERS, labels)
            obj = torch.from_numpy(out.reshape(-1, 2)).to("cuda")
            if world > 1:
                B.gather_results(labels, obj, n, count)
            return float(out[0]), float(out[1]), []

        hu = torch.cat([torch.from_numpy(gg.edges_u.astype(np.int32)) for gg in graphs]).pin_memory()
        hv = torch.cat([torch.from_numpy(gg.edges_v.astype(np.int32)) for gg in graphs]).pin_memory()
        hc = torch.cat([torch.from_numpy(gg.costs) for gg in graphs]).pin_memory()
        hl = torch.empty(labels.numel(), dtype=torch.int32).pin_memory()
        eu, ev, ec = torch.empty_like(du), torch.empty_like(dv), torch.empty_like(dc)

        def e2e_step():  # host COO in, host labels out
            eu.copy_(hu, non_blocking=True)
            ev.copy_(hv, non_blocking=True)
            ec.copy_(hc, non_blocking=True)
            _, out = P.solve_batch_device(node_off, edge_off, eu, ev, ec, cfg, BATCH_WORKERS, labels)
            hl.copy_(labels, non_blocking=True)
            torch.cuda.current_stream().synchronize()

        e2e_h2d, e2e_d2h = int(m * 16), int(labels.numel() * 4 + 16 * (hi - lo))
        e2e_host = "pinned torch tensors copied by the caller, labels copied back"
        job = {"instances_per_step": count, "instances_per_gpu": hi - lo, "nodes_per_instance": n,
               "edges_per_instance": m_inst, "union_groups_per_gpu": BATCH_WORKERS}
    else:
        n, u, v, c = instances.make(args.workload, seed=rank)
        g = P.WeightedGraph(n, u, v, c)  # canonicalised on the GPU (not timed)
        m = g.num_edges
        m_step = world * m
        du, dv, dc = g.device()
        labels = torch.empty(n, dtype=torch.int32, device="cuda")
        gathered = objs = None
        if world > 1:
            gathered = torch.empty(world * n, dtype=torch.int32, device="cuda")
            objs = torch.empty(world * 2, dtype=torch.float64, device="cuda")

        def step():
            _, primal, lb, trace = P.solve_device(n, du, dv, dc, m, cfg, labels)
            if world > 1:  # NCCL gather of labels and objectives (the only exchange)
                torch.distributed.all_gather_into_tensor(gathered, labels)
                mine = torch.tensor([primal, lb], dtype=torch.float64, device="cuda")
                torch.distributed.all_gather_into_tensor(objs, mine)
            return primal, lb, trace

        # plain (pageable) numpy arrays, as the parcut-side binding of
        # INTEGRATION.md passes them; rama_solve_host stages them itself
        hu = np.ascontiguousarray(g.edges_u, dtype=np.int32)
        hv = np.ascontiguousarray(g.edges_v, dtype=np.int32)
        hc = np.ascontiguousarray(g.costs, dtype=np.float64)
        hlab = np.empty(max(n, 1), dtype=np.int32)

        def e2e_step():  # rama_solve_host: H2D + solve + D2H inside the C ABI call
            P.solve_host(n, hu, hv, hc, cfg, labels=hlab)

        e2e_h2d, e2e_d2h = int(m * (4 + 4 + 8)), int(n * 4 + 16)
        e2e_host = "pageable numpy arrays (rama_solve_host stages them through pinned chunks)"
        job = {"instances_per_step": world, "seed": "rank"}

    for _ in range(args.warmup):
        step()
        flush.zero_()
    barrier()
    clocks = ClockSampler(local)
    launches0 = _lib.launches
    ms = []
    for _ in range(args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        primal, lb, trace = step()
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
        flush.zero_()
    barrier()
    launches = _lib.launches - launches0  # our kernels in the timed region (all steps)
    clk = clocks.stop()
    t_local = sum(ms)
    t = torch.tensor([t_local], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    t_max = float(t.item())
    value = m_step * args.steps / (t_max / 1e3)

    # the same steps again with per-kernel CUDA events (kept out of the timed
    # region above): kernel and family device times for the roofline
    _lib.profile_enable(True)
    p_ms = 0.0
    for _ in range(args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        p_ms += e0.elapsed_time(e1)
        flush.zero_()
    fam = _lib.profile_read()
    kern, fam_kern = _lib.profile_kernels(by_family=True)
    _lib.profile_enable(False)

    # end to end through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        for _ in range(max(1, args.warmup)):
            e2e_step()
        barrier()
        e_ms = []
        for _ in range(args.steps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            e2e_step()
            e1.record(stream)
            e1.synchronize()
            e_ms.append(e0.elapsed_time(e1))
            flush.zero_()
        barrier()
        te = torch.tensor([sum(e_ms)], dtype=torch.float64, device="cuda")
        if world > 1:
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        e2e = {"value": m_step * args.steps / (float(te.item()) / 1e3), "unit": "edges/s",
               "h2d_bytes_per_step": e2e_h2d, "d2h_bytes_per_step": e2e_d2h,
               "ms_per_step": float(te.item()) / args.steps, "host_memory": e2e_host}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    # roofline of the dominant kernel (largest device time in the profiled
    # steps); algorithmic bytes per launch are defined in DESIGN.md section 4
    peak, peak_src = peak_hbm()
    ranked = sorted(kern.items(), key=lambda kv: -kv[1][0])
    roof = None
    if ranked:
        name, (k_ms, k_bytes, k_cnt) = ranked[0]
        dominant = name
        if k_bytes <= 0:  # no defined bytes: report the top kernel that has them, and say so
            with_bytes = [kv for kv in ranked if kv[1][1] > 0]
            if with_bytes:
                name, (k_ms, k_bytes, k_cnt) = with_bytes[0]
        achieved = k_bytes / (k_ms / 1e3) / 1e9 if k_ms > 0 else 0.0
        roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_source": peak_src, "traffic": traffic_from_profiles(name, args.workload),
                "algorithmic_bytes_per_launch": k_bytes / max(k_cnt, 1), "launches_per_step": k_cnt / args.steps,
                "avg_launch_us": 1e3 * k_ms / max(k_cnt, 1), "share_of_step": k_ms / p_ms,
                "dominant_kernel": dominant}
    kernels = [{"kernel": k, "ms_per_step": v[0] / args.steps, "share": v[0] / p_ms, "launches_per_step": v[2] / args.steps,
                "GB_per_s": (v[1] / (v[0] / 1e3) / 1e9) if v[1] > 0 and v[0] > 0 else None}
               for k, v in ranked[:40]]
    families = {k: {"ms_per_step": vv[0] / args.steps, "kernel_ms_per_step": fam_kern.get(k, (0.0,))[0] / args.steps,
                    "alg_GB_per_step": vv[1] / args.steps / 1e9,
                    "scopes_per_step": vv[2] / args.steps} for k, vv in fam.items() if vv[2]}

    gap = None
    refp = os.path.join(ROOT, "tests", "golden", "c2_reference.json")
    if args.workload == "c2" and rank == 0 and os.path.exists(refp):
        with open(refp) as fh:
            ref = json.load(fh)
        gap = {"primal_pct": 100.0 * (primal - ref["primal"]) / abs(ref["primal"]),
               "lb_pct": 100.0 * (lb - ref["lower_bound"]) / abs(ref["lower_bound"]),
               "reference_primal": ref["primal"], "reference_lb": ref["lower_bound"]}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.workload)

    line = {
        "metric": "multicut solve throughput (edges/s)", "value": value, "unit": "edges/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.workload == "c5batch" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict({"workload": WORKLOAD_DESC[args.workload], "nodes": n, "edges": m, "mode": mode,
                   "l2": "inputs %.0f MB > 126 MB L2, and a 256 MiB buffer is written between steps" % (m * 16 / 1e6),
                   "parallelism": ("instances sharded over %d GPUs, NCCL gather" % world) if world > 1 else "single GPU",
                   "scaling_note": ("strong: 64 instances per step whatever N" if args.workload == "c5batch"
                                    else "weak: one instance per GPU")}, **job),
        "solve_time_s": t_max / args.steps / 1e3,
        "objective": {"primal": primal, "lower_bound": lb, "rounds": len(trace), "gap_vs_cpu_reference": gap},
        "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "clocks": clk, "gpu_launches": launches,
        "top_kernels": kernels, "kernel_families": families,
        "device_busy": {"kernel_ms_per_step": sum(v[0] for v in kern.values()) / args.steps,
                        "profiled_step_ms": p_ms / args.steps,
                        "note": "sum of our kernels' event-timed durations vs the profiled step (per-kernel events "
                                "add small gaps); the rest is launch latency and host round trips.  With concurrent "
                                "streams (c5batch) kernels overlap and the sum exceeds the step"},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def spawn_ranks(args):
    """--gpus N > 1 without a torchrun environment: re-exec under
    torch.distributed.run (one process per GPU, NCCL, 127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    if args.impl == "reference":
        reference_arm(args)
    else:
        b200_arm(args)


if __name__ == "__main__":
    main()
