// extern "C" boundary (include/rama_b200.h).  Every entry point runs inside
// `guarded`, which owns the per-call context, converts exceptions to status
// codes and records the message for rama_last_error().
#include "../../include/rama_b200.h"
#include "internal.h"

#include <atomic>
#include <cmath>
#include <mutex>
#include <thread>
#include <limits>
#include <new>
#include <string>
#include <vector>

using namespace rama;

namespace {

thread_local std::string g_err;
thread_local int64_t g_launches = 0;

template <class F>
int guarded(void* stream, F&& f) {
  g_err.clear();
  g_launches = 0;
  try {
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
      cudaGetLastError();
      throw Error(kCuda, "no CUDA device available (the B200 build has no CPU fallback)");
    }
    Ctx ctx((cudaStream_t)stream);
    f(ctx);
    ctx.sync();
    RAMA_CUDA(cudaGetLastError());
    g_launches = ctx.launches;
    return RAMA_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return RAMA_ERR_NOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RAMA_ERR_INTERNAL;
  }
}

GraphView view_of(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m) {
  GraphView g;
  g.n = n; g.m = m; g.u = u; g.v = v; g.c = c;
  return g;
}

void check_sizes(int64_t n, int64_t m) {
  RAMA_REQUIRE(n >= 0 && m >= 0, "sizes must be non-negative");
  RAMA_REQUIRE(n < (1LL << 31) && m < (1LL << 31), "graph too large for int32 ids");
}

void export_graph(Ctx& ctx, const Graph& g, int32_t* ou, int32_t* ov, double* oc, int64_t* om) {
  copy_d2d(ctx, ou, g.u.p, g.m);
  copy_d2d(ctx, ov, g.v.p, g.m);
  copy_d2d(ctx, oc, g.c.p, g.m);
  *om = g.m;
}

SolveConfig to_cfg(const rama_cfg* cfg) {
  RAMA_REQUIRE(cfg != nullptr, "cfg is NULL");
  SolveConfig c;
  c.mode = cfg->mode;
  c.mp_iterations = cfg->mp_iterations;
  c.max_cycle_length = cfg->max_cycle_length;
  c.max_rounds = cfg->max_rounds;
  c.separation_rounds = cfg->separation_rounds;
  c.switch_fraction = cfg->matching_switch_fraction;
  // SolverConfig.validate (solver.py:50-62)
  RAMA_REQUIRE(c.mode >= 0 && c.mode <= 4, "unknown mode");
  RAMA_REQUIRE(!(c.mode >= 1 && c.mode <= 3) || c.mp_iterations >= 1, "mp_iterations must be at least 1 for dual modes");
  RAMA_REQUIRE(c.max_cycle_length >= 3, "max_cycle_length must be at least 3");
  RAMA_REQUIRE(c.switch_fraction > 0.0 && c.switch_fraction <= 1.0, "matching_switch_fraction must be in (0, 1]");
  RAMA_REQUIRE(c.max_rounds >= 1, "max_rounds must be at least 1");
  RAMA_REQUIRE(c.separation_rounds >= 1, "separation_rounds must be at least 1");
  return c;
}

rama_round to_round(const RoundInfo& r) {
  rama_round o;
  o.round_index = r.round_index;
  o.phase = r.phase;
  o.nodes = r.nodes;
  o.edges = r.edges;
  o.triplets = r.triplets;
  o.lb = r.lb;
  o.lb_valid = r.lb_valid;
  o.reserved = 0;
  o.contracted = r.contracted;
  o.time_ms = r.time_ms;
  return o;
}

void run_solve(Ctx& ctx, int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m,
               const rama_cfg* cfg, int32_t* labels, double* primal_lb, rama_round* trace, int32_t max_trace,
               int32_t* n_rounds) {
  check_sizes(n, m);
  SolveConfig sc = to_cfg(cfg);
  GraphView g = view_of(n, u, v, c, m);
  Graph canon;
  if (m > 0 && !is_canonical(ctx, g)) {
    canon = canonicalize(ctx, n, u, v, c, m);
    g = canon.view();
  }
  std::vector<RoundInfo> tr(max_trace > 0 ? max_trace : 0);
  SolveResult res;
  solve(ctx, g, sc, labels, res, tr.data(), (int)tr.size());
  primal_lb[0] = res.primal;
  primal_lb[1] = res.lb_finite ? res.lb : -std::numeric_limits<double>::infinity();
  int written = res.n_rounds < max_trace ? res.n_rounds : max_trace;
  for (int i = 0; trace && i < written; i++) trace[i] = to_round(tr[i]);
  if (n_rounds) *n_rounds = res.n_rounds;
}

// DualState over caller arrays (copied; slot lists rebuilt)
void load_state(Ctx& ctx, DualState& st, int64_t m_aug, const double* base, int64_t T, const int32_t* tri_edges,
                const double* lam) {
  st.m_aug = m_aug;
  st.T = T;
  st.base.alloc(m_aug > 0 ? m_aug : 1, ctx.s);
  copy_d2d(ctx, st.base.p, base, m_aug);
  st.tri_edges.alloc(T > 0 ? 3 * T : 1, ctx.s);
  copy_d2d(ctx, st.tri_edges.p, tri_edges, 3 * T);
  st.lam.alloc(T > 0 ? 3 * T : 1, ctx.s);
  copy_d2d(ctx, st.lam.p, lam, 3 * T);
  build_slot_lists(ctx, st);
}

__global__ void k_handle_check(const int32_t* __restrict__ te, int64_t S, int64_t m_aug, int32_t* bad) {
  GRID_STRIDE(s, S) {
    if (te[s] < 0 || te[s] >= m_aug) atomicOr(bad, 1);
  }
}

void check_handles(Ctx& ctx, const int32_t* te, int64_t T, int64_t m_aug) {
  if (T <= 0) return;
  Buf<int32_t> bad(1, ctx);
  bad.zero();
  RAMA_KERNEL(ctx, k_handle_check, 3 * T, te, 3 * T, m_aug, bad.p);
  RAMA_REQUIRE(read_scalar(ctx, bad.p) == 0, "triplet edge handle out of range");
}

}  // namespace

extern "C" {

int rama_version(void) { return 1 * 10000 + 0 * 100 + 0; }

const char* rama_last_error(void) { return g_err.c_str(); }

int64_t rama_last_launch_count(void) { return g_launches; }

int rama_profile_enable(int32_t on) {
  return guarded(nullptr, [&](Ctx&) { prof_set(on != 0); });
}

int rama_profile_read(double* ms, double* bytes, int64_t* count) {
  return guarded(nullptr, [&](Ctx&) { prof_read(ms, bytes, count); });
}

int64_t rama_profile_kernels(char* out, int64_t cap) { return prof_kernels_json(out, cap); }

int rama_solve(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m, const rama_cfg* cfg,
               int32_t* labels, double* primal_lb, rama_round* trace, int32_t max_trace, int32_t* n_rounds,
               void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    run_solve(ctx, n, u, v, c, m, cfg, labels, primal_lb, trace, max_trace, n_rounds);
  });
}

int rama_solve_ws(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m, const rama_cfg* cfg,
                  int32_t* labels, double* primal_lb, rama_round* trace, int32_t max_trace, int32_t* n_rounds,
                  void* ws, uint64_t ws_bytes, uint64_t* ws_peak, void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    RAMA_REQUIRE(ws != nullptr || ws_bytes == 0, "workspace pointer is NULL");
    Arena arena(ws, (size_t)ws_bytes);
    {
      ArenaScope scope(&arena);
      run_solve(ctx, n, u, v, c, m, cfg, labels, primal_lb, trace, max_trace, n_rounds);
      ctx.sync();  // the workspace's ranges are in use until the stream drains
    }
    if (ws_peak) *ws_peak = arena.peak;
  });
}

uint64_t rama_ws_bytes(int64_t n, int64_t m, const rama_cfg* cfg) {
  const int L = cfg ? cfg->max_cycle_length : 5;
  const double per_edge = 400.0 + 96.0 * (L > 5 ? L - 5 : 0);
  return (uint64_t)(per_edge * (double)(m > 0 ? m : 0) + 96.0 * (double)(n > 0 ? n : 0)) + ((uint64_t)64 << 20);
}

int rama_release_cache(void) {
  return guarded(nullptr, [&](Ctx&) { dev_release_all(); });
}

int rama_solve_host(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m, const rama_cfg* cfg,
                    int32_t* labels, double* primal_lb, rama_round* trace, int32_t max_trace, int32_t* n_rounds,
                    void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    check_sizes(n, m);
    Buf<int32_t> du(m > 0 ? m : 1, ctx), dv(m > 0 ? m : 1, ctx), dl(n > 0 ? n : 1, ctx);
    Buf<double> dc(m > 0 ? m : 1, ctx);
    if (m > 0) {
      copy_h2d(ctx, du.p, u, sizeof(int32_t) * m);
      copy_h2d(ctx, dv.p, v, sizeof(int32_t) * m);
      copy_h2d(ctx, dc.p, c, sizeof(double) * m);
    }
    run_solve(ctx, n, du.p, dv.p, dc.p, m, cfg, dl.p, primal_lb, trace, max_trace, n_rounds);
    if (n > 0) copy_d2h(ctx, labels, dl.p, sizeof(int32_t) * n);
  });
}

int rama_canonicalize(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m, int32_t* out_u,
                      int32_t* out_v, double* out_c, int64_t* out_m, void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    check_sizes(n, m);
    Graph g = canonicalize(ctx, n, u, v, c, m);
    export_graph(ctx, g, out_u, out_v, out_c, out_m);
  });
}

int rama_clustering_cost(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m,
                         const int32_t* labels, double* cost, void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    check_sizes(n, m);
    *cost = clustering_cost(ctx, view_of(n, u, v, c, m), labels);
  });
}

int rama_components(int64_t n, const int32_t* su, const int32_t* sv, int64_t k, int32_t* map, int64_t* num_targets,
                    void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    check_sizes(n, k);
    *num_targets = components(ctx, n, su, sv, k, map, true);
  });
}

int rama_contract(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m, const int32_t* map,
                  int64_t n_targets, int32_t* out_u, int32_t* out_v, double* out_c, int64_t* out_m, double* joined,
                  void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    check_sizes(n, m);
    Graph g = contract(ctx, view_of(n, u, v, c, m), map, n_targets, joined);
    export_graph(ctx, g, out_u, out_v, out_c, out_m);
  });
}

int rama_select_matching(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m, int32_t rounds,
                         int32_t* su, int32_t* sv, int64_t* k, void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    check_sizes(n, m);
    Buf<int32_t> a, b;
    *k = select_matching(ctx, view_of(n, u, v, c, m), rounds, a, b);
    copy_d2d(ctx, su, a.p, *k);
    copy_d2d(ctx, sv, b.p, *k);
  });
}

int rama_select_max_edge(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m, int64_t* edge,
                         void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    check_sizes(n, m);
    *edge = select_max_edge(ctx, view_of(n, u, v, c, m));
  });
}

int rama_select_forest(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m, int32_t* su,
                       int32_t* sv, int64_t* k, void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    check_sizes(n, m);
    Buf<int32_t> a, b;
    *k = select_forest(ctx, view_of(n, u, v, c, m), a, b);
    copy_d2d(ctx, su, a.p, *k);
    copy_d2d(ctx, sv, b.p, *k);
  });
}

int rama_contraction_step(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m, int32_t policy,
                          double switch_fraction, int32_t* map, int32_t* out_u, int32_t* out_v, double* out_c,
                          int64_t* info, double* joined, void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    check_sizes(n, m);
    RAMA_REQUIRE(policy >= 0 && policy <= 3, "unknown contraction policy");
    GraphView g = view_of(n, u, v, c, m);
    StepResult st;
    contraction_step(ctx, g, policy, switch_fraction, st, true);
    info[1] = st.num_selected;
    info[3] = st.used_forest ? 1 : 0;
    *joined = st.joined;
    if (st.identity) {
      iota(ctx, map, n);
      copy_d2d(ctx, out_u, u, m);
      copy_d2d(ctx, out_v, v, m);
      copy_d2d(ctx, out_c, c, m);
      info[0] = n;
      info[2] = m;
    } else {
      copy_d2d(ctx, map, st.map.p, n);
      int64_t mo = 0;
      export_graph(ctx, st.next, out_u, out_v, out_c, &mo);
      info[0] = st.num_targets;
      info[2] = mo;
    }
  });
}

int rama_separate(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m, int32_t L,
                  int32_t* out_len, int32_t* out_nodes, int64_t* rows, void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    check_sizes(n, m);
    CycleRows cyc;
    separate(ctx, view_of(n, u, v, c, m), L, cyc);
    copy_d2d(ctx, out_len, cyc.len.p, cyc.rows);
    copy_d2d(ctx, out_nodes, cyc.nodes.p, cyc.rows * (int64_t)L);
    *rows = cyc.rows;
  });
}

int rama_triangulate(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m, const int32_t* len,
                     const int32_t* nodes, int64_t rows, int32_t L, int32_t* aug_u, int32_t* aug_v, double* base,
                     int64_t* m_aug, int32_t* tri_nodes, int32_t* tri_edges, int64_t* T, int32_t* coverage,
                     void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    check_sizes(n, m);
    RAMA_REQUIRE(L >= 3 && rows >= 0, "bad cycle rows");
    CycleRows cyc;
    cyc.rows = rows;
    cyc.L = L;
    cyc.len.alloc(rows > 0 ? rows : 1, ctx.s);
    cyc.nodes.alloc(rows > 0 ? rows * L : 1, ctx.s);
    copy_d2d(ctx, cyc.len.p, len, rows);
    copy_d2d(ctx, cyc.nodes.p, nodes, rows * (int64_t)L);
    DualState st;
    triangulate(ctx, view_of(n, u, v, c, m), cyc, st);
    copy_d2d(ctx, aug_u, st.eu.p, st.m_aug);
    copy_d2d(ctx, aug_v, st.ev.p, st.m_aug);
    copy_d2d(ctx, base, st.base.p, st.m_aug);
    copy_d2d(ctx, coverage, st.coverage.p, st.m_aug);
    copy_d2d(ctx, tri_nodes, st.tri_nodes.p, 3 * st.T);
    copy_d2d(ctx, tri_edges, st.tri_edges.p, 3 * st.T);
    *m_aug = st.m_aug;
    *T = st.T;
  });
}

int rama_extend_separation(int64_t n, int64_t m_aug, const int32_t* eu, const int32_t* ev, const double* base,
                           int64_t T, const int32_t* tri_nodes, const int32_t* tri_edges, const double* lam,
                           int32_t L, int64_t cap_edges, int64_t cap_triplets, int32_t* out_eu, int32_t* out_ev,
                           double* out_base, int64_t* out_m_aug, int32_t* out_tri_nodes, int32_t* out_tri_edges,
                           double* out_lam, int64_t* out_T, int32_t* out_coverage, int64_t* added, void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    check_sizes(n, m_aug);
    RAMA_REQUIRE(L >= 3, "max_len must be at least 3");
    check_handles(ctx, tri_edges, T, m_aug);
    DualState st;
    st.n = n;
    st.m_orig = m_aug;
    st.m_aug = m_aug;
    st.chords_sorted = false;  // caller's edge order is arbitrary
    st.eu.alloc(m_aug > 0 ? m_aug : 1, ctx.s);
    st.ev.alloc(m_aug > 0 ? m_aug : 1, ctx.s);
    copy_d2d(ctx, st.eu.p, eu, m_aug);
    copy_d2d(ctx, st.ev.p, ev, m_aug);
    st.tri_nodes.alloc(T > 0 ? 3 * T : 1, ctx.s);
    copy_d2d(ctx, st.tri_nodes.p, tri_nodes, 3 * T);
    load_state(ctx, st, m_aug, base, T, tri_edges, lam);
    int64_t k = extend_separation(ctx, st, L);
    RAMA_REQUIRE(st.m_aug <= cap_edges && st.T <= cap_triplets, "output capacity too small");
    copy_d2d(ctx, out_eu, st.eu.p, st.m_aug);
    copy_d2d(ctx, out_ev, st.ev.p, st.m_aug);
    copy_d2d(ctx, out_base, st.base.p, st.m_aug);
    copy_d2d(ctx, out_coverage, st.coverage.p, st.m_aug);
    copy_d2d(ctx, out_tri_nodes, st.tri_nodes.p, 3 * st.T);
    copy_d2d(ctx, out_tri_edges, st.tri_edges.p, 3 * st.T);
    copy_d2d(ctx, out_lam, st.lam.p, 3 * st.T);
    *out_m_aug = st.m_aug;
    *out_T = st.T;
    *added = k;
  });
}

int rama_check_agreement(int64_t m_aug, const double* base, int64_t T, const int32_t* tri_edges, const double* lam,
                         double eps, int32_t* agree, void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    check_sizes(0, m_aug);
    check_handles(ctx, tri_edges, T, m_aug);
    DualState st;
    load_state(ctx, st, m_aug, base, T, tri_edges, lam);
    *agree = check_edge_triangle_agreement(ctx, st, eps) ? 1 : 0;
  });
}

int rama_message_passing(int64_t m_aug, const double* base, int64_t T, const int32_t* tri_edges, double* lam,
                         int32_t iters, int32_t phases, void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    check_sizes(0, m_aug);
    RAMA_REQUIRE(phases >= 1 && phases <= 3, "phases must be 1, 2 or 3");
    check_handles(ctx, tri_edges, T, m_aug);
    DualState st;
    load_state(ctx, st, m_aug, base, T, tri_edges, lam);
    for (int it = 0; it < iters; it++) {
      if (phases == 3) message_passing(ctx, st, 1);
      else mp_phases(ctx, st, phases == 1, phases == 2);
    }
    copy_d2d(ctx, lam, st.lam.p, 3 * T);
  });
}

int rama_reparam_costs(int64_t m_aug, const double* base, int64_t T, const int32_t* tri_edges, const double* lam,
                       double* cl, void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    check_sizes(0, m_aug);
    check_handles(ctx, tri_edges, T, m_aug);
    DualState st;
    load_state(ctx, st, m_aug, base, T, tri_edges, lam);
    reparam_costs(ctx, st, cl);
  });
}

int rama_lower_bound(int64_t m_aug, const double* base, int64_t T, const int32_t* tri_edges, const double* lam,
                     double* lb, void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    check_sizes(0, m_aug);
    check_handles(ctx, tri_edges, T, m_aug);
    DualState st;
    load_state(ctx, st, m_aug, base, T, tri_edges, lam);
    *lb = lower_bound(ctx, st);
  });
}

int rama_solve_batch(int64_t count, const int64_t* node_off, const int64_t* edge_off, const int32_t* u,
                     const int32_t* v, const double* c, const rama_cfg* cfg, int32_t* labels, double* primal_lb,
                     rama_round* trace, int32_t max_trace, int32_t* n_rounds, int32_t workers, void* stream) {
  return guarded(stream, [&](Ctx& ctx) {
    RAMA_REQUIRE(count >= 0, "count must be non-negative");
    if (count == 0) return;
    RAMA_REQUIRE(node_off && edge_off && primal_lb, "offset / result arrays must not be NULL");
    const SolveConfig sc = to_cfg(cfg);
    for (int64_t i = 0; i < count; i++) {
      RAMA_REQUIRE(node_off[i + 1] >= node_off[i] && edge_off[i + 1] >= edge_off[i], "offsets must be non-decreasing");
      check_sizes(node_off[i + 1] - node_off[i], edge_off[i + 1] - edge_off[i]);
    }
    if (max_trace < 0 || !trace) max_trace = 0;
    // modes P / PD / PD+: contiguous groups of instances, each solved as one
    // disjoint union (batch.cu); modes D / GAEC: one instance per job
    const bool uni = sc.mode <= 2;
    int W = workers > 0 ? workers : 1;
    if (W > count) W = (int)count;
    std::vector<int64_t> job_lo, job_hi;
    if (uni) {
      for (int w = 0; w < W; w++) {
        job_lo.push_back(count * w / W);
        job_hi.push_back(count * (w + 1) / W);
      }
    } else {
      for (int64_t i = 0; i < count; i++) {
        job_lo.push_back(i);
        job_hi.push_back(i + 1);
      }
    }
    int dev = 0;
    RAMA_CUDA(cudaGetDevice(&dev));
    cudaEvent_t start;
    RAMA_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    RAMA_CUDA(cudaEventRecord(start, ctx.s));
    std::vector<cudaStream_t> streams(W);
    for (int w = 0; w < W; w++) {
      RAMA_CUDA(cudaStreamCreateWithFlags(&streams[w], cudaStreamNonBlocking));
      RAMA_CUDA(cudaStreamWaitEvent(streams[w], start, 0));
    }
    std::atomic<int64_t> next(0), launches(0);
    const int64_t njobs = (int64_t)job_lo.size();
    std::mutex mu;
    int err_code = 0;
    std::string err_msg;
    auto worker = [&](int w) {
      try {
        RAMA_CUDA(cudaSetDevice(dev));
        Ctx wc(streams[w]);
        std::vector<RoundInfo> tr;
        while (true) {
          const int64_t j = next.fetch_add(1);
          if (j >= njobs) break;
          const int64_t lo = job_lo[j], hi = job_hi[j], k = hi - lo;
          const int64_t no = node_off[lo], eo = edge_off[lo];
          if (uni) {
            tr.assign((size_t)k * max_trace, RoundInfo());
            std::vector<int32_t> nr(k, 0);
            solve_union(wc, k, node_off + lo, edge_off + lo, u + eo, v + eo, c + eo, sc, labels + no,
                        primal_lb + 2 * lo, max_trace ? tr.data() : nullptr, max_trace, nr.data());
            for (int64_t i = 0; i < k; i++) {
              const int written = nr[i] < max_trace ? nr[i] : max_trace;
              for (int r = 0; r < written; r++)
                trace[(lo + i) * max_trace + r] = to_round(tr[(size_t)i * max_trace + r]);
              if (n_rounds) n_rounds[lo + i] = nr[i];
            }
          } else {
            run_solve(wc, node_off[lo + 1] - no, u + eo, v + eo, c + eo, edge_off[lo + 1] - eo, cfg, labels + no,
                      primal_lb + 2 * lo, max_trace ? trace + lo * max_trace : nullptr, max_trace,
                      n_rounds ? n_rounds + lo : nullptr);
          }
        }
        wc.sync();
        launches += wc.launches;
      } catch (const Error& e) {
        std::lock_guard<std::mutex> lk(mu);
        if (!err_code) { err_code = e.code; err_msg = e.what(); }
        next = njobs;
      } catch (const std::exception& e) {
        std::lock_guard<std::mutex> lk(mu);
        if (!err_code) { err_code = kInternal; err_msg = e.what(); }
        next = njobs;
      }
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < W; w++) pool.emplace_back(worker, w);
    worker(0);
    for (auto& t : pool) t.join();
    for (int w = 0; w < W; w++) {
      cudaEvent_t done;
      RAMA_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
      RAMA_CUDA(cudaEventRecord(done, streams[w]));
      RAMA_CUDA(cudaStreamWaitEvent(ctx.s, done, 0));
      cudaEventDestroy(done);
      dev_release_stream(streams[w]);
      cudaStreamDestroy(streams[w]);
    }
    cudaEventDestroy(start);
    ctx.launches += (int)launches.load();
    if (err_code) throw Error(err_code, "batch instance failed: " + err_msg);
  });
}

}  // extern "C"
