// Batch of independent instances solved as ONE disjoint union (SURVEY.md
// 7.3.5 and 8(e), config C5).
//
// A batch of small graphs solved one by one is launch-bound: a 512x512 grid
// takes ~650 launches and ~100 host read-backs per solve, so 64 of them
// spend most of the step issuing work.  Here the instances are renumbered
// into one graph whose node ranges are contiguous per instance, and every
// kernel of the round loop (separation, triangulation, message passing,
// contraction, cleanup) runs once per round over all of them.  Every one of
// those operators is local to a connected component and keeps the
// instance's relative order (canonical (u, v) sorting, triplets sorted by
// node, canonical relabelling by smallest member), so each instance's
// result is the single solve's bit for bit.  What is NOT local in the
// reference loop is done per instance here (solver.py:147-208):
//   * the auto contraction policy (contraction.py:384-387): matching on the
//     union, |S_i| counted per instance, the forest run on the edges of the
//     instances with |S_i| < fraction * n_i only;
//   * termination: an instance stops when its S_i is empty or it has one
//     node left; its edges then leave the working graph (its nodes stay, as
//     singletons);
//   * the trace (n_i, m_i, T_i, |S_i| per round), the first-round lower
//     bound and the primal: segment bounds by binary search over the
//     instance node ranges, and the sums in exactly the single solve's
//     reduction order (device_sums), so objectives match bit for bit.
// Modes D and GAEC keep the per-instance path in capi.cu (mode D grows the
// triplet list out of instance order; GAEC joins one global max edge).
#include "internal.h"
#include "compact.cuh"

#include <chrono>
#include <cmath>
#include <vector>

namespace rama {

namespace {

using clk = std::chrono::steady_clock;

double ms_since(clk::time_point t0) { return std::chrono::duration<double, std::milli>(clk::now() - t0).count(); }

// largest i in [0, K) with off[i] <= x (the instance holding x; empty
// instances share their offset with the next one and are skipped)
__device__ __forceinline__ int32_t inst_of(const int64_t* __restrict__ off, int32_t K, int64_t x) {
  int32_t lo = 0, hi = K - 1;
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (off[mid] <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// union ids: local ids of slice i shifted by its node offset (range-checked)
__global__ void k_union_ids(const int32_t* __restrict__ u, const int32_t* __restrict__ v, int64_t m,
                            const int64_t* __restrict__ eoff, const int64_t* __restrict__ noff, int32_t K,
                            int32_t* __restrict__ ou, int32_t* __restrict__ ov, int32_t* __restrict__ bad) {
  GRID_STRIDE(e, m) {
    const int32_t i = inst_of(eoff, K, e);
    const int64_t nl = noff[i + 1] - noff[i];
    const int32_t a = u[e], b = v[e];
    if (a < 0 || a >= nl || b < 0 || b >= nl) atomicOr(bad, 1);
    ou[e] = (int32_t)(a + noff[i]);
    ov[e] = (int32_t)(b + noff[i]);
  }
}

// out[i] = #{j : keys[j * stride] < noff[i]} for i in [0, K] (keys ascending)
__global__ void k_bounds(const int32_t* __restrict__ keys, int64_t stride, int64_t len,
                         const int64_t* __restrict__ noff, int32_t K, int64_t* __restrict__ out) {
  GRID_STRIDE(i, (int64_t)K + 1) {
    const int64_t x = noff[i];
    int64_t lo = 0, hi = len;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid * stride] < x) lo = mid + 1; else hi = mid;
    }
    out[i] = lo;
  }
}

// pairs per instance; neighbouring pairs mostly share an instance, so one
// atomic per run of equal instance ids in a warp
__global__ void k_count_inst(const int32_t* __restrict__ su, int64_t k, const int64_t* __restrict__ noff, int32_t K,
                             int32_t* __restrict__ cnt) {
  GRID_STRIDE(p, k) {
    const int32_t i = inst_of(noff, K, su[p]);
    const unsigned same = __match_any_sync(__activemask(), i);
    if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(cnt + i, __popc(same));
  }
}

// out[i] = f(noff[i]) for i < K (the instance's first node's new id), nt past the end
__global__ void k_map_offsets(const int64_t* __restrict__ noff, int32_t K, int64_t n, const int32_t* __restrict__ f,
                              int64_t nt, int64_t* __restrict__ out) {
  GRID_STRIDE(i, (int64_t)K + 1) out[i] = (i < K && noff[i] < n) ? (int64_t)f[noff[i]] : nt;
}

struct UInInst {  // u[i] lies in an instance with flag set
  const int32_t* u;
  const int64_t* noff;
  int32_t K;
  const uint8_t* flag;
  __device__ __forceinline__ bool operator()(int32_t i) const { return flag[inst_of(noff, K, u[i])] != 0; }
};

__global__ void k_gather_edges(const int32_t* __restrict__ idx, int64_t k, const int32_t* __restrict__ u,
                               const int32_t* __restrict__ v, const double* __restrict__ c, int32_t* __restrict__ ou,
                               int32_t* __restrict__ ov, double* __restrict__ oc) {
  GRID_STRIDE(p, k) {
    const int32_t e = idx[p];
    ou[p] = u[e];
    ov[p] = v[e];
    if (oc) oc[p] = c[e];
  }
}

// neg over [originals | chords] -> per instance [its originals | its chords]
// (the single solve's augmented edge order), plus the segment bounds
__global__ void k_lb_layout(const double* __restrict__ neg, int64_t m_orig, int64_t m_aug,
                            const int64_t* __restrict__ O, const int64_t* __restrict__ C, int32_t K,
                            double* __restrict__ out) {
  GRID_STRIDE(e, m_aug) {
    int64_t pos;
    if (e < m_orig) {
      const int32_t i = inst_of(O, K, e);
      pos = e + C[i] - m_orig;
    } else {
      const int32_t i = inst_of(C, K, e);
      pos = O[i + 1] + e - m_orig;
    }
    out[pos] = neg[e];
  }
}

__global__ void k_lb_segments(const int64_t* __restrict__ O, const int64_t* __restrict__ C, int64_t m_orig, int32_t K,
                              int64_t* __restrict__ start, int64_t* __restrict__ len) {
  GRID_STRIDE(i, (int64_t)K) {
    start[i] = O[i] + C[i] - m_orig;
    len[i] = (O[i + 1] - O[i]) + (C[i + 1] - C[i]);
  }
}

__global__ void k_diff_segments(const int64_t* __restrict__ off, int32_t K, int64_t* __restrict__ start,
                                int64_t* __restrict__ len) {
  GRID_STRIDE(i, (int64_t)K) {
    start[i] = off[i];
    len[i] = off[i + 1] - off[i];
  }
}

// union canonical labels -> labels local to each instance (first-occurrence
// order inside an instance is the union's order shifted by its first label)
__global__ void k_local_labels(int32_t* __restrict__ lab, int64_t n0, const int64_t* __restrict__ noff, int32_t K,
                               const int64_t* __restrict__ first) {
  GRID_STRIDE(x, n0) lab[x] -= (int32_t)first[inst_of(noff, K, x)];
}

template <class T>
void upload(Ctx& ctx, T* dev, const std::vector<T>& h) {
  if (!h.empty()) RAMA_CUDA(cudaMemcpyAsync(dev, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, ctx.s));
  ctx.sync();  // pageable source: keep the host vector alive until the copy is done
}

template <class T>
std::vector<T> download(Ctx& ctx, const T* dev, size_t count) {
  std::vector<T> h(count);
  if (count) RAMA_CUDA(cudaMemcpyAsync(h.data(), dev, sizeof(T) * count, cudaMemcpyDeviceToHost, ctx.s));
  ctx.sync();
  return h;
}

// bounds of the instances' node ranges `d_noff` in a sorted id column
std::vector<int64_t> bounds(Ctx& ctx, const int32_t* keys, int64_t stride, int64_t len, const int64_t* d_noff,
                            int32_t K, Buf<int64_t>& d_out) {
  d_out.alloc(K + 1, ctx.s);
  RAMA_KERNEL(ctx, k_bounds, K + 1, keys, stride, len, d_noff, K, d_out.p);
  return download(ctx, d_out.p, K + 1);
}

// edges of the flagged instances (a canonical sub-list of g)
Graph edges_of(Ctx& ctx, const GraphView& g, const int64_t* d_noff, int32_t K, const uint8_t* d_flag) {
  Graph out;
  out.n = g.n;
  Buf<int32_t> idx;
  const int64_t k = g.m > 0 ? compact_if(ctx, g.m, UInInst{g.u, d_noff, K, d_flag}, idx) : 0;
  out.m = k;
  out.u.alloc(k > 0 ? k : 1, ctx.s);
  out.v.alloc(k > 0 ? k : 1, ctx.s);
  out.c.alloc(k > 0 ? k : 1, ctx.s);
  RAMA_KERNEL(ctx, k_gather_edges, k, idx.p, k, g.u, g.v, g.c, out.u.p, out.v.p, out.c.p);
  return out;
}

}  // namespace

void solve_union(Ctx& ctx, int64_t K64, const int64_t* node_off, const int64_t* edge_off, const int32_t* u,
                 const int32_t* v, const double* c, const SolveConfig& cfg, int32_t* labels, double* primal_lb,
                 RoundInfo* traces, int max_trace, int32_t* n_rounds) {
  RAMA_REQUIRE(cfg.mode == 0 || cfg.mode == 1 || cfg.mode == 2, "union batch solve: modes P, PD, PD+");
  RAMA_REQUIRE(K64 >= 1 && K64 < (1 << 20), "batch size out of range");
  const int32_t K = (int32_t)K64;
  const int64_t n0 = node_off[K] - node_off[0];
  const int64_t m0 = edge_off[K] - edge_off[0];
  RAMA_REQUIRE(n0 < (int64_t)INT32_MAX && m0 < (int64_t)INT32_MAX, "batch too large for int32 ids");
  const bool dual = cfg.mode != 0;
  const double nan = std::nan("");
  reserve_pool(ctx, (size_t)256 * (size_t)m0 + (size_t)64 * (size_t)n0);

  // ---- the union graph (canonical per instance => canonical union)
  std::vector<int64_t> noff(K + 1), eoff(K + 1);
  for (int32_t i = 0; i <= K; i++) {
    noff[i] = node_off[i] - node_off[0];
    eoff[i] = edge_off[i] - edge_off[0];
  }
  Buf<int64_t> d_noff0(K + 1, ctx), d_noff(K + 1, ctx), d_tmp(K + 1, ctx);
  upload(ctx, d_noff0.p, noff);
  copy_d2d(ctx, d_noff.p, d_noff0.p, K + 1);
  Graph g;
  g.n = n0;
  g.m = m0;
  g.u.alloc(m0 > 0 ? m0 : 1, ctx.s);
  g.v.alloc(m0 > 0 ? m0 : 1, ctx.s);
  if (m0 > 0) {
    Buf<int64_t> d_eoff(K + 1, ctx);
    upload(ctx, d_eoff.p, eoff);
    Buf<int32_t> bad(1, ctx);
    bad.zero();
    RAMA_KERNEL(ctx, k_union_ids, m0, u, v, m0, d_eoff.p, d_noff0.p, K, g.u.p, g.v.p, bad.p);
    RAMA_REQUIRE(read_scalar(ctx, bad.p) == 0, "node id out of range for its instance");
  }
  GraphView gv = g.view();
  gv.c = c;
  Graph canon;
  if (m0 > 0 && !is_canonical(ctx, gv)) {  // disjoint ranges: canonicalising the union = each instance
    canon = canonicalize(ctx, n0, g.u.p, g.v.p, c, m0);
    gv = canon.view();
  }
  Buf<int64_t> d_E0;
  const std::vector<int64_t> E0 = bounds(ctx, gv.u, 1, gv.m, d_noff0.p, K, d_E0);  // original edge ranges

  // ---- round loop (solver.py:113-144 / 147-208), all instances at once
  std::vector<uint8_t> active(K, 1);
  std::vector<int32_t> nr(K, 0);
  std::vector<double> lb1(K, nan);
  auto push = [&](int32_t i, const RoundInfo& r) {
    if (traces && nr[i] < max_trace) traces[(int64_t)i * max_trace + nr[i]] = r;
    nr[i]++;
  };
  Buf<uint8_t> d_flag(K, ctx);
  iota(ctx, labels, n0);  // f_total over the union
  Graph cur;
  cur.n = n0;
  cur.m = gv.m;
  cur.u.alloc(gv.m > 0 ? gv.m : 1, ctx.s);
  cur.v.alloc(gv.m > 0 ? gv.m : 1, ctx.s);
  cur.c.alloc(gv.m > 0 ? gv.m : 1, ctx.s);
  copy_d2d(ctx, cur.u.p, gv.u, gv.m);
  copy_d2d(ctx, cur.v.p, gv.v, gv.m);
  copy_d2d(ctx, cur.c.p, gv.c, gv.m);
  for (int rnd = 1; rnd <= cfg.max_rounds; rnd++) {
    bool any = false;
    for (int32_t i = 0; i < K; i++) any = any || active[i];
    if (!any) break;
    auto t0 = clk::now();
    Buf<int64_t> d_E;
    const std::vector<int64_t> E = bounds(ctx, cur.u.p, 1, cur.m, d_noff.p, K, d_E);
    std::vector<int64_t> Tn(K + 1, 0);
    std::vector<double> lb(K, nan);
    Graph rep_own;
    GraphView work = cur.view();
    if (dual) {
      CycleRows cyc;
      separate(ctx, cur.view(), cfg.max_cycle_length, cyc);
      DualState st;
      triangulate(ctx, cur.view(), cyc, st);
      message_passing(ctx, st, cfg.mp_iterations);
      Buf<double> cl(st.m_aug > 0 ? st.m_aug : 1, ctx);
      {  // per-instance bound in the single solve's summation order
        ProfScope prof(ctx.s, kFamBound);
        Buf<double> neg(st.m_aug > 0 ? st.m_aug : 1, ctx), negp(st.m_aug > 0 ? st.m_aug : 1, ctx);
        Buf<double> tm(st.T > 0 ? st.T : 1, ctx);
        lower_bound_terms(ctx, st, cl.p, neg.p, tm.p);
        Buf<int64_t> d_C, d_T;
        bounds(ctx, st.eu.p + st.m_orig, 1, st.m_aug - st.m_orig, d_noff.p, K, d_C);
        Tn = bounds(ctx, st.tri_nodes.p, 3, st.T, d_noff.p, K, d_T);
        Buf<int64_t> d_Cabs(K + 1, ctx), start(K, ctx), len(K, ctx);
        std::vector<int64_t> Cabs = download(ctx, d_C.p, K + 1);
        for (auto& x : Cabs) x += st.m_orig;
        upload(ctx, d_Cabs.p, Cabs);
        RAMA_KERNEL(ctx, k_lb_layout, st.m_aug, neg.p, st.m_orig, st.m_aug, d_E.p, d_Cabs.p, K, negp.p);
        RAMA_KERNEL(ctx, k_lb_segments, K, d_E.p, d_Cabs.p, st.m_orig, K, start.p, len.p);
        Buf<double> s_neg(K, ctx), s_tm(K, ctx);
        device_sums(ctx, negp.p, start.p, len.p, K, s_neg.p);
        RAMA_KERNEL(ctx, k_diff_segments, K, d_T.p, K, start.p, len.p);
        device_sums(ctx, tm.p, start.p, len.p, K, s_tm.p);
        const std::vector<double> hn = download(ctx, s_neg.p, K), ht = download(ctx, s_tm.p, K);
        for (int32_t i = 0; i < K; i++) {
          double total = 0.0;
          if ((E[i + 1] - E[i]) + (Cabs[i + 1] - Cabs[i]) > 0) total = hn[i];
          if (Tn[i + 1] - Tn[i] > 0) total += ht[i];
          lb[i] = total;
        }
      }
      rep_own = reparametrized_graph(ctx, st, cl.p);
      work = rep_own.view();
    }
    // ---- contraction step with the auto policy per instance (contraction.py:369-394)
    Buf<int32_t> su, sv;
    int64_t k = select_matching(ctx, work, 5, su, sv);
    Buf<int32_t> cnt(K, ctx);
    cnt.zero();
    RAMA_KERNEL(ctx, k_count_inst, k, su.p, k, d_noff.p, K, cnt.p);
    std::vector<int32_t> ks = download(ctx, cnt.p, K);
    std::vector<uint8_t> forest(K, 0);
    bool any_forest = false, all_forest = true;
    for (int32_t i = 0; i < K; i++) {
      const int64_t ni = noff[i + 1] - noff[i];
      forest[i] = active[i] && (double)ks[i] < cfg.switch_fraction * (double)ni;
      any_forest = any_forest || forest[i];
      all_forest = all_forest && (forest[i] || !active[i]);
    }
    if (any_forest) {
      Buf<int32_t> fu, fv;
      int64_t kf;
      if (all_forest) {
        kf = select_forest(ctx, work, fu, fv);
        su = std::move(fu);
        sv = std::move(fv);
        k = kf;
      } else {
        upload(ctx, d_flag.p, forest);
        Graph sub = edges_of(ctx, work, d_noff.p, K, d_flag.p);
        kf = select_forest(ctx, sub.view(), fu, fv);
        // matching pairs of the other instances + the forest pairs
        std::vector<uint8_t> keep(K);
        for (int32_t i = 0; i < K; i++) keep[i] = !forest[i];
        upload(ctx, d_flag.p, keep);
        Buf<int32_t> idx;
        const int64_t km = k > 0 ? compact_if(ctx, k, UInInst{su.p, d_noff.p, K, d_flag.p}, idx) : 0;
        Buf<int32_t> nu(km + kf > 0 ? km + kf : 1, ctx), nv(km + kf > 0 ? km + kf : 1, ctx);
        RAMA_KERNEL(ctx, k_gather_edges, km, idx.p, km, su.p, sv.p, (const double*)nullptr, nu.p, nv.p,
                    (double*)nullptr);
        copy_d2d(ctx, nu.p + km, fu.p, kf);
        copy_d2d(ctx, nv.p + km, fv.p, kf);
        su = std::move(nu);
        sv = std::move(nv);
        k = km + kf;
      }
      cnt.zero();
      RAMA_KERNEL(ctx, k_count_inst, k, su.p, k, d_noff.p, K, cnt.p);
      ks = download(ctx, cnt.p, K);
    }
    std::vector<int64_t> noff_next = noff;
    Buf<int32_t> map;
    Graph next;
    if (k > 0) {
      map.alloc(work.n, ctx.s);
      const int64_t nt = components(ctx, work.n, su.p, sv.p, k, map.p);
      next = contract(ctx, work, map.p, nt, nullptr);
      RAMA_KERNEL(ctx, k_map_offsets, K + 1, d_noff.p, K, work.n, map.p, nt, d_tmp.p);
      noff_next = download(ctx, d_tmp.p, K + 1);
    }
    const double t_ms = ms_since(t0);
    bool drop = false;
    for (int32_t i = 0; i < K; i++) {
      if (!active[i]) continue;
      const int64_t ni = noff[i + 1] - noff[i], ni_next = noff_next[i + 1] - noff_next[i];
      push(i, RoundInfo{rnd, dual ? 1 : 0, ni, E[i + 1] - E[i], Tn[i + 1] - Tn[i], dual ? lb[i] : nan,
                        (dual && rnd == 1) ? 1 : 0, ni - ni_next, t_ms});
      if (dual && rnd == 1) lb1[i] = lb[i];
      if (ks[i] == 0 || ni_next <= 1) {  // identity step, or one node left: this instance is done
        active[i] = 0;
        drop = drop || (ks[i] == 0 && E[i + 1] > E[i]);
      }
    }
    if (k == 0) break;
    compose(ctx, labels, n0, map.p);
    cur = std::move(next);
    noff = noff_next;
    upload(ctx, d_noff.p, noff);
    if (drop) {  // finished instances leave the working graph (their nodes stay as singletons)
      upload(ctx, d_flag.p, active);
      cur = edges_of(ctx, cur.view(), d_noff.p, K, d_flag.p);
    }
  }

  // ---- cleanup (solver.py:187-207, deviation D1) on the union of the quotients
  if (dual) {
    auto t0 = clk::now();
    Graph quotient = contract(ctx, gv, labels, cur.n, nullptr);
    Buf<int64_t> d_Q;
    const std::vector<int64_t> Q = bounds(ctx, quotient.u.p, 1, quotient.m, d_noff.p, K, d_Q);
    Buf<int32_t> fc(quotient.n > 0 ? quotient.n : 1, ctx);
    const int64_t nt = handshake_cleanup(ctx, quotient.view(), fc.p);
    compose(ctx, labels, n0, fc.p);
    RAMA_KERNEL(ctx, k_map_offsets, K + 1, d_noff.p, K, quotient.n, fc.p, nt, d_tmp.p);
    const std::vector<int64_t> after = download(ctx, d_tmp.p, K + 1);
    const double t_ms = ms_since(t0);
    for (int32_t i = 0; i < K; i++) {
      const int64_t qi = noff[i + 1] - noff[i];
      push(i, RoundInfo{nr[i] + 1, 2, qi, Q[i + 1] - Q[i], 0, nan, 0, qi - (after[i + 1] - after[i]), t_ms});
    }
  }

  // ---- objectives per instance (graph.py:134-145) in device_sum's order
  Buf<double> x(gv.m > 0 ? gv.m : 1, ctx), s_cost(K, ctx);
  cut_costs(ctx, gv, labels, x.p);
  Buf<int64_t> start(K, ctx), len(K, ctx);
  RAMA_KERNEL(ctx, k_diff_segments, K, d_E0.p, K, start.p, len.p);
  device_sums(ctx, x.p, start.p, len.p, K, s_cost.p);
  const std::vector<double> cost = download(ctx, s_cost.p, K);
  // labels local to each instance
  Buf<int64_t> first(K + 1, ctx);
  RAMA_KERNEL(ctx, k_map_offsets, K + 1, d_noff0.p, K, n0, labels, 0, first.p);
  RAMA_KERNEL(ctx, k_local_labels, n0, labels, n0, d_noff0.p, K, first.p);
  for (int32_t i = 0; i < K; i++) {
    primal_lb[2 * i] = cost[i];
    primal_lb[2 * i + 1] = dual ? lb1[i] : -INFINITY;
    if (n_rounds) n_rounds[i] = nr[i];
  }
  ctx.sync();
}

}  // namespace rama
