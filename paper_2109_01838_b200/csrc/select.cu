// Contraction-set selection.
//
// Matching (contraction.py:179-228): each handshake round is two atomic
// vote passes over the positive edges -- atomicMax of the cost bits (positive
// fp64 orders like its uint64 bit pattern), then atomicMin of the neighbour
// id among edges attaining the max -- which reproduces the reference's
// lexsort((nbr, -cost, node)) target exactly.  Mutual pairs match.  A round
// that adds nothing leaves the state unchanged, so running all rounds
// without a host check is equivalent to the reference's early exit.
//
// Forest (contraction.py:287-366): GPU Boruvka under the strict order
// (cost desc, u asc, v asc) gives the unique maximum spanning forest, i.e.
// the reference's forest bit for bit.  The conflict pass
// (_remove_conflict_edges, contraction.py:231-284) is order dependent in
// the reference (one repulsive edge at a time, ascending (u, v)); here it is
// resolved EXACTLY in parallel:
//   * every repulsive edge q inside one tree has a fixed tree path P_q and a
//     fixed cheapest edge e_q on it (Euler tour + list ranking roots the
//     forest; binary lifting answers LCA / path-min queries);
//   * q cuts e_q iff no earlier cutting q' < q has e_q' on P_q (a cut
//     disconnects, and a forest path is unique);
//   * passes decide candidates whose earlier dependencies are decided (a
//     path-min over "earliest cutting candidate per edge" and "earliest
//     undecided candidate per edge"); each pass decides at least the
//     smallest undecided candidate.
#include "internal.h"
#include "compact.cuh"

#include <cooperative_groups.h>
#include <cub/cub.cuh>

namespace rama {

__device__ __forceinline__ int32_t sf_find(int32_t* p, int32_t x) {
  while (true) {
    int32_t px = __ldcg(p + x);
    if (px == x) return x;
    int32_t gp = __ldcg(p + px);
    if (gp != px) p[x] = gp;
    x = px;
  }
}

__device__ __forceinline__ void sf_union(int32_t* p, int32_t a, int32_t b) {
  while (true) {
    a = sf_find(p, a);
    b = sf_find(p, b);
    if (a == b) return;
    int32_t lo = a < b ? a : b, hi = a < b ? b : a;
    int32_t old = atomicCAS(p + hi, hi, lo);
    if (old == hi) return;
    a = lo;
    b = old;
  }
}

// ----------------------------------------------------------------- matching

// one pass of votes: every unmatched endpoint keeps the max of
// (cost bits, ~neighbour id) as one 128-bit value -- the best positive edge,
// ties toward the smaller neighbour (contraction.py:207)
__global__ void k_match_vote(const int32_t* __restrict__ P, const int32_t* __restrict__ np_dev,
                             const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                             const double* __restrict__ c, const uint8_t* __restrict__ matched,
                             ulonglong2* __restrict__ vote) {
  const int64_t np = *np_dev;  // positive edges (compacted on the device, count not read back)
  GRID_STRIDE(i, np) {
    int32_t e = P[i];
    int32_t a = u[e], b = v[e];
    if (matched[a] | matched[b]) continue;
    unsigned long long bits = dbits(c[e]);
    vote_max_pair(vote + a, 0xffffffffULL - (uint32_t)b, vote + b, 0xffffffffULL - (uint32_t)a, bits);
  }
}

__global__ void k_match_init(int64_t n, uint8_t* __restrict__ matched, int32_t* __restrict__ partner,
                             ulonglong2* __restrict__ vote) {
  GRID_STRIDE(x, n) {
    matched[x] = 0;
    partner[x] = -1;
    vote[x] = make_ulonglong2(0ULL, 0ULL);
  }
}

// (clear: the other vote buffer, zeroed here for the next round instead of
// by a memset)
__global__ void k_match_pair(int64_t n, const ulonglong2* __restrict__ vote, uint8_t* __restrict__ matched,
                             int32_t* __restrict__ partner, ulonglong2* __restrict__ clear) {
  GRID_STRIDE(x, n) {
    if (clear) clear[x] = make_ulonglong2(0ULL, 0ULL);
    ulonglong2 vx = vote[x];
    if (vx.y == 0ULL) continue;
    int32_t t = (int32_t)(0xffffffffULL - vx.x);
    if ((int32_t)x < t && vote[t].x == 0xffffffffULL - (uint32_t)x) {
      partner[x] = t;
      partner[t] = (int32_t)x;  // (the pair's root is x: components straight from the partners)
      matched[x] = 1;
      matched[t] = 1;
    }
  }
}

__global__ void k_match_out(const int32_t* __restrict__ idx, int64_t k, const int32_t* __restrict__ partner,
                            int32_t* __restrict__ su, int32_t* __restrict__ sv) {
  GRID_STRIDE(i, k) {
    int32_t x = idx[i];
    su[i] = x;
    sv[i] = partner[x];
  }
}

__global__ void k_flag_lower(const int32_t* __restrict__ partner, int64_t n, uint8_t* __restrict__ f) {
  GRID_STRIDE(x, n) f[x] = partner[x] > (int32_t)x;
}

// the handshake rounds: partner[x] = x's mate (both ends) or -1
static void matching_rounds(Ctx& ctx, const GraphView& g, int rounds, ProfScope& prof, Buf<int32_t>& partner) {
  const int64_t n = g.n, m = g.m;
  Buf<int32_t> P, npd;
  compact_if_dev(ctx, m, PosCost{g.c}, P, npd);
  // algorithmic bytes: costs scanned once (8 m), then SURVEY.md 8(d)'s
  // 34 m+ + 17 n per handshake round over the positive edges (m+ ~ m / 2
  // here: the count stays on the device)
  prof.add_bytes(8.0 * (double)m + (double)rounds * (34.0 * 0.5 * (double)m + 17.0 * (double)n));
  Buf<uint8_t> matched(n, ctx);
  Buf<ulonglong2> vote(n, ctx);
  partner.alloc(n, ctx.s);
  RAMA_KERNEL(ctx, k_match_init, n, n, matched.p, partner.p, vote.p);  // one pass instead of three memsets
  // votes alternate between two buffers; each pair pass clears the other
  Buf<ulonglong2> vote1(rounds > 1 ? n : 1, ctx);
  for (int r = 0; r < rounds; r++) {
    ulonglong2* cur = (r & 1) ? vote1.p : vote.p;
    ulonglong2* nxt = r + 1 < rounds ? ((r & 1) ? vote.p : vote1.p) : nullptr;
    RAMA_KERNEL(ctx, k_match_vote, m, P.p, npd.p, g.u, g.v, g.c, matched.p, cur);
    RAMA_KERNEL(ctx, k_match_pair, n, n, cur, matched.p, partner.p, nxt);
  }
}

int64_t select_matching(Ctx& ctx, const GraphView& g, int rounds, Buf<int32_t>& su, Buf<int32_t>& sv) {
  ProfScope prof(ctx.s, kFamMatching);
  int64_t n = g.n, m = g.m;
  su.alloc(1, ctx.s);
  sv.alloc(1, ctx.s);
  if (n == 0 || m == 0) return 0;
  Buf<int32_t> partner;
  matching_rounds(ctx, g, rounds, prof, partner);
  Buf<uint8_t> lf(n, ctx);
  RAMA_KERNEL(ctx, k_flag_lower, n, partner.p, n, lf.p);
  Buf<int32_t> idx;
  int64_t k = compact_indices(ctx, lf.p, n, idx);
  su.alloc(k > 0 ? k : 1, ctx.s);
  sv.alloc(k > 0 ? k : 1, ctx.s);
  RAMA_KERNEL(ctx, k_match_out, k, idx.p, k, partner.p, su.p, sv.p);
  return k;
}

// The matching's contraction mapping without the pair list and the
// union-find: a pair's smaller node is its component's root (the smallest
// member, as components() roots it), so flags, one scan and one gather give
// the same canonical labels (contraction.py:101-111).  Returns the pairs;
// *nt = the number of targets.
__global__ void k_pair_roots(const int32_t* __restrict__ partner, int64_t n, int32_t* __restrict__ flag) {
  GRID_STRIDE(x, n) {
    const int32_t p = partner[x];
    flag[x] = !(p >= 0 && p < (int32_t)x);
  }
}
__global__ void k_pair_label(const int32_t* __restrict__ partner, const int32_t* __restrict__ rank, int64_t n,
                             int32_t* __restrict__ map) {
  GRID_STRIDE(x, n) {
    const int32_t p = partner[x];
    map[x] = rank[p >= 0 && p < (int32_t)x ? p : (int32_t)x];
  }
}

int64_t select_matching_map(Ctx& ctx, const GraphView& g, int rounds, int32_t* map, int64_t* nt) {
  int64_t n = g.n, m = g.m;
  *nt = n;
  if (n == 0 || m == 0) return 0;
  Buf<int32_t> partner;
  {
    ProfScope prof(ctx.s, kFamMatching);
    matching_rounds(ctx, g, rounds, prof, partner);
  }
  ProfScope prof(ctx.s, kFamComponents, 12.0 * (double)n);
  Buf<int32_t> flag(n, ctx), rank(n + 1, ctx);
  RAMA_KERNEL(ctx, k_pair_roots, n, partner.p, n, flag.p);
  *nt = exclusive_scan(ctx, flag.p, rank.p, n, true);
  RAMA_KERNEL(ctx, k_pair_label, n, partner.p, rank.p, n, map);
  return n - *nt;
}

// ----------------------------------------------------------------- max edge

__global__ void k_max_bits(const double* __restrict__ c, int64_t m, unsigned long long* best) {
  GRID_STRIDE(i, m) {
    if (c[i] > 0.0) atomicMax(best, dbits(c[i]));
  }
}

__global__ void k_argmax(const double* __restrict__ c, int64_t m, const unsigned long long* best, int32_t* idx) {
  GRID_STRIDE(i, m) {
    if (c[i] > 0.0 && dbits(c[i]) == *best) atomicMin(idx, (int32_t)i);
  }
}

int64_t select_max_edge(Ctx& ctx, const GraphView& g) {
  if (g.m == 0) return -1;
  Buf<unsigned long long> best(1, ctx);
  Buf<int32_t> idx(1, ctx);
  best.zero();
  idx.fill_bytes(0x7f);
  RAMA_KERNEL(ctx, k_max_bits, g.m, g.c, g.m, best.p);
  RAMA_KERNEL(ctx, k_argmax, g.m, g.c, g.m, best.p, idx.p);
  int32_t i = read_scalar(ctx, idx.p);
  return i == 0x7f7f7f7f ? -1 : (int64_t)i;
}

// ------------------------------------------------------------------- forest

__global__ void k_neg_bits(const int32_t* __restrict__ P, int64_t np, const double* __restrict__ c,
                           uint64_t* __restrict__ key, int32_t* __restrict__ val) {
  GRID_STRIDE(i, np) {
    key[i] = ~dbits(c[P[i]]);  // descending cost
    val[i] = (int32_t)i;
  }
}

__global__ void k_scatter_rank(const int32_t* __restrict__ sorted_val, int64_t np, int32_t* __restrict__ rank) {
  GRID_STRIDE(r, np) rank[sorted_val[r]] = (int32_t)r;
}

__global__ void k_bv_vote(const int32_t* __restrict__ P, int64_t np, const int32_t* __restrict__ u,
                          const int32_t* __restrict__ v, const int32_t* __restrict__ rank, int32_t* comp,
                          uint32_t* __restrict__ best, int32_t* __restrict__ any) {
  GRID_STRIDE(i, np) {
    int32_t e = P[i];
    int32_t a = sf_find(comp, u[e]), b = sf_find(comp, v[e]);
    if (a == b) continue;
    uint32_t r = (uint32_t)rank[i];
    atomicMin(best + a, r);
    atomicMin(best + b, r);
    *any = 1;
  }
}

__global__ void k_bv_hook(int64_t n, const uint32_t* __restrict__ best, const int32_t* __restrict__ order,
                          const int32_t* __restrict__ P, const int32_t* __restrict__ u,
                          const int32_t* __restrict__ v, int32_t* comp, uint8_t* __restrict__ in_forest) {
  GRID_STRIDE(x, n) {
    uint32_t r = best[x];
    if (r == 0xffffffffu) continue;
    int32_t pi = order[r];
    in_forest[pi] = 1;
    int32_t e = P[pi];
    sf_union(comp, u[e], v[e]);
  }
}

// read-only find for flattening (no path halving, see graph.cu k_cc_flatten)
__global__ void k_flatten(int32_t* comp, int64_t n) {
  GRID_STRIDE(x, n) {
    int32_t r = (int32_t)x;
    while (true) {
      int32_t p = __ldcg(comp + r);
      if (p == r) break;
      r = p;
    }
    comp[x] = r;
  }
}

// repulsive edges whose endpoints share a tree
__global__ void k_flag_conflicts(const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                                 const double* __restrict__ c, int64_t m, const int32_t* __restrict__ comp,
                                 uint8_t* __restrict__ f) {
  GRID_STRIDE(i, m) f[i] = (c[i] < 0.0) && comp[u[i]] == comp[v[i]];
}

// the forest's nodes get local ids 0..nf-1 (ascending node order), so the
// Euler tour, the lifting tables and the path queries scale with the forest,
// not the graph (late rounds: a few thousand forest nodes in a graph of 10^5-10^6)
__global__ void k_mark_fnodes(const int32_t* __restrict__ Fi, int64_t kf, const int32_t* __restrict__ P,
                              const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                              uint8_t* __restrict__ isf) {
  GRID_STRIDE(i, kf) {
    int32_t e = P[Fi[i]];
    isf[u[e]] = 1;
    isf[v[e]] = 1;
  }
}

__global__ void k_scatter_loc(const int32_t* __restrict__ FN, int64_t nf, int32_t* __restrict__ loc) {
  GRID_STRIDE(i, nf) loc[FN[i]] = (int32_t)i;
}

__global__ void k_comp_local(const int32_t* __restrict__ FN, int64_t nf, const int32_t* __restrict__ comp,
                             const int32_t* __restrict__ loc, int32_t* __restrict__ comp_loc) {
  GRID_STRIDE(i, nf) comp_loc[i] = loc[comp[FN[i]]];  // a tree's root (its smallest node) is a forest node
}

// largest tree (node count): bounds the depth, so the lifting tables need
// log2(largest tree) levels instead of log2(forest size)
__global__ void k_tree_sizes(const int32_t* __restrict__ comp_loc, int64_t nf, int32_t* __restrict__ sz,
                             int32_t* __restrict__ maxsz) {
  GRID_STRIDE(i, nf) atomicMax(maxsz, atomicAdd(sz + comp_loc[i], 1) + 1);
}

__global__ void k_forest_edges(const int32_t* __restrict__ Fi, int64_t kf, const int32_t* __restrict__ P,
                               const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                               const int32_t* __restrict__ loc, const double* __restrict__ c,
                               int32_t* __restrict__ fu, int32_t* __restrict__ fv,
                               uint64_t* __restrict__ fkey_bits, int32_t* __restrict__ fval) {
  GRID_STRIDE(i, kf) {
    int32_t e = P[Fi[i]];
    fu[i] = loc[u[e]];
    fv[i] = loc[v[e]];
    fkey_bits[i] = dbits(c[e]);  // ascending cost, ties keep (u, v) order
    fval[i] = (int32_t)i;
  }
}

__global__ void k_arcs(const int32_t* __restrict__ fu, const int32_t* __restrict__ fv, int64_t kf,
                       int32_t* __restrict__ row, uint64_t* __restrict__ key) {
  GRID_STRIDE(a, 2 * kf) {
    int32_t f = (int32_t)(a >> 1);
    int32_t s = (a & 1) ? fv[f] : fu[f];
    int32_t d = (a & 1) ? fu[f] : fv[f];
    row[a] = s;
    key[a] = ((uint64_t)(uint32_t)d << 32) | (uint64_t)a;
  }
}

__global__ void k_arc_pos(const int32_t* __restrict__ arc_at, int64_t na, int32_t* __restrict__ pos) {
  GRID_STRIDE(p, na) pos[arc_at[p]] = (int32_t)p;
}

// Euler successor: after arc (x->y) comes the arc following (y->x) in y's
// cyclic adjacency list; the tour of each tree starts at its root's first
// arc and is cut before returning to it.
__global__ void k_euler_succ(int64_t na, const int32_t* __restrict__ arc_at, const int32_t* __restrict__ pos,
                             const int32_t* __restrict__ arow, const int32_t* __restrict__ ptr,
                             const int32_t* __restrict__ comp, int32_t* __restrict__ succ) {
  GRID_STRIDE(a, na) {
    int32_t t = (int32_t)a ^ 1;
    int32_t pt = pos[t];
    int32_t y = arow[pt];
    int32_t p = pt + 1;
    if (p == ptr[y + 1]) p = ptr[y];
    int32_t nx = arc_at[p];
    // cut: the arc whose successor is the root's first arc ends the tour
    int32_t r = comp[y];
    if (y == r && p == ptr[y]) nx = -1;
    succ[a] = nx;
  }
}

__global__ void k_rank_init(const int32_t* __restrict__ succ, int64_t na, int32_t* __restrict__ d) {
  GRID_STRIDE(a, na) d[a] = succ[a] < 0 ? 0 : 1;
}

__global__ void k_root_init(int64_t n, int32_t* __restrict__ par, int32_t* __restrict__ pedge,
                            int32_t* __restrict__ enter, int32_t* __restrict__ exit_) {
  GRID_STRIDE(x, n) {
    par[x] = (int32_t)x;
    pedge[x] = -1;
    enter[x] = 0x7fffffff;
    exit_[x] = -1;
  }
}

// a down arc (x->y) precedes its twin in the tour (larger remaining distance)
__global__ void k_orient(int64_t na, const int32_t* __restrict__ dist, const int32_t* __restrict__ fu,
                         const int32_t* __restrict__ fv, int32_t* __restrict__ par, int32_t* __restrict__ pedge,
                         int32_t* __restrict__ enter, int32_t* __restrict__ exit_) {
  GRID_STRIDE(a, na) {
    int32_t da = dist[a], dt = dist[a ^ 1];
    if (da > dt) {
      int32_t f = (int32_t)(a >> 1);
      int32_t x = (a & 1) ? fv[f] : fu[f];
      int32_t y = (a & 1) ? fu[f] : fv[f];
      par[y] = x;
      pedge[y] = f;
      enter[y] = da;
      exit_[y] = dt;
    }
  }
}

__device__ __forceinline__ bool is_anc(const int32_t* enter, const int32_t* exit_, int32_t x, int32_t w) {
  if (x == w) return true;
  int32_t ew = enter[w];
  return exit_[x] < ew && ew < enter[x];
}

// ---- cooperative (one launch, grid.sync() between levels) -----------------
// Binary-lifting tables and list ranking are level-synchronous pointer
// jumping: one persistent launch replaces LOG (or log2 |arcs|) launches and
// their gaps.  Reads of the previous level bypass L1 (written by other SMs).

// level 0 from the parent links, then levels 1..LOG-1; up (if build_up) and
// up to two min tables over edge values va / vb (nullptr = skip)
__global__ void k_lift_coop(int64_t n, int LOG, const int32_t* __restrict__ par, const int32_t* __restrict__ pedge,
                            int build_up, int32_t* up, const int32_t* __restrict__ va, int32_t* mna,
                            const int32_t* __restrict__ vb, int32_t* mnb) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  GRID_STRIDE(x, n) {
    if (build_up) up[x] = par[x];
    int32_t f = pedge[x];
    if (mna) mna[x] = f < 0 ? 0x7fffffff : va[f];
    if (mnb) mnb[x] = f < 0 ? 0x7fffffff : vb[f];
  }
  grid.sync();
  for (int j = 1; j < LOG; j++) {
    const int32_t* uj = up + (int64_t)(j - 1) * n;
    GRID_STRIDE(x, n) {
      int32_t y = __ldcg(uj + x);
      if (build_up) up[(int64_t)j * n + x] = __ldcg(uj + y);
      if (mna) {
        const int32_t* mj = mna + (int64_t)(j - 1) * n;
        mna[(int64_t)j * n + x] = min(__ldcg(mj + x), __ldcg(mj + y));
      }
      if (mnb) {
        const int32_t* mj = mnb + (int64_t)(j - 1) * n;
        mnb[(int64_t)j * n + x] = min(__ldcg(mj + x), __ldcg(mj + y));
      }
    }
    grid.sync();
  }
}

// Wyllie list ranking: d = distance to the list end, in `steps` jumps
__global__ void k_rank_coop(int64_t na, int steps, int32_t* d1, int32_t* n1, int32_t* d2, int32_t* n2) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  for (int s = 0; s < steps; s++) {
    const int32_t* d = (s & 1) ? d2 : d1;
    const int32_t* nx = (s & 1) ? n2 : n1;
    int32_t* dd = (s & 1) ? d1 : d2;
    int32_t* nn = (s & 1) ? n1 : n2;
    GRID_STRIDE(a, na) {
      int32_t t = __ldcg(nx + a);
      if (t >= 0) {
        dd[a] = __ldcg(d + a) + __ldcg(d + t);
        nn[a] = __ldcg(nx + t);
      } else {
        dd[a] = __ldcg(d + a);
        nn[a] = -1;
      }
    }
    grid.sync();
  }
}

static unsigned coop_blocks(const void* fn) {
  const int sms = num_sms();  // per device
  int per_sm = 0;
  RAMA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBlock, 0));
  return (unsigned)(sms * (per_sm < 4 ? per_sm : 4));
}

static void launch_coop(Ctx& ctx, const void* fn, const char* name, void** args, int64_t work) {
  KernelScope ks(ctx.s, name, 0.0);
  int64_t want = (work + kBlock - 1) / kBlock;  // ~1 item per thread per level
  unsigned cap = coop_blocks(fn);
  unsigned blocks = (unsigned)(want < 1 ? 1 : (want < cap ? want : cap));
  RAMA_CUDA(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(kBlock), args, 0, ctx.s));
  ctx.launches++;
}

struct Lift {
  int LOG = 0;
  int64_t n = 0;
  Buf<int32_t> up;  // LOG * n
};

__device__ __forceinline__ int32_t climb_min(const int32_t* up, const int32_t* mn, int LOG, int64_t n,
                                             const int32_t* enter, const int32_t* exit_, int32_t x, int32_t l) {
  int32_t acc = 0x7fffffff;
  for (int j = LOG - 1; j >= 0; j--) {
    int32_t y = up[(int64_t)j * n + x];
    if (x != l && is_anc(enter, exit_, l, y)) {
      int32_t v = mn[(int64_t)j * n + x];
      acc = v < acc ? v : acc;
      x = y;
    }
  }
  return acc;
}

__device__ __forceinline__ int32_t lca(const int32_t* up, int LOG, int64_t n, const int32_t* enter,
                                       const int32_t* exit_, int32_t a, int32_t b) {
  if (is_anc(enter, exit_, a, b)) return a;
  if (is_anc(enter, exit_, b, a)) return b;
  int32_t x = a;
  for (int j = LOG - 1; j >= 0; j--) {
    int32_t y = up[(int64_t)j * n + x];
    if (!is_anc(enter, exit_, y, b)) x = y;
  }
  return up[x];
}

__global__ void k_cand_paths(const int32_t* __restrict__ Q, int64_t nq, const int32_t* __restrict__ u,
                             const int32_t* __restrict__ v, const int32_t* __restrict__ loc,
                             const int32_t* __restrict__ up,
                             const int32_t* __restrict__ mn, int LOG, int64_t n, const int32_t* __restrict__ enter,
                             const int32_t* __restrict__ exit_, const int32_t* __restrict__ key_inv,
                             int32_t* __restrict__ qa, int32_t* __restrict__ qb, int32_t* __restrict__ ql,
                             int32_t* __restrict__ qe) {
  GRID_STRIDE(q, nq) {
    int32_t e = Q[q];
    int32_t a = loc[u[e]], b = loc[v[e]];  // both ends lie in one tree: forest nodes
    int32_t l = lca(up, LOG, n, enter, exit_, a, b);
    int32_t m1 = climb_min(up, mn, LOG, n, enter, exit_, a, l);
    int32_t m2 = climb_min(up, mn, LOG, n, enter, exit_, b, l);
    int32_t mk = m1 < m2 ? m1 : m2;
    qa[q] = a;
    qb[q] = b;
    ql[q] = l;
    qe[q] = key_inv[mk];
  }
}

__global__ void k_fill_i32(int32_t* x, int64_t n, int32_t v) {
  GRID_STRIDE(i, n) x[i] = v;
}

// state: 0 undecided, 1 cuts, 2 does not cut
__global__ void k_earliest(const int32_t* __restrict__ qe, const uint8_t* __restrict__ state, int64_t nq,
                           int32_t* __restrict__ rf, int32_t* __restrict__ ru) {
  GRID_STRIDE(q, nq) {
    uint8_t s = state[q];
    if (s == 1) atomicMin(rf + qe[q], (int32_t)q);
    else if (s == 0) atomicMin(ru + qe[q], (int32_t)q);
  }
}

__global__ void k_resolve(int64_t nq, const int32_t* __restrict__ qa, const int32_t* __restrict__ qb,
                          const int32_t* __restrict__ ql, const int32_t* __restrict__ up,
                          const int32_t* __restrict__ mf, const int32_t* __restrict__ mu, int LOG, int64_t n,
                          const int32_t* __restrict__ enter, const int32_t* __restrict__ exit_,
                          uint8_t* __restrict__ state, int32_t* __restrict__ left) {
  GRID_STRIDE(q, nq) {
    if (state[q] != 0) continue;
    int32_t a = qa[q], b = qb[q], l = ql[q];
    int32_t pf = min(climb_min(up, mf, LOG, n, enter, exit_, a, l), climb_min(up, mf, LOG, n, enter, exit_, b, l));
    if (pf < (int32_t)q) {
      state[q] = 2;
      continue;
    }
    int32_t pu = min(climb_min(up, mu, LOG, n, enter, exit_, a, l), climb_min(up, mu, LOG, n, enter, exit_, b, l));
    if (pu < (int32_t)q) {
      atomicAdd(left, 1);
      continue;
    }
    state[q] = 1;
  }
}

__global__ void k_mark_removed(const int32_t* __restrict__ qe, const uint8_t* __restrict__ state, int64_t nq,
                               uint8_t* __restrict__ removed) {
  GRID_STRIDE(q, nq) {
    if (state[q] == 1) removed[qe[q]] = 1;
  }
}

// ---- small trees: the reference's sequential loop, one thread per tree ----
// When every tree of the forest has at most kSmallTree nodes (grid-like
// graphs' late forest rounds), the conflict loop of _remove_conflict_edges
// (contraction.py:231-284) runs as written, per tree: a repulsive edge only
// meets removals inside its own tree, so each tree's queries in ascending
// (u, v) order are independent of every other tree's.  A thread holds its
// tree (<= 32 nodes, <= 31 edges) in local memory, roots it once, walks
// each query's unique path up to the meeting node (a removed edge on it:
// already separated, as the reference's BFS finds) and cuts the path's
// cheapest edge (ties: smallest (u, v)).  This
// replaces the Euler tour, the lifting tables and the dependency passes of
// the general path (~40 launches and ~6 read-backs per forest round).
constexpr int kSmallTree = 32;

// combined items per tree: its forest edges (key i) then its queries (key 2^32 + q)
__global__ void k_tree_items(const int32_t* __restrict__ Fi, int64_t kf, const int32_t* __restrict__ Q, int64_t nq,
                             const int32_t* __restrict__ P, const int32_t* __restrict__ u,
                             const int32_t* __restrict__ loc, const int32_t* __restrict__ comp_loc,
                             int32_t* __restrict__ row, uint64_t* __restrict__ key) {
  GRID_STRIDE(i, kf + nq) {
    if (i < kf) {
      row[i] = comp_loc[loc[u[P[Fi[i]]]]];
      key[i] = (uint64_t)i;
    } else {
      const int64_t q = i - kf;
      row[i] = comp_loc[loc[u[Q[q]]]];
      key[i] = (1ull << 32) | (uint64_t)q;
    }
  }
}

__device__ __forceinline__ int tree_slot(int32_t* node, int& nn, int32_t x, bool add) {
  for (int i = 0; i < nn; i++)
    if (node[i] == x) return i;
  if (!add) return -1;
  node[nn] = x;
  return nn++;
}

__global__ void k_tree_resolve(const int32_t* __restrict__ rptr, const uint64_t* __restrict__ key, int64_t R,
                               const int32_t* __restrict__ Fi, const int32_t* __restrict__ P,
                               const int32_t* __restrict__ Q, const int32_t* __restrict__ u,
                               const int32_t* __restrict__ v, const double* __restrict__ c,
                               uint8_t* __restrict__ removed) {
  // one warp per tree: every lane builds the same rooted tree (broadcast
  // loads), the lanes take 32 queries at a time and find their paths and
  // cheapest edges in parallel -- both depend on the tree alone -- then the
  // warp applies them in query order: a query whose path meets an edge
  // already cut is separated, otherwise its cheapest edge is cut
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp0; r < R; r += W) {
    const int32_t b = rptr[r], e = rptr[r + 1];
    if (e - b < 2 || (key[e - 1] >> 32) == 0) continue;  // no edge or no query (warp-uniform)
    int32_t node[kSmallTree];
    int8_t ea[kSmallTree], eb[kSmallTree];
    int32_t fid[kSmallTree], fu[kSmallTree], fv[kSmallTree];
    double fc[kSmallTree];
    int nn = 0, ne = 0;
    int32_t p = b;
    for (; p < e && (key[p] >> 32) == 0; p++) {
      const int32_t i = (int32_t)(uint32_t)key[p];
      const int32_t ed = P[Fi[i]];
      fu[ne] = u[ed];
      fv[ne] = v[ed];
      fc[ne] = c[ed];
      ea[ne] = (int8_t)tree_slot(node, nn, fu[ne], true);
      eb[ne] = (int8_t)tree_slot(node, nn, fv[ne], true);
      fid[ne] = i;
      ne++;
    }
    // root the tree at its first node once: parent edge and depth per node
    int8_t pe[kSmallTree], dep[kSmallTree];
    {
      uint32_t vis = 1u;
      dep[0] = 0;
      pe[0] = -1;
      bool grew = true;
      while (grew) {
        grew = false;
        for (int k = 0; k < ne; k++) {
          const bool ia = (vis >> ea[k]) & 1u, ib = (vis >> eb[k]) & 1u;
          if (ia != ib) {
            const int y = ia ? eb[k] : ea[k], x = ia ? ea[k] : eb[k];
            vis |= 1u << y;
            pe[y] = (int8_t)k;
            dep[y] = (int8_t)(dep[x] + 1);
            grew = true;
          }
        }
      }
    }
    uint32_t rem = 0;  // removed tree edges (identical in every lane)
    for (int32_t p0 = p; p0 < e; p0 += 32) {
      uint32_t path = 0;
      int best = -1;
      if (p0 + lane < e) {
        const int32_t ed = Q[(int32_t)(uint32_t)key[p0 + lane]];
        int x = tree_slot(node, nn, u[ed], false), y = tree_slot(node, nn, v[ed], false);
        // the unique tree path: climb from the deeper end until the ends meet
        while (x >= 0 && y >= 0 && x != y) {
          int& w = dep[x] >= dep[y] ? x : y;
          const int k = pe[w];
          path |= 1u << k;
          w = ea[k] == w ? eb[k] : ea[k];
        }
        double bc = 0.0;
        int32_t bu = 0, bv = 0;
        for (uint32_t bits = path; bits; bits &= bits - 1) {
          const int k = __ffs(bits) - 1;
          const double ck = fc[k];
          const int32_t uk = fu[k], vk = fv[k];
          if (best < 0 || ck < bc || (ck == bc && (uk < bu || (uk == bu && vk < bv)))) {
            best = k;
            bc = ck;
            bu = uk;
            bv = vk;
          }
        }
      }
      const int cnt = min(32, e - p0);
      for (int j = 0; j < cnt; j++) {  // in query order
        const uint32_t pj = __shfl_sync(0xffffffffu, path, j);
        const int bj = __shfl_sync(0xffffffffu, best, j);
        if (pj && !(pj & rem)) {
          rem |= 1u << bj;
          if (lane == 0) removed[fid[bj]] = 1;
        }
      }
    }
  }
}

__global__ void k_forest_keep(const int32_t* __restrict__ Fi, int64_t kf, const uint8_t* __restrict__ removed,
                              uint8_t* __restrict__ keep_pos) {
  GRID_STRIDE(i, kf) keep_pos[Fi[i]] = !removed[i];
}

__global__ void k_gather_pairs(const int32_t* __restrict__ idx, int64_t k, const int32_t* __restrict__ P,
                               const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                               int32_t* __restrict__ su, int32_t* __restrict__ sv) {
  GRID_STRIDE(i, k) {
    int32_t e = P[idx[i]];
    su[i] = u[e];
    sv[i] = v[e];
  }
}

// All Boruvka iterations in one cooperative launch (reset, vote, hook,
// flatten with grid barriers; stop when no edge crosses components) instead
// of 2 memsets, 3 launches and a read-back per iteration.  any2: two
// alternating "an edge crossed" flags (zero on entry); iters: iterations run.
__global__ void __launch_bounds__(kBlock) k_boruvka_coop(const int32_t* __restrict__ P, int64_t np,
                                                         const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                                                         const int32_t* __restrict__ rank,
                                                         const int32_t* __restrict__ order, int32_t* comp,
                                                         uint32_t* best, uint8_t* __restrict__ in_forest, int64_t n,
                                                         int32_t* any2, int32_t* iters) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, GT = (int64_t)gridDim.x * blockDim.x;
  for (int it = 0;; it++) {
    for (int64_t x = gtid; x < n; x += GT) best[x] = 0xffffffffu;
    if (gtid == 0) any2[(it + 1) & 1] = 0;  // the next iteration's flag (this one's was cleared before)
    grid.sync();
    bool crossed = false;
    for (int64_t i = gtid; i < np; i += GT) {
      const int32_t e = P[i];
      const int32_t a = sf_find(comp, u[e]), b = sf_find(comp, v[e]);
      if (a == b) continue;
      const uint32_t r = (uint32_t)rank[i];
      atomicMin(best + a, r);
      atomicMin(best + b, r);
      crossed = true;
    }
    if (__any_sync(0xffffffffu, crossed) && (threadIdx.x & 31) == 0) any2[it & 1] = 1;
    grid.sync();
    if (__ldcg(any2 + (it & 1)) == 0) {  // uniform: read after the barrier
      if (gtid == 0) *iters = it + 1;
      break;
    }
    for (int64_t x = gtid; x < n; x += GT) {
      const uint32_t r = __ldcg(best + x);
      if (r == 0xffffffffu) continue;
      const int32_t pi = order[r];
      in_forest[pi] = 1;
      const int32_t e = P[pi];
      sf_union(comp, u[e], v[e]);
    }
    grid.sync();
    for (int64_t x = gtid; x < n; x += GT) {
      int32_t r = (int32_t)x;
      while (true) {
        const int32_t p = __ldcg(comp + r);
        if (p == r) break;
        r = p;
      }
      comp[x] = r;
    }
    grid.sync();
  }
}

int64_t select_forest(Ctx& ctx, const GraphView& g, Buf<int32_t>& su, Buf<int32_t>& sv) {
  int64_t n = g.n, m = g.m;
  // algorithmic bytes: the graph read once, the selected pairs written
  ProfScope prof(ctx.s, kFamForest, 16.0 * (double)m + 8.0 * (double)n);
  su.alloc(1, ctx.s);
  sv.alloc(1, ctx.s);
  if (n == 0 || m == 0) return 0;
  static const bool phase_prof = getenv("RAMA_ROUND_PROF") != nullptr;
  double ph[8] = {0};
  int bv_iters = 0, rs_iters = 0;
  auto tp = std::chrono::steady_clock::now();
  auto mark = [&](int i) {
    if (!phase_prof) return;
    ctx.sync();
    auto t = std::chrono::steady_clock::now();
    ph[i] += std::chrono::duration<double, std::milli>(t - tp).count();
    tp = t;
  };
  Buf<int32_t> P;
  int64_t np = compact_if(ctx, m, PosCost{g.c}, P);
  if (np == 0) return 0;

  // strict rank: cost desc, (u, v) asc == stable sort of the canonical order
  Buf<uint64_t> k1(np, ctx), k2(np, ctx);
  Buf<int32_t> v1(np, ctx), order(np, ctx), rank(np, ctx);
  RAMA_KERNEL(ctx, k_neg_bits, np, P.p, np, g.c, k1.p, v1.p);
  radix_sort_pairs(ctx, k1.p, v1.p, k2.p, order.p, np);
  RAMA_KERNEL(ctx, k_scatter_rank, np, order.p, np, rank.p);
  mark(0);

  // Boruvka
  Buf<int32_t> comp(n, ctx), any(1, ctx);
  Buf<uint32_t> best(n, ctx);
  Buf<uint8_t> in_forest(np, ctx);
  in_forest.zero();
  iota(ctx, comp.p, n);
  static const bool bv_launches = getenv("RAMA_BORUVKA_LAUNCHES") != nullptr;  // A/B: one launch set per iteration
  if (bv_launches) {
    while (true) {
      best.fill_bytes(0xff);
      any.zero();
      RAMA_KERNEL(ctx, k_bv_vote, np, P.p, np, g.u, g.v, rank.p, comp.p, best.p, any.p);
      bv_iters++;
      if (read_scalar(ctx, any.p) == 0) break;
      RAMA_KERNEL(ctx, k_bv_hook, n, n, best.p, order.p, P.p, g.u, g.v, comp.p, in_forest.p);
      RAMA_KERNEL(ctx, k_flatten, n, comp.p, n);
    }
  } else {
    Buf<int32_t> flags(3, ctx);  // any2 | iterations
    flags.zero();
    const int32_t *pP = P.p, *pu = g.u, *pv = g.v, *prank = rank.p, *porder = order.p;
    int32_t *pcomp = comp.p, *pany = flags.p, *piters = flags.p + 2;
    uint32_t* pbest = best.p;
    uint8_t* pin = in_forest.p;
    int64_t np_ = np, n_ = n;
    void* args[] = {&pP, &np_, &pu, &pv, &prank, &porder, &pcomp, &pbest, &pin, &n_, &pany, &piters};
    launch_coop(ctx, (const void*)k_boruvka_coop, "k_boruvka_coop", args, std::max<int64_t>(n, np));
    if (phase_prof) bv_iters = read_scalar(ctx, piters);
  }
  RAMA_KERNEL(ctx, k_flatten, n, comp.p, n);

  Buf<int32_t> Fi;
  int64_t kf = compact_indices(ctx, in_forest.p, np, Fi);
  Buf<uint8_t> keep(np, ctx);
  keep.zero();

  // repulsive edges inside one tree, ascending (u, v) order
  Buf<uint8_t> cflag(m, ctx);
  RAMA_KERNEL(ctx, k_flag_conflicts, m, g.u, g.v, g.c, m, comp.p, cflag.p);
  Buf<int32_t> Q;
  int64_t nq = compact_indices(ctx, cflag.p, m, Q);
  mark(1);

  Buf<uint8_t> removed(kf > 0 ? kf : 1, ctx);
  removed.zero();
  if (nq > 0 && kf > 0) {
    Buf<uint8_t> isf(n, ctx);
    isf.zero();
    RAMA_KERNEL(ctx, k_mark_fnodes, kf, Fi.p, kf, P.p, g.u, g.v, isf.p);
    Buf<int32_t> FN;
    const int64_t nf = compact_indices(ctx, isf.p, n, FN);
    Buf<int32_t> loc(n, ctx), comp_loc(nf, ctx);
    RAMA_KERNEL(ctx, k_scatter_loc, nf, FN.p, nf, loc.p);
    RAMA_KERNEL(ctx, k_comp_local, nf, FN.p, nf, comp.p, loc.p, comp_loc.p);
    int64_t maxsz = nf;  // largest tree: bounds tour lengths and depths
    {
      Buf<int32_t> sz(nf + 1, ctx);
      sz.zero();
      RAMA_KERNEL(ctx, k_tree_sizes, nf, comp_loc.p, nf, sz.p, sz.p + nf);
      maxsz = (int64_t)read_scalar(ctx, sz.p + nf);
    }
    static const bool tour_only = getenv("RAMA_FOREST_TOUR") != nullptr;  // A/B: always the general path
    if (maxsz <= kSmallTree && !tour_only) {
      const int64_t ni = kf + nq;
      Buf<int32_t> irow(ni, ctx);
      Buf<uint64_t> ikey(ni, ctx);
      RAMA_KERNEL(ctx, k_tree_items, ni, Fi.p, kf, Q.p, nq, P.p, g.u, loc.p, comp_loc.p, irow.p, ikey.p);
      BucketSorted ts;
      bucket_sort(ctx, nf, ni, irow.p, ikey.p, ts, false);
      RAMA_KERNEL(ctx, k_tree_resolve, 32 * nf, ts.row_ptr.p, ts.key.p, nf, Fi.p, P.p, Q.p, g.u, g.v, g.c,
                  removed.p);  // a warp per tree
      mark(4);
      if (phase_prof)
        fprintf(stderr, "[rama]   forest n %lld m+ %lld kf %lld conflicts %lld trees <= %lld nodes: rank sort %.2f "
                "boruvka %.2f (%d) per-tree resolve %.2f ms\n", (long long)n, (long long)np, (long long)kf,
                (long long)nq, (long long)maxsz, ph[0], ph[1], bv_iters, ph[4]);
    } else {
    const int64_t maxdepth = maxsz - 1;
    Buf<int32_t> fu(kf, ctx), fv(kf, ctx), fval(kf, ctx), fsorted(kf, ctx), fkey(kf, ctx);
    Buf<uint64_t> fbits(kf, ctx), fbits2(kf, ctx);
    RAMA_KERNEL(ctx, k_forest_edges, kf, Fi.p, kf, P.p, g.u, g.v, loc.p, g.c, fu.p, fv.p, fbits.p, fval.p);
    radix_sort_pairs(ctx, fbits.p, fval.p, fbits2.p, fsorted.p, kf);  // key_inv: rank -> forest edge
    RAMA_KERNEL(ctx, k_scatter_rank, kf, fsorted.p, kf, fkey.p);  // fkey: forest edge -> rank

    // arcs, sorted adjacency, Euler tour
    int64_t na = 2 * kf;
    Buf<int32_t> arow(na, ctx);
    Buf<uint64_t> akey(na, ctx);
    RAMA_KERNEL(ctx, k_arcs, na, fu.p, fv.p, kf, arow.p, akey.p);
    BucketSorted bs;
    bucket_sort(ctx, nf, na, arow.p, akey.p, bs, true);
    Buf<int32_t> pos(na, ctx), succ(na, ctx);
    RAMA_KERNEL(ctx, k_arc_pos, na, bs.src.p, na, pos.p);
    RAMA_KERNEL(ctx, k_euler_succ, na, na, bs.src.p, pos.p, bs.row.p, bs.row_ptr.p, comp_loc.p, succ.p);
    Buf<int32_t> d1(na, ctx), d2(na, ctx), n1(na, ctx), n2(na, ctx);
    RAMA_KERNEL(ctx, k_rank_init, na, succ.p, na, d1.p);
    copy_d2d(ctx, n1.p, succ.p, na);
    int steps = 0;  // pointer jumping over the longest tour (2 (|T| - 1) arcs)
    while ((1LL << steps) < 2 * maxsz) steps++;
    steps += 1;
    {
      int64_t na_ = na;
      int32_t *pd1 = d1.p, *pn1 = n1.p, *pd2 = d2.p, *pn2 = n2.p;
      void* args[] = {&na_, &steps, &pd1, &pn1, &pd2, &pn2};
      launch_coop(ctx, (const void*)k_rank_coop, "k_rank_coop", args, na);
      if (steps & 1) {  // result lives in the second buffer pair
        std::swap(d1, d2);
        std::swap(n1, n2);
      }
    }
    Buf<int32_t> par(nf, ctx), pedge(nf, ctx), enter(nf, ctx), exit_(nf, ctx);
    RAMA_KERNEL(ctx, k_root_init, nf, nf, par.p, pedge.p, enter.p, exit_.p);
    RAMA_KERNEL(ctx, k_orient, na, na, d1.p, fu.p, fv.p, par.p, pedge.p, enter.p, exit_.p);
    mark(2);

    // binary lifting tables (depth < largest tree)
    int LOG = 1;
    while ((1LL << LOG) <= maxdepth) LOG++;
    Buf<int32_t> up((size_t)LOG * nf, ctx);
    Buf<int32_t> mn((size_t)LOG * nf, ctx);
    {
      int64_t n_ = nf;
      int build = 1;
      int32_t *pup = up.p, *pmn = mn.p, *pnull = nullptr;
      const int32_t *ppar = par.p, *ppe = pedge.p, *pva = fkey.p, *pvnull = nullptr;
      void* args[] = {&n_, &LOG, &ppar, &ppe, &build, &pup, &pva, &pmn, &pvnull, &pnull};
      launch_coop(ctx, (const void*)k_lift_coop, "k_lift_coop", args, nf);
    }

    Buf<int32_t> qa(nq, ctx), qb(nq, ctx), ql(nq, ctx), qe(nq, ctx);
    RAMA_KERNEL(ctx, k_cand_paths, nq, Q.p, nq, g.u, g.v, loc.p, up.p, mn.p, LOG, nf, enter.p, exit_.p, fsorted.p,
                qa.p, qb.p, ql.p, qe.p);
    mn.release();
    mark(3);

    Buf<uint8_t> state(nq, ctx);
    state.zero();
    Buf<int32_t> rf(kf, ctx), ru(kf, ctx), left(1, ctx), mf, mu;
    while (true) {
      RAMA_KERNEL(ctx, k_fill_i32, kf, rf.p, kf, 0x7fffffff);
      RAMA_KERNEL(ctx, k_fill_i32, kf, ru.p, kf, 0x7fffffff);
      RAMA_KERNEL(ctx, k_earliest, nq, qe.p, state.p, nq, rf.p, ru.p);
      mf.alloc((size_t)LOG * nf, ctx.s);
      mu.alloc((size_t)LOG * nf, ctx.s);
      {
        int64_t n_ = nf;
        int build = 0;
        int32_t *pup = up.p, *pmf = mf.p, *pmu = mu.p;
        const int32_t *ppar = par.p, *ppe = pedge.p, *prf = rf.p, *pru = ru.p;
        void* args[] = {&n_, &LOG, &ppar, &ppe, &build, &pup, &prf, &pmf, &pru, &pmu};
        launch_coop(ctx, (const void*)k_lift_coop, "k_lift_coop", args, nf);
      }
      left.zero();
      RAMA_KERNEL(ctx, k_resolve, nq, nq, qa.p, qb.p, ql.p, up.p, mf.p, mu.p, LOG, nf, enter.p, exit_.p, state.p,
                  left.p);
      rs_iters++;
      if (read_scalar(ctx, left.p) == 0) break;
    }
    RAMA_KERNEL(ctx, k_mark_removed, nq, qe.p, state.p, nq, removed.p);
    mark(4);
    if (phase_prof)
      fprintf(stderr, "[rama]   forest n %lld m+ %lld kf %lld conflicts %lld LOG %d: rank sort %.2f boruvka %.2f (%d) "
              "euler %.2f lift+paths %.2f resolve %.2f (%d) ms\n", (long long)n, (long long)np, (long long)kf,
              (long long)nq, LOG, ph[0], ph[1], bv_iters, ph[2], ph[3], ph[4], rs_iters);
    }
  }
  RAMA_KERNEL(ctx, k_forest_keep, kf, Fi.p, kf, removed.p, keep.p);
  Buf<int32_t> idx;
  int64_t k = compact_indices(ctx, keep.p, np, idx);
  su.alloc(k > 0 ? k : 1, ctx.s);
  sv.alloc(k > 0 ? k : 1, ctx.s);
  RAMA_KERNEL(ctx, k_gather_pairs, k, idx.p, k, P.p, g.u, g.v, su.p, sv.p);
  return k;
}

// ------------------------------------------------------- contraction step

void contraction_step(Ctx& ctx, const GraphView& g, int policy, double switch_fraction, StepResult& out,
                      bool want_joined) {
  Buf<int32_t> su, sv;
  int64_t k = 0;
  out.used_forest = false;
  if (policy == 0) {
    int64_t e = select_max_edge(ctx, g);
    if (e >= 0) {
      su.alloc(1, ctx.s);
      sv.alloc(1, ctx.s);
      copy_d2d(ctx, su.p, g.u + e, 1);
      copy_d2d(ctx, sv.p, g.v + e, 1);
      k = 1;
    }
  } else if (policy == 2) {
    k = select_forest(ctx, g, su, sv);
    out.used_forest = true;
  } else {  // matching (1), auto (3): the matching's mapping comes straight from the partners
    out.map.alloc(g.n > 0 ? g.n : 1, ctx.s);
    int64_t nt = g.n;
    k = select_matching_map(ctx, g, 5, out.map.p, &nt);
    if (policy == 3 && (double)k < switch_fraction * (double)g.n) {
      k = select_forest(ctx, g, su, sv);
      out.used_forest = true;
    } else {
      out.num_selected = k;
      out.joined = 0.0;
      out.identity = k == 0;
      out.num_targets = nt;
      if (k == 0) return;
      out.next = contract(ctx, g, out.map.p, nt, want_joined ? &out.joined : nullptr);
      return;
    }
  }
  out.num_selected = k;
  out.joined = 0.0;
  if (k == 0) {
    out.identity = true;
    out.num_targets = g.n;
    return;
  }
  out.identity = false;
  out.map.alloc(g.n, ctx.s);
  // the component count stays on the device and returns with the
  // contraction's edge count (one read-back for both)
  Buf<int32_t> rank;
  components(ctx, g.n, su.p, sv.p, k, out.map.p, false, &rank);
  out.next = contract(ctx, g, out.map.p, g.n, want_joined ? &out.joined : nullptr, rank.p + g.n);
  out.num_targets = out.next.n;
}

}  // namespace rama
