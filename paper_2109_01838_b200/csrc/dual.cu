// Dual machinery.
//
// Separation (dual.py:109-197).  The reference runs one BFS per repulsive
// edge (a, b), a < b, over the attractive subgraph with neighbours expanded
// in ascending id order, and reports the BFS parent chain.  That parent
// chain has a closed form over sorted CSR rows, which is what each thread
// evaluates here (one thread per repulsive edge, no queues, no visited set):
//   level 1  N(a);  px(y) = min(N(a) & N(y)) is the BFS parent of a level-2
//   node y, and level-2 nodes are dequeued in (px(y), y) order;
//   3-cycle: x* = min(N(a) & N(b));
//   4-cycle: y* = argmin_(y in N(b), dist(y) = 2) (px(y), y);
//   5-cycle: for level-3 z, py(z) = argmin_(y in N(z), dist 2) (px(y), y) and
//            z* = argmin_(z in N(b), dist(z) = 3) (px(py), py, z).
// This is the BFS tie-break exactly (checked against the reference on the
// golden fixtures and by the oracle parity tests).
//
// Message passing (dual.py:309-392).  Per iteration two kernels:
//   edge phase  : cl[e] = base[e] + sum of lam over e's slots in ascending
//                 slot order (== np.bincount), delta[e] = cl[e] / cov[e];
//   triplet pass: lam[t,s] -= delta[e(t,s)]; then the damped six-step
//                 schedule in registers.
// All arithmetic is explicitly rounded (__dadd_rn/__dmul_rn/__ddiv_rn), so
// nvcc cannot contract into FMAs and lam is bit-identical to numpy's.
#include "internal.h"
#include "compact.cuh"
#include "sortreduce.cuh"

namespace rama {

// slot lists longer than kLongCov (hub edges) are summed a warp per edge
// (message passing section)
constexpr int32_t kLongCov = 64;

struct LongCov {  // edge with more than kLongCov slots
  const int32_t* ptr;
  __device__ __forceinline__ bool operator()(int32_t e) const { return ptr[e + 1] - ptr[e] > kLongCov; }
};

// ---------------------------------------------------------------- CSR

// Rows of at most kSmallRow int32 values (grid-like graphs: the positive
// CSR, the edge->slot lists) are built without a general sort: a
// run-aggregated count hands every item its offset in its row, the values
// are scattered into place and each row is insertion-sorted in registers.
// A row beyond kSmallRow (power-law hubs) sends the build to the bucket sort.
constexpr int32_t kSmallRow = 32;

__device__ __forceinline__ void cswap(int32_t& a, int32_t& b) {
  const int32_t lo = min(a, b), hi = max(a, b);
  a = lo;
  b = hi;
}

__global__ void k_rowsort_i32(const int32_t* __restrict__ ptr, int64_t m, int32_t* __restrict__ vals) {
  GRID_STRIDE(e, m) {
    const int32_t b = ptr[e], len = ptr[e + 1] - b;
    if (len < 2) continue;
    if (len <= 8) {  // registers: an 8-wide sorting network, padded
      int32_t x0 = vals[b], x1 = vals[b + 1];
      int32_t x2 = len > 2 ? vals[b + 2] : INT32_MAX, x3 = len > 3 ? vals[b + 3] : INT32_MAX;
      int32_t x4 = len > 4 ? vals[b + 4] : INT32_MAX, x5 = len > 5 ? vals[b + 5] : INT32_MAX;
      int32_t x6 = len > 6 ? vals[b + 6] : INT32_MAX, x7 = len > 7 ? vals[b + 7] : INT32_MAX;
      cswap(x0, x2); cswap(x1, x3); cswap(x4, x6); cswap(x5, x7);
      cswap(x0, x4); cswap(x1, x5); cswap(x2, x6); cswap(x3, x7);
      cswap(x0, x1); cswap(x2, x3); cswap(x4, x5); cswap(x6, x7);
      cswap(x2, x4); cswap(x3, x5);
      cswap(x1, x4); cswap(x3, x6);
      cswap(x1, x2); cswap(x3, x4); cswap(x5, x6);
      vals[b] = x0;
      vals[b + 1] = x1;
      if (len > 2) vals[b + 2] = x2;
      if (len > 3) vals[b + 3] = x3;
      if (len > 4) vals[b + 4] = x4;
      if (len > 5) vals[b + 5] = x5;
      if (len > 6) vals[b + 6] = x6;
      if (len > 7) vals[b + 7] = x7;
      continue;
    }
    int32_t x[kSmallRow];
    for (int32_t k = 0; k < len; k++) x[k] = vals[b + k];
    for (int32_t k = 1; k < len; k++) {
      const int32_t y = x[k];
      int32_t h = k - 1;
      while (h >= 0 && x[h] > y) {
        x[h + 1] = x[h];
        h--;
      }
      x[h + 1] = y;
    }
    for (int32_t k = 0; k < len; k++) vals[b + k] = x[k];
  }
}

// both arcs of every positive edge: counts per node with offsets
__global__ void k_pcsr_count(const int32_t* __restrict__ P, int64_t np, const int32_t* __restrict__ u,
                             const int32_t* __restrict__ v, int32_t* __restrict__ cnt, int32_t* __restrict__ off,
                             int32_t* __restrict__ long_flag) {
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x - lane; i0 < np;
       i0 += (int64_t)gridDim.x * blockDim.x) {  // warp-uniform trip count
    const int64_t i = i0 + lane;
    const int32_t e = i < np ? P[i] : -1;
    const int32_t a = e >= 0 ? u[e] : -1, b = e >= 0 ? v[e] : -1;
    const int32_t oa = run_atomic_add(cnt, a, 1);  // sorted by u: runs aggregate
    const int32_t ob = run_atomic_add(cnt, b, 1);
    if (e >= 0) {
      off[2 * i] = oa;
      off[2 * i + 1] = ob;
      if (oa >= kSmallRow || ob >= kSmallRow) *long_flag = 1;
    }
  }
}

__global__ void k_pcsr_scatter(const int32_t* __restrict__ P, int64_t np, const int32_t* __restrict__ u,
                               const int32_t* __restrict__ v, const int32_t* __restrict__ ptr,
                               const int32_t* __restrict__ off, int32_t* __restrict__ adj) {
  GRID_STRIDE(i, np) {
    const int32_t e = P[i], a = u[e], b = v[e];
    adj[ptr[a] + off[2 * i]] = b;
    adj[ptr[b] + off[2 * i + 1]] = a;
  }
}



__global__ void k_pos_arcs(const int32_t* __restrict__ P, int64_t np, const int32_t* __restrict__ u,
                           const int32_t* __restrict__ v, int32_t* __restrict__ row, uint64_t* __restrict__ key) {
  GRID_STRIDE(i, np) {
    int32_t e = P[i];
    row[2 * i] = u[e];
    key[2 * i] = (uint64_t)(uint32_t)v[e];
    row[2 * i + 1] = v[e];
    key[2 * i + 1] = (uint64_t)(uint32_t)u[e];
  }
}

__global__ void k_key_lo(const uint64_t* __restrict__ key, int64_t n, int32_t* __restrict__ out) {
  GRID_STRIDE(i, n) out[i] = (int32_t)(uint32_t)key[i];
}

struct PosCSR {
  Buf<int32_t> ptr;  // n + 1
  Buf<int32_t> adj;  // 2 m+
  int64_t arcs = 0;
};

// _positive_csr (dual.py:155-166): symmetric CSR of E+ sorted by (head, tail)
// (P: the np positive edges, ascending)
static void positive_csr(Ctx& ctx, const GraphView& g, const Buf<int32_t>& P, int64_t np, PosCSR& out) {
  int64_t na = 2 * np;
  if (np > 0) {  // short rows: count, scatter, sort each row in registers
    Buf<int32_t> cnt(g.n + 1, ctx), off(na, ctx);  // counts | long-row flag: one memset
    cnt.zero();
    int32_t* flag = cnt.p + g.n;
    RAMA_KERNEL(ctx, k_pcsr_count, np, P.p, np, g.u, g.v, cnt.p, off.p, flag);
    out.ptr.alloc(g.n + 1, ctx.s);
    exclusive_scan(ctx, cnt.p, out.ptr.p, g.n, false);
    if (read_scalar(ctx, flag) == 0) {
      out.adj.alloc(na, ctx.s);
      RAMA_KERNEL(ctx, k_pcsr_scatter, np, P.p, np, g.u, g.v, out.ptr.p, off.p, out.adj.p);
      RAMA_KERNEL(ctx, k_rowsort_i32, g.n, out.ptr.p, g.n, out.adj.p);
      out.arcs = na;
      return;
    }
  }
  Buf<int32_t> row(na > 0 ? na : 1, ctx);
  Buf<uint64_t> key(na > 0 ? na : 1, ctx);
  RAMA_KERNEL(ctx, k_pos_arcs, np, P.p, np, g.u, g.v, row.p, key.p);
  BucketSorted bs;
  bucket_sort(ctx, g.n, na, row.p, key.p, bs, false);
  out.ptr = std::move(bs.row_ptr);
  out.adj.alloc(na > 0 ? na : 1, ctx.s);
  RAMA_KERNEL(ctx, k_key_lo, na, bs.key.p, na, out.adj.p);
  out.arcs = na;
}

// ----------------------------------------------------------- separation

__device__ __forceinline__ bool in_sorted(const int32_t* a, int32_t len, int32_t y) {
  int32_t lo = 0, hi = len;
  while (lo < hi) {
    int32_t mid = (lo + hi) >> 1;
    int32_t x = a[mid];
    if (x < y) lo = mid + 1;
    else if (x > y) hi = mid;
    else return true;
  }
  return false;
}

// smallest common element of two ascending lists, or -1.  Skewed sizes
// (power-law hubs) walk the short list and binary-search the long one.
__device__ __forceinline__ int32_t first_common(const int32_t* a, int32_t la, const int32_t* b, int32_t lb) {
  if (la > 16 * lb || lb > 16 * la) {
    const int32_t* s = la < lb ? a : b;
    const int32_t* l = la < lb ? b : a;
    int32_t ls = la < lb ? la : lb, ll = la < lb ? lb : la;
    int32_t lo = 0;
    for (int32_t k = 0; k < ls; k++) {
      int32_t y = s[k], hi = ll;
      while (lo < hi) {
        int32_t mid = (lo + hi) >> 1;
        if (l[mid] < y) lo = mid + 1; else hi = mid;
      }
      if (lo == ll) return -1;
      if (l[lo] == y) return y;
    }
    return -1;
  }
  int32_t i = 0, j = 0;
  while (i < la && j < lb) {
    int32_t x = a[i], y = b[j];
    if (x == y) return x;
    if (x < y) i++; else j++;
  }
  return -1;
}

// position in a of the smallest common element of two ascending lists, or -1
__device__ __forceinline__ int32_t first_common_pos(const int32_t* a, int32_t la, const int32_t* b, int32_t lb) {
  if (la > 16 * lb) {  // short b: binary-search its elements in a
    int32_t lo = 0;
    for (int32_t k = 0; k < lb; k++) {
      int32_t y = b[k], hi = la;
      while (lo < hi) {
        int32_t mid = (lo + hi) >> 1;
        if (a[mid] < y) lo = mid + 1; else hi = mid;
      }
      if (lo == la) return -1;
      if (a[lo] == y) return lo;
    }
    return -1;
  }
  if (lb > 16 * la) {  // short a: binary-search its elements in b
    int32_t lo = 0;
    for (int32_t k = 0; k < la; k++) {
      int32_t y = a[k], hi = lb;
      while (lo < hi) {
        int32_t mid = (lo + hi) >> 1;
        if (b[mid] < y) lo = mid + 1; else hi = mid;
      }
      if (lo == lb) return -1;
      if (b[lo] == y) return k;
    }
    return -1;
  }
  int32_t i = 0, j = 0;
  while (i < la && j < lb) {
    int32_t x = a[i], y = b[j];
    if (x == y) return i;
    if (x < y) i++; else j++;
  }
  return -1;
}

__global__ void k_gather_i32_dev(const int32_t* __restrict__ src, const int32_t* __restrict__ idx,
                                 const int32_t* __restrict__ n_dev, int32_t* __restrict__ out) {
  const int64_t n = *n_dev;
  GRID_STRIDE(i, n) out[i] = src[idx[i]];
}

__global__ void k_gather_i32(const int32_t* __restrict__ src, const int32_t* __restrict__ idx, int64_t n,
                             int32_t* __restrict__ dst) {
  GRID_STRIDE(i, n) dst[i] = src[idx[i]];
}

// Three convergent passes instead of one divergent kernel: every repulsive
// edge tries the 3-cycle; the misses are compacted and try the 4-cycle; the
// remaining misses try the 5-cycle.  (One fused kernel made nearly every
// warp wait for its slowest 5-cycle lane.)
__global__ void k_sep3(const int32_t* __restrict__ Q, int64_t nq, const int32_t* __restrict__ NQ,
                       const int32_t* __restrict__ u, const int32_t* __restrict__ v, const int32_t* __restrict__ ptr,
                       const int32_t* __restrict__ adj, int L, int32_t* __restrict__ out_len,
                       int32_t* __restrict__ out_nodes, uint8_t* __restrict__ miss,
                       uint8_t* __restrict__ zero_flags, int32_t* __restrict__ zero_cnt) {
  // (zero_flags[nq], zero_cnt[4]: the later passes' flags and list counters,
  // cleared here instead of by memsets)
  if (zero_cnt && blockIdx.x == 0 && threadIdx.x < 4) zero_cnt[threadIdx.x] = 0;
  GRID_STRIDE(i, nq) {
    if (zero_flags) zero_flags[i] = 0;
    int32_t q = Q ? Q[i] : (int32_t)i;
    int32_t e = NQ[q];
    int32_t a = u[e], b = v[e];
    int32_t pa = ptr[a], pb = ptr[b];
    int32_t la = ptr[a + 1] - pa, lb = ptr[b + 1] - pb;
    int32_t x = first_common(adj + pa, la, adj + pb, lb);
    int32_t* row = out_nodes + q * (int64_t)L;
    if (x >= 0) {
      out_len[q] = 3;
      row[0] = a; row[1] = x; row[2] = b;
      for (int j = 3; j < L; j++) row[j] = 0;
    } else {
      out_len[q] = 0;
      for (int j = 0; j < L; j++) row[j] = 0;
    }
    if (miss) miss[i] = x < 0 && la > 0 && lb > 0;  // a longer cycle needs both ends on E+
  }
}

// px(y) for a level-2 candidate y (y not a, not in N(a)); -1 if y is not at distance 2
__device__ __forceinline__ int32_t level2_parent(const int32_t* __restrict__ ptr, const int32_t* __restrict__ adj,
                                                 int32_t a, const int32_t* Na, int32_t la, int32_t y) {
  if (y == a || in_sorted(Na, la, y)) return -1;
  return first_common(Na, la, adj + ptr[y], ptr[y + 1] - ptr[y]);
}

// 4- and 5-cycle passes: a group of kSepLanes lanes per repulsive edge; the
// lanes split the candidate neighbours and the group takes the
// lexicographic argmin with shuffles (keys packed as (parent << 32 | node)).
constexpr int kSepLanes = 8;

// Dense / power-law neighbourhoods only: the pull-style 5-cycle search
// (per z in N(b), scan N(z)) looks at no more than kHubCap neighbours z of b
// and stops at candidates z with more than kHubCap positive neighbours,
// bounding the per-edge work at kHubCap^2 lookups; a search that hit a cap
// is flagged and answered again by the exact ordered search
// (k_sep5_ordered), which stops at its first hit.  Grid-like graphs (C1-C3,
// C5) never reach the caps.
constexpr int32_t kHubCap = 128;


__device__ __forceinline__ uint64_t group_min(uint64_t x) {
#pragma unroll
  for (int o = kSepLanes / 2; o > 0; o >>= 1) {
    uint64_t y = __shfl_xor_sync(0xffffffffu, x, o, kSepLanes);
    x = y < x ? y : x;
  }
  return x;
}

__device__ __forceinline__ int32_t warp_max(int32_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

__device__ __forceinline__ uint64_t pack2(int32_t hi, int32_t lo) {
  return ((uint64_t)(uint32_t)hi << 32) | (uint64_t)(uint32_t)lo;
}

// 4-cycles for sources whose BFS levels overflow the shared tables (dense or
// hub neighbourhoods).  Ordered search, exact: the answer's parent p* is the
// smallest x in N(a) with some y in N(x) & N(b), y not in {a} u N(a) (every
// such y has px(y) = x because no smaller x qualifies), and y* is the
// smallest of those.  Scanning x ascending usually stops at the first x, so
// the cost is one row intersection instead of |N(b)| of them.
// (Q: repulsive edge ids, *nq_dev of them; the misses are appended to miss_list)
__global__ void k_sep4(const int32_t* __restrict__ Q, const int32_t* __restrict__ nq_dev,
                       const int32_t* __restrict__ NQ, const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                       const int32_t* __restrict__ ptr, const int32_t* __restrict__ adj, int L,
                       int32_t* __restrict__ out_len, int32_t* __restrict__ out_nodes, int32_t* __restrict__ miss_list,
                       int32_t* __restrict__ miss_cnt) {
  const int64_t nq = *nq_dev;
  const int g = threadIdx.x % kSepLanes;
  const int64_t per_warp = 32 / kSepLanes;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * per_warp; base < nq; base += nwarps * per_warp) {  // warp-uniform
    const int64_t i = base + (threadIdx.x & 31) / kSepLanes;
    bool live = i < nq;
    uint64_t best = ~0ULL;
    int32_t a = 0, b = 0, q = 0, la = 0, pb = 0, lb = 0;
    const int32_t* Na = adj;
    if (live) {
      q = Q[i];
      int32_t e = NQ[q];
      a = u[e];
      b = v[e];
      Na = adj + ptr[a];
      la = ptr[a + 1] - ptr[a];
      pb = ptr[b];
      lb = ptr[b + 1] - pb;
    }
    bool done = !live;
    // hub sources (|N(a)| >> |N(b)|): the same answer from b's side,
    // argmin over y in N(b) of (px(y), y), one level-2 test per y
    const bool bside = live && la > 4 * lb;
    const int32_t lb_max = warp_max(bside ? lb : 0);
    if (lb_max > 0) {
      // keys (position of px(y) in N(a), y).  px(y) is searched in a growing
      // prefix of N(a) (64, 512, ... positions): if any y has a parent in the
      // prefix, the minimum does, so the walks never pass it (hub rows: two
      // long rows are never merged end to end); a prefix with no parent
      // for any y grows x8 for all of them.
      uint64_t bb = ~0ULL;
      int32_t lim = min(la, 64);
      bool need = bside;
      while (__any_sync(0xffffffffu, need)) {
        for (int32_t k0 = 0; k0 < lb_max; k0 += kSepLanes) {
          const int32_t k = k0 + g;
          if (need && k < lb) {
            const int32_t y = adj[pb + k];
            if (y != a && !in_sorted(Na, la, y)) {
              const int32_t p = first_common_pos(Na, lim, adj + ptr[y], ptr[y + 1] - ptr[y]);
              if (p >= 0) {
                const uint64_t key = pack2(p, y);
                bb = key < bb ? key : bb;
              }
            }
          }
        }
        bb = group_min(bb);
        if (need && (bb != ~0ULL || lim >= la)) need = false;
        if (need) lim = (int32_t)min((int64_t)la, (int64_t)lim * 8);
      }
      if (bb != ~0ULL) bb = pack2(Na[(int32_t)(bb >> 32)], (int32_t)(uint32_t)bb);  // position -> node
      if (bside) {
        best = bb;
        done = true;
      }
    }
    const int32_t la_max = warp_max(done ? 0 : la);
    for (int32_t xi = 0; xi < la_max; xi++) {
      int32_t cand = 0x7fffffff, x = 0;
      if (!done && xi < la) {
        x = Na[xi];
        const int32_t px = ptr[x], lx = ptr[x + 1] - px;
        const bool xs = lx <= lb;
        const int32_t* S = xs ? adj + px : adj + pb;
        const int32_t* G = xs ? adj + pb : adj + px;
        const int32_t ls = xs ? lx : lb, lg = xs ? lb : lx;
        for (int32_t k = g; k < ls; k += kSepLanes) {
          int32_t y = S[k];
          if (y != a && in_sorted(G, lg, y) && !in_sorted(Na, la, y)) {
            cand = y;
            break;  // S ascending: the lane's first hit is its minimum
          }
        }
      }
      uint64_t c = group_min((uint64_t)(uint32_t)cand);
      if (!done && c != 0x7fffffffULL) {
        best = pack2(x, (int32_t)c);
        done = true;
      }
      if (__all_sync(0xffffffffu, done)) break;
    }
    if (live && g == 0) {
      bool found = best != ~0ULL;
      if (found) {
        int32_t* row = out_nodes + q * (int64_t)L;
        out_len[q] = 4;
        row[0] = a; row[1] = (int32_t)(best >> 32); row[2] = (int32_t)(uint32_t)best; row[3] = b;
      }
      if (miss_list && !found) miss_list[atomicAdd(miss_cnt, 1)] = q;
    }
  }
}

__global__ void k_sep5(const int32_t* __restrict__ Q, const int32_t* __restrict__ nq_dev,
                       const int32_t* __restrict__ NQ, const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                       const int32_t* __restrict__ ptr, const int32_t* __restrict__ adj, int L,
                       int32_t* __restrict__ out_len, int32_t* __restrict__ out_nodes, uint8_t* __restrict__ capped) {
  const int64_t nq = *nq_dev;
  const int g = threadIdx.x % kSepLanes;
  const int64_t per_warp = 32 / kSepLanes;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * per_warp; base < nq; base += nwarps * per_warp) {  // warp-uniform
    const int64_t i = base + (threadIdx.x & 31) / kSepLanes;
    bool live = i < nq;
    int32_t a = 0, b = 0, q = 0, la = 0, pb = 0, lb = 0;
    const int32_t* Na = adj;
    if (live) {
      q = Q[i];
      int32_t e = NQ[q];
      a = u[e];
      b = v[e];
      Na = adj + ptr[a];
      la = ptr[a + 1] - ptr[a];
      pb = ptr[b];
      lb = ptr[b + 1] - pb;
    }
    // level-3 neighbours z of b ranked by (px(py(z)), py(z), z); each z's
    // best level-2 neighbour py(z) is a group argmin over N(z)
    uint64_t bx_y = ~0ULL;
    int32_t bz = 0x7fffffff;
    // trip counts are warp-uniform: the group shuffles below use the full mask
    int32_t lbmax = warp_max(min(lb, kHubCap));
    if (capped && live && g == 0 && lb > kHubCap) capped[q] = 1;  // truncated: answered again exactly
    for (int32_t k = 0; k < lbmax; k++) {
      bool zok = live && k < lb;
      int32_t z = zok ? adj[pb + k] : 0;
      int32_t pz = 0, lz = 0;
      if (zok) {
        if (z == a || in_sorted(Na, la, z)) zok = false;
      }
      if (zok) {
        pz = ptr[z];
        lz = ptr[z + 1] - pz;
        if (lz > kHubCap) {  // hub candidate skipped: flagged for the exact search
          zok = false;
          if (capped) capped[q] = 1;
        } else if (first_common(Na, la, adj + pz, lz) >= 0) {
          zok = false;  // z at distance 2
        }
      }
      uint64_t zbest = ~0ULL;
      int32_t lzmax = warp_max(zok ? lz : 0);
      for (int32_t j0 = 0; j0 < lzmax; j0 += kSepLanes) {
        int32_t j = j0 + g;
        if (zok && j < lz) {
          int32_t y = adj[pz + j];
          int32_t py = level2_parent(ptr, adj, a, Na, la, y);
          if (py >= 0) {
            uint64_t key = pack2(py, y);
            zbest = key < zbest ? key : zbest;
          }
        }
      }
      zbest = group_min(zbest);
      if (zok && zbest != ~0ULL && (zbest < bx_y || (zbest == bx_y && z < bz))) {
        bx_y = zbest;
        bz = z;
      }
    }
    if (live && g == 0 && bx_y != ~0ULL) {
      int32_t* row = out_nodes + q * (int64_t)L;
      out_len[q] = 5;
      row[0] = a; row[1] = (int32_t)(bx_y >> 32); row[2] = (int32_t)(uint32_t)bx_y; row[3] = bz; row[4] = b;
    }
  }
}

// Exact 5-cycles for the searches the capped passes truncated (hub
// neighbourhoods).  At this stage (a, b) has no 3- or 4-cycle, so every
// z in N(b) is at BFS level >= 3 and the reference's answer
// z* = argmin_(z in N(b)) (px(py(z)), py(z), z) is the FIRST (x, y) in
// lexicographic order -- x in N(a) ascending, y in N(x) ascending, y not in
// {a} u N(a) -- with N(y) & N(b) non-empty, and z* = min(N(y) & N(b)).  (A y
// met again under a larger x was already tested under px(y) and failed, so
// the first hit has px(y) = x.)  One warp per edge, lanes over N(x) in
// ascending chunks; the scan stops at the first hit, which on power-law
// graphs comes within the first hub rows.
__global__ void k_sep5_ordered(const uint8_t* __restrict__ flags, int64_t nq, const int32_t* __restrict__ NQ,
                               const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                               const int32_t* __restrict__ ptr, const int32_t* __restrict__ adj, int L,
                               int32_t* __restrict__ out_len, int32_t* __restrict__ out_nodes) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c0 = w0 * 32; c0 < nq; c0 += W * 32) {  // a warp scans 32 flags, then takes the flagged edges
    unsigned todo = __ballot_sync(0xffffffffu, c0 + lane < nq && flags[c0 + lane]);
    while (todo) {
      const int32_t q = (int32_t)(c0 + __ffs(todo) - 1);
      todo &= todo - 1;
      const int32_t e = NQ[q];
      const int32_t a = u[e], b = v[e];
      const int32_t* Na = adj + ptr[a];
      const int32_t la = ptr[a + 1] - ptr[a];
      const int32_t* Nb = adj + ptr[b];
      const int32_t lb = ptr[b + 1] - ptr[b];
      int32_t hx = -1, hy = -1, hz = -1;
      for (int32_t xi = 0; xi < la && hx < 0; xi++) {
        const int32_t x = Na[xi];
        const int32_t* Nx = adj + ptr[x];
        const int32_t lx = ptr[x + 1] - ptr[x];
        for (int32_t j0 = 0; j0 < lx; j0 += 32) {
          const int32_t j = j0 + lane;
          int32_t z = -1, y = -1;
          if (j < lx) {
            y = Nx[j];
            if (y != a && !in_sorted(Na, la, y)) z = first_common(adj + ptr[y], ptr[y + 1] - ptr[y], Nb, lb);
          }
          const unsigned hit = __ballot_sync(0xffffffffu, z >= 0);
          if (hit) {
            const int src = __ffs(hit) - 1;
            hx = x;
            hy = __shfl_sync(0xffffffffu, y, src);
            hz = __shfl_sync(0xffffffffu, z, src);
            break;
          }
        }
      }
      if (lane == 0) {
        int32_t* row = out_nodes + (int64_t)q * L;
        if (hx >= 0) {
          out_len[q] = 5;
          row[0] = a; row[1] = hx; row[2] = hy; row[3] = hz; row[4] = b;
          for (int j = 5; j < L; j++) row[j] = 0;
        } else {
          out_len[q] = 0;
          for (int j = 0; j < L; j++) row[j] = 0;
        }
      }
    }
  }
}

// ---- source-grouped separation ------------------------------------------
//
// 4/5-cycles.  Repulsive edges without a triangle are grouped by their
// source a (the smaller endpoint; the list is (u, v)-sorted, so a source's
// edges are contiguous) and each source gets a group of kGrp lanes.  The
// group builds a's BFS levels once -- L1 = N+(a) in shared memory and
// L2 = {y : dist(a, y) = 2} with px(y) = min(N+(a) & N+(y)) in a shared hash
// table, filled by scanning N+(x) for x in ascending order so the first
// insertion is the BFS parent -- and answers all of a's edges (a, b) by
// table lookups instead of sorted-row intersections:
//   4-cycle  y* = argmin_(y in N(b) & L2) (px(y), y)
//   5-cycle  z* = argmin_(z in N(b), z not in {a} u L1 u L2) (px(py), py, z)
//            with py(z) = argmin_(y in N(z) & L2) (px(y), y).
// Table sizes: tier 1 (8 lanes per source, 16 sources per block, |N+(a)|
// <= 16) fits grid-like neighbourhoods; tier 1.5 takes its overflow with
// twice the L1 and L2 tables; the rest go to tier 2 (a warp per source, 128
// L1 entries, 16x the L2 table); what overflows tier 2 (hubs) is flagged for
// the row-intersection kernels above.  Tiers 1 / 1.5 walk the build's
// (x, y in N+(x)) pairs and each 5-cycle candidate batch's (z, y in N+(z))
// pairs flattened over the group's lanes (row offsets in shared memory), so
// short and uneven rows do not leave lanes idle.
// A group answers its source's edges one after another, so sources with
// very many repulsive edges (power-law hubs' neighbours) would serialize a
// whole launch behind one group: tier 2 passes those to the per-edge kernels.
template <int G, int NL1, int HBITS, int BUILD, int EDGES, bool ABORT>
struct SrcTier {
  static constexpr bool kAbort = ABORT;       // shared L2 counter: stop building on overflow
  static constexpr int kGrp = G;              // lanes per source
  static constexpr int kL1 = NL1;             // |N+(a)| capacity
  static constexpr int kHashBits = HBITS;
  static constexpr int kHash = 1 << HBITS;    // per-source L2 table; used at load <= 1/2
  static constexpr int kBuild = BUILD;        // max sum of |N+(x)| over x in N+(a)
  static constexpr int kEdges = EDGES;        // max repulsive edges of the source
};
#ifndef RAMA_T1_L1
#define RAMA_T1_L1 16
#endif
using SrcTier1 = SrcTier<8, RAMA_T1_L1, 6, 256, 1 << 30, false>;
using SrcTier15 = SrcTier<8, 32, 7, 512, 64, false>;  // tier 1's overflow, twice the L2 table
using SrcTier2 = SrcTier<32, 128, 10, 1024, 64, true>;
constexpr int kSrcThreads1 = 128, kSrcThreads2 = 128;

template <int HBITS>
__device__ __forceinline__ int32_t src_slot(int32_t y) {
  return (int32_t)(((uint32_t)y * 0x9E3779B1u) >> (32 - HBITS));
}

template <int HBITS>
__device__ __forceinline__ int32_t src_lookup(const int32_t* hk, const int32_t* hv, int32_t y) {
  constexpr int H = 1 << HBITS;
  int32_t h = src_slot<HBITS>(y);
  for (int t = 0; t < H; t++) {
    int32_t k = hk[h];
    if (k == y) return hv[h];
    if (k < 0) return -1;
    h = (h + 1) & (H - 1);
  }
  return -1;
}

// 128-bit membership filters held in registers (no false negatives): a
// miss skips the shared-memory binary search / hash probe
struct Bloom128 {
  uint64_t lo = 0, hi = 0;
  __device__ __forceinline__ static uint32_t bit(int32_t y) { return ((uint32_t)y * 0x2545F491u) >> 25; }
  __device__ __forceinline__ void add(int32_t y) {
    const uint32_t b = bit(y);
    const uint64_t m = 1ULL << (b & 63);
    lo |= b < 64 ? m : 0ULL;
    hi |= b < 64 ? 0ULL : m;
  }
  __device__ __forceinline__ bool maybe(int32_t y) const {
    uint32_t b = bit(y);
    return ((b < 64 ? lo : hi) >> (b & 63)) & 1ULL;
  }
  template <int G>
  __device__ __forceinline__ void group_or(unsigned mask) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      lo |= __shfl_xor_sync(mask, lo, o, G);
      hi |= __shfl_xor_sync(mask, hi, o, G);
    }
  }
};

__device__ __forceinline__ bool src_in_l1(const int32_t* l1, int32_t la, int32_t y) {
  int32_t lo = 0, hi = la;
  while (lo < hi) {
    int32_t mid = (lo + hi) >> 1;
    int32_t x = l1[mid];
    if (x < y) lo = mid + 1;
    else if (x > y) hi = mid;
    else return true;
  }
  return false;
}

template <int G>
__device__ __forceinline__ uint64_t grp_min_u64(uint64_t x, unsigned mask) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    uint64_t y = __shfl_xor_sync(mask, x, o, G);
    x = y < x ? y : x;
  }
  return x;
}

template <int G>
__device__ __forceinline__ int32_t grp_min_i32(int32_t x, unsigned mask) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) x = min(x, __shfl_xor_sync(mask, x, o, G));
  return x;
}

template <int G>
__device__ __forceinline__ int32_t grp_sum_i32(int32_t x, unsigned mask) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) x += __shfl_xor_sync(mask, x, o, G);
  return x;
}

// gstart[k] = first index (into Q2) of source group k (source gsrc[k]);
// groups end at gstart[k+1] (or n2).  qb[i] = target b of the i-th miss.
// glist (tier 2): the groups to run, else all ng.  A group that overflows
// the tables sets gover[k] (tier 1, when given) or fb of its edges.
// Table values are POSITIONS in N+(a) (ascending = node order), so the
// parent is the atomicMin over the positions that reach y and every row of
// the level can be walked at once (no sequential x loop).
// Lists are appended on the device (no host read-back between the tiers):
// the next tier reads *over_cnt groups of over_list, the row-intersection
// kernels *fb_cnt repulsive edges of fb_list.
template <class T, int THREADS, int MINB, bool kListed>
__global__ void __launch_bounds__(THREADS, MINB) k_sep_src(
    const int32_t* __restrict__ gstart, const int32_t* __restrict__ gsrc, const int32_t* __restrict__ glist,
    int64_t nlist_host, const int32_t* __restrict__ nlist_dev, const int32_t* __restrict__ ng_dev,
    const int32_t* __restrict__ n2_dev, const int32_t* __restrict__ Q2, const int32_t* __restrict__ qb, const int32_t* __restrict__ ptr,
    const int32_t* __restrict__ adj, int L, int32_t* __restrict__ out_len, int32_t* __restrict__ out_nodes,
    int32_t* __restrict__ over_list, int32_t* __restrict__ over_cnt, int32_t* __restrict__ fb_list,
    int32_t* __restrict__ fb_cnt, int force_fallback, uint8_t* __restrict__ capped) {
  const int64_t ng = *ng_dev, n2 = *n2_dev;  // source groups, listed repulsive edges (counts on the device)
  int64_t nlist = nlist_host < 0 ? ng : nlist_host;
  if constexpr (kListed) nlist = *nlist_dev;
  constexpr int kGrp = T::kGrp, kPer = THREADS / T::kGrp, kH = T::kHash;
  __shared__ int32_t s_l1[kPer][T::kL1];
  __shared__ int32_t s_hk[kPer][kH];
  __shared__ int32_t s_hv[kPer][kH];
  __shared__ int32_t s_fill[kPer];
  // flattened walks: row starts and cumulative row lengths of the build's
  // N+(x) rows (tiers 1 / 1.5), reused for one batch of 5-cycle candidates z
  constexpr int kFlat = T::kAbort ? kGrp : T::kL1;  // tier 2 builds row by row (it stops early)
  __shared__ int32_t s_rs[kPer][kFlat];
  __shared__ int32_t s_cum[kPer][kFlat + 1];
  __shared__ int32_t s_zz[kPer][kGrp];
  const int gi = threadIdx.x / kGrp, lane = threadIdx.x % kGrp;
  const unsigned mask = kGrp == 32 ? 0xffffffffu : ((1u << kGrp) - 1u) << ((threadIdx.x & 31) & ~(kGrp - 1));
  int32_t* l1 = s_l1[gi];
  int32_t* hk = s_hk[gi];
  int32_t* hv = s_hv[gi];
  int32_t* rs = s_rs[gi];
  int32_t* cum = s_cum[gi];
  int32_t* zz = s_zz[gi];
  const int64_t ngroups = (int64_t)gridDim.x * kPer;
  for (int64_t j = (int64_t)blockIdx.x * kPer + gi; j < nlist; j += ngroups) {
    const int64_t k = kListed ? glist[j] : j;
    const int32_t e0 = gstart[k], e1 = k + 1 < ng ? gstart[k + 1] : (int32_t)n2;
    const int32_t a = gsrc[k];
    const int32_t pa = ptr[a], la = ptr[a + 1] - pa;
    bool over = la > T::kL1 || e1 - e0 > T::kEdges || force_fallback;
    Bloom128 f1, f2;  // L1 and L2 members
    __syncwarp(mask);  // the previous source's lookups are done before the table is reset
    if (!over) {
      // lane owns kL1 / kGrp consecutive positions of N+(a): x, row start,
      // row length (cum, turned into exclusive offsets below)
      constexpr int kOwn = T::kL1 / kGrp;
      int32_t own = 0;
#pragma unroll
      for (int r = 0; r < kOwn; r++) {
        const int32_t xi = lane * kOwn + r;
        if (xi < la) {
          const int32_t x = adj[pa + xi];
          l1[xi] = x;
          f1.add(x);
          const int32_t px = ptr[x], lx = ptr[x + 1] - px;
          if constexpr (!T::kAbort) {
            rs[xi] = px;
            cum[xi] = lx;
          }
          own += lx;
        }
      }
      f1.group_or<kGrp>(mask);
      int32_t incl = own;
#pragma unroll
      for (int o = 1; o < kGrp; o <<= 1) {
        const int32_t t = __shfl_up_sync(mask, incl, o, kGrp);
        if (lane >= o) incl += t;
      }
      const int32_t work = __shfl_sync(mask, incl, kGrp - 1, kGrp);
      if constexpr (!T::kAbort) {
        int32_t run = incl - own;
#pragma unroll
        for (int r = 0; r < kOwn; r++) {
          const int32_t xi = lane * kOwn + r;
          if (xi < la) {
            const int32_t lx = cum[xi];
            cum[xi] = run;
            run += lx;
          }
        }
        if (lane == 0) cum[la] = work;
      }
      for (int32_t t = lane; t < kH; t += kGrp) {
        hk[t] = -1;
        hv[t] = 0x7fffffff;
      }
      if (T::kAbort && lane == 0) s_fill[gi] = 0;
      __syncwarp(mask);
      over = work > T::kBuild;
      if (!over) {
        if (T::kAbort) {
          // tier 2: the group's L2 count is shared, so a source whose L2
          // outgrows the table stops building at once instead of finishing
          // its rows (power-law neighbourhoods)
          volatile int32_t* fill = s_fill + gi;
          for (int32_t xi = lane; xi < la && *fill <= kH / 2; xi += kGrp) {
            const int32_t x = l1[xi];
            const int32_t px = ptr[x], lx = ptr[x + 1] - px;
            for (int32_t t = 0; t < lx; t++) {
              const int32_t y = adj[px + t];
              if (y == a || (f1.maybe(y) && src_in_l1(l1, la, y))) continue;
              int32_t h = src_slot<T::kHashBits>(y);
              for (int r = 0; r < kH; r++) {
                int32_t kk = atomicCAS(hk + h, -1, y);
                if (kk == -1 || kk == y) {
                  if (kk == -1) {
                    atomicAdd(s_fill + gi, 1);
                    f2.add(y);
                  }
                  atomicMin(hv + h, xi);  // BFS parent = smallest position reaching y
                  break;
                }
                h = (h + 1) & (kH - 1);
              }
              if (*fill > kH / 2) break;
            }
          }
          __syncwarp(mask);
          over = *fill > kH / 2;
        } else {
          // the (x, y in N+(x)) pairs flattened over the group's lanes:
          // pair w lies in row xi with cum[xi] <= w < cum[xi + 1]
          int32_t mine = 0;
          int32_t xi = 0;
          for (int32_t w = lane; w < work; w += kGrp) {
            while (cum[xi + 1] <= w) xi++;
            const int32_t y = adj[rs[xi] + (w - cum[xi])];
            if (y == a || (f1.maybe(y) && src_in_l1(l1, la, y))) continue;
            int32_t h = src_slot<T::kHashBits>(y);
            for (int r = 0; r < kH; r++) {
              int32_t kk = atomicCAS(hk + h, -1, y);
              if (kk == -1 || kk == y) {
                if (kk == -1) {  // a lane that finds y present: its inserter added it
                  mine++;
                  f2.add(y);
                }
                atomicMin(hv + h, xi);  // BFS parent = smallest position reaching y
                break;
              }
              h = (h + 1) & (kH - 1);
            }
          }
          mine = grp_sum_i32<kGrp>(mine, mask);
          over = mine > kH / 2;
        }
        f2.group_or<kGrp>(mask);
      }
      __syncwarp(mask);  // table complete before the lookups
    }
    if (over) {
      if constexpr (!T::kAbort) {  // tiers 1 / 1.5: the next tier takes the source
        if (lane == 0) over_list[atomicAdd(over_cnt, 1)] = (int32_t)k;
      } else {  // last tier: its edges go to the row-intersection kernels
        int32_t at = 0;
        if (lane == 0) at = atomicAdd(fb_cnt, e1 - e0);
        at = __shfl_sync(mask, at, 0, kGrp);
        for (int32_t i = e0 + lane; i < e1; i += kGrp) fb_list[at + (i - e0)] = Q2[i];
      }
      __syncwarp(mask);
      continue;
    }
    for (int32_t i = e0; i < e1; i++) {
      const int32_t q = Q2[i];
      const int32_t b = qb[i];
      const int32_t pb = ptr[b], lb = ptr[b + 1] - pb;
      int32_t len = 0, r1 = 0, r2 = 0, r3 = 0;
      uint64_t best = ~0ULL;
      for (int32_t t = lane; t < lb; t += kGrp) {
        int32_t y = adj[pb + t];
        int32_t p = f2.maybe(y) ? src_lookup<T::kHashBits>(hk, hv, y) : -1;
        if (p >= 0) {
          uint64_t key = ((uint64_t)(uint32_t)p << 32) | (uint32_t)y;
          best = key < best ? key : best;
        }
      }
      best = grp_min_u64<kGrp>(best, mask);
      if (best != ~0ULL) {
        len = 4; r1 = l1[(int32_t)(best >> 32)]; r2 = (int32_t)(uint32_t)best;
      } else if (L >= 5) {
        // min over the pairs (z, y in N+(z) & L2) of ((px(y), y), z), which
        // is the per-z minimum followed by the (key, z) minimum over z; a
        // batch of kGrp candidates z is filtered, then its pairs are walked
        // flattened over the lanes
        uint64_t bk = ~0ULL;
        int32_t bz = 0x7fffffff;
        const int32_t lbc = min(lb, kHubCap);
        if (capped && lane == 0 && lb > kHubCap) capped[q] = 1;  // truncated: answered again exactly
        for (int32_t base = 0; base < lbc; base += kGrp) {
          const int32_t t = base + lane;
          int32_t z = 0, pz = 0, lz = 0;
          if (t < lbc) {
            z = adj[pb + t];
            if (!(z == a || (f1.maybe(z) && src_in_l1(l1, la, z)) ||
                  (f2.maybe(z) && src_lookup<T::kHashBits>(hk, hv, z) >= 0))) {
              pz = ptr[z];
              lz = ptr[z + 1] - pz;
              if (lz > kHubCap) {  // hub candidate skipped: flagged for the exact search
                if (capped) capped[q] = 1;
                lz = 0;
              }
            }
          }
          int32_t zi = lz;
#pragma unroll
          for (int o = 1; o < kGrp; o <<= 1) {
            const int32_t v = __shfl_up_sync(mask, zi, o, kGrp);
            if (lane >= o) zi += v;
          }
          const int32_t tot = __shfl_sync(mask, zi, kGrp - 1, kGrp);
          if (tot == 0) continue;
          cum[lane] = zi - lz;
          rs[lane] = pz;
          zz[lane] = z;
          if (lane == 0) cum[kGrp] = tot;
          __syncwarp(mask);
          int32_t c = 0;
          for (int32_t w = lane; w < tot; w += kGrp) {
            while (cum[c + 1] <= w) c++;
            const int32_t y = adj[rs[c] + (w - cum[c])];
            const int32_t p = f2.maybe(y) ? src_lookup<T::kHashBits>(hk, hv, y) : -1;
            if (p >= 0) {
              const uint64_t key = ((uint64_t)(uint32_t)p << 32) | (uint32_t)y;
              const int32_t zc = zz[c];
              if (key < bk || (key == bk && zc < bz)) { bk = key; bz = zc; }
            }
          }
          __syncwarp(mask);  // the batch is read before the next one is written
        }
        uint64_t mn = grp_min_u64<kGrp>(bk, mask);
        int32_t zc = grp_min_i32<kGrp>(bk == mn ? bz : 0x7fffffff, mask);
        if (mn != ~0ULL) {
          len = 5; r1 = l1[(int32_t)(mn >> 32)]; r2 = (int32_t)(uint32_t)mn; r3 = zc;
        }
      }
      if (lane == 0 && len) {
        int32_t* row = out_nodes + (int64_t)q * L;
        out_len[q] = len;
        row[0] = a; row[1] = r1; row[2] = r2;
        if (len == 4) row[3] = b;
        else { row[3] = r3; row[4] = b; }
      }
    }
    __syncwarp(mask);
  }
}

// over the first *n2_dev of cap list entries (heads of the rest cleared)
__global__ void k_src_heads(const int32_t* __restrict__ Q2, const int32_t* __restrict__ n2_dev, int64_t cap,
                            const int32_t* __restrict__ NQ, const int32_t* __restrict__ u,
                            const int32_t* __restrict__ v, uint8_t* __restrict__ head, int32_t* __restrict__ qa,
                            int32_t* __restrict__ qb) {
  const int64_t n2 = *n2_dev;
  GRID_STRIDE(i, cap) {
    if (i >= n2) {
      head[i] = 0;
      continue;
    }
    int32_t e = NQ[Q2[i]];
    int32_t a = u[e];
    qa[i] = a;
    qb[i] = v[e];
    head[i] = (i == 0) || a != u[NQ[Q2[i - 1]]];
  }
}

// ---- generic BFS separation (L >= 6, mode PD+) ----------------------------
//
// The reference BFS itself, source-grouped: one warp per source a runs the
// BFS of dual.py:109-152 level by level in per-warp global scratch and then
// answers all of a's repulsive edges.  Queue order is reproduced exactly:
// level k+1 is discovered by scanning the level-k queue in order and each
// row in ascending id order; a node's parent is the first queue position
// that reaches it (atomicMin over the position), and the winners are
// appended in (position, row index) order with warp ballots.
// key[y] = ((0xffffffff - tick) << 32) | c: c = 0 discovered, c = p + 1
// candidate from queue position p; a fresh tick compares below stale keys.
__device__ __forceinline__ uint64_t bfs_key(uint32_t tick, uint32_t c) {
  return ((uint64_t)(0xffffffffu - tick) << 32) | c;
}

// BFS state of one warp, per node: the candidate key K (atomicMin), BFS
// parent, queue position and depth.  Dense: node-indexed arrays of n
// entries (any graph).  Hashed: tick-tagged open addressing over H slots --
// a slot whose tag carries another source's tick is free, so nothing is
// cleared between sources, and stale keys (older ticks) compare above any
// current one; a source whose BFS outgrows H/2 slots is handed to the dense
// pass.
struct BfsDense {
  unsigned long long* K;
  int32_t *Pa, *Po, *Dp;
  __device__ __forceinline__ int32_t ins(int32_t y, uint32_t) { return y; }
  __device__ __forceinline__ int32_t find(int32_t y, uint32_t) const { return y; }
};

struct BfsHash {
  unsigned long long* tag;  // (tick << 32) | node
  unsigned long long* K;
  int32_t *Pa, *Po, *Dp;
  uint32_t mask;
  int32_t* claims;          // slots claimed for the current source (shared memory)
  __device__ __forceinline__ static uint32_t slot(int32_t y) {  // mixed: the low bits index the table
    uint32_t x = (uint32_t)y * 0x9E3779B1u;
    x ^= x >> 15;
    x *= 0x85EBCA6Bu;
    return x ^ (x >> 13);
  }
  __device__ __forceinline__ int32_t ins(int32_t y, uint32_t tick) {
    const unsigned long long want = ((unsigned long long)tick << 32) | (uint32_t)y;
    uint32_t h = slot(y) & mask;
    for (uint32_t probes = 0; probes <= mask;) {
      const unsigned long long t = __ldcg(tag + h);
      if (t == want) return (int32_t)h;
      if ((uint32_t)(t >> 32) != tick) {  // free for this source
        const unsigned long long old = atomicCAS(tag + h, t, want);
        if (old == t) {
          atomicAdd(claims, 1);
          return (int32_t)h;
        }
        if (old == want) return (int32_t)h;
        if ((uint32_t)(old >> 32) != tick) continue;  // another stale value: retry the slot
      }
      h = (h + 1) & mask;
      probes++;
    }
    return -1;
  }
  __device__ __forceinline__ int32_t find(int32_t y, uint32_t tick) const {
    const unsigned long long want = ((unsigned long long)tick << 32) | (uint32_t)y;
    uint32_t h = slot(y) & mask;
    for (uint32_t probes = 0; probes <= mask; probes++) {
      const unsigned long long t = __ldcg(tag + h);
      if (t == want) return (int32_t)h;
      if ((uint32_t)(t >> 32) != tick) return -1;
      h = (h + 1) & mask;
    }
    return -1;
  }
};

// One warp per source group (glist: the groups to run, *gcount of them; else
// all ng).  qcap: queue capacity per warp; limit: claimed slots after which a
// source is abandoned to `over` (hashed state only).
constexpr int32_t kBfsLaneRow = 12;  // rows up to this long are walked by one lane (longer: the whole warp)

// tick: this source's stamp, increasing along each warp's sources (stale
// keys of earlier sources must compare above the current ones)
template <class S>
__device__ __forceinline__ void bfs_source(S& st, int32_t* Qu, int64_t k, uint32_t tick, int64_t ng, int64_t n2,
                                           const int32_t* __restrict__ gstart, const int32_t* __restrict__ Q2,
                                           const int32_t* __restrict__ NQ, const int32_t* __restrict__ u,
                                           const int32_t* __restrict__ v, const int32_t* __restrict__ ptr,
                                           const int32_t* __restrict__ adj, int L, int32_t* __restrict__ out_len,
                                           int32_t* __restrict__ out_nodes, int32_t limit, int32_t* claims,
                                           int32_t* __restrict__ over_list, int32_t* __restrict__ over_cnt) {
  const int lane = threadIdx.x & 31;
  const uint64_t done = bfs_key(tick, 0);
  const int32_t i0 = gstart[k], i1 = (k + 1 < ng) ? gstart[k + 1] : (int32_t)n2;
  const int32_t a = u[NQ[Q2[i0]]];
  if (lane == 0) {
    *claims = 0;
    const int32_t sa = st.ins(a, tick);
    Qu[0] = a;
    st.K[sa] = done;
    st.Pa[sa] = -1;
    st.Po[sa] = 0;
    st.Dp[sa] = 0;
  }
  __syncwarp();
  int32_t s = 0, e = 1;  // current level's queue range
  int32_t qlen = 1;
  for (int lev = 0; lev <= L - 3 && s < e; lev++) {  // discover levels 1 .. L-2
    // 32 queue positions at a time: a lane per position walks its row (grid
    // degrees: most lanes busy), or, when a row in the chunk is long, the
    // whole warp walks one row after the other
    bool full = false;
    for (int32_t p0 = s; p0 < e; p0 += 32) {  // candidates: atomicMin over the position
      const int32_t p = p0 + lane;
      const int32_t x = p < e ? __ldcg(Qu + p) : 0;
      const int32_t b0 = p < e ? ptr[x] : 0, dx = p < e ? ptr[x + 1] - b0 : 0;
      if (!__any_sync(0xffffffffu, dx > kBfsLaneRow)) {
        for (int32_t j = 0; j < dx; j++) {
          const int32_t sy = st.ins(adj[b0 + j], tick);
          if (sy < 0) full = true;
          else atomicMin(st.K + sy, (unsigned long long)bfs_key(tick, (uint32_t)p + 1));
        }
        continue;
      }
      for (int32_t pp = p0; pp < min(p0 + 32, e); pp++) {
        const int32_t xx = __ldcg(Qu + pp);
        const int32_t bb = ptr[xx], dd = ptr[xx + 1] - bb;
        for (int32_t j = lane; j < dd; j += 32) {
          const int32_t sy = st.ins(adj[bb + j], tick);
          if (sy < 0) full = true;
          else atomicMin(st.K + sy, (unsigned long long)bfs_key(tick, (uint32_t)pp + 1));
        }
      }
    }
    __syncwarp();
    if (__any_sync(0xffffffffu, full) || *(volatile int32_t*)claims > limit) {  // hashed state outgrown
      if (lane == 0) over_list[atomicAdd(over_cnt, 1)] = (int32_t)k;
      return;
    }
    for (int32_t p0 = s; p0 < e; p0 += 32) {  // winners in (position, row) order
      const int32_t p = p0 + lane;
      const int32_t x = p < e ? __ldcg(Qu + p) : 0;
      const int32_t b0 = p < e ? ptr[x] : 0, dx = p < e ? ptr[x + 1] - b0 : 0;
      if (!__any_sync(0xffffffffu, dx > kBfsLaneRow)) {
        // a lane per position: count its winners, offsets by a warp scan
        // (lane order = position order), then write them in row order
        const unsigned long long mine = bfs_key(tick, (uint32_t)p + 1);
        int32_t cnt = 0;
        for (int32_t j = 0; j < dx; j++) {
          const int32_t sy = st.find(adj[b0 + j], tick);
          cnt += sy >= 0 && __ldcg(st.K + sy) == mine;
        }
        int32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        int32_t at = qlen + incl - cnt;
        for (int32_t j = 0; j < dx && cnt > 0; j++) {
          const int32_t y = adj[b0 + j];
          const int32_t sy = st.find(y, tick);
          if (sy >= 0 && __ldcg(st.K + sy) == mine) {
            Qu[at] = y;
            st.Pa[sy] = x;
            st.Po[sy] = at;
            st.Dp[sy] = lev + 1;
            at++;
            cnt--;
          }
        }
        qlen += __shfl_sync(0xffffffffu, incl, 31);
        continue;
      }
      for (int32_t pp = p0; pp < min(p0 + 32, e); pp++) {
        const int32_t xx = __ldcg(Qu + pp);
        const int32_t bb = ptr[xx], dd = ptr[xx + 1] - bb;
        for (int32_t j0 = 0; j0 < dd; j0 += 32) {
          const int32_t j = j0 + lane;
          const int32_t y = j < dd ? adj[bb + j] : 0;
          const int32_t sy = j < dd ? st.find(y, tick) : -1;
          const bool win = sy >= 0 && __ldcg(st.K + sy) == bfs_key(tick, (uint32_t)pp + 1);
          const unsigned bal = __ballot_sync(0xffffffffu, win);
          if (win) {
            const int32_t at = qlen + __popc(bal & ((1u << lane) - 1u));
            Qu[at] = y;
            st.Pa[sy] = xx;
            st.Po[sy] = at;
            st.Dp[sy] = lev + 1;
          }
          qlen += __popc(bal);
        }
      }
    }
    __syncwarp();
    for (int32_t i = e + lane; i < qlen; i += 32) st.K[st.find(__ldcg(Qu + i), tick)] = done;
    __syncwarp();
    s = e;
    e = qlen;
  }
  const int32_t last = L - 2;  // deepest stored level
  for (int32_t i = i0; i < i1; i++) {
    const int32_t q = Q2[i];
    const int32_t b = v[NQ[q]];
    int32_t tail = -1, len = 0;
    const int32_t sb = st.find(b, tick);
    if (sb >= 0 && __ldcg(st.K + sb) == done) {  // b itself reached at level <= L-2
      len = __ldcg(st.Dp + sb) + 1;
      tail = b;
    } else {  // b at level L-1: parent = first queue position among N(b) at level L-2
      const int32_t b0 = ptr[b], db = ptr[b + 1] - b0;
      int32_t best = 0x7fffffff;
      for (int32_t j = lane; j < db; j += 32) {
        const int32_t sy = st.find(adj[b0 + j], tick);
        if (sy >= 0 && __ldcg(st.K + sy) == done && __ldcg(st.Dp + sy) == last) best = min(best, __ldcg(st.Po + sy));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
      if (best != 0x7fffffff) {
        len = L;
        tail = -2 - best;  // marks: b appended after the queue node at `best`
      }
    }
    if (lane == 0 && len >= 3) {
      int32_t* row = out_nodes + (int64_t)q * L;
      out_len[q] = len;
      int32_t idx = len - 1, x;
      if (tail >= 0) {
        x = tail;
      } else {
        row[idx--] = b;
        x = __ldcg(Qu + (-2 - tail));
      }
      for (; idx >= 0; idx--) {
        row[idx] = x;
        x = __ldcg(st.Pa + st.find(x, tick));
      }
    }
    __syncwarp();
  }
}

// dense state: n-sized slices per warp (glist: an overflow list, *gcount
// groups; else every group)
__global__ void __launch_bounds__(256) k_sep_bfs(const int32_t* __restrict__ gstart, int64_t ng, int64_t n2,
                                                 const int32_t* __restrict__ glist, const int32_t* __restrict__ gcount,
                                                 const int32_t* __restrict__ Q2, const int32_t* __restrict__ NQ,
                                                 const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                                                 const int32_t* __restrict__ ptr, const int32_t* __restrict__ adj,
                                                 int L, int32_t* __restrict__ out_len,
                                                 int32_t* __restrict__ out_nodes, unsigned long long* keys,
                                                 int32_t* par, int32_t* pos, int32_t* queue, int32_t* depth,
                                                 int64_t n) {
  __shared__ int32_t s_claims[8];
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  BfsDense st{keys + w * n, par + w * n, pos + w * n, depth + w * n};
  const int64_t nl = glist ? (int64_t)*gcount : ng;
  for (int64_t j = w; j < nl; j += W) {
    const int64_t k = glist ? glist[j] : j;  // the list is unordered: stamp by position j
    bfs_source(st, queue + w * n, k, (uint32_t)(j + 1), ng, n2, gstart, Q2, NQ, u, v, ptr, adj, L, out_len, out_nodes, 0x7fffffff,
               s_claims + (threadIdx.x >> 5), nullptr, nullptr);
  }
}

// hashed state: H = mask + 1 slots per warp; sources that outgrow H / 2 go
// to over_list for the dense kernel
__global__ void __launch_bounds__(256) k_sep_bfs_hash(const int32_t* __restrict__ gstart, int64_t ng, int64_t n2,
                                                      const int32_t* __restrict__ glist,
                                                      const int32_t* __restrict__ gcount,
                                                      const int32_t* __restrict__ Q2, const int32_t* __restrict__ NQ,
                                                      const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                                                      const int32_t* __restrict__ ptr,
                                                      const int32_t* __restrict__ adj, int L,
                                                      int32_t* __restrict__ out_len, int32_t* __restrict__ out_nodes,
                                                      unsigned long long* tags, unsigned long long* keys,
                                                      int32_t* par, int32_t* pos, int32_t* queue, int32_t* depth,
                                                      uint32_t mask, int32_t* __restrict__ over_list,
                                                      int32_t* __restrict__ over_cnt) {
  __shared__ int32_t s_claims[8];
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t H = (int64_t)mask + 1;
  BfsHash st{tags + w * H, keys + w * H, par + w * H, pos + w * H, depth + w * H, mask, s_claims + (threadIdx.x >> 5)};
  const int64_t nl = glist ? (int64_t)*gcount : ng;
  for (int64_t j = w; j < nl; j += W) {
    const int64_t k = glist ? glist[j] : j;
    bfs_source(st, queue + w * H, k, (uint32_t)(j + 1), ng, n2, gstart, Q2, NQ, u, v, ptr, adj, L, out_len,
               out_nodes, (int32_t)(H / 2), st.claims, over_list, over_cnt);
  }
}

// no cycle of up to 5 edges found, and both ends have attractive neighbours
__global__ void k_needs_bfs(const int32_t* __restrict__ len, int64_t nq, const int32_t* __restrict__ NQ,
                            const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                            const int32_t* __restrict__ ptr, uint8_t* __restrict__ deep) {
  GRID_STRIDE(q, nq) {
    const int32_t e = NQ[q], a = u[e], b = v[e];
    deep[q] = len[q] == 0 && ptr[a + 1] > ptr[a] && ptr[b + 1] > ptr[b];
  }
}

// The exact BFS over the repulsive edges Qx (indices into NQ, ascending):
// grouped by source, one warp per source with 24 n bytes of scratch per warp.
__global__ void k_bfs_heads(const int32_t* __restrict__ Qx, int64_t nx, const int32_t* __restrict__ NQ,
                            const int32_t* __restrict__ u, uint8_t* __restrict__ head) {
  GRID_STRIDE(i, nx) head[i] = (i == 0) || u[NQ[Qx[i]]] != u[NQ[Qx[i - 1]]];
}

static void run_sep_bfs(Ctx& ctx, const GraphView& g, const int32_t* ptr, const int32_t* adj, const int32_t* NQ,
                        const int32_t* Qx, int64_t nx, int L, CycleRows& out) {
  if (nx == 0) return;
  Buf<uint8_t> head(nx, ctx);
  RAMA_KERNEL(ctx, k_bfs_heads, nx, Qx, nx, NQ, g.u, head.p);
  Buf<int32_t> gstart;
  const int64_t ng = compact_indices(ctx, head.p, nx, gstart);
  // hashed pass, one warp per source, 1 K slots (32 KB) per warp: the small
  // balls of grid-like graphs stay in L2-resident tables; the balls that
  // outgrow them take the dense pass (measured, PD+: C2 293 -> 152 ms and
  // 83 -> 6 GB; C3 34.6 s with the dense pass alone -> 29 s; 16 K-slot tables:
  // C2 162 ms, C3 83 s) -- RAMA_BFS_HASH_BITS resizes the table (tests)
  static const int kHashBits = [] {
    const char* e = getenv("RAMA_BFS_HASH_BITS");
    const int b = e ? atoi(e) : 10;
    return b < 4 ? 4 : (b > 20 ? 20 : b);
  }();
  Buf<int32_t> over(ng, ctx), ocnt(1, ctx);
  ocnt.zero();
  for (int pass = 0; pass < 1; pass++) {
    const int bits = kHashBits;
    const int64_t H = (int64_t)1 << bits;
    const int64_t budget = std::max<int64_t>(8, ((int64_t)4 << 30) / (32 * H));  // ~4 GB of tables at most
    int64_t W = std::min<int64_t>(std::min<int64_t>((int64_t)num_sms() * 8, ng), budget);
    W = (W + 7) / 8 * 8;  // whole 8-warp blocks
    Buf<unsigned long long> tags((size_t)W * H, ctx), keys((size_t)W * H, ctx);
    Buf<int32_t> par((size_t)W * H, ctx), pos((size_t)W * H, ctx), queue((size_t)W * H, ctx),
        depth((size_t)W * H, ctx);
    tags.fill_bytes(0xff);
    keys.fill_bytes(0xff);
    KernelScope ks(ctx.s, "k_sep_bfs_hash", 0.0);
    k_sep_bfs_hash<<<(unsigned)(W / 8), 256, 0, ctx.s>>>(
        gstart.p, ng, nx, (const int32_t*)nullptr, ocnt.p, Qx, NQ, g.u, g.v, ptr, adj, L, out.len.p, out.nodes.p,
        tags.p, keys.p, par.p, pos.p, queue.p, depth.p, (uint32_t)(H - 1), over.p, ocnt.p);
    RAMA_LAUNCH_CHECK();
    ctx.launches++;
  }
  const int64_t no = read_scalar(ctx, ocnt.p);
  if (getenv("RAMA_SEP_STATS"))
    fprintf(stderr, "[rama] sep bfs: %lld edges, %lld sources, %lld beyond the hashed table\n", (long long)nx,
            (long long)ng, (long long)no);
  if (no == 0) return;
  // dense pass for the sources whose ball outgrew the table: n-sized slices,
  // at most ~16 GB of them
  const int64_t per_warp = 24 * g.n;
  int64_t Wd = std::min<int64_t>((int64_t)num_sms() * 8, no);
  const int64_t budget = std::max<int64_t>(8, ((int64_t)16 << 30) / (per_warp > 0 ? per_warp : 1));
  if (Wd > budget) Wd = budget;
  Wd = (Wd + 7) / 8 * 8;
  Buf<unsigned long long> keys((size_t)Wd * g.n, ctx);
  Buf<int32_t> par((size_t)Wd * g.n, ctx), pos((size_t)Wd * g.n, ctx), queue((size_t)Wd * g.n, ctx),
      depth((size_t)Wd * g.n, ctx);
  keys.fill_bytes(0xff);
  KernelScope ks(ctx.s, "k_sep_bfs", 0.0);
  k_sep_bfs<<<(unsigned)(Wd / 8), 256, 0, ctx.s>>>(gstart.p, ng, nx, over.p, ocnt.p, Qx, NQ, g.u, g.v, ptr, adj, L,
                                                   out.len.p, out.nodes.p, keys.p, par.p, pos.p, queue.p, depth.p,
                                                   g.n);
  RAMA_LAUNCH_CHECK();
  ctx.launches++;
}

// RAMA_SEP_FALLBACK=1 routes every source through the row-intersection
// kernels, =2 every source through the tier-2 tables (tests use them to
// check all executions against the oracle)
static int sep_force_fallback() {
  static const int v = [] {
    const char* e = getenv("RAMA_SEP_FALLBACK");
    return (e && (e[0] == '1' || e[0] == '2')) ? e[0] - '0' : 0;
  }();
  return v;
}

// RAMA_SEP_STATS=1: per call, miss edges by outcome and neighbourhood sizes
__global__ void k_sep_stats(const int32_t* __restrict__ Q2, const int32_t* __restrict__ qa,
                            const int32_t* __restrict__ qb, int64_t n2, const int32_t* __restrict__ ptr,
                            const int32_t* __restrict__ len, unsigned long long* st) {
  GRID_STRIDE(i, n2) {
    int32_t l = len[Q2[i]];
    atomicAdd(st + (l == 4 ? 1 : l == 5 ? 2 : 0), 1ULL);
    atomicAdd(st + 3, (unsigned long long)(ptr[qa[i] + 1] - ptr[qa[i]]));
    atomicAdd(st + 4, (unsigned long long)(ptr[qb[i] + 1] - ptr[qb[i]]));
  }
}

static void separate_tables(Ctx& ctx, const GraphView& g, int L, CycleRows& out, const PosCSR& csr,
                            const Buf<int32_t>& NQ, int64_t nq, uint8_t* capped);

void separate(Ctx& ctx, const GraphView& g, int L, CycleRows& out) {
  // algorithmic bytes: the graph read once (16 m),
  // the positive CSR written and read once (2 x (4 (n + 1) + 4 arcs)), one
  // cycle row per repulsive edge written (4 + 4 L)
  ProfScope prof(ctx.s, kFamSeparate, 16.0 * (double)g.m + 8.0 * (double)(g.n + 1));
  RAMA_REQUIRE(L >= 3, "max_len must be at least 3");
  Buf<int32_t> NQ, PE;
  int64_t nq = 0, npos = 0;
  partition2(ctx, g.m, NegCost{g.c}, PosCost{g.c}, NQ, PE, nq, npos);  // repulsive and attractive edges, one pass
  prof.add_bytes((4.0 + 4.0 * L) * (double)nq);
  out.rows = nq;
  out.L = L;
  out.len.alloc(nq > 0 ? nq : 1, ctx.s);
  out.nodes.alloc(nq > 0 ? nq * L : 1, ctx.s);
  if (nq == 0) return;
  PosCSR csr;
  positive_csr(ctx, g, PE, npos, csr);
  prof.add_bytes(8.0 * (double)csr.arcs);
  if (csr.arcs == 0) {
    out.len.zero();
    out.nodes.zero();
    return;
  }
  // searches the capped 5-cycle passes truncate are flagged and rerun
  // exactly; the exact pass scans the flags itself (no compaction, no read-back)
  Buf<uint8_t> capped;
  if (L >= 5) capped.alloc(nq, ctx.s);  // zeroed by k_sep3
  separate_tables(ctx, g, L, out, csr, NQ, nq, capped.p);
  if (capped.p) {
    KernelScope ks(ctx.s, "k_sep5_ordered", 0.0);
    const int64_t warps = (nq + 31) / 32;
    const unsigned blocks = (unsigned)std::min<int64_t>((warps + 7) / 8, (int64_t)num_sms() * 16);
    k_sep5_ordered<<<blocks, 256, 0, ctx.s>>>(capped.p, nq, NQ.p, g.u, g.v, csr.ptr.p, csr.adj.p, L, out.len.p,
                                              out.nodes.p);
    RAMA_LAUNCH_CHECK();
    ctx.launches++;
  }
  if (L >= 6) {
    // PD+ and longer: cycles of up to 5 edges came from the passes above --
    // the BFS reaches b at the same level with the same parents whatever L
    // is -- so only the edges without one (both ends on E+) run the exact
    // source-grouped BFS for lengths 6..L
    Buf<uint8_t> deep(nq, ctx);
    RAMA_KERNEL(ctx, k_needs_bfs, nq, out.len.p, nq, NQ.p, g.u, g.v, csr.ptr.p, deep.p);
    Buf<int32_t> Qx;
    const int64_t nx = compact_indices(ctx, deep.p, nq, Qx);
    run_sep_bfs(ctx, g, csr.ptr.p, csr.adj.p, NQ.p, Qx.p, nx, L, out);
  }
}

// triangles, then 4/5-cycles from the source tables / row intersections
static void separate_tables(Ctx& ctx, const GraphView& g, int L, CycleRows& out, const PosCSR& csr,
                            const Buf<int32_t>& NQ, int64_t nq, uint8_t* capped) {
  // triangles: thread per edge, sorted-row intersection
  Buf<uint8_t> miss(nq, ctx);
  Buf<int32_t> cnt(4, ctx);  // G15 | G2 | fall-back | misses (zeroed by k_sep3)
  RAMA_KERNEL(ctx, k_sep3, nq, (const int32_t*)nullptr, nq, NQ.p, g.u, g.v, csr.ptr.p, csr.adj.p, L, out.len.p,
              out.nodes.p, L >= 4 ? miss.p : (uint8_t*)nullptr, capped, cnt.p);
  if (L < 4) return;
  // the edges without a triangle and their sources' group starts stay on
  // the device (counts n2c / ngc): grids are sized by nq, no read-back
  Buf<int32_t> Q2, n2c, gstart, ngc;
  compact_if_dev(ctx, nq, FlagSet{miss.p}, Q2, n2c);
  // 4/5-cycles: source-grouped BFS levels in shared memory
  Buf<uint8_t> head(nq, ctx);
  Buf<int32_t> qa(nq, ctx), qb(nq, ctx);
  RAMA_KERNEL(ctx, k_src_heads, nq, Q2.p, n2c.p, nq, NQ.p, g.u, g.v, head.p, qa.p, qb.p);
  compact_if_dev(ctx, nq, FlagSet{head.p}, gstart, ngc);
  Buf<int32_t> gsrc(nq, ctx);
  RAMA_KERNEL(ctx, k_gather_i32_dev, nq, qa.p, gstart.p, ngc.p, gsrc.p);
  const int64_t n2 = nq, ng = nq;  // upper bounds of both counts (grid sizes, list capacities)
  // overflow lists, appended on the device: tier 1 -> 1.5 -> 2 sources, then
  // the fall-back edges and the 4-cycle misses of the row-intersection pass
  Buf<int32_t> G15(ng, ctx), G2(ng, ctx), FB(n2, ctx), M4(n2, ctx);
  static const int64_t cap = [] {  // RAMA_SEP_BLOCKS overrides the grid cap (tests)
    const char* e = getenv("RAMA_SEP_BLOCKS");
    return e ? (int64_t)atoll(e) : (int64_t)148 * 12 * 8;  // 8 waves of 12 CTAs per SM
  }();
  const int force = sep_force_fallback();
  {
    constexpr int kPer = kSrcThreads1 / SrcTier1::kGrp;
    int64_t blocks = std::min<int64_t>((ng + kPer - 1) / kPer, cap);
    if (trace_print()) fprintf(stderr, "[rama] k_sep_src groups=%lld\n", (long long)ng);
    // algorithmic bytes: the positive CSR once, the miss list and its
    // edges' endpoints, the cycle rows written
    // (the miss count is on the device: profiled runs read it for the bytes)
    const double n2_alg = prof_enabled() ? (double)read_scalar(ctx, n2c.p) : 0.0;
    KernelScope ks(ctx.s, "k_sep_src",
                   4.0 * (double)(g.n + 1) + 4.0 * (double)csr.arcs + (16.0 + 4.0 * L) * n2_alg);
    k_sep_src<SrcTier1, kSrcThreads1, 12, false><<<(unsigned)blocks, kSrcThreads1, 0, ctx.s>>>(
        gstart.p, gsrc.p, (const int32_t*)nullptr, -1, (const int32_t*)nullptr, ngc.p, n2c.p, Q2.p, qb.p, csr.ptr.p,
        csr.adj.p, L, out.len.p, out.nodes.p, G15.p, cnt.p, (int32_t*)nullptr, (int32_t*)nullptr, force ? 1 : 0,
        capped);
    RAMA_LAUNCH_CHECK();
    ctx.launches++;
  }
  // sources too large for tier 1: 8 lanes with a 128-entry table, then a warp
  // each with 4x/16x tables (grids of one wave: the lists are short or empty)
  const unsigned wave = (unsigned)num_sms() * 12;
  {
    KernelScope ks(ctx.s, "k_sep_src_mid", 0.0);
    k_sep_src<SrcTier15, kSrcThreads1, 12, true><<<wave, kSrcThreads1, 0, ctx.s>>>(
        gstart.p, gsrc.p, G15.p, 0, cnt.p, ngc.p, n2c.p, Q2.p, qb.p, csr.ptr.p, csr.adj.p, L, out.len.p, out.nodes.p,
        G2.p, cnt.p + 1, (int32_t*)nullptr, (int32_t*)nullptr, force ? 1 : 0, capped);
    RAMA_LAUNCH_CHECK();
    ctx.launches++;
  }
  {
    KernelScope ks(ctx.s, "k_sep_src_wide", 0.0);
    k_sep_src<SrcTier2, kSrcThreads2, 6, true><<<(unsigned)num_sms() * 6, kSrcThreads2, 0, ctx.s>>>(
        gstart.p, gsrc.p, G2.p, 0, cnt.p + 1, ngc.p, n2c.p, Q2.p, qb.p, csr.ptr.p, csr.adj.p, L, out.len.p, out.nodes.p,
        (int32_t*)nullptr, (int32_t*)nullptr, FB.p, cnt.p + 2, force == 1 ? 1 : 0, capped);
    RAMA_LAUNCH_CHECK();
    ctx.launches++;
  }
  if (getenv("RAMA_SEP_STATS")) {
    Buf<unsigned long long> st(5, ctx);
    st.zero();
    const int64_t n2 = read_scalar(ctx, n2c.p), ng = read_scalar(ctx, ngc.p);
    RAMA_KERNEL(ctx, k_sep_stats, n2, Q2.p, qa.p, qb.p, n2, csr.ptr.p, out.len.p, st.p);
    unsigned long long h[5];
    int32_t nf = 0;
    RAMA_CUDA(cudaMemcpy(h, st.p, sizeof(h), cudaMemcpyDeviceToHost));
    RAMA_CUDA(cudaMemcpy(&nf, cnt.p + 2, sizeof(nf), cudaMemcpyDeviceToHost));
    fprintf(stderr, "[rama] sep n=%lld m=%lld arcs+=%lld nq=%lld n2=%lld sources=%lld fallback=%d | none %llu c4 %llu c5 %llu (before the fall-back) | avg deg+ a %.2f b %.2f\n",
            (long long)g.n, (long long)g.m, (long long)csr.arcs, (long long)nq, (long long)n2, (long long)ng,
            nf, h[0], h[1], h[2], (double)h[3] / n2, (double)h[4] / n2);
  }
  // sources that did not fit the tables: sorted-row intersections over the
  // device lists (4-cycles, then 5-cycles for the misses)
  RAMA_KERNEL(ctx, k_sep4, n2 * kSepLanes, FB.p, cnt.p + 2, NQ.p, g.u, g.v, csr.ptr.p, csr.adj.p, L, out.len.p,
              out.nodes.p, L >= 5 ? M4.p : (int32_t*)nullptr, cnt.p + 3);
  if (L < 5) return;
  RAMA_KERNEL(ctx, k_sep5, n2 * kSepLanes, M4.p, cnt.p + 3, NQ.p, g.u, g.v, csr.ptr.p, csr.adj.p, L, out.len.p,
              out.nodes.p, capped);
}

// --------------------------------------------------------- triangulation

// per cycle row: triplets (high word) and chords (low word) of its fan, one
// 64-bit value so one scan gives both offsets (neither sum reaches 2^32);
// entry `rows` is 0, so the scan's last entry is both totals
__global__ void k_fan_counts(const int32_t* __restrict__ len, int64_t rows, uint64_t* __restrict__ cnt) {
  GRID_STRIDE(r, rows + 1) {
    const int32_t l = r < rows ? len[r] : 0;
    const uint64_t nt = l >= 3 ? (uint64_t)(l - 2) : 0, nc = l >= 4 ? (uint64_t)(l - 3) : 0;
    cnt[r] = (nt << 32) | nc;
  }
}

// _fan_arrays (dual.py:228-252): triplets {v0, v_j, v_j+1} and chords (v0, v_j)
__global__ void k_fan_emit(const int32_t* __restrict__ len, const int32_t* __restrict__ nodes, int64_t rows, int L,
                           const uint64_t* __restrict__ off,
                           int32_t* __restrict__ trow, uint64_t* __restrict__ tkey, int32_t* __restrict__ crow,
                           uint64_t* __restrict__ ckey, uint64_t ctag) {
  GRID_STRIDE(r, rows) {
    int32_t l = len[r];
    if (l < 3) continue;
    const int32_t* row = nodes + r * (int64_t)L;
    int32_t v0 = row[0];
    const uint64_t o = off[r];
    int32_t t = (int32_t)(o >> 32);
    for (int j = 1; j < l - 1; j++) {
      int32_t a = v0, b = row[j], c = row[j + 1], s;
      if (a > b) { s = a; a = b; b = s; }
      if (b > c) { s = b; b = c; c = s; }
      if (a > b) { s = a; a = b; b = s; }
      trow[t] = a;
      tkey[t] = ((uint64_t)(uint32_t)b << 32) | (uint64_t)(uint32_t)c;
      t++;
    }
    int32_t h = (int32_t)(uint32_t)o;
    for (int j = 2; j < l - 1; j++) {
      int32_t a = v0 < row[j] ? v0 : row[j];
      int32_t b = v0 < row[j] ? row[j] : v0;
      crow[h] = a;
      ckey[h] = ctag | (uint64_t)(uint32_t)b;
      h++;
    }
  }
}

__device__ __forceinline__ int32_t find_in_row(const int32_t* __restrict__ rptr, const int32_t* __restrict__ ev,
                                               int32_t a, int32_t b) {
  int32_t lo = rptr[a], hi = rptr[a + 1];
  while (lo < hi) {
    int32_t mid = (lo + hi) >> 1;
    int32_t x = ev[mid];
    if (x < b) lo = mid + 1;
    else if (x > b) hi = mid;
    else return mid;
  }
  return -1;
}

// triangulate's combined sort: chords carry kChordTag in the key (after the
// row's triplets), triplets (b << 32 | c) with b < 2^31
constexpr uint64_t kChordTag = 1ull << 63;

// kind of each sorted item: 1 first of a run of equal triplets, 2 first of
// a run of equal chords that is not an edge of g, 0 otherwise (one thread
// per item, so the graph-row searches overlap at full occupancy)
__global__ void k_tri_kinds(const int32_t* __restrict__ row, const uint64_t* __restrict__ key, int64_t N,
                            const int32_t* __restrict__ rptr, const int32_t* __restrict__ gv,
                            uint8_t* __restrict__ kind) {
  GRID_STRIDE(p, N) {
    const uint64_t k = key[p];
    const int32_t r = row[p];
    uint8_t out = 0;
    if (p == 0 || row[p - 1] != r || key[p - 1] != k)
      out = !(k & kChordTag) ? 1 : (find_in_row(rptr, gv, r, (int32_t)(uint32_t)k) < 0 ? 2 : 0);
    kind[p] = out;
  }
}
struct KindIs {
  const uint8_t* kind;
  uint8_t want;
  __device__ __forceinline__ bool operator()(int32_t p) const { return kind[p] == want; }
};

// unique chords that are not already edges of g (extend_separation)
__global__ void k_chord_new(const int32_t* __restrict__ heads, int64_t nh, const int32_t* __restrict__ row,
                            const uint64_t* __restrict__ key, const int32_t* __restrict__ rptr,
                            const int32_t* __restrict__ gv, uint8_t* __restrict__ is_new) {
  GRID_STRIDE(i, nh) {
    int32_t p = heads[i];
    is_new[i] = find_in_row(rptr, gv, row[p], (int32_t)key[p]) < 0;
  }
}

__global__ void k_chord_out(const int32_t* __restrict__ sel, int64_t C, const int32_t* __restrict__ heads,
                            const int32_t* __restrict__ row, const uint64_t* __restrict__ key, int64_t m,
                            int32_t* __restrict__ eu, int32_t* __restrict__ ev, double* __restrict__ base,
                            uint64_t* __restrict__ ckeys) {
  GRID_STRIDE(i, C) {
    int32_t p = heads[sel ? sel[i] : (int32_t)i];
    int32_t a = row[p], b = (int32_t)key[p];
    eu[m + i] = a;
    ev[m + i] = b;
    base[m + i] = 0.0;
    ckeys[i] = ((uint64_t)(uint32_t)a << 32) | (uint64_t)(uint32_t)b;
  }
}

__global__ void k_tri_out(const int32_t* __restrict__ heads, int64_t T, const int32_t* __restrict__ row,
                          const uint64_t* __restrict__ key, int32_t* __restrict__ tn) {
  GRID_STRIDE(t, T) {
    int32_t p = heads[t];
    tn[3 * t] = row[p];
    tn[3 * t + 1] = (int32_t)(key[p] >> 32);
    tn[3 * t + 2] = (int32_t)(uint32_t)key[p];
  }
}

__device__ __forceinline__ int32_t edge_handle(const int32_t* rptr, const int32_t* gv, const int32_t* crptr,
                                               const int32_t* cv, int64_t m, int32_t a, int32_t b) {
  int32_t e = find_in_row(rptr, gv, a, b);
  if (e >= 0) return e;
  return (int32_t)(m + find_in_row(crptr, cv, a, b));  // a chord: present by construction
}

__global__ void k_tri_handles(const int32_t* __restrict__ tn, int64_t T, const int32_t* __restrict__ rptr,
                              const int32_t* __restrict__ gv, const int32_t* __restrict__ crptr,
                              const int32_t* __restrict__ cv, int64_t m, int32_t* __restrict__ te) {
  GRID_STRIDE(t, T) {
    int32_t i = tn[3 * t], j = tn[3 * t + 1], k = tn[3 * t + 2];
    te[3 * t] = edge_handle(rptr, gv, crptr, cv, m, i, j);
    te[3 * t + 1] = edge_handle(rptr, gv, crptr, cv, m, i, k);
    te[3 * t + 2] = edge_handle(rptr, gv, crptr, cv, m, j, k);
  }
}

// k_tri_out + k_tri_handles in one pass over the kept triplets
__global__ void k_tri_out_handles(const int32_t* __restrict__ heads, int64_t T, const int32_t* __restrict__ row,
                                  const uint64_t* __restrict__ key, const int32_t* __restrict__ rptr,
                                  const int32_t* __restrict__ gv, const int32_t* __restrict__ crptr,
                                  const int32_t* __restrict__ cv, int64_t m, int32_t* __restrict__ tn,
                                  int32_t* __restrict__ te, double* __restrict__ lam) {
  GRID_STRIDE(t, T) {
    lam[3 * t] = 0.0;  // the multipliers start at zero (no memset)
    lam[3 * t + 1] = 0.0;
    lam[3 * t + 2] = 0.0;
    const int32_t p = heads[t];
    const uint64_t k = key[p];
    const int32_t i = row[p], j = (int32_t)(k >> 32), l = (int32_t)(uint32_t)k;
    tn[3 * t] = i;
    tn[3 * t + 1] = j;
    tn[3 * t + 2] = l;
    // the three edges' searches in the graph's rows run interleaved (ILP);
    // an edge not in g is a chord (present by construction)
    const int32_t ra[3] = {i, i, j}, rb[3] = {j, l, l};
    int32_t lo[3], hi[3], end[3];
#pragma unroll
    for (int q = 0; q < 3; q++) {
      lo[q] = rptr[ra[q]];
      end[q] = hi[q] = rptr[ra[q] + 1];
    }
    while (lo[0] < hi[0] || lo[1] < hi[1] || lo[2] < hi[2]) {
#pragma unroll
      for (int q = 0; q < 3; q++) {
        if (lo[q] < hi[q]) {
          const int32_t mid = (lo[q] + hi[q]) >> 1;
          if (gv[mid] < rb[q]) lo[q] = mid + 1;
          else hi[q] = mid;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 3; q++)
      te[3 * t + q] = lo[q] < end[q] && gv[lo[q]] == rb[q] ? lo[q]
                                                          : (int32_t)(m + find_in_row(crptr, cv, ra[q], rb[q]));
  }
}

__global__ void k_slot_items(const int32_t* __restrict__ te, int64_t S, uint64_t* __restrict__ key) {
  GRID_STRIDE(s, S) key[s] = (uint64_t)s;
}

// edge -> slot lists without a general sort: count the slots per edge (the
// run-aggregated atomics also hand every slot its offset in the row), scan,
// scatter the slot ids, then order each row -- rows hold 1-3 slots on grids,
// so an insertion sort per row in registers replaces the bucket sort's
// 16-byte items, key arrays and ranking.  If any row exceeds kSmallRow the
// bucket sort (with its hub paths) builds the lists instead.

__global__ void k_slot_count(const int32_t* __restrict__ te, int64_t S, int32_t* __restrict__ cov,
                             int32_t* __restrict__ off, int32_t* __restrict__ long_flag) {
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x - lane; i0 < S;
       i0 += (int64_t)gridDim.x * blockDim.x) {  // warp-uniform trip count
    const int64_t s = i0 + lane;
    const int32_t e = s < S ? te[s] : -1;
    const int32_t o = run_atomic_add(cov, e, 1);
    if (e >= 0) {
      off[s] = o;
      if (o >= kSmallRow) *long_flag = 1;
    }
  }
}

__global__ void k_slot_scatter(const int32_t* __restrict__ te, int64_t S, const int32_t* __restrict__ ptr,
                               const int32_t* __restrict__ off, int32_t* __restrict__ slots) {
  GRID_STRIDE(s, S) slots[ptr[te[s]] + off[s]] = (int32_t)s;
}

void build_slot_lists(Ctx& ctx, DualState& st) {
  int64_t S = 3 * st.T;
  st.coverage.alloc(st.m_aug + 1, ctx.s);  // coverage | long-row flag: one memset
  st.slots.alloc(S > 0 ? S : 1, ctx.s);
  st.long_e.release();
  st.n_long.release();
  st.coverage.zero();
  {
    Buf<int32_t> off(S > 0 ? S : 1, ctx);
    int32_t* flag = st.coverage.p + st.m_aug;
    RAMA_KERNEL(ctx, k_slot_count, S, st.tri_edges.p, S, st.coverage.p, off.p, flag);
    st.slot_ptr.alloc(st.m_aug + 1, ctx.s);
    exclusive_scan(ctx, st.coverage.p, st.slot_ptr.p, st.m_aug, false);
    if (read_scalar(ctx, flag) == 0) {
      RAMA_KERNEL(ctx, k_slot_scatter, S, st.tri_edges.p, S, st.slot_ptr.p, off.p, st.slots.p);
      RAMA_KERNEL(ctx, k_rowsort_i32, st.m_aug, st.slot_ptr.p, st.m_aug, st.slots.p);
      return;
    }
  }
  // rows beyond kSmallRow (power-law hubs): the bucket sort
  Buf<uint64_t> key(S > 0 ? S : 1, ctx);
  RAMA_KERNEL(ctx, k_slot_items, S, st.tri_edges.p, S, key.p);
  BucketSorted bs;
  bucket_sort(ctx, st.m_aug, S, st.tri_edges.p, key.p, bs, false);
  st.slot_ptr = std::move(bs.row_ptr);
  RAMA_KERNEL(ctx, k_key_lo, S, bs.key.p, S, st.slots.p);
  // hub slot lists (only when the sort saw rows > 256: grids never have them)
  if (bs.big_rows > 0) compact_if_dev(ctx, st.m_aug, LongCov{st.slot_ptr.p}, st.long_e, st.n_long);
}

void triangulate(Ctx& ctx, const GraphView& g, const CycleRows& cyc, DualState& st, Graph* steal) {
  ProfScope prof(ctx.s, kFamTriangulate);
  int64_t rows = cyc.rows, m = g.m, n = g.n;
  st.n = n;
  st.m_orig = m;
  Buf<uint64_t> fcnt(rows + 1, ctx), foff(rows + 1, ctx);
  RAMA_KERNEL(ctx, k_fan_counts, rows + 1, cyc.len.p, rows, fcnt.p);
  exclusive_scan64(ctx, (const int64_t*)fcnt.p, (int64_t*)foff.p, rows + 1);
  int64_t traw = 0, craw = 0;
  {
    uint64_t tot;
    memcpy(&tot, fetch(ctx, {{foff.p + rows, 8}}), 8);
    traw = (int64_t)(tot >> 32);
    craw = (int64_t)(uint32_t)tot;
  }
  // triplets and chords in one list, sorted once (chords tagged after each
  // row's triplets); one partition then keeps the first triplet of each run
  // and the first chord of each run that is not an edge of g, both in
  // sorted order, with one read-back for both counts
  const int64_t N = traw + craw;
  Buf<int32_t> irow(N > 0 ? N : 1, ctx);
  Buf<uint64_t> ikey(N > 0 ? N : 1, ctx);
  RAMA_KERNEL(ctx, k_fan_emit, rows, cyc.len.p, cyc.nodes.p, rows, cyc.L, foff.p, irow.p, ikey.p,
              irow.p + traw, ikey.p + traw, kChordTag);

  st.orig_ptr.alloc(n + 1, ctx.s);
  int32_t* rptr_p = st.orig_ptr.p;
  row_ptr_from_sorted(ctx, g.u, m, n, rptr_p);
  int64_t C = 0, T = 0;
  Buf<uint64_t> ckeys(1, ctx);
  const size_t cap = (size_t)(m + craw > 0 ? m + craw : 1);
  if (steal && steal->u.p == g.u && steal->v.p == g.v && steal->c.p == g.c && steal->u.n >= cap &&
      steal->v.n >= cap && steal->c.n >= cap) {
    // the caller's graph has room for the chords after its edges (a
    // contraction's output is sized by its input): take its buffers
    // instead of copying the m edges (g's pointers stay valid: same memory)
    st.eu = std::move(steal->u);
    st.ev = std::move(steal->v);
    st.base = std::move(steal->c);
  } else {
    st.eu.alloc(cap, ctx.s);
    st.ev.alloc(cap, ctx.s);
    st.base.alloc(cap, ctx.s);
    copy_d2d(ctx, st.eu.p, g.u, m);
    copy_d2d(ctx, st.ev.p, g.v, m);
    copy_d2d(ctx, st.base.p, g.c, m);
  }
  BucketSorted bs;
  Buf<int32_t> hc, ht;
  if (N > 0) {
    bucket_sort(ctx, n, N, irow.p, ikey.p, bs, true);
    Buf<uint8_t> kind(bs.total > 0 ? bs.total : 1, ctx);
    RAMA_KERNEL(ctx, k_tri_kinds, bs.total, bs.row.p, bs.key.p, bs.total, rptr_p, g.v, kind.p);
    partition2(ctx, bs.total, KindIs{kind.p, 2}, KindIs{kind.p, 1}, hc, ht, C, T);
  }
  irow.release();
  ikey.release();
  if (C > 0) {
    ckeys.alloc(C, ctx.s);
    RAMA_KERNEL(ctx, k_chord_out, C, (const int32_t*)nullptr, C, hc.p, bs.row.p, bs.key.p, m, st.eu.p, st.ev.p,
                st.base.p, ckeys.p);
  }
  st.m_aug = m + C;
  st.chords_sorted = true;
  st.chord_ptr.alloc(n + 1, ctx.s);
  row_ptr_from_sorted(ctx, st.eu.p + m, C, n, st.chord_ptr.p);

  // triplets: handles
  st.lam.alloc(T > 0 ? 3 * T : 1, ctx.s);
  if (T > 0) {
    st.tri_nodes.alloc(3 * T, ctx.s);
    st.tri_edges.alloc(3 * T, ctx.s);
    RAMA_KERNEL(ctx, k_tri_out_handles, T, ht.p, T, bs.row.p, bs.key.p, rptr_p, g.v, st.chord_ptr.p, st.ev.p + m, m,
                st.tri_nodes.p, st.tri_edges.p, st.lam.p);
  } else {
    st.tri_nodes.alloc(1, ctx.s);
    st.tri_edges.alloc(1, ctx.s);
    st.lam.zero();
  }
  st.T = T;
  build_slot_lists(ctx, st);
  // algorithmic bytes: cycle rows read (4 + 4 L), the
  // originals' (u, v) read for the handles (8 m), augmented edges written
  // (eu, ev, base, coverage, slot pointer: 24 m_aug), triplets written
  // (nodes 12, handles 12, lambda 24, slot list 12: 60 T)
  prof.add_bytes((4.0 + 4.0 * cyc.L) * (double)rows + 8.0 * (double)m + 24.0 * (double)st.m_aug +
                 60.0 * (double)st.T);
}


// ------------------------------------------------------ extend_separation
//
// dual.py:414-474 (mode D, separation_rounds > 1): separate on the current
// reparametrized graph, append the new chords (base 0) and the new
// triplets (zero multipliers) in the reference's order -- chords and
// triplets sorted lexicographically, existing triplets skipped.

__global__ void k_ext_tri_keys(const int32_t* __restrict__ tn, int64_t T, int32_t* __restrict__ row,
                               uint64_t* __restrict__ key) {
  GRID_STRIDE(t, T) {
    row[t] = tn[3 * t];
    key[t] = ((uint64_t)(uint32_t)tn[3 * t + 1] << 32) | (uint64_t)(uint32_t)tn[3 * t + 2];
  }
}

// new (deduped) triplet at sorted slot hp[i] is kept unless present in the
// existing triplets (bucket-sorted by row i with key (j << 32 | k))
__global__ void k_ext_tri_new(const int32_t* __restrict__ hp, int64_t nh, const int32_t* __restrict__ row,
                              const uint64_t* __restrict__ key, const int32_t* __restrict__ eptr,
                              const uint64_t* __restrict__ ekey, int64_t T, uint8_t* __restrict__ keep) {
  GRID_STRIDE(i, nh) {
    int32_t p = hp[i];
    int32_t r = row[p];
    uint64_t k = key[p];
    bool found = false;
    if (T > 0) {
      int32_t lo = eptr[r], hi = eptr[r + 1];
      while (lo < hi) {
        int32_t mid = (lo + hi) >> 1;
        uint64_t x = ekey[mid];
        if (x < k) lo = mid + 1;
        else if (x > k) hi = mid;
        else { found = true; break; }
      }
    }
    keep[i] = !found;
  }
}

__global__ void k_ext_tri_out(const int32_t* __restrict__ sel, int64_t k, const int32_t* __restrict__ hp,
                              const int32_t* __restrict__ row, const uint64_t* __restrict__ key, int64_t T0,
                              int32_t* __restrict__ tn) {
  GRID_STRIDE(i, k) {
    int32_t p = hp[sel[i]];
    int64_t t = T0 + i;
    tn[3 * t] = row[p];
    tn[3 * t + 1] = (int32_t)(key[p] >> 32);
    tn[3 * t + 2] = (int32_t)(uint32_t)key[p];
  }
}

__global__ void k_ext_edge_keys(const int32_t* __restrict__ eu, const int32_t* __restrict__ ev, int64_t m,
                                int32_t* __restrict__ row, uint64_t* __restrict__ key) {
  GRID_STRIDE(i, m) {
    row[i] = eu[i];
    key[i] = ((uint64_t)(uint32_t)ev[i] << 32) | (uint64_t)i;
  }
}

__device__ __forceinline__ int32_t ext_handle(const int32_t* eptr, const uint64_t* ekey, int32_t a, int32_t b) {
  uint64_t k = (uint64_t)(uint32_t)b << 32;
  int32_t lo = eptr[a], hi = eptr[a + 1];
  while (lo < hi) {
    int32_t mid = (lo + hi) >> 1;
    if (ekey[mid] < k) lo = mid + 1; else hi = mid;
  }
  return (int32_t)(uint32_t)ekey[lo];  // present by construction
}

__global__ void k_ext_handles(const int32_t* __restrict__ tn, int64_t T0, int64_t k, const int32_t* __restrict__ eptr,
                              const uint64_t* __restrict__ ekey, int32_t* __restrict__ te) {
  GRID_STRIDE(i, k) {
    int64_t t = T0 + i;
    int32_t a = tn[3 * t], b = tn[3 * t + 1], c = tn[3 * t + 2];
    te[3 * t] = ext_handle(eptr, ekey, a, b);
    te[3 * t + 1] = ext_handle(eptr, ekey, a, c);
    te[3 * t + 2] = ext_handle(eptr, ekey, b, c);
  }
}

template <class T>
static void grow(Ctx& ctx, Buf<T>& b, int64_t old_n, int64_t new_n) {
  Buf<T> nb(new_n > 0 ? new_n : 1, ctx);
  copy_d2d(ctx, nb.p, b.p, old_n);
  b = std::move(nb);
}

int64_t extend_separation(Ctx& ctx, DualState& st, int L) {
  ProfScope prof(ctx.s, kFamTriangulate);
  const int64_t n = st.n;
  Graph rep = reparametrized_graph(ctx, st);  // canonical merge of the augmented edges, c^lambda
  CycleRows cyc;
  separate(ctx, rep.view(), L, cyc);
  const int64_t rows = cyc.rows;
  if (rows == 0) return 0;
  Buf<uint64_t> fcnt(rows + 1, ctx), foff(rows + 1, ctx);
  RAMA_KERNEL(ctx, k_fan_counts, rows + 1, cyc.len.p, rows, fcnt.p);
  exclusive_scan64(ctx, (const int64_t*)fcnt.p, (int64_t*)foff.p, rows + 1);
  const uint64_t tot = read_scalar(ctx, foff.p + rows);
  const int64_t traw = (int64_t)(tot >> 32), craw = (int64_t)(uint32_t)tot;
  if (traw == 0) return 0;  // no cycle: nothing changes (dual.py:428-429)
  Buf<int32_t> trow(traw, ctx), crow(craw > 0 ? craw : 1, ctx);
  Buf<uint64_t> tkey(traw, ctx), ckey(craw > 0 ? craw : 1, ctx);
  RAMA_KERNEL(ctx, k_fan_emit, rows, cyc.len.p, cyc.nodes.p, rows, cyc.L, foff.p, trow.p, tkey.p, crow.p,
              ckey.p, 0ull);
  // new chords (sorted, unique, not yet augmented edges) join at base 0
  int64_t C = 0;
  Buf<int32_t> sel_c, hp_c;
  BucketSorted cs;
  if (craw > 0) {
    Buf<int32_t> rptr(n + 1, ctx);
    row_ptr_from_sorted(ctx, rep.u.p, rep.m, n, rptr.p);
    bucket_sort(ctx, n, craw, crow.p, ckey.p, cs, true);
    int64_t nh = compact_if(ctx, craw, SortedHead{cs.row.p, cs.key.p}, hp_c);
    Buf<uint8_t> isnew(nh > 0 ? nh : 1, ctx);
    RAMA_KERNEL(ctx, k_chord_new, nh, hp_c.p, nh, cs.row.p, cs.key.p, rptr.p, rep.v.p, isnew.p);
    C = compact_indices(ctx, isnew.p, nh, sel_c);
  }
  const int64_t m0 = st.m_aug;
  if (C > 0) {
    grow(ctx, st.eu, m0, m0 + C);
    grow(ctx, st.ev, m0, m0 + C);
    grow(ctx, st.base, m0, m0 + C);
    Buf<uint64_t> unused(C, ctx);
    RAMA_KERNEL(ctx, k_chord_out, C, sel_c.p, C, hp_c.p, cs.row.p, cs.key.p, m0, st.eu.p, st.ev.p, st.base.p,
                unused.p);
    st.m_aug = m0 + C;
    if (m0 > st.m_orig) {
      st.chords_sorted = false;
    } else if (st.chords_sorted && st.chord_ptr.p) {  // the new chords are the only run: refresh its rows
      row_ptr_from_sorted(ctx, st.eu.p + st.m_orig, st.m_aug - st.m_orig, n, st.chord_ptr.p);
    }
  }
  // new triplets: fan dedupe, then drop those already present
  BucketSorted ts;
  bucket_sort(ctx, n, traw, trow.p, tkey.p, ts, true);
  Buf<int32_t> hp;
  int64_t nh = compact_if(ctx, traw, SortedHead{ts.row.p, ts.key.p}, hp);
  const int64_t T0 = st.T;
  BucketSorted es;
  Buf<int32_t> erow(T0 > 0 ? T0 : 1, ctx);
  Buf<uint64_t> ekey(T0 > 0 ? T0 : 1, ctx);
  if (T0 > 0) {
    RAMA_KERNEL(ctx, k_ext_tri_keys, T0, st.tri_nodes.p, T0, erow.p, ekey.p);
    bucket_sort(ctx, n, T0, erow.p, ekey.p, es, false);
  }
  Buf<uint8_t> keep(nh > 0 ? nh : 1, ctx);
  RAMA_KERNEL(ctx, k_ext_tri_new, nh, hp.p, nh, ts.row.p, ts.key.p, T0 > 0 ? es.row_ptr.p : (const int32_t*)nullptr,
              T0 > 0 ? es.key.p : (const uint64_t*)nullptr, T0, keep.p);
  Buf<int32_t> sel;
  const int64_t k = compact_indices(ctx, keep.p, nh, sel);
  if (k > 0) {
    grow(ctx, st.tri_nodes, 3 * T0, 3 * (T0 + k));
    grow(ctx, st.tri_edges, 3 * T0, 3 * (T0 + k));
    Buf<double> lam(3 * (T0 + k), ctx);
    lam.zero();
    copy_d2d(ctx, lam.p, st.lam.p, 3 * T0);
    st.lam = std::move(lam);
    RAMA_KERNEL(ctx, k_ext_tri_out, k, sel.p, k, hp.p, ts.row.p, ts.key.p, T0, st.tri_nodes.p);
    // handles into the augmented edge list (originals, earlier chords, new chords)
    Buf<int32_t> arow(st.m_aug, ctx);
    Buf<uint64_t> akey(st.m_aug, ctx);
    RAMA_KERNEL(ctx, k_ext_edge_keys, st.m_aug, st.eu.p, st.ev.p, st.m_aug, arow.p, akey.p);
    BucketSorted as;
    bucket_sort(ctx, n, st.m_aug, arow.p, akey.p, as, false);
    RAMA_KERNEL(ctx, k_ext_handles, k, st.tri_nodes.p, T0, k, as.row_ptr.p, as.key.p, st.tri_edges.p);
    st.T = T0 + k;
  }
  build_slot_lists(ctx, st);  // coverage over the grown edge list
  return k;
}

// ------------------------------------------------------ message passing

__device__ __forceinline__ double mn2(double a, double b) { return a < b ? a : b; }  // np.minimum

__device__ __forceinline__ double edge_sum(const int32_t* __restrict__ ptr, const int32_t* __restrict__ slots,
                                           const double* __restrict__ lam, int64_t e, int32_t* cov) {
  int32_t b = ptr[e], en = ptr[e + 1];
  double acc = 0.0;
  for (int32_t p = b; p < en; p++) acc = __dadd_rn(acc, lam[slots[p]]);
  *cov = en - b;
  return acc;
}

// Edges covered by more than kLongCov slots (power-law hubs: C4 round 1 has
// edges covered ~1e5 times) would serialise one thread over a long chain of
// dependent gathers.  Their sum must stay sequential in slot order
// (np.bincount), so a warp gathers 32 multipliers at a time -- the next
// chunk's loads in flight while the current one is folded -- and every lane
// folds them in order from registers: the critical path is one fp64 add per
// slot instead of a dependent load.
__device__ __forceinline__ double warp_edge_sum(const int32_t* __restrict__ ptr, const int32_t* __restrict__ slots,
                                                const double* __restrict__ lam, int32_t e, int32_t& cov) {
  const int lane = threadIdx.x & 31;
  const int32_t b = ptr[e], en = ptr[e + 1];
  cov = en - b;
  double acc = 0.0;
  double x = b + lane < en ? lam[slots[b + lane]] : 0.0;
  for (int32_t p0 = b; p0 < en; p0 += 32) {
    const int32_t pn = p0 + 32 + lane;
    const double xn = pn < en ? lam[slots[pn]] : 0.0;  // next chunk in flight
    const int32_t cnt = min(32, en - p0);
    for (int32_t j = 0; j < cnt; j++) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, x, j));
    x = xn;
  }
  return acc;
}

__global__ void k_mp_edge(int64_t m, const double* __restrict__ base, const int32_t* __restrict__ ptr,
                          const int32_t* __restrict__ slots, const double* __restrict__ lam,
                          double* __restrict__ delta, int32_t long_cov) {
  GRID_STRIDE(e, m) {
    if (ptr[e + 1] - ptr[e] > long_cov) continue;  // k_mp_edge_long
    int32_t cov;
    double acc = edge_sum(ptr, slots, lam, e, &cov);
    if (cov == 0) continue;
    double cl = __dadd_rn(base[e], acc);
    delta[e] = __ddiv_rn(cl, (double)cov);
  }
}

__global__ void k_mp_edge_long(const int32_t* __restrict__ list, const int32_t* __restrict__ count,
                               const double* __restrict__ base, const int32_t* __restrict__ ptr,
                               const int32_t* __restrict__ slots, const double* __restrict__ lam,
                               double* __restrict__ delta) {
  const int32_t nl = *count;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < nl; i += W) {
    const int32_t e = list[i];
    int32_t cov;
    const double acc = warp_edge_sum(ptr, slots, lam, e, cov);
    if ((threadIdx.x & 31) == 0) delta[e] = __ddiv_rn(__dadd_rn(base[e], acc), (double)cov);
  }
}

// the same edge pass reached through the slots (late rounds: a few
// triplets over a large graph): the first slot of each covered edge computes it
__global__ void k_mp_edge_by_slot(int64_t S, const int32_t* __restrict__ te, const double* __restrict__ base,
                                  const int32_t* __restrict__ ptr, const int32_t* __restrict__ slots,
                                  const double* __restrict__ lam, double* __restrict__ delta, int32_t long_cov) {
  GRID_STRIDE(s, S) {
    const int32_t e = te[s];
    const int32_t b = ptr[e];
    if (slots[b] != (int32_t)s || ptr[e + 1] - b > long_cov) continue;
    int32_t cov;
    const double acc = edge_sum(ptr, slots, lam, e, &cov);
    delta[e] = __ddiv_rn(__dadd_rn(base[e], acc), (double)cov);
  }
}

// the edge phase: short lists a thread per edge (or per first slot when the
// slots are far fewer than the edges), hub lists a warp per edge
static void edge_phase(Ctx& ctx, const DualState& st, double* delta) {
  const int32_t long_cov = st.n_long.p ? kLongCov : INT32_MAX;
  if (3 * st.T < st.m_aug) {
    RAMA_KERNEL(ctx, k_mp_edge_by_slot, 3 * st.T, 3 * st.T, st.tri_edges.p, st.base.p, st.slot_ptr.p, st.slots.p,
                st.lam.p, delta, long_cov);
  } else {
    RAMA_KERNEL(ctx, k_mp_edge, st.m_aug, st.m_aug, st.base.p, st.slot_ptr.p, st.slots.p, st.lam.p, delta,
                long_cov);
  }
  if (st.n_long.p) {
    KernelScope ks(ctx.s, "k_mp_edge_long", 0.0);
    k_mp_edge_long<<<(unsigned)num_sms() * 8, kBlock, 0, ctx.s>>>(st.long_e.p, st.n_long.p, st.base.p,
                                                                  st.slot_ptr.p, st.slots.p, st.lam.p, delta);
    RAMA_LAUNCH_CHECK();
    ctx.launches++;
  }
}

__device__ __forceinline__ double slot_marginal(double l0, double l1, double l2, int slot) {
  double c110 = -__dadd_rn(l0, l1);
  double c101 = -__dadd_rn(l0, l2);
  double c011 = -__dadd_rn(l1, l2);
  double c111 = -__dadd_rn(__dadd_rn(l0, l1), l2);
  if (slot == 0) return __dsub_rn(mn2(mn2(c110, c101), c111), mn2(0.0, c011));
  if (slot == 1) return __dsub_rn(mn2(mn2(c110, c011), c111), mn2(0.0, c101));
  return __dsub_rn(mn2(mn2(c101, c011), c111), mn2(0.0, c110));
}

__device__ __forceinline__ void triplet_schedule(double& l0, double& l1, double& l2) {
  // _SCHEDULE (dual.py:371): (0,1/3) (1,1/2) (2,1) (0,1/2) (1,1) (0,1)
  l0 = __dadd_rn(l0, __dmul_rn(1.0 / 3.0, slot_marginal(l0, l1, l2, 0)));
  l1 = __dadd_rn(l1, __dmul_rn(0.5, slot_marginal(l0, l1, l2, 1)));
  l2 = __dadd_rn(l2, __dmul_rn(1.0, slot_marginal(l0, l1, l2, 2)));
  l0 = __dadd_rn(l0, __dmul_rn(0.5, slot_marginal(l0, l1, l2, 0)));
  l1 = __dadd_rn(l1, __dmul_rn(1.0, slot_marginal(l0, l1, l2, 1)));
  l0 = __dadd_rn(l0, __dmul_rn(1.0, slot_marginal(l0, l1, l2, 0)));
}

__global__ void k_mp_triplet(int64_t T, const int32_t* __restrict__ te, const double* __restrict__ delta,
                             double* __restrict__ lam, int do_edge, int do_tri) {
  GRID_STRIDE(t, T) {
    double l0 = lam[3 * t], l1 = lam[3 * t + 1], l2 = lam[3 * t + 2];
    if (do_edge) {
      l0 = __dsub_rn(l0, delta[te[3 * t]]);
      l1 = __dsub_rn(l1, delta[te[3 * t + 1]]);
      l2 = __dsub_rn(l2, delta[te[3 * t + 2]]);
    }
    if (do_tri) triplet_schedule(l0, l1, l2);
    lam[3 * t] = l0;
    lam[3 * t + 1] = l1;
    lam[3 * t + 2] = l2;
  }
}

void mp_phases(Ctx& ctx, DualState& st, bool do_edge, bool do_triplet) {
  if (st.T == 0) return;
  Buf<double> delta;
  if (do_edge) {
    delta.alloc(st.m_aug, ctx.s);
    edge_phase(ctx, st, delta.p);
  }
  RAMA_KERNEL(ctx, k_mp_triplet, st.T, st.T, st.tri_edges.p, delta.p, st.lam.p, do_edge ? 1 : 0,
              do_triplet ? 1 : 0);
}

void message_passing(Ctx& ctx, DualState& st, int iters) {
  if (st.T == 0) return;
  // algorithmic bytes per iteration: 132 T + 20 m_aug
  ProfScope prof(ctx.s, kFamMP, (double)iters * (132.0 * (double)st.T + 20.0 * (double)st.m_aug));
  Buf<double> delta(st.m_aug, ctx);
  for (int it = 0; it < iters; it++) {
    prof_set_bytes(20.0 * (double)st.m_aug + 36.0 * (double)st.T);
    edge_phase(ctx, st, delta.p);
    prof_set_bytes(84.0 * (double)st.T);
    RAMA_KERNEL(ctx, k_mp_triplet, st.T, st.T, st.tri_edges.p, delta.p, st.lam.p, 1, 1);
  }
}

// merge position of originals [0, m) and chords [m, m_aug) (both sorted):
// the count of the other list's keys below (a, b) is that list's row start
// plus a search inside its (short) row a
__device__ __forceinline__ int32_t row_lower(const int32_t* ptr, const int32_t* col, int32_t a, int32_t b) {
  int32_t lo = ptr[a], hi = ptr[a + 1];
  while (lo < hi) {
    int32_t mid = (lo + hi) >> 1;
    if (col[mid] < b) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// the reparametrized graph written directly by the bound's edge pass: c^lambda
// of augmented edge e goes to its merged canonical position (k_merge_scatter)
struct MergeOut {
  int32_t* ou = nullptr;
  int32_t* ov = nullptr;
  double* oc = nullptr;
  const int32_t* eu = nullptr;
  const int32_t* ev = nullptr;
  const int32_t* optr = nullptr;
  const int32_t* cptr = nullptr;
  int64_t m = 0;  // originals [0, m), chords after
  __device__ __forceinline__ void put(int64_t i, double x) const {
    const int32_t a = eu[i], b = ev[i];
    const int64_t pos = i < m ? i + row_lower(cptr, ev + m, a, b) : (i - m) + row_lower(optr, ev, a, b);
    ou[pos] = a;
    ov[pos] = b;
    oc[pos] = x;
  }
};

__global__ void k_reparam(int64_t m, const double* __restrict__ base, const int32_t* __restrict__ ptr,
                          const int32_t* __restrict__ slots, const double* __restrict__ lam,
                          double* __restrict__ cl, double* __restrict__ negpart, int32_t long_cov, MergeOut mo) {
  GRID_STRIDE(e, m) {
    if (ptr != nullptr && ptr[e + 1] - ptr[e] > long_cov) continue;  // k_reparam_long
    int32_t cov;
    double acc = (ptr != nullptr) ? edge_sum(ptr, slots, lam, e, &cov) : 0.0;
    double x = __dadd_rn(base[e], acc);
    if (cl) cl[e] = x;
    if (mo.ou) mo.put(e, x);
    if (negpart) negpart[e] = mn2(x, 0.0);
  }
}

__global__ void k_reparam_long(const int32_t* __restrict__ list, const int32_t* __restrict__ count,
                               const double* __restrict__ base, const int32_t* __restrict__ ptr,
                               const int32_t* __restrict__ slots, const double* __restrict__ lam,
                               double* __restrict__ cl, double* __restrict__ negpart, MergeOut mo) {
  const int32_t nl = *count;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < nl; i += W) {
    const int32_t e = list[i];
    int32_t cov;
    const double x = __dadd_rn(base[e], warp_edge_sum(ptr, slots, lam, e, cov));
    if ((threadIdx.x & 31) == 0) {
      if (cl) cl[e] = x;
      if (mo.ou) mo.put(e, x);
      if (negpart) negpart[e] = mn2(x, 0.0);
    }
  }
}

// c^lambda (and its negative part): short slot lists a thread per edge, hub lists a warp per edge
static void reparam_pass(Ctx& ctx, const DualState& st, double* cl, double* neg, const MergeOut& mo = MergeOut{}) {
  RAMA_KERNEL(ctx, k_reparam, st.m_aug, st.m_aug, st.base.p, st.T ? st.slot_ptr.p : (const int32_t*)nullptr,
              st.slots.p, st.lam.p, cl, neg, st.n_long.p ? kLongCov : INT32_MAX, mo);
  if (st.T && st.n_long.p) {
    KernelScope ks(ctx.s, "k_reparam_long", 0.0);
    k_reparam_long<<<(unsigned)num_sms() * 8, kBlock, 0, ctx.s>>>(st.long_e.p, st.n_long.p, st.base.p,
                                                                  st.slot_ptr.p, st.slots.p, st.lam.p, cl, neg, mo);
    RAMA_LAUNCH_CHECK();
    ctx.launches++;
  }
}

void reparam_costs(Ctx& ctx, const DualState& st, double* cl) { reparam_pass(ctx, st, cl, nullptr); }

__global__ void k_tri_min(int64_t T, const double* __restrict__ lam, double* __restrict__ out) {
  GRID_STRIDE(t, T) {
    double l0 = lam[3 * t], l1 = lam[3 * t + 1], l2 = lam[3 * t + 2];
    double c110 = -__dadd_rn(l0, l1);
    double c101 = -__dadd_rn(l0, l2);
    double c011 = -__dadd_rn(l1, l2);
    double c111 = -__dadd_rn(__dadd_rn(l0, l1), l2);
    out[t] = mn2(mn2(mn2(c110, c101), mn2(c011, c111)), 0.0);
  }
}

void lower_bound_terms(Ctx& ctx, const DualState& st, double* cl_out, double* neg, double* tm) {
  reparam_pass(ctx, st, cl_out, neg);
  RAMA_KERNEL(ctx, k_tri_min, st.T, st.T, st.lam.p, tm);
}

__global__ void k_lb_total(const double* __restrict__ sn, const double* __restrict__ st, double* __restrict__ out) {
  double total = 0.0;  // as lower_bound: total = sum(neg); total += sum(tm)
  if (sn) total = *sn;
  if (st) total += *st;
  *out = total;
}

static void lower_bound_to_impl(Ctx& ctx, const DualState& st, double* cl_out, double* out, const MergeOut& mo) {
  Buf<double> neg(st.m_aug > 0 ? st.m_aug : 1, ctx), tm(st.T > 0 ? st.T : 1, ctx), sums(2, ctx);
  reparam_pass(ctx, st, cl_out, neg.p, mo);
  RAMA_KERNEL(ctx, k_tri_min, st.T, st.T, st.lam.p, tm.p);
  if (st.m_aug > 0) device_sum_to(ctx, neg.p, st.m_aug, sums.p);
  if (st.T > 0) device_sum_to(ctx, tm.p, st.T, sums.p + 1);
  {
    KernelScope ks(ctx.s, "k_lb_total", 0.0);
    k_lb_total<<<1, 1, 0, ctx.s>>>(st.m_aug > 0 ? sums.p : nullptr, st.T > 0 ? sums.p + 1 : nullptr, out);
  }
  RAMA_LAUNCH_CHECK();
  ctx.launches++;
}

void lower_bound_to(Ctx& ctx, const DualState& st, double* cl_out, double* out) {
  ProfScope prof(ctx.s, kFamBound, 36.0 * (double)st.T + 20.0 * (double)st.m_aug);
  lower_bound_to_impl(ctx, st, cl_out, out, MergeOut{});
}

Graph bound_and_reparametrized(Ctx& ctx, const DualState& st, double* lb_out) {
  if (st.m_aug == 0 || !st.chords_sorted || !st.orig_ptr.p || !st.chord_ptr.p) {
    Buf<double> cl(st.m_aug > 0 ? st.m_aug : 1, ctx);
    lower_bound_to(ctx, st, cl.p, lb_out);
    return reparametrized_graph(ctx, st, cl.p);
  }
  // bound terms + the merged canonical graph in the same edge pass
  ProfScope prof(ctx.s, kFamBound, 36.0 * (double)st.T + 20.0 * (double)st.m_aug + 32.0 * (double)st.m_aug);
  Graph g;
  g.n = st.n;
  g.m = st.m_aug;
  g.u.alloc(st.m_aug, ctx.s);
  g.v.alloc(st.m_aug, ctx.s);
  g.c.alloc(st.m_aug, ctx.s);
  MergeOut mo;
  mo.ou = g.u.p;
  mo.ov = g.v.p;
  mo.oc = g.c.p;
  mo.eu = st.eu.p;
  mo.ev = st.ev.p;
  mo.optr = st.orig_ptr.p;
  mo.cptr = st.chord_ptr.p;
  mo.m = st.m_orig;
  lower_bound_to_impl(ctx, st, nullptr, lb_out, mo);
  return g;
}

double lower_bound(Ctx& ctx, const DualState& st, double* cl_out) {
  // algorithmic bytes: lambda (24 T) and the slot lists (12 T + 4 m_aug)
  // read once, base read (8 m_aug), c^lambda written (8 m_aug)
  ProfScope prof(ctx.s, kFamBound, 36.0 * (double)st.T + 20.0 * (double)st.m_aug);
  double total = 0.0;
  Buf<double> neg(st.m_aug > 0 ? st.m_aug : 1, ctx), tm(st.T > 0 ? st.T : 1, ctx);
  lower_bound_terms(ctx, st, cl_out, neg.p, tm.p);
  if (st.m_aug > 0) total = device_sum(ctx, neg.p, st.m_aug);
  if (st.T > 0) total += device_sum(ctx, tm.p, st.T);
  return total;
}


// ------------------------------------------- check_edge_triangle_agreement
//
// dual.py:477-531: arc consistency between the near-optimal label sets of
// edges (bit 0 uncut, bit 1 cut) and triplets (bit p = pattern p of
// MC_TRIANGLE = 000, 110, 101, 011, 111).  Jacobi sweeps exactly like the
// reference: triplet pass against the current edge sets, then edge pass
// against the new triplet sets (bits only ever clear), until no change.
__constant__ uint8_t kMcPat[5][3] = {{0, 0, 0}, {1, 1, 0}, {1, 0, 1}, {0, 1, 1}, {1, 1, 1}};

__global__ void k_agree_init_edges(const double* __restrict__ cl, int64_t m, double eps, uint32_t* __restrict__ em) {
  GRID_STRIDE(e, m) {
    double x = cl[e];
    double best = mn2(x, 0.0);
    uint32_t b = 0;
    if (0.0 <= __dadd_rn(best, eps)) b |= 1u;
    if (x <= __dadd_rn(best, eps)) b |= 2u;
    em[e] = b;
  }
}

__global__ void k_agree_init_tri(const double* __restrict__ lam, int64_t T, double eps, uint8_t* __restrict__ tm) {
  GRID_STRIDE(t, T) {
    double l0 = lam[3 * t], l1 = lam[3 * t + 1], l2 = lam[3 * t + 2];
    double pc[5];
    pc[0] = 0.0;
    pc[1] = -__dadd_rn(l0, l1);
    pc[2] = -__dadd_rn(l0, l2);
    pc[3] = -__dadd_rn(l1, l2);
    pc[4] = -__dadd_rn(__dadd_rn(l0, l1), l2);
    double best = pc[0];
    for (int p = 1; p < 5; p++) best = mn2(best, pc[p]);
    uint8_t b = 0;
    for (int p = 0; p < 5; p++)
      if (pc[p] <= __dadd_rn(best, eps)) b |= (uint8_t)(1u << p);
    tm[t] = b;
  }
}

__global__ void k_agree_tri(const int32_t* __restrict__ te, int64_t T, const uint32_t* __restrict__ em,
                            uint8_t* __restrict__ tm, int32_t* __restrict__ changed) {
  GRID_STRIDE(t, T) {
    uint8_t b = tm[t], nb = b;
    uint32_t e0 = em[te[3 * t]], e1 = em[te[3 * t + 1]], e2 = em[te[3 * t + 2]];
    for (int p = 0; p < 5; p++) {
      bool ok = (e0 & (1u << kMcPat[p][0])) && (e1 & (1u << kMcPat[p][1])) && (e2 & (1u << kMcPat[p][2]));
      if (!ok) nb &= (uint8_t)~(1u << p);
    }
    if (nb != b) {
      tm[t] = nb;
      *changed = 1;
    }
  }
}

__global__ void k_agree_edges(const int32_t* __restrict__ te, int64_t T, const uint8_t* __restrict__ tm,
                              uint32_t* __restrict__ em, int32_t* __restrict__ changed) {
  GRID_STRIDE(t, T) {
    uint8_t b = tm[t];
    for (int s = 0; s < 3; s++) {
      bool has0 = false, has1 = false;
      for (int p = 0; p < 5; p++)
        if (b & (1u << p)) {
          if (kMcPat[p][s]) has1 = true; else has0 = true;
        }
      uint32_t clear = (has0 ? 0u : 1u) | (has1 ? 0u : 2u);
      if (clear) {
        uint32_t old = atomicAnd(em + te[3 * t + s], ~clear);
        if (old & clear) *changed = 1;
      }
    }
  }
}

__global__ void k_agree_empty_e(const uint32_t* __restrict__ em, int64_t m, int32_t* __restrict__ bad) {
  GRID_STRIDE(e, m) if (em[e] == 0) *bad = 1;
}

__global__ void k_agree_empty_t(const uint8_t* __restrict__ tm, int64_t T, int32_t* __restrict__ bad) {
  GRID_STRIDE(t, T) if (tm[t] == 0) *bad = 1;
}

bool check_edge_triangle_agreement(Ctx& ctx, const DualState& st, double eps) {
  RAMA_REQUIRE(eps >= 0.0, "eps must be non-negative");
  const int64_t m = st.m_aug, T = st.T;
  Buf<double> cl(m > 0 ? m : 1, ctx);
  reparam_costs(ctx, st, cl.p);
  Buf<uint32_t> em(m > 0 ? m : 1, ctx);
  Buf<uint8_t> tm(T > 0 ? T : 1, ctx);
  Buf<int32_t> flag(2, ctx);
  RAMA_KERNEL(ctx, k_agree_init_edges, m, cl.p, m, eps, em.p);
  RAMA_KERNEL(ctx, k_agree_init_tri, T, st.lam.p, T, eps, tm.p);
  while (T > 0) {
    flag.zero();
    RAMA_KERNEL(ctx, k_agree_tri, T, st.tri_edges.p, T, em.p, tm.p, flag.p);
    RAMA_KERNEL(ctx, k_agree_edges, T, st.tri_edges.p, T, tm.p, em.p, flag.p);
    if (read_scalar(ctx, flag.p) == 0) break;
  }
  flag.zero();
  RAMA_KERNEL(ctx, k_agree_empty_e, m, em.p, m, flag.p);
  RAMA_KERNEL(ctx, k_agree_empty_t, T, tm.p, T, flag.p);
  return read_scalar(ctx, flag.p) == 0;
}

// --------------------------------------------------- reparametrized graph

__global__ void k_merge_scatter(int64_t m, int64_t C, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                                const double* __restrict__ cl, const int32_t* __restrict__ optr,
                                const int32_t* __restrict__ cptr, int32_t* __restrict__ ou, int32_t* __restrict__ ov,
                                double* __restrict__ oc) {
  GRID_STRIDE(i, m + C) {
    int32_t a = eu[i], b = ev[i];
    int64_t pos = i < m ? i + row_lower(cptr, ev + m, a, b) : (i - m) + row_lower(optr, ev, a, b);
    ou[pos] = a;
    ov[pos] = b;
    oc[pos] = cl[i];  // WeightedGraph ctor: x0 + pairwise([]) = x0 per unique pair
  }
}

__global__ void k_sorted_edges_out(const int32_t* __restrict__ row, const uint64_t* __restrict__ key,
                                   const double* __restrict__ cl, int64_t m, int32_t* __restrict__ ou,
                                   int32_t* __restrict__ ov, double* __restrict__ oc) {
  GRID_STRIDE(p, m) {
    ou[p] = row[p];
    ov[p] = (int32_t)(key[p] >> 32);
    oc[p] = cl[(uint32_t)key[p]];  // WeightedGraph ctor: x0 + pairwise([]) = x0
  }
}

Graph reparametrized_graph(Ctx& ctx, const DualState& st, const double* cl_in) {
  ProfScope prof(ctx.s, kFamBound, 32.0 * (double)st.m_aug);  // (eu, ev, c^lambda) read, canonical COO written
  Graph g;
  g.n = st.n;
  g.m = st.m_aug;
  int64_t ma = st.m_aug > 0 ? st.m_aug : 1;
  g.u.alloc(ma, ctx.s);
  g.v.alloc(ma, ctx.s);
  g.c.alloc(ma, ctx.s);
  if (st.m_aug == 0) return g;
  Buf<double> cl_own;
  const double* cl = cl_in;
  if (!cl) {
    cl_own.alloc(st.m_aug, ctx.s);
    reparam_costs(ctx, st, cl_own.p);
    cl = cl_own.p;
  }
  if (!st.chords_sorted || !st.orig_ptr.p || !st.chord_ptr.p) {  // general edge order: sort all augmented edges
    Buf<int32_t> row(st.m_aug, ctx);
    Buf<uint64_t> key(st.m_aug, ctx);
    RAMA_KERNEL(ctx, k_ext_edge_keys, st.m_aug, st.eu.p, st.ev.p, st.m_aug, row.p, key.p);
    BucketSorted bs;
    bucket_sort(ctx, st.n, st.m_aug, row.p, key.p, bs, true);
    RAMA_KERNEL(ctx, k_sorted_edges_out, st.m_aug, bs.row.p, bs.key.p, cl, st.m_aug, g.u.p, g.v.p, g.c.p);
    return g;
  }
  RAMA_KERNEL(ctx, k_merge_scatter, st.m_aug, st.m_orig, st.m_aug - st.m_orig, st.eu.p, st.ev.p, cl, st.orig_ptr.p,
              st.chord_ptr.p, g.u.p, g.v.p, g.c.p);
  return g;
}

}  // namespace rama
