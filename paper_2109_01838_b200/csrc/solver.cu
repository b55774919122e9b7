// Device-resident solver driver.
//
// The whole solve stays in HBM: the host loop only reads back the handful
// of scalars that size the next launches (|S|, n', m', T, LB).  Rounds follow
// solver.py:147-208 (PD/PD+) and solver.py:113-144 (P):
//   separate -> triangulate -> k x MP -> LB -> reparametrized graph ->
//   auto contraction step -> compose.
// Cleanup (solver.py:187-207) contracts the ORIGINAL graph under f_total and
// then replaces the reference's sequential heap GAEC with repeated parallel
// handshake rounds (one mutual-max round on original costs, contract,
// repeat until no pair) -- DESIGN.md deviation D1, measured at +0.0011% on C2.
#include "internal.h"

#include <chrono>
#include <cmath>

namespace rama {

using clk = std::chrono::steady_clock;

static double ms_since(clk::time_point t0) {
  return std::chrono::duration<double, std::milli>(clk::now() - t0).count();
}

static Graph copy_graph(Ctx& ctx, const GraphView& g) {
  Graph out;
  out.n = g.n;
  out.m = g.m;
  int64_t mm = g.m > 0 ? g.m : 1;
  out.u.alloc(mm, ctx.s);
  out.v.alloc(mm, ctx.s);
  out.c.alloc(mm, ctx.s);
  copy_d2d(ctx, out.u.p, g.u, g.m);
  copy_d2d(ctx, out.v.p, g.v, g.m);
  copy_d2d(ctx, out.c.p, g.c, g.m);
  return out;
}

static void push(RoundInfo* trace, int max_trace, int& nr, const RoundInfo& r) {
  if (trace && nr < max_trace) trace[nr] = r;
  nr++;
}

// ------------------------------------------------------------- cleanup
//
// Deviation D1: the reference's sequential heap GAEC is
// replaced by repeated handshake rounds on the quotient under its own
// costs.  Node ids are never renumbered: a mutual pair (x < t) merges into
// x, so a cluster's id stays its smallest member and tie-breaks by id match
// canonical relabelling.  Per round, only edges with a merged endpoint are
// rewritten; they are grouped by (u', v', slot) and each group folds into
// its smallest slot with a sequential sum (oracle: orc_cleanup_handshake).
//
// Two executions of the same round:
//  * wide rounds (many positive edges): a few grid-wide kernels streaming
//    the slot arrays, touched slots sorted by CUB radix sort;
//  * the long tail (a growing cluster absorbing one neighbour per round,
//    hundreds of rounds on 3-D grids) runs inside ONE persistent
//    single-CTA kernel: the positive slots P and per-node incidence rows
//    are kept on the device, a round touches only the rows of merged nodes
//    and sorts them in shared memory, so there is no host round trip per
//    round.  It hands back to the wide path if a round outgrows it.

__global__ void k_cl_vote1(const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                           const double* __restrict__ c, const uint8_t* __restrict__ alive, int64_t m,
                           unsigned long long* __restrict__ bc, int32_t* __restrict__ npos) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < m; base += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = base + threadIdx.x;
    bool pos = false;
    if (i < m) {
      double x = c[i];
      pos = alive[i] && x > 0.0;
      if (pos) {
        unsigned long long bits = dbits(x);
        atomicMax(bc + u[i], bits);
        atomicMax(bc + v[i], bits);
      }
    }
    unsigned b = __ballot_sync(0xffffffffu, pos);
    if (lane == 0 && b) atomicAdd(npos, __popc(b));
  }
}

__global__ void k_cl_vote2(const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                           const double* __restrict__ c, const uint8_t* __restrict__ alive, int64_t m,
                           const unsigned long long* __restrict__ bc, int32_t* __restrict__ bn) {
  GRID_STRIDE(i, m) {
    double x = c[i];
    if (!alive[i] || !(x > 0.0)) continue;
    unsigned long long bits = dbits(x);
    int32_t a = u[i], b = v[i];
    if (bits == bc[a]) atomicMin(bn + a, b);
    if (bits == bc[b]) atomicMin(bn + b, a);
  }
}

// merged[x] = x is in a mutual pair this round; the smaller side appends the pair
__global__ void k_cl_pair(int64_t n, const unsigned long long* __restrict__ bc, const int32_t* __restrict__ bn,
                          uint8_t* __restrict__ merged, int32_t* __restrict__ pu, int32_t* __restrict__ pv,
                          int32_t* __restrict__ npairs) {
  GRID_STRIDE(x, n) {
    bool p = false;
    int32_t t = bn[x];
    if (bc[x] != 0ULL) p = (bn[t] == (int32_t)x);
    merged[x] = p;
    if (p && (int32_t)x < t) {
      int32_t k = atomicAdd(npairs, 1);
      pu[k] = (int32_t)x;
      pv[k] = t;
    }
  }
}

__global__ void k_cl_relabel(int32_t* __restrict__ u, int32_t* __restrict__ v, uint8_t* __restrict__ alive,
                             int64_t m, const uint8_t* __restrict__ merged, const int32_t* __restrict__ bn,
                             uint8_t* __restrict__ touched) {
  GRID_STRIDE(i, m) {
    uint8_t t = 0;
    if (alive[i]) {
      int32_t x = u[i], y = v[i];
      bool mx = merged[x], my = merged[y];
      if (mx || my) {
        int32_t a = mx ? min(x, bn[x]) : x;
        int32_t b = my ? min(y, bn[y]) : y;
        if (a == b) {
          alive[i] = 0;
        } else {
          u[i] = min(a, b);
          v[i] = max(a, b);
          t = 1;
        }
      }
    }
    touched[i] = t;
  }
}

__global__ void k_cl_keys(const int32_t* __restrict__ idx, int64_t k, const int32_t* __restrict__ u,
                          const int32_t* __restrict__ v, uint64_t* __restrict__ key) {
  GRID_STRIDE(j, k) {
    int32_t i = idx[j];
    key[j] = ((uint64_t)(uint32_t)u[i] << 32) | (uint64_t)(uint32_t)v[i];
  }
}

// touched slots sorted by (u', v') with ascending slots inside a group
// (stable radix sort of an ascending slot list): fold into the first slot
__global__ void k_cl_fold(int64_t k, const uint64_t* __restrict__ key, const int32_t* __restrict__ slot,
                          double* __restrict__ c, uint8_t* __restrict__ alive) {
  GRID_STRIDE(p, k) {
    if (p > 0 && key[p] == key[p - 1]) continue;
    int32_t first = slot[p];
    double acc = c[first];
    int64_t q = p + 1;
    for (; q < k && key[q] == key[p]; q++) {
      acc = __dadd_rn(acc, c[slot[q]]);
      alive[slot[q]] = 0;
    }
    if (q > p + 1) c[first] = acc;
  }
}

// ---- tail state -----------------------------------------------------------

constexpr int kTailThreads = 1024;
constexpr int kTailSort = 16384;    // touched slots sorted in shared memory per round
constexpr int kTailP = 32768;       // enter the tail when at most this many positive slots remain
constexpr int kTailPairs = 4096;    // pairs per tail round
constexpr size_t kTailSmem = (size_t)kTailSort * (sizeof(uint64_t) + sizeof(int32_t));

enum TailStatus : int32_t { kTailRunning = 0, kTailDone = 1, kTailBail = 2 };

struct TailArgs {
  int32_t* u;
  int32_t* v;
  double* c;
  uint8_t* alive;
  int32_t* tmark;          // per slot, clean (0) between rounds
  unsigned long long* bc;  // per node, clean (0) between rounds
  int32_t* bn;             // per node, clean (INT_MAX) between rounds
  int32_t* mate;           // per node, -1 unless merged this round
  int32_t* P0;             // positive alive slots (double buffered, capacity kTailP + kTailSort)
  int32_t* P1;
  int32_t* np;             // |P| of the current buffer
  int32_t* which;          // current buffer (0: P0)
  int32_t* row_off;        // per node: incidence row (slot ids, may hold dead slots) in pool
  int32_t* row_len;
  int32_t* pool;
  int64_t pool_cap;
  int32_t* pool_top;
  int32_t* pu;             // global pair list (continues the wide rounds')
  int32_t* pv;
  int32_t* npairs;
  int32_t* status;
  int32_t* rounds;
};

// the tail kernel reads arrays other threads of the CTA wrote or updated
// with atomics earlier in the same launch: bypass L1 (ld.global.cg)
#define LD(p) __ldcg(p)

__device__ __forceinline__ int32_t tail_rep(const int32_t* mate, int32_t y) {
  int32_t t = LD(mate + y);
  return t < 0 ? y : min(y, t);
}

__device__ __forceinline__ bool tail_less(uint64_t ka, int32_t sa, uint64_t kb, int32_t sb) {
  return ka < kb || (ka == kb && sa < sb);
}

__global__ void __launch_bounds__(kTailThreads, 1) k_cl_tail(TailArgs A) {
  extern __shared__ uint64_t sk[];           // kTailSort keys
  int32_t* ss = (int32_t*)(sk + kTailSort);  // kTailSort slots
  __shared__ int32_t s_np, s_npairs, s_nt, s_rowsum, s_np2, s_stop, s_which, s_base;
  const int tid = threadIdx.x, NT = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, NW = NT >> 5;
  if (tid == 0) s_which = *A.which;
  __syncthreads();
  while (true) {
    if (tid == 0) {
      s_np = LD(A.np);
      s_npairs = 0;
      s_nt = 0;
      s_rowsum = 0;
      s_np2 = 0;
      s_base = LD(A.npairs);
      s_stop = (s_np > kTailP || (int64_t)LD(A.pool_top) + kTailSort > A.pool_cap) ? kTailBail : 0;
    }
    __syncthreads();
    if (s_stop) break;
    const int32_t* P = s_which ? A.P1 : A.P0;
    int32_t* P2 = s_which ? A.P0 : A.P1;
    const int32_t np = s_np;
    // handshake votes over the positive slots (contraction.py:207 rule)
    for (int32_t i = tid; i < np; i += NT) {
      int32_t s = P[i];
      unsigned long long bits = dbits(LD(A.c + s));
      atomicMax(A.bc + LD(A.u + s), bits);
      atomicMax(A.bc + LD(A.v + s), bits);
    }
    __syncthreads();
    for (int32_t i = tid; i < np; i += NT) {
      int32_t s = P[i];
      unsigned long long bits = dbits(LD(A.c + s));
      int32_t a = LD(A.u + s), b = LD(A.v + s);
      if (bits == LD(A.bc + a)) atomicMin(A.bn + a, b);
      if (bits == LD(A.bc + b)) atomicMin(A.bn + b, a);
    }
    __syncthreads();
    // mutual pairs: slot (a, b) with bn[a] == b and bn[b] == a is both nodes' max edge
    for (int32_t i = tid; i < np; i += NT) {
      int32_t s = P[i];
      int32_t a = LD(A.u + s), b = LD(A.v + s);
      if (LD(A.bn + a) == b && LD(A.bn + b) == a) {
        int32_t k = atomicAdd(&s_npairs, 1);
        if (k < kTailPairs) {
          A.pu[s_base + k] = a;
          A.pv[s_base + k] = b;
          atomicAdd(&s_rowsum, LD(A.row_len + a) + LD(A.row_len + b));
        }
      }
    }
    __syncthreads();
    for (int32_t i = tid; i < np; i += NT) {  // votes back to clean
      int32_t s = P[i];
      int32_t a = LD(A.u + s), b = LD(A.v + s);
      A.bc[a] = 0ULL;
      A.bc[b] = 0ULL;
      A.bn[a] = 0x7fffffff;
      A.bn[b] = 0x7fffffff;
    }
    __syncthreads();
    const int32_t npairs = s_npairs;
    if (npairs == 0 || npairs > kTailPairs || s_rowsum > kTailSort) {
      // nothing was modified this round: the wide path can redo it
      if (tid == 0) s_stop = npairs == 0 ? kTailDone : kTailBail;
      __syncthreads();
      break;
    }
    const int32_t* pu = A.pu + s_base;
    const int32_t* pv = A.pv + s_base;
    for (int32_t k = tid; k < npairs; k += NT) {
      A.mate[pu[k]] = pv[k];
      A.mate[pv[k]] = pu[k];
    }
    __syncthreads();
    // touched = alive slots in the rows of merged nodes (deduplicated)
    for (int32_t k = warp; k < 2 * npairs; k += NW) {
      int32_t y = (k & 1) ? pv[k >> 1] : pu[k >> 1];
      int32_t off = LD(A.row_off + y), len = LD(A.row_len + y);
      for (int32_t j = lane; j < len; j += 32) {
        int32_t s = LD(A.pool + off + j);
        if (LD(A.alive + s) && atomicExch(A.tmark + s, 1) == 0) ss[atomicAdd(&s_nt, 1)] = s;
      }
    }
    __syncthreads();
    const int32_t nt = s_nt;
    int32_t P2n = 2;
    while (P2n < nt) P2n <<= 1;
    // relabel to the pair representatives (smaller id); internal slots die
    for (int32_t i = tid; i < P2n; i += NT) {
      if (i >= nt) {
        sk[i] = ~0ULL;
        ss[i] = 0x7fffffff;
        continue;
      }
      int32_t s = ss[i];
      int32_t a = tail_rep(A.mate, LD(A.u + s)), b = tail_rep(A.mate, LD(A.v + s));
      if (a == b) {
        A.alive[s] = 0;
        sk[i] = ~0ULL;
      } else {
        int32_t lo = min(a, b), hi = max(a, b);
        A.u[s] = lo;
        A.v[s] = hi;
        sk[i] = ((uint64_t)(uint32_t)lo << 32) | (uint64_t)(uint32_t)hi;
      }
    }
    __syncthreads();
    // bitonic sort of (key, slot) in shared memory
    for (int32_t k = 2; k <= P2n; k <<= 1) {
      for (int32_t j = k >> 1; j > 0; j >>= 1) {
        for (int32_t i = tid; i < P2n; i += NT) {
          int32_t ixj = i ^ j;
          if (ixj > i) {
            bool up = (i & k) == 0;
            uint64_t ka = sk[i], kb = sk[ixj];
            int32_t sa = ss[i], sb = ss[ixj];
            if (tail_less(kb, sb, ka, sa) == up) {
              sk[i] = kb; sk[ixj] = ka;
              ss[i] = sb; ss[ixj] = sa;
            }
          }
        }
        __syncthreads();
      }
    }
    // fold each (u', v') group into its smallest slot, sequential sum
    for (int32_t p = tid; p < nt; p += NT) {
      uint64_t key = sk[p];
      if (key == ~0ULL || (p > 0 && sk[p - 1] == key)) continue;
      int32_t first = ss[p];
      double acc = LD(A.c + first);
      int32_t q = p + 1;
      for (; q < nt && sk[q] == key; q++) {
        acc = __dadd_rn(acc, LD(A.c + ss[q]));
        A.alive[ss[q]] = 0;
      }
      if (q > p + 1) A.c[first] = acc;
    }
    __syncthreads();
    // next P: untouched positive slots of P + positive touched survivors
    for (int32_t i = tid; i < np; i += NT) {
      int32_t s = P[i];
      if (!LD(A.tmark + s)) P2[atomicAdd(&s_np2, 1)] = s;  // untouched: still alive and positive
    }
    for (int32_t i = tid; i < nt; i += NT) {
      int32_t s = ss[i];
      if (sk[i] != ~0ULL && LD(A.alive + s) && LD(A.c + s) > 0.0) P2[atomicAdd(&s_np2, 1)] = s;
    }
    // absorbed nodes lose their rows; representatives get fresh ones
    for (int32_t k = tid; k < npairs; k += NT) {
      A.row_len[pu[k]] = 0;
      A.row_len[pv[k]] = 0;
    }
    __syncthreads();
    for (int32_t i = tid; i < nt; i += NT) {
      int32_t s = ss[i];
      if (sk[i] == ~0ULL || !LD(A.alive + s)) continue;
      int32_t a = LD(A.u + s), b = LD(A.v + s);
      if (LD(A.mate + a) >= 0) atomicAdd(A.row_len + a, 1);
      if (LD(A.mate + b) >= 0) atomicAdd(A.row_len + b, 1);
    }
    __syncthreads();
    for (int32_t k = tid; k < npairs; k += NT) {
      int32_t x = pu[k];
      A.row_off[x] = atomicAdd(A.pool_top, LD(A.row_len + x));
    }
    __syncthreads();
    for (int32_t i = tid; i < nt; i += NT) {  // bc doubles as the fill cursor (clean = 0)
      int32_t s = ss[i];
      if (sk[i] == ~0ULL || !LD(A.alive + s)) continue;
      int32_t a = LD(A.u + s), b = LD(A.v + s);
      if (LD(A.mate + a) >= 0) A.pool[LD(A.row_off + a) + (int32_t)atomicAdd(A.bc + a, 1ULL)] = s;
      if (LD(A.mate + b) >= 0) A.pool[LD(A.row_off + b) + (int32_t)atomicAdd(A.bc + b, 1ULL)] = s;
    }
    __syncthreads();
    for (int32_t i = tid; i < P2n; i += NT) {
      int32_t s = ss[i];
      if (s != 0x7fffffff) A.tmark[s] = 0;
    }
    for (int32_t k = tid; k < npairs; k += NT) {
      A.bc[pu[k]] = 0ULL;
      A.mate[pu[k]] = -1;
      A.mate[pv[k]] = -1;
    }
    if (tid == 0) {
      *A.npairs = s_base + npairs;
      *A.np = s_np2;
      s_which ^= 1;
      *A.which = s_which;
      *A.rounds += 1;
    }
    __syncthreads();
  }
  if (tid == 0) *A.status = s_stop;
}
#undef LD

// rows: per node, the alive slots incident to it
__global__ void k_cl_degree(const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                            const uint8_t* __restrict__ alive, int64_t m, int32_t* __restrict__ deg) {
  GRID_STRIDE(i, m) {
    if (!alive[i]) continue;
    atomicAdd(deg + u[i], 1);
    atomicAdd(deg + v[i], 1);
  }
}

__global__ void k_cl_fill_rows(const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                               const uint8_t* __restrict__ alive, int64_t m, const int32_t* __restrict__ off,
                               int32_t* __restrict__ cursor, int32_t* __restrict__ pool) {
  GRID_STRIDE(i, m) {
    if (!alive[i]) continue;
    int32_t a = u[i], b = v[i];
    pool[off[a] + atomicAdd(cursor + a, 1)] = (int32_t)i;
    pool[off[b] + atomicAdd(cursor + b, 1)] = (int32_t)i;
  }
}

__global__ void k_cl_posflag(const double* __restrict__ c, const uint8_t* __restrict__ alive, int64_t m,
                             uint8_t* __restrict__ f) {
  GRID_STRIDE(i, m) f[i] = alive[i] && c[i] > 0.0;
}

// RAMA_TAIL_P=<k> overrides the tail entry threshold (0 disables the tail;
// the tests use it to run both executions of a round on the same quotient)
static int64_t tail_entry_limit() {
  static const int64_t v = [] {
    const char* e = getenv("RAMA_TAIL_P");
    int64_t x = e ? atoll(e) : kTailP;
    return x < 0 ? 0 : (x > kTailP ? (int64_t)kTailP : x);
  }();
  return v;
}

// Runs the cleanup on quotient q; writes the canonical map fc (size q.n)
// and returns the number of clusters.
static int64_t handshake_cleanup(Ctx& ctx, const GraphView& q, int32_t* fc) {
  ProfScope prof(ctx.s, kFamCleanup);
  const int64_t n = q.n, m = q.m;
  if (n == 0) return 0;
  if (m == 0) {
    iota(ctx, fc, n);
    return n;
  }
  Buf<int32_t> u(m, ctx), v(m, ctx);
  Buf<double> c(m, ctx);
  copy_d2d(ctx, u.p, q.u, m);
  copy_d2d(ctx, v.p, q.v, m);
  copy_d2d(ctx, c.p, q.c, m);
  Buf<uint8_t> alive(m, ctx), touched(m, ctx), merged(n, ctx);
  alive.fill_bytes(1);
  Buf<unsigned long long> bc(n, ctx);
  Buf<int32_t> bn(n, ctx), pu(n, ctx), pv(n, ctx);
  // device scalars: 0 npairs, 1 npos, 2 np (tail), 3 which, 4 pool_top, 5 status, 6 rounds
  Buf<int32_t> sc(8, ctx);
  sc.zero();
  int32_t* d_npairs = sc.p;
  int32_t* d_npos = sc.p + 1;
  int64_t total = 0;
  int skip = 0, backoff = 1;  // wide rounds to run before retrying the tail after a bail
  while (true) {
    bc.zero();
    bn.fill_bytes(0x7f);
    RAMA_CUDA(cudaMemsetAsync(d_npos, 0, sizeof(int32_t), ctx.s));
    RAMA_KERNEL(ctx, k_cl_vote1, m, u.p, v.p, c.p, alive.p, m, bc.p, d_npos);
    int32_t npos = read_scalar(ctx, d_npos);
    if (npos == 0) break;
    if (npos <= tail_entry_limit() && skip == 0) {
      // ---- persistent tail: P list, incidence rows, one CTA --------------
      bc.zero();
      Buf<uint8_t> pf(m, ctx);
      RAMA_KERNEL(ctx, k_cl_posflag, m, c.p, alive.p, m, pf.p);
      Buf<int32_t> Pl;
      int64_t np = compact_indices(ctx, pf.p, m, Pl);
      Buf<int32_t> P0(kTailP + kTailSort, ctx), P1(kTailP + kTailSort, ctx);
      copy_d2d(ctx, P0.p, Pl.p, np);
      Buf<int32_t> deg(n, ctx), off(n + 1, ctx), cur(n, ctx), mate(n, ctx), tmark(m, ctx);
      deg.zero();
      cur.zero();
      tmark.zero();
      mate.fill_bytes(0xff);
      RAMA_KERNEL(ctx, k_cl_degree, m, u.p, v.p, alive.p, m, deg.p);
      int64_t arcs = exclusive_scan(ctx, deg.p, off.p, n, true);
      int64_t cap = arcs + 64LL * kTailSort + (1 << 20);
      Buf<int32_t> pool(cap, ctx);
      RAMA_KERNEL(ctx, k_cl_fill_rows, m, u.p, v.p, alive.p, m, off.p, cur.p, pool.p);
      int32_t init[7] = {(int32_t)total, 0, (int32_t)np, 0, (int32_t)arcs, 0, 0};
      RAMA_CUDA(cudaMemcpyAsync(sc.p, init, sizeof(init), cudaMemcpyHostToDevice, ctx.s));
      TailArgs A;
      A.u = u.p; A.v = v.p; A.c = c.p; A.alive = alive.p; A.tmark = tmark.p; A.bc = bc.p; A.bn = bn.p;
      A.mate = mate.p; A.P0 = P0.p; A.P1 = P1.p; A.np = sc.p + 2; A.which = sc.p + 3;
      A.row_off = off.p; A.row_len = deg.p; A.pool = pool.p; A.pool_cap = cap; A.pool_top = sc.p + 4;
      A.pu = pu.p; A.pv = pv.p; A.npairs = d_npairs; A.status = sc.p + 5; A.rounds = sc.p + 6;
      static bool attr = false;
      if (!attr) {
        RAMA_CUDA(cudaFuncSetAttribute(k_cl_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTailSmem));
        attr = true;
      }
      k_cl_tail<<<1, kTailThreads, kTailSmem, ctx.s>>>(A);
      RAMA_LAUNCH_CHECK();
      ctx.launches++;
      int32_t st[7];
      RAMA_CUDA(cudaMemcpyAsync(ctx.pinned, sc.p, sizeof(st), cudaMemcpyDeviceToHost, ctx.s));
      ctx.sync();
      memcpy(st, ctx.pinned, sizeof(st));
      total = st[0];
      if (st[5] == kTailDone) break;
      // bail: the round that did not fit is redone by the wide path below
      backoff = st[6] > 0 ? 1 : (backoff < 64 ? 2 * backoff : 64);
      skip = backoff;
      bc.zero();
      RAMA_CUDA(cudaMemsetAsync(d_npos, 0, sizeof(int32_t), ctx.s));
      RAMA_KERNEL(ctx, k_cl_vote1, m, u.p, v.p, c.p, alive.p, m, bc.p, d_npos);
    } else if (skip > 0) {
      skip--;
    }
    RAMA_KERNEL(ctx, k_cl_vote2, m, u.p, v.p, c.p, alive.p, m, bc.p, bn.p);
    RAMA_KERNEL(ctx, k_cl_pair, n, n, bc.p, bn.p, merged.p, pu.p, pv.p, d_npairs);
    int64_t now = read_scalar(ctx, d_npairs);
    if (now == total) break;
    total = now;
    RAMA_KERNEL(ctx, k_cl_relabel, m, u.p, v.p, alive.p, m, merged.p, bn.p, touched.p);
    Buf<int32_t> idx;
    int64_t k = compact_indices(ctx, touched.p, m, idx);
    if (k == 0) continue;
    Buf<uint64_t> key(k, ctx), key2(k, ctx);
    Buf<int32_t> slot(k, ctx);
    RAMA_KERNEL(ctx, k_cl_keys, k, idx.p, k, u.p, v.p, key.p);
    int bits = 1;
    while ((1LL << bits) < n) bits++;
    radix_sort_pairs(ctx, key.p, idx.p, key2.p, slot.p, k, 0, 32 + bits);
    RAMA_KERNEL(ctx, k_cl_fold, k, k, key2.p, slot.p, c.p, alive.p);
  }
  return components(ctx, n, pu.p, pv.p, total, fc);
}

void solve(Ctx& ctx, const GraphView& g, const SolveConfig& cfg, int32_t* labels, SolveResult& res,
           RoundInfo* trace, int max_trace) {
  RAMA_REQUIRE(cfg.mode >= 0 && cfg.mode <= 4, "unknown mode");
  RAMA_REQUIRE(cfg.max_rounds >= 1, "max_rounds must be at least 1");
  RAMA_REQUIRE(cfg.max_cycle_length >= 3, "max_cycle_length must be at least 3");
  const int64_t n0 = g.n;
  int nr = 0;
  res = SolveResult();
  const double nan = std::nan("");

  if (cfg.mode == 3) {  // D: solver.py:211-240
    RAMA_REQUIRE(cfg.separation_rounds == 1,
                 "separation_rounds > 1 (extend_separation) is not implemented in the B200 build yet");
    auto t0 = clk::now();
    CycleRows cyc;
    separate(ctx, g, cfg.max_cycle_length, cyc);
    DualState st;
    triangulate(ctx, g, cyc, st);
    message_passing(ctx, st, cfg.mp_iterations);
    double lb = lower_bound(ctx, st);
    iota(ctx, labels, n0);
    push(trace, max_trace, nr, RoundInfo{1, 3, n0, st.m_aug, st.T, lb, 1, 0, ms_since(t0)});
    res.lb = lb;
    res.lb_finite = true;
    res.primal = clustering_cost(ctx, g, labels);
    res.n_rounds = nr;
    return;
  }

  if (cfg.mode == 4) {  // GAEC: iterated max-edge contraction (contraction.py:397, one join per round)
    auto t0 = clk::now();
    iota(ctx, labels, n0);
    Graph cur = copy_graph(ctx, g);
    while (true) {
      StepResult step;
      contraction_step(ctx, cur.view(), 0, cfg.switch_fraction, step);
      if (step.identity) break;
      compose(ctx, labels, n0, step.map.p);
      cur = std::move(step.next);
    }
    push(trace, max_trace, nr, RoundInfo{1, 4, n0, g.m, 0, nan, 0, n0 - cur.n, ms_since(t0)});
    res.primal = clustering_cost(ctx, g, labels);
    res.n_rounds = nr;
    return;
  }

  const bool dual = (cfg.mode == 1 || cfg.mode == 2);
  iota(ctx, labels, n0);  // f_total
  Graph cur = copy_graph(ctx, g);
  double lb = nan;
  for (int rnd = 1; rnd <= cfg.max_rounds; rnd++) {
    auto t0 = clk::now();
    int64_t nodes_before = cur.n, edges_before = cur.m, T = 0;
    double lb_r = nan;
    StepResult step;
    if (dual) {
      CycleRows cyc;
      separate(ctx, cur.view(), cfg.max_cycle_length, cyc);
      DualState st;
      triangulate(ctx, cur.view(), cyc, st);
      message_passing(ctx, st, cfg.mp_iterations);
      lb_r = lower_bound(ctx, st);
      T = st.T;
      if (rnd == 1) lb = lb_r;
      Graph rep = reparametrized_graph(ctx, st);
      contraction_step(ctx, rep.view(), 3, cfg.switch_fraction, step);
    } else {
      contraction_step(ctx, cur.view(), 3, cfg.switch_fraction, step);
    }
    ctx.sync();
    push(trace, max_trace, nr,
         RoundInfo{rnd, dual ? 1 : 0, nodes_before, edges_before, T, lb_r, (dual && rnd == 1) ? 1 : 0,
                   nodes_before - step.num_targets, ms_since(t0)});
    if (step.identity) break;
    compose(ctx, labels, n0, step.map.p);
    cur = std::move(step.next);
    if (cur.n <= 1) break;
  }
  if (dual) {
    auto t0 = clk::now();
    Graph quotient = contract(ctx, g, labels, cur.n, nullptr);
    Buf<int32_t> fc(quotient.n > 0 ? quotient.n : 1, ctx);
    int64_t nt = handshake_cleanup(ctx, quotient.view(), fc.p);
    compose(ctx, labels, n0, fc.p);
    ctx.sync();
    push(trace, max_trace, nr,
         RoundInfo{nr + 1, 2, quotient.n, quotient.m, 0, nan, 0, quotient.n - nt, ms_since(t0)});
    res.lb = lb;
    res.lb_finite = true;
  }
  res.primal = clustering_cost(ctx, g, labels);
  res.n_rounds = nr;
}

}  // namespace rama
