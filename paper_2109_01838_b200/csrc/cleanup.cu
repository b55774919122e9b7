// PD cleanup (solver.py:187-207) -- DESIGN.md
// deviation D1.
//
// The reference finishes PD with a sequential lazy-heap GAEC on the
// quotient (contraction.py:397-452).  Here the quotient is contracted by
// repeated handshake rounds under its own costs, which is GAEC's parallel
// form: a pair is merged when its edge is the maximum positive edge at both
// ends (the select_matching rule, contraction.py:207: ties toward the
// smaller neighbour id).  Semantics (oracle: orc_cleanup_handshake):
//   * a cluster is named by its smallest member ("canonical id", minid);
//     every tie-break compares canonical ids;
//   * parallel edges created by a merge fold into their smallest edge slot
//     with a sequential sum in ascending slot order.
//
// Execution: ONE cooperative persistent kernel (one CTA per SM, grid.sync()
// between phases) runs round after round with no host round trip.  State:
//   * edge slots (u, v, c, alive) over INTERNAL cluster ids.  A pair's
//     internal representative is the larger cluster (member count, ties by
//     canonical id), so only the smaller side's edges are rewritten
//     (union-by-size: O(m log n) rewrites even when one cluster absorbs a
//     neighbour per round for hundreds of rounds, as on 3-D grids);
//   * P, the alive positive slots (the only ones that vote);
//   * per-cluster incidence rows in a bump-allocated pool (lazy: dead slots
//     are skipped, representatives get a compacted row when they merge).
// A round: votes over P, mutual pairs, R = alive slots of the absorbed
// clusters, rewrite R to the representatives, group equal (u', v') in a
// global hash table (the one slot outside R with the same key, if any, is
// found in the representative's row), fold each group in slot order,
// rebuild the representatives' rows.  The host only rebuilds P and the rows
// when the pool runs out.
#include "internal.h"

#include <cooperative_groups.h>

#include <chrono>

namespace rama {

// representative ordering: larger cluster first, then smaller canonical id
__device__ __forceinline__ bool rep_first(int32_t sa, int32_t ma, int32_t sb, int32_t mb) {
  return sa > sb || (sa == sb && ma < mb);
}

__device__ __forceinline__ uint64_t pair_key(int32_t a, int32_t b) {
  int32_t lo = a < b ? a : b, hi = a < b ? b : a;
  return ((uint64_t)(uint32_t)lo << 32) | (uint64_t)(uint32_t)hi;
}

__device__ __forceinline__ uint32_t key_hash(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  return (uint32_t)k;
}

constexpr int kThreads = 512;
constexpr uint64_t kEmpty = ~0ULL;

enum CleanupStatus : int32_t { kRunning = 0, kDone = 1, kPoolFull = 2 };

// device scalars (int32)
enum {
  SC_NPAIRS = 0,  // committed pairs (pair list length)
  SC_NP = 1,      // |P| of the current buffer
  SC_WHICH = 2,   // current P buffer
  SC_POOL = 3,    // pool top
  SC_STATUS = 4,
  SC_ROUNDS = 5,
  SC_RPAIRS = 6,  // this round: pairs found
  SC_RNT = 7,     // this round: |R|
  SC_RSUM = 8,    // this round: sum of absorbed row lengths
  SC_RREP = 9,    // this round: sum of representative row lengths
  SC_RNP2 = 10,   // this round: next |P|
  SC_MEM = 11,    // this round: member-list top
  SC_COUNT = 16
};

struct Args {
  int32_t* u;
  int32_t* v;
  double* c;
  uint8_t* alive;
  int32_t* tmark;          // per slot, clean (0) between rounds
  unsigned long long* bc;  // per node, clean (0) between rounds; also the row fill cursor
  int32_t* bn;             // per node, "none" (>= n) between rounds
  int32_t* rp;             // per node, -1 unless in a pair this round
  int32_t* minid;          // per node: canonical id of the cluster
  int32_t* size;           // per node: member count
  int32_t* P0;             // positive alive slots (double buffered, capacity m)
  int32_t* P1;
  int32_t* row_off;        // per node: incidence row (slot ids, may hold dead slots) in pool
  int32_t* row_len;
  int32_t* pool;
  int64_t pool_cap;
  int32_t* pr;             // global pair list (representative, absorbed)
  int32_t* pa;
  int32_t* ooff;           // per pair of the round: representative's old row
  int32_t* olen;
  int32_t* apref;          // prefix of absorbed row lengths (npairs + 1)
  int32_t* rpref;          // prefix of representative row lengths
  int32_t* R;              // rewritten slots of the round
  uint64_t* Rk;            // their new keys (kEmpty: became internal)
  int32_t* Rg;             // their group (hash position)
  uint64_t* hkey;          // group hash table (capacity hcap, power of two)
  int32_t* hcnt;           // R members per group
  int32_t* hhead;          // smallest R slot per group
  int32_t* hext;           // the slot outside R with the same key, or -1
  int32_t* hoff;           // member list offset (groups with >= 2 R members)
  int32_t* hfill;
  int32_t* mem;            // member lists
  uint32_t hmask;
  int32_t* sc;             // device scalars, SC_*
};

// arrays written or updated with atomics earlier in the same launch by
// other SMs are read around L1
#define LD(p) __ldcg(p)

__device__ __forceinline__ int32_t rep_of(const int32_t* rp, int32_t y) {
  int32_t r = LD(rp + y);
  return r < 0 ? y : r;
}

// owner k of flattened position i: pref[k] <= i < pref[k + 1]
__device__ __forceinline__ int32_t owner_of(const int32_t* pref, int32_t n, int32_t i) {
  int32_t lo = 0, hi = n;
  while (hi - lo > 1) {
    int32_t mid = (lo + hi) >> 1;
    if (LD(pref + mid) <= i) lo = mid; else hi = mid;
  }
  return lo;
}

// CTA-wide exclusive scan of f(k), k < n, into pref[0..n]
template <class F>
__device__ void block_prefix(int32_t* pref, int32_t n, F f) {
  __shared__ int32_t part[kThreads / 32 + 1];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int32_t b0 = 0; b0 < n; b0 += blockDim.x) {
    int32_t k = b0 + threadIdx.x;
    int32_t x = k < n ? f(k) : 0;
    int32_t incl = x;
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) part[w] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      int32_t acc = 0;
      for (int i = 0; i < nw; i++) { int32_t t = part[i]; part[i] = acc; acc += t; }
      part[nw] = acc;
    }
    __syncthreads();
    if (k < n) pref[k] = carry + part[w] + incl - x;
    __syncthreads();
    if (threadIdx.x == 0) carry += part[nw];
    __syncthreads();
  }
  if (threadIdx.x == 0) pref[n] = carry;
}

// group position of key k, inserting it
__device__ __forceinline__ int32_t h_insert(const Args& A, uint64_t k) {
  uint32_t h = key_hash(k) & A.hmask;
  while (true) {
    unsigned long long old = atomicCAS((unsigned long long*)(A.hkey + h), (unsigned long long)kEmpty,
                                       (unsigned long long)k);
    if (old == kEmpty || old == k) return (int32_t)h;
    h = (h + 1) & A.hmask;
  }
}

// group position of an existing key, or -1
__device__ __forceinline__ int32_t h_find(const Args& A, uint64_t k) {
  uint32_t h = key_hash(k) & A.hmask;
  while (true) {
    uint64_t x = LD(A.hkey + h);
    if (x == k) return (int32_t)h;
    if (x == kEmpty) return -1;
    h = (h + 1) & A.hmask;
  }
}

__global__ void __launch_bounds__(kThreads, 1) k_cl_rounds(Args A) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  int32_t* sc = A.sc;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t GT = (int64_t)gridDim.x * blockDim.x;
  while (true) {
    const int32_t np = LD(sc + SC_NP);
    const int32_t which = LD(sc + SC_WHICH);
    const int32_t base = LD(sc + SC_NPAIRS);
    const int32_t* P = which ? A.P1 : A.P0;
    int32_t* P2 = which ? A.P0 : A.P1;
    // ---- handshake votes over the positive slots (contraction.py:207 rule)
    for (int64_t i = gtid; i < np; i += GT) {
      int32_t s = LD(P + i);
      unsigned long long bits = dbits(LD(A.c + s));
      atomicMax(A.bc + LD(A.u + s), bits);
      atomicMax(A.bc + LD(A.v + s), bits);
    }
    grid.sync();
    for (int64_t i = gtid; i < np; i += GT) {
      int32_t s = LD(P + i);
      unsigned long long bits = dbits(LD(A.c + s));
      int32_t a = LD(A.u + s), b = LD(A.v + s);
      if (bits == LD(A.bc + a)) atomicMin(A.bn + a, LD(A.minid + b));
      if (bits == LD(A.bc + b)) atomicMin(A.bn + b, LD(A.minid + a));
    }
    grid.sync();
    for (int64_t i = gtid; i < np; i += GT) {  // mutual pairs: their slot is both ends' best
      int32_t s = LD(P + i);
      int32_t a = LD(A.u + s), b = LD(A.v + s);
      int32_t ma = LD(A.minid + a), mb = LD(A.minid + b);
      if (LD(A.bn + a) == mb && LD(A.bn + b) == ma) {
        int32_t r = rep_first(LD(A.size + a), ma, LD(A.size + b), mb) ? a : b;
        int32_t t = r == a ? b : a;
        int32_t k = atomicAdd(sc + SC_RPAIRS, 1);
        A.pr[base + k] = r;
        A.pa[base + k] = t;
        atomicAdd(sc + SC_RSUM, LD(A.row_len + t));
        atomicAdd(sc + SC_RREP, LD(A.row_len + r));
      }
    }
    grid.sync();
    for (int64_t i = gtid; i < np; i += GT) {  // votes back to clean
      int32_t s = LD(P + i);
      int32_t a = LD(A.u + s), b = LD(A.v + s);
      A.bc[a] = 0ULL;
      A.bc[b] = 0ULL;
      A.bn[a] = 0x7fffffff;
      A.bn[b] = 0x7fffffff;
    }
    const int32_t npairs = LD(sc + SC_RPAIRS);
    int32_t stop = 0;
    if (npairs == 0) stop = kDone;
    else if ((int64_t)LD(sc + SC_POOL) + LD(sc + SC_RREP) + LD(sc + SC_RSUM) > A.pool_cap) stop = kPoolFull;
    if (stop) {  // nothing was modified: the host rebuilds the rows and the round is redone
      grid.sync();
      if (gtid == 0) {
        sc[SC_STATUS] = stop;
        sc[SC_RPAIRS] = 0; sc[SC_RSUM] = 0; sc[SC_RREP] = 0;
      }
      break;
    }
    const int32_t* pr = A.pr + base;
    const int32_t* pa = A.pa + base;
    for (int64_t k = gtid; k < npairs; k += GT) {
      int32_t r = LD(pr + k), t = LD(pa + k);
      A.rp[r] = r;
      A.rp[t] = r;
      A.ooff[k] = LD(A.row_off + r);
      A.olen[k] = LD(A.row_len + r);
    }
    if (blockIdx.x == 0) {
      block_prefix(A.apref, npairs, [&](int32_t k) { return LD(A.row_len + LD(pa + k)); });
      block_prefix(A.rpref, npairs, [&](int32_t k) { return LD(A.row_len + LD(pr + k)); });
    }
    grid.sync();
    const int32_t asum = LD(A.apref + npairs), rsum = LD(A.rpref + npairs);
    // ---- R = alive slots of the absorbed clusters (deduplicated), flattened
    for (int64_t i = gtid; i < asum; i += GT) {
      int32_t k = owner_of(A.apref, npairs, (int32_t)i);
      int32_t y = LD(pa + k);
      int32_t s = LD(A.pool + LD(A.row_off + y) + ((int32_t)i - LD(A.apref + k)));
      if (LD(A.alive + s) && atomicExch(A.tmark + s, 1) == 0) A.R[atomicAdd(sc + SC_RNT, 1)] = s;
    }
    grid.sync();
    const int32_t nt = LD(sc + SC_RNT);
    // ---- rewrite R to the representatives (internal slots die) and group
    // equal keys.  tmark = 1 | mask of the new endpoints the slot was already
    // incident to (2: low, 4: high): the row update appends only where new.
    for (int64_t i = gtid; i < nt; i += GT) {
      int32_t s = LD(A.R + i);
      int32_t x = LD(A.u + s), y = LD(A.v + s);
      int32_t a = rep_of(A.rp, x), b = rep_of(A.rp, y);
      if (a == b) {
        A.alive[s] = 0;
        A.Rk[i] = kEmpty;
        A.Rg[i] = -1;
      } else {
        int32_t lo = min(a, b), hi = max(a, b);
        A.u[s] = lo;
        A.v[s] = hi;
        A.tmark[s] = 1 | ((lo == x || lo == y) ? 2 : 0) | ((hi == x || hi == y) ? 4 : 0);
        uint64_t key = pair_key(lo, hi);
        A.Rk[i] = key;
        int32_t g = h_insert(A, key);
        A.Rg[i] = g;
        atomicAdd(A.hcnt + g, 1);
        atomicMin(A.hhead + g, s);
      }
    }
    grid.sync();
    // ---- the slot outside R with a group's key: it joins a representative
    // with a cluster that is not absorbed, keeps its key, and sits in that
    // representative's row (at most one per key).  Groups with >= 2 R
    // members reserve their member list.
    for (int64_t i = gtid; i < rsum; i += GT) {
      int32_t k = owner_of(A.rpref, npairs, (int32_t)i);
      int32_t s = LD(A.pool + LD(A.ooff + k) + ((int32_t)i - LD(A.rpref + k)));
      if (!LD(A.alive + s) || LD(A.tmark + s)) continue;
      int32_t g = h_find(A, pair_key(LD(A.u + s), LD(A.v + s)));
      if (g >= 0 && atomicCAS(A.hext + g, -1, s) == -1) A.tmark[s] = 8;
    }
    for (int64_t i = gtid; i < nt; i += GT) {
      int32_t g = LD(A.Rg + i);
      if (g < 0 || LD(A.hhead + g) != LD(A.R + i)) continue;
      int32_t cnt = LD(A.hcnt + g);
      if (cnt >= 2) A.hoff[g] = atomicAdd(sc + SC_MEM, cnt);
    }
    grid.sync();
    for (int64_t i = gtid; i < nt; i += GT) {
      int32_t g = LD(A.Rg + i);
      if (g < 0 || LD(A.hcnt + g) < 2) continue;
      A.mem[LD(A.hoff + g) + atomicAdd(A.hfill + g, 1)] = LD(A.R + i);
    }
    grid.sync();
    // ---- fold each group (R members + the outside slot) into its smallest
    // slot, sequential sum in slot order; survivors enter the next P when
    // positive, untouched positive slots stay
    for (int64_t i = gtid; i < nt; i += GT) {
      const int32_t g = LD(A.Rg + i);
      const int32_t s0 = LD(A.R + i);
      if (g < 0 || LD(A.hhead + g) != s0) continue;
      const int32_t cnt = LD(A.hcnt + g), ext = LD(A.hext + g);
      if (cnt == 1 && ext < 0) {
        if (LD(A.c + s0) > 0.0) P2[atomicAdd(sc + SC_RNP2, 1)] = s0;
        continue;
      }
      const int32_t* list = cnt >= 2 ? A.mem + LD(A.hoff + g) : nullptr;
      const int32_t total = cnt + (ext >= 0 ? 1 : 0);
      int32_t surv = s0;
      if (total <= 16) {  // small groups: insertion sort in registers / local memory
        int32_t buf[16];
        int32_t k = 0;
        if (list) {
          for (int32_t j = 0; j < cnt; j++) buf[k++] = LD(list + j);
        } else {
          buf[k++] = s0;
        }
        if (ext >= 0) buf[k++] = ext;
        for (int32_t a = 1; a < k; a++) {
          int32_t x = buf[a], b = a - 1;
          while (b >= 0 && buf[b] > x) { buf[b + 1] = buf[b]; b--; }
          buf[b + 1] = x;
        }
        surv = buf[0];
        double acc = LD(A.c + buf[0]);
        for (int32_t j = 1; j < k; j++) {
          acc = __dadd_rn(acc, LD(A.c + buf[j]));
          A.alive[buf[j]] = 0;
        }
        A.c[surv] = acc;
      } else {  // large group (rare): repeated minimum extraction over the list
        int32_t prev = -1;
        double acc = 0.0;
        for (int32_t j = 0; j < total; j++) {
          int32_t nxt = 0x7fffffff;
          for (int32_t t = 0; t < cnt; t++) {
            int32_t x = LD(list + t);
            if (x > prev && x < nxt) nxt = x;
          }
          if (ext > prev && ext < nxt) nxt = ext;
          if (j == 0) {
            surv = nxt;
            acc = LD(A.c + nxt);
          } else {
            acc = __dadd_rn(acc, LD(A.c + nxt));
            A.alive[nxt] = 0;
          }
          prev = nxt;
        }
        A.c[surv] = acc;
      }
      if (LD(A.c + surv) > 0.0) P2[atomicAdd(sc + SC_RNP2, 1)] = surv;
    }
    for (int64_t i = gtid; i < np; i += GT) {
      int32_t s = LD(P + i);
      if (!LD(A.tmark + s)) P2[atomicAdd(sc + SC_RNP2, 1)] = s;
    }
    grid.sync();
    // ---- rows: a representative keeps its alive slots and gains the R
    // survivors new to it (bc counts, then serves as the fill cursor)
    for (int64_t i = gtid; i < rsum; i += GT) {
      int32_t k = owner_of(A.rpref, npairs, (int32_t)i);
      int32_t s = LD(A.pool + LD(A.ooff + k) + ((int32_t)i - LD(A.rpref + k)));
      if (LD(A.alive + s)) atomicAdd(A.bc + LD(pr + k), 1ULL);
    }
    for (int64_t i = gtid; i < nt; i += GT) {
      int32_t s = LD(A.R + i);
      if (LD(A.Rk + i) == kEmpty || !LD(A.alive + s)) continue;
      int32_t mk = LD(A.tmark + s);
      int32_t a = LD(A.u + s), b = LD(A.v + s);
      if (LD(A.rp + a) == a && !(mk & 2)) atomicAdd(A.bc + a, 1ULL);
      if (LD(A.rp + b) == b && !(mk & 4)) atomicAdd(A.bc + b, 1ULL);
    }
    grid.sync();
    for (int64_t k = gtid; k < npairs; k += GT) {  // new rows past the pool top
      int32_t x = LD(pr + k);
      int32_t cnt = (int32_t)LD(A.bc + x);
      A.row_off[x] = atomicAdd(sc + SC_POOL, cnt);
      A.row_len[x] = cnt;
      A.bc[x] = 0ULL;
    }
    grid.sync();
    for (int64_t i = gtid; i < rsum; i += GT) {
      int32_t k = owner_of(A.rpref, npairs, (int32_t)i);
      int32_t s = LD(A.pool + LD(A.ooff + k) + ((int32_t)i - LD(A.rpref + k)));
      int32_t x = LD(pr + k);
      if (LD(A.alive + s)) A.pool[LD(A.row_off + x) + (int32_t)atomicAdd(A.bc + x, 1ULL)] = s;
    }
    for (int64_t i = gtid; i < nt; i += GT) {
      int32_t s = LD(A.R + i);
      if (LD(A.Rk + i) == kEmpty || !LD(A.alive + s)) continue;
      int32_t mk = LD(A.tmark + s);
      int32_t a = LD(A.u + s), b = LD(A.v + s);
      if (LD(A.rp + a) == a && !(mk & 2)) A.pool[LD(A.row_off + a) + (int32_t)atomicAdd(A.bc + a, 1ULL)] = s;
      if (LD(A.rp + b) == b && !(mk & 4)) A.pool[LD(A.row_off + b) + (int32_t)atomicAdd(A.bc + b, 1ULL)] = s;
    }
    grid.sync();
    // ---- back to clean; cluster bookkeeping
    for (int64_t i = gtid; i < nt; i += GT) {
      A.tmark[LD(A.R + i)] = 0;
      int32_t g = LD(A.Rg + i);
      if (g < 0) continue;
      int32_t e = LD(A.hext + g);
      if (e >= 0) A.tmark[e] = 0;
    }
    for (int64_t k = gtid; k < npairs; k += GT) {
      int32_t x = LD(pr + k), t = LD(pa + k);
      A.bc[x] = 0ULL;
      A.row_len[t] = 0;
      A.size[x] = LD(A.size + x) + LD(A.size + t);
      A.minid[x] = min(LD(A.minid + x), LD(A.minid + t));
    }
    grid.sync();
    for (int64_t i = gtid; i < nt; i += GT) {  // hash groups back to empty (after the ext reads)
      int32_t g = LD(A.Rg + i);
      if (g < 0) continue;
      A.hkey[g] = kEmpty;
      A.hcnt[g] = 0;
      A.hhead[g] = 0x7fffffff;
      A.hext[g] = -1;
      A.hfill[g] = 0;
    }
    for (int64_t k = gtid; k < npairs; k += GT) {
      A.rp[LD(pr + k)] = -1;
      A.rp[LD(pa + k)] = -1;
    }
    if (gtid == 0) {
      sc[SC_NPAIRS] = base + npairs;
      sc[SC_NP] = LD(sc + SC_RNP2);
      sc[SC_WHICH] = which ^ 1;
      sc[SC_ROUNDS] += 1;
      sc[SC_RPAIRS] = 0; sc[SC_RNT] = 0; sc[SC_RSUM] = 0; sc[SC_RNP2] = 0; sc[SC_RREP] = 0; sc[SC_MEM] = 0;
    }
    grid.sync();
  }
}
#undef LD

__global__ void k_cl_fill_i32(int32_t* x, int64_t n, int32_t val) {
  GRID_STRIDE(i, n) x[i] = val;
}

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

// RAMA_CLEANUP_POOL=<k>: pool slack in entries (tests shrink it to force the
// rebuild path); default max(8 * arcs, 4M)
static int64_t pool_slack_override() {
  static const int64_t v = [] {
    const char* e = getenv("RAMA_CLEANUP_POOL");
    return e ? (int64_t)atoll(e) : (int64_t)-1;
  }();
  return v;
}

int64_t handshake_cleanup(Ctx& ctx, const GraphView& q, int32_t* fc) {
  ProfScope prof(ctx.s, kFamCleanup);
  const int64_t n = q.n, m = q.m;
  if (n == 0) return 0;
  if (m == 0) {
    iota(ctx, fc, n);
    return n;
  }
  auto t_start = std::chrono::steady_clock::now();
  Buf<int32_t> u(m, ctx), v(m, ctx);
  Buf<double> c(m, ctx);
  copy_d2d(ctx, u.p, q.u, m);
  copy_d2d(ctx, v.p, q.v, m);
  copy_d2d(ctx, c.p, q.c, m);
  Buf<uint8_t> alive(m, ctx);
  alive.fill_bytes(1);
  Buf<unsigned long long> bc(n, ctx);
  bc.zero();
  Buf<int32_t> bn(n, ctx), pr(n, ctx), pa(n, ctx), rp(n, ctx), minid(n, ctx), size(n, ctx), tmark(m, ctx);
  bn.fill_bytes(0x7f);
  rp.fill_bytes(0xff);
  tmark.zero();
  iota(ctx, minid.p, n);
  RAMA_KERNEL(ctx, k_cl_fill_i32, n, size.p, n, 1);
  Buf<int32_t> P0(m, ctx), P1(m, ctx), ooff(n, ctx), olen(n, ctx), apref(n + 1, ctx), rpref(n + 1, ctx);
  Buf<int32_t> R(m, ctx), Rg(m, ctx), mem(m, ctx);
  Buf<uint64_t> Rk(m, ctx);
  uint32_t hcap = 1024;
  while ((int64_t)hcap < 2 * m) hcap <<= 1;
  Buf<uint64_t> hkey(hcap, ctx);
  Buf<int32_t> hcnt(hcap, ctx), hhead(hcap, ctx), hext(hcap, ctx), hoff(hcap, ctx), hfill(hcap, ctx);
  hkey.fill_bytes(0xff);
  hcnt.zero();
  hfill.zero();
  hext.fill_bytes(0xff);
  RAMA_KERNEL(ctx, k_cl_fill_i32, hcap, hhead.p, hcap, 0x7fffffff);
  Buf<int32_t> sc(SC_COUNT, ctx);
  static int grid_blocks = 0;
  if (!grid_blocks) {
    int dev = 0, sms = 0, per_sm = 0;
    RAMA_CUDA(cudaGetDevice(&dev));
    RAMA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    RAMA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cl_rounds, kThreads, 0));
    RAMA_REQUIRE(per_sm >= 1, "cleanup kernel cannot be resident");
    grid_blocks = sms;  // one CTA per SM
  }
  int64_t total = 0;
  int launches = 0, rounds = 0;
  while (true) {
    // P and the rows, from the current slots
    Buf<uint8_t> pf(m, ctx);
    RAMA_KERNEL(ctx, k_cl_posflag, m, c.p, alive.p, m, pf.p);
    Buf<int32_t> Pl;
    int64_t np = compact_indices(ctx, pf.p, m, Pl);
    if (np == 0) break;
    copy_d2d(ctx, P0.p, Pl.p, np);
    Buf<int32_t> deg(n, ctx), off(n + 1, ctx), cur(n, ctx);
    deg.zero();
    cur.zero();
    RAMA_KERNEL(ctx, k_cl_degree, m, u.p, v.p, alive.p, m, deg.p);
    int64_t arcs = exclusive_scan(ctx, deg.p, off.p, n, true);
    int64_t slack = pool_slack_override() >= 0 ? pool_slack_override() : std::max<int64_t>(8 * arcs, 1 << 22);
    int64_t cap = 2 * arcs + slack;
    if (cap > 0x7fffffffLL) cap = 0x7fffffffLL;
    Buf<int32_t> pool(cap, ctx);
    RAMA_KERNEL(ctx, k_cl_fill_rows, m, u.p, v.p, alive.p, m, off.p, cur.p, pool.p);
    int32_t init[SC_COUNT] = {0};
    init[SC_NPAIRS] = (int32_t)total;
    init[SC_NP] = (int32_t)np;
    init[SC_POOL] = (int32_t)arcs;
    RAMA_CUDA(cudaMemcpyAsync(sc.p, init, sizeof(init), cudaMemcpyHostToDevice, ctx.s));
    Args A;
    A.u = u.p; A.v = v.p; A.c = c.p; A.alive = alive.p; A.tmark = tmark.p; A.bc = bc.p; A.bn = bn.p;
    A.rp = rp.p; A.minid = minid.p; A.size = size.p; A.P0 = P0.p; A.P1 = P1.p;
    A.row_off = off.p; A.row_len = deg.p; A.pool = pool.p; A.pool_cap = cap;
    A.pr = pr.p; A.pa = pa.p; A.ooff = ooff.p; A.olen = olen.p; A.apref = apref.p; A.rpref = rpref.p;
    A.R = R.p; A.Rk = Rk.p; A.Rg = Rg.p; A.hkey = hkey.p; A.hcnt = hcnt.p; A.hhead = hhead.p; A.hext = hext.p;
    A.hoff = hoff.p; A.hfill = hfill.p; A.mem = mem.p; A.hmask = hcap - 1; A.sc = sc.p;
    if (trace_print()) fprintf(stderr, "[rama] k_cl_rounds np=%lld\n", (long long)np);
    {
      KernelScope ks(ctx.s, "k_cl_rounds", 0.0);
      void* kargs[] = {&A};
      RAMA_CUDA(cudaLaunchCooperativeKernel((const void*)k_cl_rounds, dim3(grid_blocks), dim3(kThreads), kargs, 0,
                                            ctx.s));
    }
    ctx.launches++;
    launches++;
    int32_t st[SC_COUNT];
    RAMA_CUDA(cudaMemcpyAsync(ctx.pinned, sc.p, sizeof(st), cudaMemcpyDeviceToHost, ctx.s));
    ctx.sync();
    memcpy(st, ctx.pinned, sizeof(st));
    total = st[SC_NPAIRS];
    rounds += st[SC_ROUNDS];
    if (st[SC_STATUS] == kDone) break;
    RAMA_REQUIRE(st[SC_STATUS] == kPoolFull, "cleanup kernel ended in an unknown state");
  }
  if (getenv("RAMA_CLEANUP_STATS"))
    fprintf(stderr, "[rama] cleanup n %lld m %lld: %d rounds in %d launches, %lld pairs, %.2f ms\n", (long long)n,
            (long long)m, rounds, launches, (long long)total,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
  return components(ctx, n, pr.p, pa.p, total, fc);
}

}  // namespace rama
