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
//     internal representative is the cluster with the longer incidence row
//     (ties by canonical id), so only the shorter row is rewritten -- cheap
//     even when one cluster absorbs a neighbour per round for hundreds of
//     rounds, as on 3-D grids.  Internal ids never reach the results: every
//     tie-break compares canonical ids;
//   * P, the alive positive slots (the only ones that vote);
//   * per-cluster incidence rows in a bump-allocated pool (lazy: dead slots
//     stay until the row is reallocated; rows grow by doubling);
//   * an edge hash holding every alive slot under its current key.
// A round is five phases: (1) votes over P, one 128-bit atomic max of
// (cost, neighbour id) per endpoint; (2) mutual pairs, each getting its
// index and the offset of its absorbed row from one warp-aggregated packed
// atomic; (3) R = alive slots of the absorbed clusters, and representatives
// whose row could overflow get a larger one; (4) rewrite R to the
// representatives, group equal keys in a hash table, find each group's slot
// outside R in the edge hash; (5) fold each group in slot order, append
// survivors to the representatives' rows.  The round's marks are cleared in
// the next round's phase 1.  The host only rebuilds P, the rows and the
// edge hash when the pool or the hash runs out.
#include "internal.h"
#include "compact.cuh"

#include <cooperative_groups.h>

#include <chrono>
#include <vector>

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
constexpr int32_t kBigRow = 2048;  // rows longer than this are copied by a whole CTA

enum CleanupStatus : int32_t { kRunning = 0, kDone = 1, kPoolFull = 2 };

// device scalars (int32).  Per-round counters live in two banks (round
// parity): a bank is zeroed one round after its last use, so no extra grid
// barrier is needed for the reset.
enum {
  SC_NPAIRS = 0,  // committed pairs (pair list length)
  SC_NP = 1,      // |P| at launch
  SC_POOL = 2,    // pool top
  SC_STATUS = 3,
  SC_ROUNDS = 4,  // rounds run by the launch
  SC_EFILL = 5,   // edge hash entries (upper bound)
  SC_RREP = 6,    // + bank: sum of representative row lengths
  SC_RNT = 8,     // + bank: |R|
  SC_RNP2 = 10,   // + bank: next |P|
  SC_COUNT = 16
};

struct alignas(32) Group {  // one sector per group
  unsigned long long key;
  int32_t cnt;   // R members
  int32_t head;  // smallest R slot
  int32_t ext;   // the slot outside R with the same key, or -1
  int32_t list;  // first member (R index) of the group's list, or -1
  int32_t pad[2];
  __host__ __device__ static Group empty() { return Group{~0ULL, 0, 0x7fffffff, -1, -1, {0, 0}}; }
};

struct Args {
  int32_t* u;
  int32_t* v;
  double* c;
  uint8_t* alive;
  int32_t* tmark;          // per slot, clean (0) between rounds; R: 1 | 2/4 (endpoint kept); ext: 8
  ulonglong2* vote;        // per node, 0 between rounds: max of (cost bits, ~canonical id of the neighbour)
  int32_t* rp;             // per node, -1 unless in a pair of this round
  int32_t* minid;          // per node: canonical id of the cluster
  int32_t* size;           // per node: member count
  int32_t* P0;             // positive alive slots (double buffered, capacity m)
  int32_t* P1;
  int32_t* row_off;        // per node: incidence row (slot ids, may hold dead slots) in pool
  int32_t* row_len;
  int32_t* row_cap;
  int32_t* pool;
  int64_t pool_cap;
  int32_t* pr;             // global pair list (representative, absorbed)
  int32_t* pa;
  int32_t* apref;          // per pair of the round: offset of its absorbed row in the flattened R scan
  unsigned long long* pk;  // per bank: (pairs << 32) | sum of absorbed row lengths
  int32_t* R;              // rewritten slots of the round
  int32_t* Rg;             // their group (hash position), -1: became internal
  int32_t* Rnext;          // group member list (R indices, linked)
  Group* grp;              // group hash table (capacity hmask + 1), clean between rounds; a round
  uint32_t hmask;          //   uses only its first 2 |R| entries or so, which stay in L2
  int32_t* eh;             // edge hash of slot ids: every alive slot under its current key (stale entries
                           //   of dead or re-keyed slots stay and are skipped)
  uint32_t emask;
  int32_t* sc;             // device scalars, SC_*
  long long* trace;        // RAMA_CLEANUP_STATS=2: per round {np, npairs, nt, asum, rrep, t_ns}
  long long* ptrace;       // RAMA_CLEANUP_STATS=3: per round, the end time of each of the 5 phases
  int32_t trace_cap;
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

// the group table positions a round uses: 2 |R| rounded up (|R| <= asum)
__device__ __forceinline__ uint32_t round_mask(int32_t asum, uint32_t hmask) {
  uint32_t m = 4095;
  while ((int64_t)m + 1 < 2 * (int64_t)asum && m < hmask) m = 2 * m + 1;
  return m < hmask ? m : hmask;
}

// group position of key k, inserting it
__device__ __forceinline__ int32_t h_insert(const Args& A, uint64_t k, uint32_t mask) {
  uint32_t h = key_hash(k) & mask;
  while (true) {
    unsigned long long old = atomicCAS((unsigned long long*)&A.grp[h].key, (unsigned long long)kEmpty,
                                       (unsigned long long)k);
    if (old == kEmpty || old == k) return (int32_t)h;
    h = (h + 1) & mask;
  }
}

// edge hash: a new entry (entries of dead or re-keyed slots stay; readers validate)
__device__ __forceinline__ void e_insert(const Args& A, uint64_t k, int32_t s) {
  uint32_t h = key_hash(k) & A.emask;
  while (atomicCAS(A.eh + h, -1, s) != -1) h = (h + 1) & A.emask;
}

// the alive slot outside R whose current key is k, or -1 (at most one: alive
// keys are unique between rounds)
__device__ __forceinline__ int32_t e_find(const Args& A, uint64_t k) {
  uint32_t h = key_hash(k) & A.emask;
  while (true) {
    int32_t s = LD(A.eh + h);
    if (s < 0) return -1;
    if (pair_key(LD(A.u + s), LD(A.v + s)) == k && LD(A.alive + s) && !(LD(A.tmark + s) & 1)) return s;
    h = (h + 1) & A.emask;
  }
}

__device__ __forceinline__ unsigned lanes_below() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// warp-aggregated slot in a global list: every lane with `take` gets a
// distinct index (all 32 lanes must call)
__device__ __forceinline__ int32_t warp_claim(int32_t* counter, bool take) {
  const unsigned bal = __ballot_sync(0xffffffffu, take);
  if (!bal) return -1;
  const int leader = __ffs(bal) - 1;
  int32_t b = 0;
  if ((int)(threadIdx.x & 31) == leader) b = atomicAdd(counter, __popc(bal));
  b = __shfl_sync(0xffffffffu, b, leader);
  return take ? b + __popc(bal & lanes_below()) : -1;
}

// the vote a node casts for neighbour y over a slot of cost bits `bits`:
// larger cost first, then smaller canonical id (contraction.py:207)
__device__ __forceinline__ unsigned long long vote_lo(int32_t minid_y) {
  return (unsigned long long)(0xffffffffu - (uint32_t)minid_y);
}

// RAMA_CLEANUP_STATS=3: the time each phase of each round ends
#define PHASE_MARK(k)                                                                        \
  do {                                                                                       \
    if (A.ptrace && gtid == 0 && round0 + rounds < A.trace_cap) {                            \
      unsigned long long tns_;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tns_));                             \
      A.ptrace[5 * (int64_t)(round0 + rounds) + (k)] = (long long)tns_;                      \
    }                                                                                        \
  } while (0)

__global__ void __launch_bounds__(kThreads, 1) k_cl_rounds(Args A) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ int32_t s_small[kThreads], s_big[kThreads];
  __shared__ int32_t s_nsmall, s_nbig, s_cnt, s_off;
  int32_t* sc = A.sc;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t GT = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  // loop state, identical in every thread
  int32_t base = LD(sc + SC_NPAIRS), np = LD(sc + SC_NP), efill = LD(sc + SC_EFILL);
  const int32_t round0 = LD(sc + SC_ROUNDS);
  int32_t prev_base = base, prev_nt = 0, which = 0, rounds = 0;
  while (true) {
    const int q = rounds & 1;
    const int32_t* P = which ? A.P1 : A.P0;
    int32_t* P2 = which ? A.P0 : A.P1;
    // ---- 1. the last round's marks back to clean (the group's head resets
    // the group); handshake votes over the positive slots
    for (int64_t k = prev_base + gtid; k < base; k += GT) {
      A.rp[LD(A.pr + k)] = -1;
      A.rp[LD(A.pa + k)] = -1;
    }
    for (int64_t i = gtid; i < prev_nt; i += GT) {
      const int32_t s = LD(A.R + i), g = LD(A.Rg + i);
      A.tmark[s] = 0;
      if (g >= 0 && LD(&A.grp[g].head) == s) {
        int32_t e = LD(&A.grp[g].ext);
        if (e >= 0) A.tmark[e] = 0;
        A.grp[g] = Group::empty();
      }
    }
    for (int64_t i = gtid; i < np; i += GT) {
      int32_t s = LD(P + i);
      unsigned long long bits = dbits(LD(A.c + s));
      int32_t a = LD(A.u + s), b = LD(A.v + s);
      vote_max_pair(A.vote + a, vote_lo(LD(A.minid + b)), A.vote + b, vote_lo(LD(A.minid + a)), bits);
    }
    grid.sync();
    PHASE_MARK(0);
    // ---- 2. mutual pairs: the slot is both ends' vote.  One packed atomic
    // per warp gives each pair its index and the offset of its absorbed row.
    if (gtid == 0) {
      A.pk[q ^ 1] = 0ULL;
      sc[SC_RREP + (q ^ 1)] = 0;
      sc[SC_RNT + (q ^ 1)] = 0;
      sc[SC_RNP2 + (q ^ 1)] = 0;
    }
    for (int64_t i0 = gtid - lane; i0 < np; i0 += GT) {
      const int64_t i = i0 + lane;
      bool found = false;
      int32_t r = 0, t = 0, len = 0, rlen = 0;
      if (i < np) {
        int32_t s = LD(P + i);
        unsigned long long bits = dbits(LD(A.c + s));
        int32_t a = LD(A.u + s), b = LD(A.v + s);
        int32_t ma = LD(A.minid + a), mb = LD(A.minid + b);
        ulonglong2 va = __ldcg(A.vote + a), vb = __ldcg(A.vote + b);
        if (va.y == bits && va.x == vote_lo(mb) && vb.y == bits && vb.x == vote_lo(ma)) {
          found = true;
          r = rep_first(LD(A.row_len + a), ma, LD(A.row_len + b), mb) ? a : b;  // the longer row stays
          t = r == a ? b : a;
          len = LD(A.row_len + t);
          rlen = LD(A.row_len + r);
          A.rp[r] = r;
          A.rp[t] = r;
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, found);
      if (!bal) continue;
      int32_t incl = len, rsum = rlen;
      for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      for (int o = 16; o > 0; o >>= 1) rsum += __shfl_xor_sync(0xffffffffu, rsum, o);
      const int32_t wsum = __shfl_sync(0xffffffffu, incl, 31);
      const int leader = __ffs(bal) - 1;
      unsigned long long old = 0;
      if (lane == leader) {
        old = atomicAdd(A.pk + q, ((unsigned long long)__popc(bal) << 32) | (unsigned long long)(uint32_t)wsum);
        atomicAdd(sc + SC_RREP + q, rsum);
      }
      old = __shfl_sync(0xffffffffu, old, leader);
      if (found) {
        const int32_t k = (int32_t)(old >> 32) + __popc(bal & lanes_below());
        A.pr[base + k] = r;
        A.pa[base + k] = t;
        A.apref[k] = (int32_t)(uint32_t)old + incl - len;
      }
    }
    grid.sync();
    PHASE_MARK(1);
    const unsigned long long pk = LD(A.pk + q);
    const int32_t npairs = (int32_t)(pk >> 32), asum = (int32_t)(uint32_t)pk;
    const int32_t rrep = LD(sc + SC_RREP + q);
    int32_t stop = 0;
    if (npairs == 0) stop = kDone;
    else if ((int64_t)LD(sc + SC_POOL) + 2 * ((int64_t)rrep + asum) + 16LL * npairs > A.pool_cap ||
             (int64_t)efill + asum > (int64_t)(A.emask >> 1) || asum > (int32_t)(A.hmask >> 1))
      stop = kPoolFull;
    const int32_t* pr = A.pr + base;
    const int32_t* pa = A.pa + base;
    for (int64_t i = gtid; i < np; i += GT) {  // votes back to clean
      int32_t s = LD(P + i);
      A.vote[LD(A.u + s)] = make_ulonglong2(0ULL, 0ULL);
      A.vote[LD(A.v + s)] = make_ulonglong2(0ULL, 0ULL);
    }
    if (stop) {  // nothing was modified: the host rebuilds P and the rows, and the round is redone
      for (int64_t k = gtid; k < npairs; k += GT) {
        A.rp[LD(pr + k)] = -1;
        A.rp[LD(pa + k)] = -1;
      }
      if (gtid == 0) {
        sc[SC_STATUS] = stop;
        sc[SC_NPAIRS] = base;
        sc[SC_ROUNDS] = round0 + rounds;
      }
      break;
    }
    // ---- 3. R = alive slots of the absorbed clusters (deduplicated)
    for (int64_t i0 = gtid - lane; i0 < asum; i0 += GT) {
      const int64_t i = i0 + lane;
      int32_t s = -1;
      bool take = false;
      if (i < asum) {
        int32_t k = owner_of(A.apref, npairs, (int32_t)i);
        int32_t y = LD(pa + k);
        s = LD(A.pool + LD(A.row_off + y) + ((int32_t)i - LD(A.apref + k)));
        take = LD(A.alive + s) && atomicExch(A.tmark + s, 1) == 0;
      }
      int32_t at = warp_claim(sc + SC_RNT + q, take);
      if (take) A.R[at] = s;
    }
    // representatives whose row could overflow (it gains at most the absorbed
    // row) get a new one, twice the bound, dead slots dropped: short rows one
    // warp each, long rows one CTA
    for (int64_t k0 = (int64_t)blockIdx.x * blockDim.x; k0 < npairs; k0 += GT) {
      if (threadIdx.x == 0) { s_nsmall = 0; s_nbig = 0; }
      __syncthreads();
      const int64_t k = k0 + threadIdx.x;
      if (k < npairs) {
        int32_t r = LD(pr + k);
        int32_t len = LD(A.row_len + r);
        int32_t need = len + LD(A.row_len + LD(pa + k));
        if (need > LD(A.row_cap + r)) {
          A.row_cap[r] = need;  // replaced below
          if (len > kBigRow) s_big[atomicAdd(&s_nbig, 1)] = (int32_t)k;
          else s_small[atomicAdd(&s_nsmall, 1)] = (int32_t)k;
        }
      }
      __syncthreads();
      for (int32_t j = warp; j < s_nsmall; j += nwarps) {
        const int32_t r = LD(pr + s_small[j]);
        const int32_t cap = max(2 * LD(A.row_cap + r), 16);
        int32_t off = 0;
        if (lane == 0) off = atomicAdd(sc + SC_POOL, cap);
        off = __shfl_sync(0xffffffffu, off, 0);
        const int32_t old = LD(A.row_off + r), len = LD(A.row_len + r);
        int32_t cnt = 0;
        for (int32_t e0 = 0; e0 < len; e0 += 128) {  // four independent loads per lane in flight
          int32_t sl[4];
          bool keep[4];
#pragma unroll
          for (int j = 0; j < 4; j++) {
            int32_t e = e0 + 32 * j + lane;
            sl[j] = e < len ? LD(A.pool + old + e) : -1;
          }
#pragma unroll
          for (int j = 0; j < 4; j++) keep[j] = sl[j] >= 0 && LD(A.alive + sl[j]);
#pragma unroll
          for (int j = 0; j < 4; j++) {
            unsigned bal = __ballot_sync(0xffffffffu, keep[j]);
            if (keep[j]) A.pool[off + cnt + __popc(bal & lanes_below())] = sl[j];
            cnt += __popc(bal);
          }
        }
        if (lane == 0) {
          A.row_off[r] = off;
          A.row_len[r] = cnt;
          A.row_cap[r] = cap;
        }
      }
      for (int32_t j = 0; j < s_nbig; j++) {
        const int32_t r = LD(pr + s_big[j]);
        if (threadIdx.x == 0) {
          int32_t cap = 2 * LD(A.row_cap + r);
          s_off = atomicAdd(sc + SC_POOL, cap);
          s_cnt = 0;
          A.row_cap[r] = cap;
        }
        __syncthreads();
        const int32_t old = LD(A.row_off + r), len = LD(A.row_len + r);
        for (int32_t e = threadIdx.x; e < len; e += blockDim.x) {
          int32_t s = LD(A.pool + old + e);
          if (LD(A.alive + s)) A.pool[s_off + atomicAdd(&s_cnt, 1)] = s;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          A.row_off[r] = s_off;
          A.row_len[r] = s_cnt;
        }
        __syncthreads();
      }
      __syncthreads();
    }
    grid.sync();
    PHASE_MARK(2);
    const int32_t nt = LD(sc + SC_RNT + q);
    const uint32_t gmask = round_mask(asum, A.hmask);
    if (gtid == 0 && A.trace && round0 + rounds < A.trace_cap) {
      unsigned long long tns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tns));
      long long* e = A.trace + 6 * (int64_t)(round0 + rounds);
      e[0] = np; e[1] = npairs; e[2] = nt; e[3] = asum; e[4] = rrep; e[5] = (long long)tns;
    }
    // ---- 4. rewrite R to the representatives (internal slots die), group
    // equal keys, and find each group's slot outside R (it joins a
    // representative with a cluster that is not absorbed and keeps its key)
    // in the edge hash.  tmark = 1 | mask of the new endpoints the slot was
    // already incident to (2: low, 4: high): rows gain it only where new.
    for (int64_t i = gtid; i < nt; i += GT) {
      int32_t s = LD(A.R + i);
      int32_t x = LD(A.u + s), y = LD(A.v + s);
      int32_t a = rep_of(A.rp, x), b = rep_of(A.rp, y);
      if (a == b) {
        A.alive[s] = 0;
        A.Rg[i] = -1;
      } else {
        int32_t lo = min(a, b), hi = max(a, b);
        A.u[s] = lo;
        A.v[s] = hi;
        A.tmark[s] = 1 | ((lo == x || lo == y) ? 2 : 0) | ((hi == x || hi == y) ? 4 : 0);
        uint64_t key = pair_key(lo, hi);
        int32_t g = h_insert(A, key, gmask);
        A.Rg[i] = g;
        atomicAdd(&A.grp[g].cnt, 1);
        atomicMin(&A.grp[g].head, s);
        A.Rnext[i] = atomicExch(&A.grp[g].list, (int32_t)i);
        int32_t e = e_find(A, key);
        if (e >= 0 && atomicCAS(&A.grp[g].ext, -1, e) == -1) A.tmark[e] = 8;
      }
    }
    for (int64_t k = gtid; k < npairs; k += GT) {  // cluster bookkeeping
      int32_t x = LD(pr + k), t = LD(pa + k);
      A.row_len[t] = 0;
      A.size[x] = LD(A.size + x) + LD(A.size + t);
      A.minid[x] = min(LD(A.minid + x), LD(A.minid + t));
    }
    grid.sync();
    PHASE_MARK(3);
    // ---- 5. fold each group (R members + the outside slot) into its smallest
    // slot, sequential sum in slot order; survivors enter the next P when
    // positive and their new representatives' rows; untouched positive slots
    // stay.  A group has at most 3 R members and one outside slot (a matching
    // merges each cluster once).
    for (int64_t i0 = gtid - lane; i0 < nt; i0 += GT) {
      const int64_t i = i0 + lane;
      int32_t surv = -1;
      bool pos = false;
      if (i < nt) {
        const int32_t g = LD(A.Rg + i);
        const int32_t s0 = LD(A.R + i);
        if (g >= 0 && LD(&A.grp[g].head) == s0) {
          const int32_t cnt = LD(&A.grp[g].cnt), ext = LD(&A.grp[g].ext);
          const uint64_t key = pair_key(LD(A.u + s0), LD(A.v + s0));
          surv = s0;
          if (cnt > 1 || ext >= 0) {
            const int32_t total = cnt + (ext >= 0 ? 1 : 0);
            if (total <= 16) {  // insertion sort in registers / local memory
              int32_t buf[16];
              int32_t k = 0;
              for (int32_t j = LD(&A.grp[g].list); j >= 0; j = LD(A.Rnext + j)) buf[k++] = LD(A.R + j);
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
            } else {  // not reachable under a matching; kept exact: repeated minimum extraction
              int32_t prev = -1;
              double acc = 0.0;
              for (int32_t j = 0; j < total; j++) {
                int32_t nxt = 0x7fffffff;
                for (int32_t t = LD(&A.grp[g].list); t >= 0; t = LD(A.Rnext + t)) {
                  int32_t x = LD(A.R + t);
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
          }
          pos = LD(A.c + surv) > 0.0;
          if (surv != ext) {  // an R slot under its new key
            e_insert(A, key, surv);
            const int32_t mk = LD(A.tmark + surv);
            const int32_t a = LD(A.u + surv), b = LD(A.v + surv);
            if (LD(A.rp + a) == a && !(mk & 2)) A.pool[LD(A.row_off + a) + atomicAdd(A.row_len + a, 1)] = surv;
            if (LD(A.rp + b) == b && !(mk & 4)) A.pool[LD(A.row_off + b) + atomicAdd(A.row_len + b, 1)] = surv;
          }
        }
      }
      const int32_t at = warp_claim(sc + SC_RNP2 + q, pos);
      if (pos) P2[at] = surv;
    }
    for (int64_t i0 = gtid - lane; i0 < np; i0 += GT) {
      const int64_t i = i0 + lane;
      int32_t s = i < np ? LD(P + i) : 0;
      const bool keep = i < np && !LD(A.tmark + s);
      const int32_t at = warp_claim(sc + SC_RNP2 + q, keep);
      if (keep) P2[at] = s;
    }
    grid.sync();
    PHASE_MARK(4);
    np = LD(sc + SC_RNP2 + q);
    prev_base = base;
    base += npairs;
    prev_nt = nt;
    efill += nt;
    which ^= 1;
    rounds++;
  }
}
#undef LD

__global__ void k_cl_group_init(Group* g, int64_t n) {
  GRID_STRIDE(i, n) g[i] = Group::empty();
}

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

// initial row capacity: room for the first merges without a copy
__global__ void k_cl_rowcap(const int32_t* __restrict__ deg, int64_t n, int32_t* __restrict__ cap) {
  GRID_STRIDE(i, n) cap[i] = 2 * deg[i] + 4;
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

__global__ void k_cl_ehash_build(const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                                 const uint8_t* __restrict__ alive, int64_t m, Args A) {
  GRID_STRIDE(i, m) {
    if (alive[i]) e_insert(A, pair_key(u[i], v[i]), (int32_t)i);
  }
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
  const int64_t n = q.n, m = q.m;
  // algorithmic bytes: the quotient read once, the map written
  ProfScope prof(ctx.s, kFamCleanup, 16.0 * (double)m + 4.0 * (double)n);
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
  Buf<ulonglong2> vote(n, ctx);
  vote.zero();
  Buf<unsigned long long> pk(2, ctx);
  Buf<int32_t> pr(n, ctx), pa(n, ctx), rp(n, ctx), minid(n, ctx), size(n, ctx), tmark(m, ctx);
  rp.fill_bytes(0xff);
  tmark.zero();
  iota(ctx, minid.p, n);
  RAMA_KERNEL(ctx, k_cl_fill_i32, n, size.p, n, 1);
  Buf<int32_t> P0(m, ctx), P1(m, ctx), apref(n, ctx);
  Buf<int32_t> R(m, ctx), Rg(m, ctx), Rnext(m, ctx);
  // group table: at most asum groups per round (checked each round); sized
  // to stay in L2 on typical rounds, grown by the host when a round needs more
  uint32_t hcap = 4096;
  while ((int64_t)hcap < m && hcap < (1u << 30)) hcap <<= 1;
  Buf<Group> grp;
  uint32_t ecap = 4096;
  while ((int64_t)ecap < 4 * m && ecap < (1u << 30)) ecap <<= 1;
  Buf<int32_t> eh;
  int64_t grow = 1;  // doubles when a launch could not run a single round
  Buf<int32_t> sc(SC_COUNT, ctx);
  static const bool resident = [] {  // thread-safe init (batch workers)
    int per_sm = 0;
    RAMA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cl_rounds, kThreads, 0));
    return per_sm >= 1;
  }();
  RAMA_REQUIRE(resident, "cleanup kernel cannot be resident");
  const int max_blocks = num_sms();  // at most one CTA per SM (per device)
  // sized by the quotient: a small cleanup (batch instances) leaves the
  // other SMs to concurrent solves instead of claiming the whole GPU
  const int grid_blocks = (int)std::min<int64_t>(max_blocks, std::max<int64_t>(8, (m + 8191) / 8192));
  int64_t total = 0;
  int launches = 0, rounds = 0;
  const char* stats_env = getenv("RAMA_CLEANUP_STATS");
  const bool round_trace = stats_env && atoi(stats_env) >= 2;
  constexpr int32_t kTraceCap = 4096;
  Buf<long long> trace(round_trace ? 6 * kTraceCap : 1, ctx);
  const bool phase_trace = stats_env && atoi(stats_env) >= 3;
  Buf<long long> ptrace(phase_trace ? 5 * kTraceCap : 1, ctx);
  Args A;
  A.u = u.p; A.v = v.p; A.c = c.p; A.alive = alive.p; A.tmark = tmark.p; A.vote = vote.p;
  A.rp = rp.p; A.minid = minid.p; A.size = size.p; A.P0 = P0.p; A.P1 = P1.p;
  A.pr = pr.p; A.pa = pa.p; A.apref = apref.p; A.pk = pk.p;
  A.R = R.p; A.Rg = Rg.p; A.Rnext = Rnext.p;
  A.sc = sc.p;
  A.trace = round_trace ? trace.p : nullptr;
  A.ptrace = phase_trace ? ptrace.p : nullptr;
  A.trace_cap = kTraceCap;
  while (true) {
    // P, the rows and the edge hash, from the current slots
    Buf<int32_t> Pl;
    int64_t np = compact_if(ctx, m, PosAlive{c.p, alive.p}, Pl);
    if (np == 0) break;
    copy_d2d(ctx, P0.p, Pl.p, np);
    Buf<int32_t> deg(n, ctx), rcap(n, ctx), off(n + 1, ctx), cur(n, ctx);
    deg.zero();
    cur.zero();
    RAMA_KERNEL(ctx, k_cl_degree, m, u.p, v.p, alive.p, m, deg.p);
    RAMA_KERNEL(ctx, k_cl_rowcap, n, deg.p, n, rcap.p);
    int64_t used = exclusive_scan(ctx, rcap.p, off.p, n, true);
    int64_t arcs = (used - 4 * n) / 2;
    int64_t slack = pool_slack_override() >= 0 ? pool_slack_override() : std::max<int64_t>(8 * arcs, 1 << 22);
    int64_t cap = used + slack * grow;
    if (cap > 0x7fffffffLL) cap = 0x7fffffffLL;
    RAMA_REQUIRE(used <= cap, "cleanup rows exceed the pool");
    Buf<int32_t> pool(cap, ctx);
    RAMA_KERNEL(ctx, k_cl_fill_rows, m, u.p, v.p, alive.p, m, off.p, cur.p, pool.p);
    if (eh.n != ecap) eh.alloc(ecap, ctx.s);
    eh.fill_bytes(0xff);
    A.eh = eh.p; A.emask = ecap - 1;
    if (grp.n != hcap) {
      grp.alloc(hcap, ctx.s);
      RAMA_KERNEL(ctx, k_cl_group_init, hcap, grp.p, hcap);
    }
    A.grp = grp.p; A.hmask = hcap - 1;
    A.row_off = off.p; A.row_len = deg.p; A.row_cap = rcap.p; A.pool = pool.p; A.pool_cap = cap;
    RAMA_KERNEL(ctx, k_cl_ehash_build, m, u.p, v.p, alive.p, m, A);
    int32_t init[SC_COUNT] = {0};
    init[SC_NPAIRS] = (int32_t)total;
    init[SC_ROUNDS] = rounds;
    init[SC_NP] = (int32_t)np;
    init[SC_POOL] = (int32_t)used;
    init[SC_EFILL] = (int32_t)m;
    RAMA_CUDA(cudaMemcpyAsync(sc.p, init, sizeof(init), cudaMemcpyHostToDevice, ctx.s));
    pk.zero();
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
    memcpy(st, fetch(ctx, {{sc.p, (int)sizeof(st)}}), sizeof(st));
    total = st[SC_NPAIRS];
    if (round_trace) {
      const int32_t k0 = std::min(rounds, kTraceCap), k1 = std::min(st[SC_ROUNDS], kTraceCap);
      std::vector<long long> h(6 * (size_t)k1);
      if (k1) RAMA_CUDA(cudaMemcpy(h.data(), trace.p, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
      for (int32_t r = k0; r < k1; r++) {
        const long long* e = &h[6 * (size_t)r];
        long long prev = r > k0 ? h[6 * (size_t)(r - 1) + 5] : e[5];
        fprintf(stderr, "[rama] cl launch %d round %d np %lld pairs %lld nt %lld asum %lld rrep %lld dt_us %.1f\n",
                launches, r, e[0], e[1], e[2], e[3], e[4], (e[5] - prev) / 1e3);
      }
      if (phase_trace && k1 > k0) {
        std::vector<long long> q(5 * (size_t)k1);
        RAMA_CUDA(cudaMemcpy(q.data(), ptrace.p, q.size() * sizeof(long long), cudaMemcpyDeviceToHost));
        for (int32_t r = k0 + 1; r < k1; r++) {
          const long long* e = &q[5 * (size_t)r];
          fprintf(stderr, "[rama] cl phases round %d np %lld: %.1f %.1f %.1f %.1f %.1f us\n", r, h[6 * (size_t)r],
                  (e[0] - q[5 * (size_t)(r - 1) + 4]) / 1e3, (e[1] - e[0]) / 1e3, (e[2] - e[1]) / 1e3,
                  (e[3] - e[2]) / 1e3, (e[4] - e[3]) / 1e3);
        }
      }
    }
    const bool progress = st[SC_ROUNDS] > rounds;
    rounds = st[SC_ROUNDS];
    if (st[SC_STATUS] == kDone) break;
    RAMA_REQUIRE(st[SC_STATUS] == kPoolFull, "cleanup kernel ended in an unknown state");
    if (!progress) {  // one round does not fit: larger pool and edge hash
      RAMA_REQUIRE(grow < (1 << 20), "cleanup cannot make progress");
      grow *= 2;
      if (ecap < (1u << 30)) ecap <<= 1;
      if (hcap < (1u << 30)) hcap <<= 1;
    }
  }
  if (stats_env)
    fprintf(stderr, "[rama] cleanup n %lld m %lld: %d rounds in %d launches, %lld pairs, %.2f ms\n", (long long)n,
            (long long)m, rounds, launches, (long long)total,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
  return components(ctx, n, pr.p, pa.p, total, fc);
}

}  // namespace rama
