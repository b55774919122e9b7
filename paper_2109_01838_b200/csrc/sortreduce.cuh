// Fused row sort + unique + reduce ("sort-reduce"): the canonical-order
// primitive behind contraction (a18) and canonicalisation (a3).  (The
// positive CSR, triangulation's dedupes and the slot lists keep the bucket
// sort of prims.cu: their rows hold 1-3 items, for which this tile kernel
// measured slower -- DESIGN.md section 4.)
//
// Items are produced on the fly by a functor over an input index space (so
// relabelling and orientation are fused into the passes instead of
// materialising row/key arrays), grouped by a 32-bit row
// and ordered by a 64-bit key inside the row:
//
//   K1 count    one pass over the inputs: row histogram (L2-resident atomics)
//   K2 scan     row pointers (CUB), + list of rows longer than kSrHuge
//   K3 scatter  second pass over the inputs: 16-byte items {key, payload}
//               into their row (a count-down atomic gives the slot)
//   K4 tiles    one CTA per tile of rows (the rows whose first item falls
//               in a kSrTile-item window): stage the items in shared memory
//               with 16-byte loads, order each row by ranking, mark group
//               heads (first item of each run of equal key >> GS), count the
//               kept heads, take the tile's output offset from a
//               decoupled look-back over the tile aggregates, and emit one
//               output per kept group at its final position -- no head
//               flags, no compaction pass, no host read-back.
//
// Determinism: the scatter order inside a row is arbitrary, but rows are
// ordered by key (keys embed the source index where equal groups must sum
// in source order), so every output is deterministic and, with the
// reduceat-order segment sum, bit-identical to numpy.
//
// Rows longer than kSrHuge items (power-law hubs only) are sorted in
// global memory by CUB's segmented sort before K4 and streamed from there;
// the host learns whether any exist from an asynchronous read-back that
// lands while K3 runs.
#pragma once

#include "common.cuh"

#include <atomic>

#include <cub/cub.cuh>

namespace rama {

struct __align__(16) SrItem {
  uint64_t key;
  double pay;
};

#ifndef RAMA_SR_THREADS
#define RAMA_SR_THREADS 512
#define RAMA_SR_TILE 4096
#define RAMA_SR_HUGE 768
#endif
constexpr int kSrThreads = RAMA_SR_THREADS;
constexpr int kSrTile = RAMA_SR_TILE;   // row window per tile (items)
constexpr int kSrHuge = RAMA_SR_HUGE;   // longer rows: pre-sorted in global memory
constexpr int kSrCap = kSrTile + kSrHuge;  // staged items per tile (max)
constexpr int kSrPer = (kSrCap + kSrThreads - 1) / kSrThreads;
// dynamic shared memory of a tile: keys, payloads, rows, sort permutation
constexpr size_t kSrSmem = (size_t)kSrCap * (8 + 8 + 4 + 2);

// payloads of a run of sorted positions through the tile's permutation
struct SrPermPay {
  const double* pay;
  const uint16_t* perm;
  __device__ __forceinline__ double operator[](int64_t i) const { return pay[perm[i]]; }
  __device__ __forceinline__ SrPermPay operator+(int64_t k) const { return SrPermPay{pay, perm + k}; }
};

// payloads of a run of items (smem or global) as a numpy-order summand list
struct SrPay {
  const SrItem* p;
  __device__ __forceinline__ double operator[](int64_t i) const { return p[i].pay; }
  __device__ __forceinline__ SrPay operator+(int64_t k) const { return SrPay{p + k}; }
};

// ---- decoupled look-back over tile aggregates --------------------------------
// status word: bits 62-63 flag (0 empty, 1 aggregate, 2 inclusive prefix),
// bits 0-61 value.  Tiles are claimed in order from a counter, so every
// predecessor is running or done.
// The status words carry their own payload, so relaxed device-scope
// accesses suffice (no fence: nothing else is published through them).
__device__ __forceinline__ void sr_store(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t sr_load(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void sr_publish(uint64_t* st, int64_t t, uint64_t flag, uint64_t v) {
  sr_store(st + t, (flag << 62) | v);
}

// called by one full warp after the tile's aggregate was published;
// returns the exclusive prefix of tile t and publishes its inclusive prefix
__device__ __forceinline__ int64_t sr_lookback(uint64_t* st, int64_t t, int64_t agg) {
  const int lane = threadIdx.x & 31;
  if (t == 0) return 0;
  int64_t excl = 0;
  int64_t base = t - 1;
  while (true) {
    const int64_t idx = base - lane;
    uint64_t s;
    int spins = 0;
    while (true) {
      s = idx >= 0 ? sr_load(st + idx) : (2ull << 62);
      if (__all_sync(0xffffffffu, (s >> 62) != 0)) break;
      if (++spins > 4) __nanosleep(64);
    }
    const unsigned incl = __ballot_sync(0xffffffffu, (s >> 62) == 2);
    const int stop = incl ? __ffs(incl) - 1 : 31;
    int64_t v = lane <= stop ? (int64_t)(s & ((1ull << 62) - 1)) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (incl) break;
    base -= 32;
  }
  if (lane == 0) sr_publish(st, t, 2ull, (uint64_t)(excl + agg));
  return excl;
}

// Block-wide look-back (all threads): one round trip reads kSrThreads
// predecessors.  Tiles run in waves of (2 CTAs x 148 SMs) that reach their
// look-back together, so the nearest inclusive prefix is usually a whole
// wave back -- one step here instead of ~10 warp-window steps.
template <int NT>
__device__ __forceinline__ int64_t sr_lookback_block(uint64_t* st, int64_t t, int32_t* s_stop, int64_t* s_sum) {
  if (t == 0) return 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t excl = 0;
  int64_t base = t - 1;
  while (true) {
    const int64_t idx = base - tid;
    uint64_t s;
    int spins = 0;
    while (true) {
      s = idx >= 0 ? sr_load(st + idx) : (2ull << 62);
      if (__syncthreads_and((s >> 62) != 0)) break;
      if (++spins > 2) __nanosleep(100);
    }
    if (tid == 0) *s_stop = 0x7fffffff;
    __syncthreads();
    if ((s >> 62) == 2) atomicMin(s_stop, tid);
    __syncthreads();
    const int stop = *s_stop;
    int64_t v = tid <= stop ? (int64_t)(s & ((1ull << 62) - 1)) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) s_sum[warp] = v;
    __syncthreads();
    int64_t tot = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; w++) tot += s_sum[w];
    excl += tot;
    __syncthreads();  // s_stop / s_sum reused by the next step
    if (stop != 0x7fffffff) break;
    base -= NT;
  }
  return excl;
}

// ---- K1 / K3 -------------------------------------------------------------------
// Src functor: `int64_t size() const` inputs, up to Src::kK items each;
// `bool item(int64_t i, int k, int32_t& row, uint64_t& key, double& pay) const`.
// (counts and slots aggregated over runs of equal rows in consecutive lanes,
// run_atomic_add: sorted inputs and hub rows take one atomic per run)
template <class Src>
__global__ void k_sr_count(Src src, int32_t* __restrict__ cnt) {
  const int64_t n = src.size();
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x - lane; i0 < n;
       i0 += (int64_t)gridDim.x * blockDim.x) {  // warp-uniform trip count
    const int64_t i = i0 + lane;
#pragma unroll
    for (int k = 0; k < Src::kK; k++) {
      int32_t row = -1;
      uint64_t key;
      double pay;
      if (!(i < n && src.item(i, k, row, key, pay))) row = -1;
      run_atomic_add(cnt, row, 1);
    }
  }
}

template <class Src>
__global__ void k_sr_scatter(Src src, const int32_t* __restrict__ rowptr, int32_t* __restrict__ cnt,
                             SrItem* __restrict__ items) {
  const int64_t n = src.size();
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x - lane; i0 < n;
       i0 += (int64_t)gridDim.x * blockDim.x) {  // warp-uniform trip count
    const int64_t i = i0 + lane;
#pragma unroll
    for (int k = 0; k < Src::kK; k++) {
      int32_t row = -1;
      uint64_t key = 0;
      double pay = 0.0;
      if (!(i < n && src.item(i, k, row, key, pay))) row = -1;
      const int32_t left = run_atomic_add(cnt, row, -1);  // count-down: slots left before this item's
      if (row >= 0) {
        const int32_t p = rowptr[row] + left - 1;
        SrItem it;
        it.key = key;
        it.pay = pay;
        items[p] = it;
      }
    }
  }
}

// rows longer than kSrHuge (listed for the global segmented sort)
static __global__ void k_sr_huge(const int32_t* __restrict__ rowptr, int64_t R, int32_t* __restrict__ list,
                          int32_t* __restrict__ count) {
  GRID_STRIDE(r, R) {
    if (rowptr[r + 1] - rowptr[r] > kSrHuge) list[atomicAdd(count, 1)] = (int32_t)r;
  }
}

// tile_row[t] = first row r in [0, R) with rowptr[r] >= t * kSrTile (R if
// none), for t in [0, tiles]: row r owns the windows (rowptr[r-1], rowptr[r]]
// (one parallel pass instead of two binary searches per tile)
static __global__ void k_sr_tilemap(const int32_t* __restrict__ rowptr, int64_t R, int64_t tiles,
                                    int32_t* __restrict__ tile_row, uint64_t* __restrict__ status,
                                    int64_t* __restrict__ total) {
  // the tiles' look-back words and the output counter start at zero (no memsets)
  GRID_STRIDE(t, tiles + 1) status[t] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) *total = 0;
  GRID_STRIDE(r, R + 1) {
    const int64_t prev = r == 0 ? -1 : (int64_t)rowptr[r - 1];
    const int64_t cur = r == R ? (int64_t)tiles * kSrTile : (int64_t)rowptr[r];
    const int64_t t0 = (prev + kSrTile) / kSrTile;  // first t with t*T > prev
    int64_t t1 = cur / kSrTile;                      // last t with t*T <= cur
    if (t1 > tiles) t1 = tiles;
    for (int64_t t = t0; t <= t1; t++) tile_row[t] = (int32_t)r;
  }
}

// ---- K4 --------------------------------------------------------------------------
// Emit functor:
//   bool keep(int32_t row, uint64_t key) const
//   template <class A> void out(int64_t idx, int32_t row, uint64_t key, A pays, int64_t len) const
// (pays: accessor of the group's payloads in order, pays[i], pays + k)
// kUnique: one output per group of equal (key >> GS) in a row, at its rank
// among the kept groups of the whole list; else one output per item at its
// sorted position (idx = position, keep() not consulted).
constexpr int kSrWarps = kSrThreads / 32;

// kDistinct: the keys of a row are pairwise distinct (they embed the source
// index), so the ranking needs no tie-break
template <int GS, bool kUnique, bool kDistinct, class Emit>
__global__ void __launch_bounds__(kSrThreads) k_sr_tiles(const SrItem* __restrict__ items,
                                                         const int32_t* __restrict__ rowptr, int64_t R,
                                                         int64_t tiles, const int32_t* __restrict__ tile_row,
                                                         uint64_t* __restrict__ status,
                                                         int32_t* __restrict__ tile_ctr, int64_t* __restrict__ total,
                                                         Emit emit, const int32_t* __restrict__ R_dev) {
  // staged items as SoA; the row order is a permutation (sorted position ->
  // staged index), so items never move
  extern __shared__ __align__(16) unsigned char s_dyn[];
  uint64_t* const s_key = (uint64_t*)s_dyn;
  double* const s_pay = (double*)(s_key + kSrCap);
  int32_t* const s_row = (int32_t*)(s_pay + kSrCap);
  uint16_t* const s_perm = (uint16_t*)(s_row + kSrCap);
  __shared__ int32_t s_meta[8];
  __shared__ int32_t s_wcnt[kSrPer * kSrWarps];  // kept heads per (slab, warp) -> exclusive offsets
  __shared__ unsigned s_hb[kSrPer * kSrWarps + 1];  // group-boundary bits of the sorted positions
  __shared__ int64_t s_prefix;
  __shared__ int32_t s_stop;
  __shared__ int64_t s_lsum[kSrWarps];
  using BlockScan = cub::BlockScan<int32_t, kSrThreads>;
  __shared__ typename BlockScan::TempStorage s_scan;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  (void)tile_ctr;

  // tiles in launch order (blocks are dispatched in index order, as in CUB's
  // single-pass scans)
  const int32_t t = blockIdx.x;
  // R_dev: the rows actually used when R only bounds them (the rest are
  // empty; the last tile must not walk them)
  const int32_t r0 = __ldg(tile_row + t), r1 = R_dev ? min(__ldg(tile_row + t + 1), max(*R_dev, r0))
                                                     : __ldg(tile_row + t + 1);
  const int32_t s0 = __ldg(rowptr + r0), s1 = __ldg(rowptr + r1);
  int32_t se = s1, rh = -1;  // staged end, huge (last) row
  if (r1 > r0) {
    const int32_t sl = __ldg(rowptr + r1 - 1);
    if (s1 - sl > kSrHuge) {
      rh = r1 - 1;
      se = sl;
    }
  }
  const int32_t S = se - s0;  // staged items (<= kSrCap)
  const int32_t rs_end = rh >= 0 ? rh : r1;  // staged rows [r0, rs_end)
  if (tid == 0) s_meta[7] = 0;
  if (tid == 0) s_hb[kSrPer * kSrWarps] = ~0u;  // sentinel past the last slab

  // stage (16-byte loads); each staged row writes its id over its items
  for (int32_t j = tid; j < S; j += kSrThreads) {
    const SrItem it = items[s0 + j];
    s_key[j] = it.key;
    s_pay[j] = it.pay;
  }
  for (int32_t r = r0 + tid; r < rs_end; r += kSrThreads) {
    const int32_t b = __ldg(rowptr + r) - s0, e = __ldg(rowptr + r + 1) - s0;
    for (int32_t j = b; j < e; j++) s_row[j] = r;
  }
  __syncthreads();
  // rank each item inside its row (ties by staged index: a permutation)
  for (int32_t j = tid; j < S; j += kSrThreads) {
    const int32_t r = s_row[j];
    const int32_t b = __ldg(rowptr + r) - s0, e = __ldg(rowptr + r + 1) - s0;
    const uint64_t k = s_key[j];
    int32_t rank = 0;
    if (kDistinct) {
      for (int32_t x = b; x < e; x++) rank += s_key[x] < k;
    } else {
      for (int32_t x = b; x < e; x++) {
        const uint64_t y = s_key[x];
        rank += (y < k) || (y == k && x < j);
      }
    }
    s_perm[b + rank] = (uint16_t)j;
  }
  __syncthreads();
  // s_row[p] is also the row of SORTED position p: ranking permutes inside a row

  if (!kUnique) {
    for (int32_t p = tid; p < S; p += kSrThreads) {
      const int32_t j = s_perm[p];
      emit.out((int64_t)s0 + p, s_row[p], s_key[j], SrPermPay{s_pay, s_perm + p}, 1);
    }
    if (rh >= 0) {  // pre-sorted huge row: straight copy
      for (int32_t p = se + tid; p < s1; p += kSrThreads) emit.out((int64_t)p, rh, items[p].key, SrPay{items + p}, 1);
    }
    return;
  }

  // kept group heads in sorted order; position p = q * kSrThreads + tid, so
  // (slab, warp, lane) order is position order and warp ballots give offsets
  unsigned bal[kSrPer];
  int32_t kept = 0;
#pragma unroll
  for (int q = 0; q < kSrPer; q++) {
    const int32_t p = q * kSrThreads + tid;
    bool kh = false, head = false;
    if (p < S) {
      const uint64_t k = s_key[s_perm[p]];
      head = p == 0 || s_row[p] != s_row[p - 1] || (s_key[s_perm[p - 1]] >> GS) != (k >> GS);
      kh = head && emit.keep(s_row[p], k);
    }
    bal[q] = __ballot_sync(0xffffffffu, kh);
    kept += __popc(bal[q]);
    const unsigned hb = __ballot_sync(0xffffffffu, head || p >= S);  // group boundaries (and the end)
    if (lane == 0) {
      s_wcnt[q * kSrWarps + warp] = __popc(bal[q]);
      s_hb[q * kSrWarps + warp] = hb;
    }
  }
  if (lane == 0 && kept) atomicAdd(&s_meta[7], kept);  // staged kept heads of the tile
  // huge row: kept heads from global memory (pre-sorted), strided over the block
  int32_t hmine = 0;
  if (rh >= 0) {
    for (int32_t p = se + tid; p < s1; p += kSrThreads) {
      const uint64_t k = items[p].key;
      if ((p == se || (items[p - 1].key >> GS) != (k >> GS)) && emit.keep(rh, k)) hmine++;
    }
  }
  __syncthreads();
  const int32_t agg = s_meta[7];
  if (rh < 0 && tid == 0) sr_publish(status, t, t == 0 ? 2ull : 1ull, (uint64_t)agg);  // as soon as known
  if (warp == 0) {  // exclusive scan of the kSrPer * kSrWarps counts (in order)
    constexpr int kC = kSrPer * kSrWarps;
    constexpr int kPerLane = (kC + 31) / 32;
    int32_t v[kPerLane];
    int32_t sum = 0;
#pragma unroll
    for (int i = 0; i < kPerLane; i++) {
      const int c = lane * kPerLane + i;
      v[i] = c < kC ? s_wcnt[c] : 0;
      sum += v[i];
    }
    int32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int32_t run = incl - sum;
#pragma unroll
    for (int i = 0; i < kPerLane; i++) {
      const int c = lane * kPerLane + i;
      if (c < kC) s_wcnt[c] = run;
      run += v[i];
    }
  }
  int32_t hoff = 0, hagg = 0;
  if (rh >= 0) {
    BlockScan(s_scan).ExclusiveSum(hmine, hoff, hagg);
    if (tid == 0) sr_publish(status, t, t == 0 ? 2ull : 1ull, (uint64_t)(agg + hagg));
  }
  __syncthreads();  // s_wcnt offsets complete
  {
    const int64_t pre = sr_lookback_block<kSrThreads>(status, t, &s_stop, s_lsum);
    if (tid == 0) {
      if (t > 0) sr_publish(status, t, 2ull, (uint64_t)(pre + agg + hagg));
      s_prefix = pre;
      if (t == tiles - 1) *total = pre + agg + hagg;
    }
  }
  __syncthreads();
  const int64_t base = s_prefix;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll 1
  for (int q = 0; q < kSrPer; q++) {
    if (bal[q] & (1u << lane)) {
      const int32_t p = q * kSrThreads + tid;
      const int64_t idx = base + s_wcnt[q * kSrWarps + warp] + __popc(bal[q] & lt);
      const int32_t row = s_row[p];
      const uint64_t k = s_key[s_perm[p]];
      // group end: the next boundary bit after p
      int32_t w = (p + 1) >> 5;
      unsigned bits = ((p + 1) & 31) ? (s_hb[w] & (~0u << ((p + 1) & 31))) : s_hb[w];
      while (!bits) bits = s_hb[++w];
      const int32_t e = min((w << 5) + __ffs(bits) - 1, S);
      emit.out(idx, row, k, SrPermPay{s_pay, s_perm + p}, e - p);
    }
  }
  if (rh >= 0) {  // outputs of the huge row follow the staged ones, in position order
    int64_t hidx = base + agg;
    for (int32_t p0 = se; p0 < s1; p0 += kSrThreads) {
      const int32_t p = p0 + tid;
      bool kh = false;
      int64_t len = 0;
      uint64_t k = 0;
      if (p < s1) {
        k = items[p].key;
        if ((p == se || (items[p - 1].key >> GS) != (k >> GS)) && emit.keep(rh, k)) {
          int64_t e = p + 1;
          while (e < s1 && (items[e].key >> GS) == (k >> GS)) e++;
          len = e - p;
          kh = true;
        }
      }
      int32_t o = 0, a = 0;
      BlockScan(s_scan).ExclusiveSum(kh ? 1 : 0, o, a);
      __syncthreads();
      if (kh) emit.out(hidx + o, rh, k, SrPay{items + p}, len);
      hidx += a;
    }
    (void)hoff;
  }
}

// ---- host driver --------------------------------------------------------------------
// CUB segmented sort (by key) of the listed rows, in place (prims.cu)
void sr_sort_huge(Ctx& ctx, const int32_t* rowptr, const int32_t* rows, int64_t nrows, SrItem* items);

struct SrResult {
  Buf<int32_t> rowptr;  // R + 1 (rowptr[R] = items kept)
  Buf<int64_t> total;   // device: outputs written (kUnique; else rowptr[R] counts them)
};

// One sort-reduce over `src` into `R` rows.  N_max: upper bound of the
// items (src.size() * kK).  Returns the number of outputs when `want` (one
// read-back), else -1 (the count stays in res.total on the device).
template <int GS, bool kUnique, bool kDistinct, class Src, class Emit>
int64_t sort_reduce(Ctx& ctx, int64_t R, int64_t N_max, const Src& src, const Emit& emit, SrResult& res,
                    bool want = true, const char* tag = "sr", const int32_t* extra_dev = nullptr,
                    int64_t* extra_out = nullptr) {
  // extra_dev: one more device word read back with the output count (want);
  // it is also the number of rows in use (R bounds it; rows beyond are empty)
  res.rowptr.alloc(R + 1, ctx.s);
  res.total.alloc(1, ctx.s);
  if (R == 0 || N_max == 0) {
    RAMA_CUDA(cudaMemsetAsync(res.total.p, 0, sizeof(int64_t), ctx.s));
    RAMA_CUDA(cudaMemsetAsync(res.rowptr.p, 0, sizeof(int32_t) * (R + 1), ctx.s));
    if (want && extra_dev) *extra_out = read_scalar(ctx, extra_dev);
    return want ? 0 : -1;
  }
  Buf<int32_t> cnt(R + 2, ctx);  // counts | huge-row counter
  RAMA_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * (R + 2), ctx.s));
  const int64_t n_in = src.size();
  if (trace_print()) {
    fprintf(stderr, "[rama] sort_reduce<%s> R %lld N_max %lld inputs %lld\n", tag, (long long)R, (long long)N_max,
            (long long)n_in);
    fflush(stderr);
  }
  {
    KernelScope ks(ctx.s, "k_sr_count");
    k_sr_count<Src><<<capped_grid(n_in), kBlock, 0, ctx.s>>>(src, cnt.p);
  }
  RAMA_LAUNCH_CHECK();
  ctx.launches++;
  exclusive_scan(ctx, cnt.p, res.rowptr.p, R, false);
  int32_t* hcount = cnt.p + R + 1;
  Buf<int32_t> hlist(R, ctx);
  {
    KernelScope ks(ctx.s, "k_sr_huge", 8.0 * (double)R);
    k_sr_huge<<<capped_grid(R), kBlock, 0, ctx.s>>>(res.rowptr.p, R, hlist.p, hcount);
  }
  RAMA_LAUNCH_CHECK();
  ctx.launches++;
  // the huge-row count travels back while the scatter runs
  int32_t* hp = (int32_t*)(ctx.pinned + 32);
  RAMA_CUDA(cudaMemcpyAsync(hp, hcount, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx.s));
  RAMA_CUDA(cudaEventRecord(ctx.ev, ctx.s));
  Buf<SrItem> items(N_max, ctx);
  {
    KernelScope ks(ctx.s, "k_sr_scatter");
    k_sr_scatter<Src><<<capped_grid(n_in), kBlock, 0, ctx.s>>>(src, res.rowptr.p, cnt.p, items.p);
  }
  RAMA_LAUNCH_CHECK();
  ctx.launches++;
  RAMA_CUDA(cudaEventSynchronize(ctx.ev));
  const int32_t nh = *hp;
  if (trace_print()) {
    fprintf(stderr, "[rama] sort_reduce huge rows %d\n", nh);
    fflush(stderr);
  }
  if (nh > 0) sr_sort_huge(ctx, res.rowptr.p, hlist.p, nh, items.p);
  const int64_t tiles = (N_max + kSrTile - 1) / kSrTile;
  Buf<uint64_t> status(tiles + 1, ctx);
  Buf<int32_t> tile_row(tiles + 1, ctx);
  {
    KernelScope ks(ctx.s, "k_sr_tilemap", 4.0 * (double)R);
    k_sr_tilemap<<<capped_grid(std::max<int64_t>(R, tiles) + 1), kBlock, 0, ctx.s>>>(res.rowptr.p, R, tiles,
                                                                                    tile_row.p, status.p,
                                                                                    res.total.p);
  }
  RAMA_LAUNCH_CHECK();
  ctx.launches++;
  {  // the dynamic shared memory opt-in is per device
    static std::atomic<uint64_t> set_on{0};
    int dev = 0;
    RAMA_CUDA(cudaGetDevice(&dev));
    const uint64_t bit = 1ull << (dev & 63);
    if (!(set_on.load() & bit)) {
      RAMA_CUDA(cudaFuncSetAttribute(k_sr_tiles<GS, kUnique, kDistinct, Emit>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSrSmem));
      set_on.fetch_or(bit);
    }
  }
  {
    KernelScope ks(ctx.s, "k_sr_tiles");
    k_sr_tiles<GS, kUnique, kDistinct, Emit><<<(unsigned)tiles, kSrThreads, kSrSmem, ctx.s>>>(
        items.p, res.rowptr.p, R, tiles, tile_row.p, status.p, (int32_t*)(status.p + tiles), res.total.p, emit,
        extra_dev);
  }
  RAMA_LAUNCH_CHECK();
  ctx.launches++;
  if (!want) return -1;
  if (extra_dev) {
    const int32_t* hp = kUnique ? (const int32_t*)fetch(ctx, {{res.total.p, 8}, {extra_dev, 4}})
                                : (const int32_t*)fetch(ctx, {{res.rowptr.p + R, 4}, {extra_dev, 4}});
    int64_t cnt;
    if (kUnique) {
      memcpy(&cnt, hp, 8);
      *extra_out = hp[2];
    } else {
      cnt = hp[0];
      *extra_out = hp[1];
    }
    return cnt;
  }
  if (!kUnique) return read_scalar(ctx, res.rowptr.p + R);  // every item is an output
  return read_scalar(ctx, res.total.p);
}

}  // namespace rama
