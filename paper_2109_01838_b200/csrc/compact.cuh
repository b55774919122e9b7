// Predicate compaction: the indices i in [0, n) with pred(i), ascending, in
// one CUB select over a counting iterator -- no flag array and no separate
// flag kernel (a launch and a pass saved per call; small solves are
// launch-bound).
#pragma once

#include "common.cuh"

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/discard_iterator.h>

namespace rama {

template <class Pred>
int64_t compact_if(Ctx& ctx, int64_t n, Pred pred, Buf<int32_t>& out) {
  out.alloc(n > 0 ? n : 1, ctx.s);
  if (n <= 0) return 0;
  Buf<int32_t> nsel(1, ctx);
  thrust::counting_iterator<int32_t> it(0);
  size_t tb = 0;
  RAMA_CUDA(cub::DeviceSelect::If(nullptr, tb, it, out.p, nsel.p, (int)n, pred, ctx.s));
  Buf<uint8_t> tmp(tb, ctx);
  {
    KernelScope ks(ctx.s, "cub::DeviceSelect", 0.0);
    RAMA_CUDA(cub::DeviceSelect::If(tmp.p, tb, it, out.p, nsel.p, (int)n, pred, ctx.s));
  }
  ctx.launches++;
  return read_scalar(ctx, nsel.p);
}

// the same, count left on the device (no read-back): consumers read *count
template <class Pred>
void compact_if_dev(Ctx& ctx, int64_t n, Pred pred, Buf<int32_t>& out, Buf<int32_t>& count) {
  out.alloc(n > 0 ? n : 1, ctx.s);
  count.alloc(1, ctx.s);
  if (n <= 0) {
    count.zero();
    return;
  }
  thrust::counting_iterator<int32_t> it(0);
  size_t tb = 0;
  RAMA_CUDA(cub::DeviceSelect::If(nullptr, tb, it, out.p, count.p, (int)n, pred, ctx.s));
  Buf<uint8_t> tmp(tb, ctx);
  {
    KernelScope ks(ctx.s, "cub::DeviceSelect", 0.0);
    RAMA_CUDA(cub::DeviceSelect::If(tmp.p, tb, it, out.p, count.p, (int)n, pred, ctx.s));
  }
  ctx.launches++;
}

// indices with c < 0 and with c > 0, each ascending, in ONE pass over the
// costs (CUB three-way partition; zero-cost edges are discarded) and one
// read-back of both counts
template <class PredA, class PredB>
void partition2(Ctx& ctx, int64_t n, PredA pa, PredB pb, Buf<int32_t>& out_a, Buf<int32_t>& out_b, int64_t& na,
                int64_t& nb) {
  out_a.alloc(n > 0 ? n : 1, ctx.s);
  out_b.alloc(n > 0 ? n : 1, ctx.s);
  na = nb = 0;
  if (n <= 0) return;
  Buf<int32_t> cnt(2, ctx);
  thrust::counting_iterator<int32_t> it(0);
  thrust::discard_iterator<> none;
  size_t tb = 0;
  RAMA_CUDA(cub::DevicePartition::If(nullptr, tb, it, out_a.p, out_b.p, none, cnt.p, (int)n, pa, pb, ctx.s));
  Buf<uint8_t> tmp(tb, ctx);
  {
    KernelScope ks(ctx.s, "cub::DevicePartition", 0.0);
    RAMA_CUDA(cub::DevicePartition::If(tmp.p, tb, it, out_a.p, out_b.p, none, cnt.p, (int)n, pa, pb, ctx.s));
  }
  ctx.launches++;
  read_pair(ctx, cnt.p, cnt.p + 1, na, nb);
}

struct NegCost {  // c_i < 0
  const double* c;
  __device__ __forceinline__ bool operator()(int32_t i) const { return c[i] < 0.0; }
};
struct PosCost {  // c_i > 0
  const double* c;
  __device__ __forceinline__ bool operator()(int32_t i) const { return c[i] > 0.0; }
};
struct PosAlive {  // alive slot with c_i > 0
  const double* c;
  const uint8_t* alive;
  __device__ __forceinline__ bool operator()(int32_t i) const { return alive[i] && c[i] > 0.0; }
};
struct FlagSet {  // flags[i] != 0
  const uint8_t* f;
  __device__ __forceinline__ bool operator()(int32_t i) const { return f[i] != 0; }
};
struct SortedHead {  // first item of each (row, key) run of a sorted list
  const int32_t* row;
  const uint64_t* key;
  __device__ __forceinline__ bool operator()(int32_t p) const {
    return p == 0 || row[p] != row[p - 1] || key[p] != key[p - 1];
  }
};

}  // namespace rama
