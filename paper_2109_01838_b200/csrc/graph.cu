// Graph core kernels: canonicalisation (a3), connected components (a17),
// contraction (a18), composition (a19) and the clustering objective (a21).
//
// Contraction = relabel + bucket sort by the contracted row u' with key
// (v' << 32 | edge index) + segmented reduce.  Sorting within a (u', v')
// segment by source edge index reproduces numpy's stable lexsort, and the
// segment sum reproduces np.add.reduceat's x0 + pairwise(x[1:]) order, so
// contracted costs are bit-identical to the reference (contraction.py:155-162).
// Merged (f(u) == f(v)) edges get row -1 and are dropped by the bucket sort,
// which avoids a separate compaction pass.
#include "internal.h"

namespace rama {

// --------------------------------------------------------------- helpers

__global__ void k_iota(int32_t* x, int64_t n) {
  GRID_STRIDE(i, n) x[i] = (int32_t)i;
}

void iota(Ctx& ctx, int32_t* x, int64_t n) { RAMA_KERNEL(ctx, k_iota, n, x, n); }

// head[p] = slot p starts a new (row, key-high) segment (p < limit)
__global__ void k_seg_heads(const int32_t* __restrict__ row, const uint64_t* __restrict__ key, int64_t limit,
                            uint8_t* __restrict__ head) {
  GRID_STRIDE(p, limit) {
    head[p] = (p == 0) || row[p] != row[p - 1] || (key[p] >> 32) != (key[p - 1] >> 32);
  }
}

// out edge j = segment [heads[j], heads[j+1]) of the sorted slots
__global__ void k_seg_reduce(const int32_t* __restrict__ heads, int64_t k, int64_t limit,
                             const int32_t* __restrict__ row, const uint64_t* __restrict__ key,
                             const double* __restrict__ c, const int32_t* __restrict__ src,
                             int32_t* __restrict__ ou, int32_t* __restrict__ ov, double* __restrict__ oc) {
  GRID_STRIDE(j, k) {
    int64_t b = heads[j];
    int64_t e = (j + 1 < k) ? heads[j + 1] : limit;
    ou[j] = row[b];
    ov[j] = (int32_t)(key[b] >> 32);
    oc[j] = seg_sum(GatherF64{c, src + b}, e - b);  // c in sorted order, gathered in place
  }
}

// reduce sorted slots [0, limit) into a canonical graph
static Graph reduce_sorted(Ctx& ctx, int64_t n_out, int64_t limit, BucketSorted& bs, const double* c) {
  Graph out;
  out.n = n_out;
  Buf<uint8_t> head(limit > 0 ? limit : 1, ctx);
  RAMA_KERNEL(ctx, k_seg_heads, limit, bs.row.p, bs.key.p, limit, head.p);
  Buf<int32_t> hp;
  int64_t k = compact_indices(ctx, head.p, limit, hp);
  out.m = k;
  out.u.alloc(k > 0 ? k : 1, ctx.s);
  out.v.alloc(k > 0 ? k : 1, ctx.s);
  out.c.alloc(k > 0 ? k : 1, ctx.s);
  RAMA_KERNEL(ctx, k_seg_reduce, k, hp.p, k, limit, bs.row.p, bs.key.p, c, bs.src.p, out.u.p, out.v.p, out.c.p);
  return out;
}

// ---------------------------------------------------------- canonicalize

__global__ void k_canon_prep(const int32_t* __restrict__ u, const int32_t* __restrict__ v, int64_t m, int64_t n,
                             int32_t* __restrict__ row, uint64_t* __restrict__ key, int32_t* __restrict__ err) {
  GRID_STRIDE(i, m) {
    int32_t a = u[i], b = v[i];
    if (a == b) atomicOr(err, 1);
    if (a < 0 || b < 0 || a >= n || b >= n) {
      atomicOr(err, 2);
      a = 0; b = 0;
    }
    int32_t lo = a < b ? a : b, hi = a < b ? b : a;
    row[i] = lo;
    key[i] = ((uint64_t)(uint32_t)hi << 32) | (uint64_t)i;
  }
}

Graph canonicalize(Ctx& ctx, int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m) {
  ProfScope prof(ctx.s, kFamCanon);
  RAMA_REQUIRE(n >= 0, "num_nodes must be non-negative");
  RAMA_REQUIRE(n < (1LL << 31) && m < (1LL << 31), "graph too large for int32 ids");
  if (m == 0) {
    Graph g;
    g.n = n;
    return g;
  }
  Buf<int32_t> row(m, ctx), err(1, ctx);
  Buf<uint64_t> key(m, ctx);
  err.zero();
  RAMA_KERNEL(ctx, k_canon_prep, m, u, v, m, n, row.p, key.p, err.p);
  int32_t e = read_scalar(ctx, err.p);
  RAMA_REQUIRE(!(e & 1), "self-loops are not allowed");
  RAMA_REQUIRE(!(e & 2), "edge endpoint out of range");
  BucketSorted bs;
  bucket_sort(ctx, n, m, row.p, key.p, bs);
  return reduce_sorted(ctx, n, m, bs, c);
}

// ------------------------------------------------------------ components

__device__ __forceinline__ int32_t uf_find(int32_t* p, int32_t x) {
  while (true) {
    int32_t px = __ldcg(p + x);
    if (px == x) return x;
    int32_t gp = __ldcg(p + px);
    if (gp != px) p[x] = gp;  // path halving; pointers only move to ancestors
    x = px;
  }
}

// hook the larger root under the smaller one => final root = component min
__device__ __forceinline__ void uf_union(int32_t* p, int32_t a, int32_t b) {
  while (true) {
    a = uf_find(p, a);
    b = uf_find(p, b);
    if (a == b) return;
    int32_t lo = a < b ? a : b, hi = a < b ? b : a;
    int32_t old = atomicCAS(p + hi, hi, lo);
    if (old == hi) return;
    a = lo;
    b = old;
  }
}

__global__ void k_cc_check(const int32_t* __restrict__ su, const int32_t* __restrict__ sv, int64_t k, int64_t n,
                           int32_t* err) {
  GRID_STRIDE(i, k) {
    if (su[i] < 0 || sv[i] < 0 || su[i] >= n || sv[i] >= n) atomicOr(err, 1);
  }
}

__global__ void k_cc_hook(const int32_t* __restrict__ su, const int32_t* __restrict__ sv, int64_t k,
                          int32_t* parent) {
  GRID_STRIDE(i, k) uf_union(parent, su[i], sv[i]);
}

// read-only find: a flatten pass must not path-halve, or another thread's
// halving store can land after `parent[x] = root` and leave x pointing at a
// non-root ancestor.
__device__ __forceinline__ int32_t uf_root(const int32_t* p, int32_t x) {
  while (true) {
    int32_t px = __ldcg(p + x);
    if (px == x) return x;
    x = px;
  }
}

__global__ void k_cc_flatten(int32_t* parent, int64_t n, int32_t* __restrict__ is_root) {
  GRID_STRIDE(x, n) {
    int32_t r = uf_root(parent, (int32_t)x);
    parent[x] = r;
    is_root[x] = (r == x);
  }
}

__global__ void k_cc_label(const int32_t* __restrict__ parent, const int32_t* __restrict__ rank, int64_t n,
                           int32_t* __restrict__ map) {
  GRID_STRIDE(x, n) map[x] = rank[parent[x]];
}

int64_t components(Ctx& ctx, int64_t n, const int32_t* su, const int32_t* sv, int64_t k, int32_t* map, bool check) {
  ProfScope prof(ctx.s, kFamComponents);
  if (n == 0) return 0;
  if (check && k > 0) {
    Buf<int32_t> err(1, ctx);
    err.zero();
    RAMA_KERNEL(ctx, k_cc_check, k, su, sv, k, n, err.p);
    RAMA_REQUIRE(read_scalar(ctx, err.p) == 0, "contraction edge endpoint out of range");
  }
  Buf<int32_t> parent(n, ctx), flag(n, ctx), rank(n + 1, ctx);
  iota(ctx, parent.p, n);
  RAMA_KERNEL(ctx, k_cc_hook, k, su, sv, k, parent.p);
  RAMA_KERNEL(ctx, k_cc_flatten, n, parent.p, n, flag.p);
  int64_t nt = exclusive_scan(ctx, flag.p, rank.p, n, true);
  RAMA_KERNEL(ctx, k_cc_label, n, parent.p, rank.p, n, map);
  return nt;
}

// -------------------------------------------------------------- contract

__global__ void k_contract_prep(const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                                const double* __restrict__ c, int64_t m, const int32_t* __restrict__ f,
                                int32_t n_out, int32_t* __restrict__ row, uint64_t* __restrict__ key,
                                double* __restrict__ jc) {
  GRID_STRIDE(i, m) {
    int32_t a = f[u[i]], b = f[v[i]];
    if (a == b) {
      row[i] = -1;  // merged edge: dropped by the bucket sort, joined mass
      key[i] = (uint64_t)i;
      if (jc) jc[i] = c[i];
    } else {
      int32_t lo = a < b ? a : b, hi = a < b ? b : a;
      row[i] = lo;
      key[i] = ((uint64_t)(uint32_t)hi << 32) | (uint64_t)i;
      if (jc) jc[i] = 0.0;
    }
  }
}

Graph contract(Ctx& ctx, const GraphView& g, const int32_t* map, int64_t n_targets, double* joined) {
  // algorithmic bytes: 24 m_in + 16 m_out
  ProfScope prof(ctx.s, kFamContract, 24.0 * (double)g.m);
  int64_t m = g.m;
  if (m == 0) {
    if (joined) *joined = 0.0;
    Graph out;
    out.n = n_targets;
    return out;
  }
  Buf<int32_t> row(m, ctx);
  Buf<uint64_t> key(m, ctx);
  Buf<double> jc;
  if (joined) jc.alloc(m, ctx.s);
  prof_set_bytes(36.0 * (double)m);
  RAMA_KERNEL(ctx, k_contract_prep, m, g.u, g.v, g.c, m, map, (int32_t)n_targets, row.p, key.p,
              joined ? jc.p : (double*)nullptr);
  if (joined) *joined = device_sum(ctx, jc.p, m);
  BucketSorted bs;
  bucket_sort(ctx, n_targets, m, row.p, key.p, bs, true);
  int64_t limit = bs.total;
  Graph out = reduce_sorted(ctx, n_targets, limit, bs, g.c);
  prof.add_bytes(16.0 * (double)out.m);
  return out;
}

// --------------------------------------------------------------- compose

__global__ void k_compose(int32_t* __restrict__ ft, int64_t n0, const int32_t* __restrict__ f) {
  GRID_STRIDE(i, n0) ft[i] = f[ft[i]];
}

void compose(Ctx& ctx, int32_t* f_total, int64_t n0, const int32_t* f) {
  RAMA_KERNEL(ctx, k_compose, n0, f_total, n0, f);
}

// ------------------------------------------------------------------ cost

__global__ void k_cut_costs(const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                            const double* __restrict__ c, int64_t m, const int32_t* __restrict__ lab,
                            double* __restrict__ x) {
  GRID_STRIDE(i, m) x[i] = (lab[u[i]] != lab[v[i]]) ? c[i] : 0.0;
}

double clustering_cost(Ctx& ctx, const GraphView& g, const int32_t* labels) {
  if (g.m == 0) return 0.0;
  Buf<double> x(g.m, ctx);
  RAMA_KERNEL(ctx, k_cut_costs, g.m, g.u, g.v, g.c, g.m, labels, x.p);
  return device_sum(ctx, x.p, g.m);
}

}  // namespace rama
