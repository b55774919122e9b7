// Graph core kernels: canonicalisation (a3), connected components (a17),
// contraction (a18), composition (a19) and the clustering objective (a21).
//
// Contraction = one fused sort-reduce (sortreduce.cuh): the relabel by f
// happens inside its count and scatter passes, items are grouped by the
// contracted row u' with key (v' << 32 | edge index), and each unique
// (u', v') group is written at its final position with its segment sum.
// Sorting within a group by source edge index reproduces numpy's stable
// lexsort, and the sum reproduces np.add.reduceat's x0 + pairwise(x[1:])
// order, so contracted costs are bit-identical to the reference
// (contraction.py:155-162).  Merged (f(u) == f(v)) edges produce no item.
#include "internal.h"
#include "sortreduce.cuh"

namespace rama {

// --------------------------------------------------------------- helpers

__global__ void k_iota(int32_t* x, int64_t n) {
  GRID_STRIDE(i, n) x[i] = (int32_t)i;
}

void iota(Ctx& ctx, int32_t* x, int64_t n) { RAMA_KERNEL(ctx, k_iota, n, x, n); }

// ---------------------------------------------------------- canonicalize

// validation pass (graph.py:31-42): raised before any work
__global__ void k_canon_check(const int32_t* __restrict__ u, const int32_t* __restrict__ v, int64_t m, int64_t n,
                              int32_t* __restrict__ err) {
  GRID_STRIDE(i, m) {
    const int32_t a = u[i], b = v[i];
    if (a == b) atomicOr(err, 1);
    if (a < 0 || b < 0 || a >= n || b >= n) atomicOr(err, 2);
  }
}

// items of a raw COO: row = min endpoint, key = (max << 32 | edge), pay = c
struct CanonSrc {
  static constexpr int kK = 1;
  const int32_t* u;
  const int32_t* v;
  const double* c;
  int64_t m;
  __host__ __device__ __forceinline__ int64_t size() const { return m; }
  __device__ __forceinline__ bool item(int64_t i, int, int32_t& row, uint64_t& key, double& pay) const {
    const int32_t a = u[i], b = v[i];
    row = a < b ? a : b;
    key = ((uint64_t)(uint32_t)(a < b ? b : a) << 32) | (uint64_t)i;
    pay = c[i];
    return true;
  }
};

// items of a contraction (contraction.py:148-160): row = min(f(u), f(v)),
// key = (max << 32 | edge); merged edges (f(u) == f(v)) produce nothing
struct ContractSrc {
  static constexpr int kK = 1;
  const int32_t* u;
  const int32_t* v;
  const double* c;
  const int32_t* f;
  int64_t m;
  __host__ __device__ __forceinline__ int64_t size() const { return m; }
  __device__ __forceinline__ bool item(int64_t i, int, int32_t& row, uint64_t& key, double& pay) const {
    const int32_t a = __ldg(f + u[i]), b = __ldg(f + v[i]);
    if (a == b) return false;
    row = a < b ? a : b;
    key = ((uint64_t)(uint32_t)(a < b ? b : a) << 32) | (uint64_t)i;
    pay = c[i];
    return true;
  }
};

// one canonical edge per (row, hi) group: cost = np.add.reduceat order over
// the group's source edges (keys embed the source index => source order)
struct GraphEmit {
  int32_t* ou;
  int32_t* ov;
  double* oc;
  __device__ __forceinline__ bool keep(int32_t, uint64_t) const { return true; }
  template <class A>
  __device__ __forceinline__ void out(int64_t idx, int32_t row, uint64_t key, A pays, int64_t len) const {
    ou[idx] = row;
    ov[idx] = (int32_t)(key >> 32);
    // reduceat: x0 + pairwise(x[1:]); two terms are x0 + x1 in either order
    oc[idx] = len == 1 ? pays[0] : len == 2 ? __dadd_rn(pays[0], pays[1]) : seg_sum(pays, len);
  }
};

template <class Src>
static Graph sort_reduce_graph(Ctx& ctx, int64_t n_out, int64_t m_in, const Src& src,
                               const int32_t* nt_dev = nullptr) {
  Graph out;
  out.n = n_out;
  out.u.alloc(m_in > 0 ? m_in : 1, ctx.s);
  out.v.alloc(m_in > 0 ? m_in : 1, ctx.s);
  out.c.alloc(m_in > 0 ? m_in : 1, ctx.s);
  SrResult sr;
  int64_t nt = n_out;
  out.m = sort_reduce<32, true, true>(ctx, n_out, m_in, src, GraphEmit{out.u.p, out.v.p, out.c.p}, sr, true, "sr",
                                      nt_dev, &nt);
  out.n = nt;
  return out;
}

Graph canonicalize(Ctx& ctx, int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m) {
  // algorithmic bytes: raw COO read once, canonical COO written (<= m)
  ProfScope prof(ctx.s, kFamCanon, 32.0 * (double)m);
  RAMA_REQUIRE(n >= 0, "num_nodes must be non-negative");
  RAMA_REQUIRE(n < (1LL << 31) && m < (1LL << 31), "graph too large for int32 ids");
  if (m == 0) {
    Graph g;
    g.n = n;
    return g;
  }
  Buf<int32_t> err(1, ctx);
  err.zero();
  RAMA_KERNEL(ctx, k_canon_check, m, u, v, m, n, err.p);
  int32_t e = read_scalar(ctx, err.p);
  RAMA_REQUIRE(!(e & 1), "self-loops are not allowed");
  RAMA_REQUIRE(!(e & 2), "edge endpoint out of range");
  return sort_reduce_graph(ctx, n, m, CanonSrc{u, v, c, m});
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

int64_t components(Ctx& ctx, int64_t n, const int32_t* su, const int32_t* sv, int64_t k, int32_t* map, bool check,
                   Buf<int32_t>* keep_rank) {
  // algorithmic bytes: the pairs read once, the map written
  ProfScope prof(ctx.s, kFamComponents, 8.0 * (double)k + 4.0 * (double)n);
  if (n == 0) return 0;
  if (check && k > 0) {
    Buf<int32_t> err(1, ctx);
    err.zero();
    RAMA_KERNEL(ctx, k_cc_check, k, su, sv, k, n, err.p);
    RAMA_REQUIRE(read_scalar(ctx, err.p) == 0, "contraction edge endpoint out of range");
  }
  Buf<int32_t> parent(n, ctx), flag(n, ctx), own_rank;
  Buf<int32_t>& rank = keep_rank ? *keep_rank : own_rank;
  rank.alloc(n + 1, ctx.s);
  iota(ctx, parent.p, n);
  RAMA_KERNEL(ctx, k_cc_hook, k, su, sv, k, parent.p);
  RAMA_KERNEL(ctx, k_cc_flatten, n, parent.p, n, flag.p);
  int64_t nt = exclusive_scan(ctx, flag.p, rank.p, n, !keep_rank);  // rank[n] = number of components
  RAMA_KERNEL(ctx, k_cc_label, n, parent.p, rank.p, n, map);
  return keep_rank ? -1 : nt;
}

__global__ void k_is_canonical(const int32_t* __restrict__ u, const int32_t* __restrict__ v, int64_t m, int64_t n,
                               int32_t* bad) {
  GRID_STRIDE(i, m) {
    bool ok = u[i] >= 0 && u[i] < v[i] && v[i] < n;
    if (ok && i > 0) ok = u[i - 1] < u[i] || (u[i - 1] == u[i] && v[i - 1] < v[i]);
    if (!ok) atomicOr(bad, 1);
  }
}

bool is_canonical(Ctx& ctx, const GraphView& g) {
  if (g.m == 0) return true;
  Buf<int32_t> bad(1, ctx);
  bad.zero();
  RAMA_KERNEL(ctx, k_is_canonical, g.m, g.u, g.v, g.m, g.n, bad.p);
  return read_scalar(ctx, bad.p) == 0;
}

// -------------------------------------------------------------- contract

// mass of the merged edges (contraction.py:151): only when a caller asks
__global__ void k_joined_mass(const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                              const double* __restrict__ c, int64_t m, const int32_t* __restrict__ f,
                              double* __restrict__ jc) {
  GRID_STRIDE(i, m) jc[i] = (f[u[i]] == f[v[i]]) ? c[i] : 0.0;
}

// ---- contraction by a device-wide radix sort (long rows) -----------------
// When the contracted rows are long (the cleanup's quotient of the original
// graph: 9.9 M edges into ~290 k clusters on C2), the row tiles of the
// sort-reduce spend their time on long in-row rankings and on waiting for
// each other's look-back.  This path sorts (min, max) target pairs packed in
// 2 * bits(R) key bits with the source index as the value by CUB's stable
// LSD onesweep passes -- equal pairs keep the canonical source order, i.e.
// exactly the reduceat order of contraction.py:142-163 -- then marks the
// heads of equal keys, compacts them, and sums each group in numpy's
// pairwise order from the gathered costs.
// self-loops (both ends in one target) are dropped before the sort: a flag
// per edge, a stable compaction, then (key, source index) of the kept edges
__global__ void k_crx_flags(const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                            const int32_t* __restrict__ f, int64_t m, uint8_t* __restrict__ cross) {
  GRID_STRIDE(i, m) cross[i] = __ldg(f + u[i]) != __ldg(f + v[i]);
}

__global__ void k_crx_keys_of(const int32_t* __restrict__ E, int64_t N, const int32_t* __restrict__ u,
                              const int32_t* __restrict__ v, const int32_t* __restrict__ f, int bits,
                              uint64_t* __restrict__ key, int32_t* __restrict__ val) {
  GRID_STRIDE(t, N) {
    const int32_t i = E[t];
    const int32_t a = __ldg(f + u[i]), b = __ldg(f + v[i]);
    key[t] = ((uint64_t)(uint32_t)(a < b ? a : b) << bits) | (uint64_t)(uint32_t)(a < b ? b : a);
    val[t] = i;
  }
}

__global__ void k_crx_heads(const uint64_t* __restrict__ key, int64_t m, int bits, uint8_t* __restrict__ head,
                            int32_t* __restrict__ nvalid) {
  const uint64_t sentinel = (1ull << (2 * bits)) - 1ull;
  GRID_STRIDE(p, m) {
    const uint64_t k = key[p];
    const bool ok = k != sentinel;
    head[p] = ok && (p == 0 || key[p - 1] != k);
    if (ok && (p + 1 == m || key[p + 1] == sentinel)) *nvalid = (int32_t)(p + 1);
  }
}

struct GatherPay {  // costs of a run of sorted positions through the source index
  const double* c;
  const int32_t* idx;
  __device__ __forceinline__ double operator[](int64_t i) const { return c[idx[i]]; }
  __device__ __forceinline__ GatherPay operator+(int64_t k) const { return GatherPay{c, idx + k}; }
};

__global__ void k_crx_emit(const int32_t* __restrict__ H, int64_t M, const int32_t* __restrict__ nvalid,
                           const uint64_t* __restrict__ key, const int32_t* __restrict__ val,
                           const double* __restrict__ c, int bits, int32_t* __restrict__ ou, int32_t* __restrict__ ov,
                           double* __restrict__ oc) {
  const int64_t end = *nvalid;
  GRID_STRIDE(gi, M) {
    const int64_t p = H[gi], e = gi + 1 < M ? H[gi + 1] : end;
    const uint64_t k = key[p];
    ou[gi] = (int32_t)(k >> bits);
    ov[gi] = (int32_t)(k & ((1ull << bits) - 1ull));
    const GatherPay pays{c, val + p};
    const int64_t len = e - p;
    oc[gi] = len == 1 ? pays[0] : len == 2 ? __dadd_rn(pays[0], pays[1]) : seg_sum(pays, len);
  }
}

static Graph contract_radix(Ctx& ctx, const GraphView& g, const int32_t* map, int64_t n_targets,
                            const int32_t* nt_dev) {
  const int64_t m = g.m;
  int bits = 1;
  while ((1ll << bits) <= n_targets) bits++;  // ids <= n_targets - 1 < 2^bits - 1
  int64_t N = m;  // edges into the sort
  Buf<int32_t> E;
  {
    Buf<uint8_t> cross(m, ctx);
    RAMA_KERNEL(ctx, k_crx_flags, m, g.u, g.v, map, m, cross.p);
    N = compact_indices(ctx, cross.p, m, E);  // ascending: the source order is kept
  }
  Buf<uint64_t> k1(N > 0 ? N : 1, ctx), k2(N > 0 ? N : 1, ctx);
  Buf<int32_t> v1(N > 0 ? N : 1, ctx), v2(N > 0 ? N : 1, ctx);
  RAMA_KERNEL(ctx, k_crx_keys_of, N, E.p, N, g.u, g.v, map, bits, k1.p, v1.p);
  E.release();
  radix_sort_pairs(ctx, k1.p, v1.p, k2.p, v2.p, N, 0, 2 * bits);
  k1.release();
  v1.release();
  Buf<uint8_t> head(N > 0 ? N : 1, ctx);
  Buf<int32_t> nvalid(1, ctx);
  nvalid.zero();
  RAMA_KERNEL(ctx, k_crx_heads, N, k2.p, N, bits, head.p, nvalid.p);
  Buf<int32_t> H;
  const int64_t M = compact_indices(ctx, head.p, N, H);
  Graph out;
  out.n = nt_dev ? (int64_t)read_scalar(ctx, nt_dev) : n_targets;  // (forced radix on a round contraction)
  out.m = M;
  out.u.alloc(M > 0 ? M : 1, ctx.s);
  out.v.alloc(M > 0 ? M : 1, ctx.s);
  out.c.alloc(M > 0 ? M : 1, ctx.s);
  RAMA_KERNEL(ctx, k_crx_emit, M, H.p, M, nvalid.p, k2.p, v2.p, g.c, bits, out.u.p, out.v.p, out.c.p);
  return out;
}

Graph contract(Ctx& ctx, const GraphView& g, const int32_t* map, int64_t n_targets, double* joined,
               const int32_t* nt_dev) {
  // algorithmic bytes: 24 m_in + 16 m_out
  ProfScope prof(ctx.s, kFamContract, 24.0 * (double)g.m);
  const int64_t m = g.m;
  if (m == 0) {
    if (joined) *joined = 0.0;
    Graph out;
    out.n = nt_dev ? (int64_t)read_scalar(ctx, nt_dev) : n_targets;
    return out;
  }
  if (joined) {
    Buf<double> jc(m, ctx);
    RAMA_KERNEL(ctx, k_joined_mass, m, g.u, g.v, g.c, m, map, jc.p);
    *joined = device_sum(ctx, jc.p, m);
  }
  // long rows on average (few targets per edge: the cleanup's quotient) take
  // the radix path; RAMA_CONTRACT_RADIX=0/1 forces either (A/B, tests)
  static const int force_radix = [] {
    const char* e = getenv("RAMA_CONTRACT_RADIX");
    return e ? atoi(e) : -1;
  }();
  const bool radix = force_radix == 1 || (force_radix < 0 && !nt_dev && m >= 16 * n_targets);
  Graph out = radix ? contract_radix(ctx, g, map, n_targets, nt_dev)
                    : sort_reduce_graph(ctx, n_targets, m, ContractSrc{g.u, g.v, g.c, map, m}, nt_dev);
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

void cut_costs(Ctx& ctx, const GraphView& g, const int32_t* labels, double* x) {
  RAMA_KERNEL(ctx, k_cut_costs, g.m, g.u, g.v, g.c, g.m, labels, x);
}

double clustering_cost(Ctx& ctx, const GraphView& g, const int32_t* labels) {
  if (g.m == 0) return 0.0;
  Buf<double> x(g.m, ctx);
  cut_costs(ctx, g, labels, x.p);
  return device_sum(ctx, x.p, g.m);
}

}  // namespace rama
