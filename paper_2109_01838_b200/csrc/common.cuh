// Common device/host infrastructure for the RAMA B200 library.
//
// * Errors: internal code throws rama::Error; the C-ABI layer (capi.cu)
//   converts it to a status code + rama_last_error() message.
// * Memory: every scratch buffer is stream-ordered (cudaMallocAsync /
//   cudaFreeAsync) from the device's default pool, whose release threshold
//   is raised once so freed blocks are cached across rounds and solves.
// * Ids are int32 (n, m < 2^31), costs and multipliers fp64 (the reference
//   is fp64 throughout, graph.py:35).
#pragma once

#include <cuda_runtime.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <initializer_list>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>

namespace rama {

enum Status : int {
  kOk = 0,
  kInvalid = 1,   // -> ValueError
  kCuda = 2,      // -> RuntimeError
  kNoMemory = 3,  // -> MemoryError
  kInternal = 4,
};

struct Error : public std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define RAMA_CUDA(call)                                                                   \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess) {                                                              \
      throw ::rama::Error(_e == cudaErrorMemoryAllocation ? ::rama::kNoMemory              \
                                                          : ::rama::kCuda,                 \
                          std::string(#call) + ": " + cudaGetErrorString(_e) + " @" +     \
                              __FILE__ + ":" + std::to_string(__LINE__));                 \
    }                                                                                     \
  } while (0)

#define RAMA_LAUNCH_CHECK() RAMA_CUDA(cudaGetLastError())

#define RAMA_REQUIRE(cond, msg)                                   \
  do {                                                            \
    if (!(cond)) throw ::rama::Error(::rama::kInvalid, (msg));    \
  } while (0)

// RAMA_HOST_STATS=2: count host syncs per call chain (backtrace), printed
// after each solve
void note_sync();
void dump_sync_sites();

constexpr int kPinSlots = 512;   // pinned read-back block (int64 slots)
constexpr int kPinTagged = 256;  // first slot of fetch()'s tagged words

// Per-call context: the stream everything is ordered on plus a small pinned
// staging area for scalar read-backs (the only host syncs in a solve).
struct Ctx {
  cudaStream_t s = nullptr;
  int64_t* pinned = nullptr;  // kPinSlots int64 slots: 0-62 read-back data, 63 the sequence, kPinTagged.. tagged words
  int64_t* pinned_dev = nullptr;  // the same block, mapped into the device
  uint32_t seq = 0;           // last read-back sequence number published
  // piggyback: 8 device bytes the next fetch() brings back as well (the
  // round's lower bound rides on the contraction's first read-back)
  const void* piggy = nullptr;
  bool piggy_done = false;
  uint64_t piggy_val = 0;
  cudaEvent_t ev = nullptr;   // asynchronous read-backs (recycled with `pinned`)
  int launches = 0;           // kernels launched through this context

  explicit Ctx(cudaStream_t st);
  ~Ctx();
  Ctx(const Ctx&) = delete;
  Ctx& operator=(const Ctx&) = delete;
  void sync() {
    note_sync();
    RAMA_CUDA(cudaStreamSynchronize(s));
  }
};

void ensure_pool_configured();
// SM count of the current device (after ensure_pool_configured)
int num_sms();
// grow the stream-ordered pool to at least `bytes` up front (one mapping
// instead of many growth steps in the middle of a solve)
void reserve_pool(Ctx& ctx, size_t bytes);

// ---- live kernel-family timing (bench.py roofline) ------------------------
// When enabled (rama_profile_enable), each ProfScope records a CUDA event
// pair on the context stream around one kernel family and the algorithmic
// bytes it moves; rama_profile_read() sums elapsed time per family.
enum Family : int {
  kFamSeparate = 0,
  kFamTriangulate = 1,
  kFamMP = 2,
  kFamBound = 3,
  kFamMatching = 4,
  kFamForest = 5,
  kFamComponents = 6,
  kFamContract = 7,
  kFamCleanup = 8,
  kFamCanon = 9,
  kNumFamilies = 10
};
bool prof_enabled();
void prof_set(bool on);
void prof_push(int fam, cudaEvent_t a, cudaEvent_t b, double bytes);
void prof_read(double* ms, double* bytes, int64_t* count);
cudaEvent_t prof_event();  // from a recycled pool (no per-scope cudaEventCreate)

// per-kernel timing (same switch): an event pair around one launch, summed
// per kernel name; `bytes` = that launch's algorithmic bytes (0 = not
// defined for this kernel).  prof_set_bytes() tags the NEXT RAMA_KERNEL.
void prof_kernel_push(const char* name, cudaEvent_t a, cudaEvent_t b, double bytes);
// the innermost open family scope on this thread (-1: none); kernel time is
// also summed per family ("@<family index>" entries of the kernel JSON)
int prof_family_swap(int fam);
void prof_set_bytes(double bytes);
double prof_take_bytes();
// JSON {"kernel": [ms, bytes, launches], ...} of the kernels timed since enable
int64_t prof_kernels_json(char* out, int64_t cap);

struct KernelScope {
  cudaStream_t s;
  const char* name;
  double bytes;
  cudaEvent_t a = nullptr, b = nullptr;
  KernelScope(cudaStream_t st, const char* nm, double by = -1.0) : s(st), name(nm) {
    bytes = by >= 0.0 ? by : prof_take_bytes();
    if (prof_enabled()) {
      a = prof_event();
      b = prof_event();
      cudaEventRecord(a, s);
    }
  }
  ~KernelScope() {
    if (a) {
      cudaEventRecord(b, s);
      prof_kernel_push(name, a, b, bytes);
    }
  }
};

struct ProfScope {
  cudaStream_t s;
  int fam;
  double bytes;
  cudaEvent_t a = nullptr, b = nullptr;
  int outer;
  ProfScope(cudaStream_t st, int f, double by = 0.0) : s(st), fam(f), bytes(by) {
    outer = prof_family_swap(f);
    if (prof_enabled()) {
      a = prof_event();
      b = prof_event();
      cudaEventRecord(a, s);
    }
  }
  void add_bytes(double by) { bytes += by; }
  ~ProfScope() {
    prof_family_swap(outer);
    if (a) {
      cudaEventRecord(b, s);
      prof_push(fam, a, b, bytes);
    }
  }
};

// host-side accounting (RAMA_HOST_STATS=1): time in stream-ordered
// allocation calls and in scalar read-back waits, per thread
struct HostStats {
  double alloc_ms = 0, sync_ms = 0;
  int64_t allocs = 0, syncs = 0;
};
HostStats& host_stats();
inline double host_ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// Stream-keyed caching allocator over cudaMallocAsync: blocks are binned in
// size classes (<= 12.5% slack) and reused on the stream that freed them
// (same-stream reuse is ordered, no events needed).  After the first solve
// of a shape every scratch buffer comes from the cache.
void* dev_alloc(size_t bytes, cudaStream_t s);

// Caller-owned workspace (rama_solve_ws, SURVEY.md 8(b) ownership): while
// an ArenaScope is open on a thread, dev_alloc carves every buffer from the
// caller's device block (first fit, 256-byte aligned, coalescing free list;
// the call's work is on one stream, so a freed range is reusable at once)
// and nothing reaches the CUDA pool.  Exhaustion throws kNoMemory.
struct Arena {
  char* base;
  size_t size;
  size_t used = 0, peak = 0;
  std::map<size_t, size_t> free_, live_;  // offset -> length
  Arena(void* p, size_t n);
  void* alloc(size_t bytes);
  void release(void* p);
  bool owns(const void* p) const;
};
struct ArenaScope {
  Arena* prev;
  explicit ArenaScope(Arena* a);
  ~ArenaScope();
};
bool arena_active();
void dev_free(void* p, size_t bytes, cudaStream_t s);
// return every cached block of stream s to the pool (before destroying s)
void dev_release_stream(cudaStream_t s);
// return every cached block (all devices, all streams) and trim the pools
void dev_release_all();

template <class T>
struct Buf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;

  Buf() = default;
  Buf(size_t count, cudaStream_t st) { alloc(count, st); }
  Buf(size_t count, const Ctx& c) { alloc(count, c.s); }
  ~Buf() { release(); }
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  Buf(Buf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  Buf& operator=(Buf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count) {
      auto t0 = std::chrono::steady_clock::now();
      p = (T*)dev_alloc(sizeof(T) * count, st);
      HostStats& hs = host_stats();
      hs.alloc_ms += host_ms_since(t0);
      hs.allocs++;
    }
  }
  void release() {
    if (p) dev_free(p, sizeof(T) * n, s);
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
  operator T*() const { return p; }
  size_t bytes() const { return n * sizeof(T); }
  void zero() {
    if (n) RAMA_CUDA(cudaMemsetAsync(p, 0, bytes(), s));
  }
  void fill_bytes(int v) {
    if (n) RAMA_CUDA(cudaMemsetAsync(p, v, bytes(), s));
  }
};

constexpr int kBlock = 256;

inline unsigned grid_for(int64_t work, int block = kBlock) {
  int64_t g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 0x7fffffff) g = 0x7fffffff;
  return (unsigned)g;
}

// Grid-stride launch helper: caps the grid at a multiple of the SM count.
unsigned capped_grid(int64_t work, int block = kBlock);

// RAMA_TRACE=1 in the environment: print every launch and synchronise after
// it (debugging hangs / faults; never set for timing)
bool trace_enabled();   // RAMA_TRACE=1: print + sync after every launch
bool trace_print();     // RAMA_TRACE=1 or 2: print launches and sync points

#define RAMA_KERNEL(ctx, kernel, work, ...)                                           \
  do {                                                                                \
    int64_t _w = (int64_t)(work);                                                     \
    if (_w <= 0) ::rama::prof_take_bytes();                                           \
    if (_w > 0) {                                                                     \
      if (::rama::trace_print()) {                                                    \
        fprintf(stderr, "[rama] %s work=%lld\n", #kernel, (long long)_w);             \
        fflush(stderr);                                                               \
      }                                                                               \
      {                                                                               \
        ::rama::KernelScope _ks((ctx).s, #kernel);                                    \
        kernel<<<::rama::capped_grid(_w), ::rama::kBlock, 0, (ctx).s>>>(__VA_ARGS__); \
      }                                                                               \
      RAMA_LAUNCH_CHECK();                                                            \
      (ctx).launches++;                                                               \
      if (::rama::trace_enabled()) (ctx).sync();                                      \
    }                                                                                 \
  } while (0)

#define GRID_STRIDE(i, n) \
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)(n); i += (int64_t)gridDim.x * blockDim.x)

// ---- scalar read-back -----------------------------------------------------
// fetch(): up to four small device ranges (whole 4-byte words, <= 126 words
// in all) are written by a one-warp kernel into the mapped pinned block, each
// word in one 8-byte store together with the call's sequence number; the
// host spins until every word carries it (no system-scope fence on the
// device) and copies the words to byte offset `at` of the block.  Measured
// on the B200 with a flag-after-fence variant: 8.7 us per read-back round
// trip against 12.4 us for cudaMemcpyAsync + cudaStreamSynchronize
// (tools/readback_probe.cu).  Returns a pointer to the fetched bytes.
struct FetchPart {
  const void* src;
  int bytes;
};
void* fetch(Ctx& ctx, std::initializer_list<FetchPart> parts, int at = 0);

template <class T>
T read_scalar(Ctx& ctx, const T* dev) {
  static_assert(sizeof(T) % 4 == 0 && sizeof(T) <= 8, "scalar");
  T v;
  memcpy(&v, fetch(ctx, {{dev, (int)sizeof(T)}}), sizeof(T));
  return v;
}

// two int32 device scalars in one round trip
inline void read_pair(Ctx& ctx, const int32_t* a, const int32_t* b, int64_t& x, int64_t& y) {
  const int32_t* hp = (const int32_t*)fetch(ctx, {{a, 4}, {b, 4}});
  x = hp[0];
  y = hp[1];
}

template <class T>
void copy_d2d(Ctx& ctx, T* dst, const T* src, int64_t count) {
  if (count > 0) RAMA_CUDA(cudaMemcpyAsync(dst, src, sizeof(T) * count, cudaMemcpyDeviceToDevice, ctx.s));
}

template <class T>
void set_scalar(Ctx& ctx, T* dev, T value) {
  RAMA_CUDA(cudaMemcpyAsync(dev, &value, sizeof(T), cudaMemcpyHostToDevice, ctx.s));
  ctx.sync();  // value lives on the host stack
}

// ---- primitives (prims.cu) --------------------------------------------------
// exclusive prefix sum of n int32 counts; out has n+1 entries, out[n] = total.
// Returns the total (one read-back) when want_total.
int64_t exclusive_scan(Ctx& ctx, const int32_t* in, int32_t* out, int64_t n, bool want_total = true);
// in-place variant on int64
void exclusive_scan64(Ctx& ctx, const int64_t* in, int64_t* out, int64_t n);

// Bucket ("segmented") sort: items i in [0, N) with row[i] in [0, R) and a
// 64-bit key.  Produces row_ptr[R+1], and for each output slot p the row,
// key and source index, grouped by row and ascending by key inside a row.
// Keys are made unique by the caller (they embed an index) so the output is
// deterministic although the scatter uses atomics.
struct BucketSorted {
  Buf<int32_t> row_ptr;  // R + 1
  Buf<int32_t> row;      // N (row of slot p)
  Buf<uint64_t> key;     // N
  Buf<int32_t> src;      // N
  int64_t total = 0;     // kept items (row >= 0) = row_ptr[R]
  int64_t big_rows = 0;  // rows longer than 256 items
};
// Items with row < 0 are dropped.  Only rows < sort_rows are sorted
// (default all); later rows keep scatter order.
void bucket_sort(Ctx& ctx, int64_t R, int64_t N, const int32_t* row, const uint64_t* key, BucketSorted& out,
                 bool want_row = true, int64_t sort_rows = -1);

// stable LSD radix sort of (key, value) pairs on key bits [begin_bit, end_bit)
// (CUB onesweep): equal keys keep their input order
void radix_sort_pairs(Ctx& ctx, const uint64_t* k_in, const int32_t* v_in, uint64_t* k_out, int32_t* v_out,
                      int64_t N, int begin_bit = 0, int end_bit = 64);

// stable compaction of indices [0, n) where flag != 0; returns the count.
int64_t compact_indices(Ctx& ctx, const uint8_t* flags, int64_t n, Buf<int32_t>& out);

// deterministic fp64 sum (fixed block order, not numpy's order)
double device_sum(Ctx& ctx, const double* x, int64_t n);
// the same sum written to a device scalar (n >= 1), no read-back
void device_sum_to(Ctx& ctx, const double* x, int64_t n, double* out);
// out[j] (device) = device_sum of x[start[j], start[j] + len[j]), bit for
// bit (start, len: device int64[K]); 0.0 for an empty segment
void device_sums(Ctx& ctx, const double* x, const int64_t* start, const int64_t* len, int64_t K, double* out);

// row pointers of a (u, v)-sorted edge list: ptr[x] = first edge with u >= x
void row_ptr_from_sorted(Ctx& ctx, const int32_t* u, int64_t m, int64_t n, int32_t* ptr);

// numpy summation orders on device (see oracle/rama_oracle.c).  The
// summands come through an accessor: a contiguous array, or values gathered
// by index (so segment sums read c[src[p]] without a gathered copy).
struct DirectF64 {
  const double* p;
  __device__ __forceinline__ double operator[](int64_t i) const { return p[i]; }
  __device__ __forceinline__ DirectF64 operator+(int64_t k) const { return DirectF64{p + k}; }
};
struct GatherF64 {
  const double* c;
  const int32_t* idx;
  __device__ __forceinline__ double operator[](int64_t i) const { return c[idx[i]]; }
  __device__ __forceinline__ GatherF64 operator+(int64_t k) const { return GatherF64{c, idx + k}; }
};

template <class A>
__device__ __forceinline__ double pw_leaf(A a, int64_t n) {
  if (n < 8) {
    double r = -0.0;  // numpy 2.x starts the short sum at -0.0 (keeps -0.0 sums)
    for (int64_t i = 0; i < n; i++) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
  int64_t i;
  for (i = 8; i < n - (n % 8); i += 8) {
    r0 = __dadd_rn(r0, a[i + 0]); r1 = __dadd_rn(r1, a[i + 1]);
    r2 = __dadd_rn(r2, a[i + 2]); r3 = __dadd_rn(r3, a[i + 3]);
    r4 = __dadd_rn(r4, a[i + 4]); r5 = __dadd_rn(r5, a[i + 5]);
    r6 = __dadd_rn(r6, a[i + 6]); r7 = __dadd_rn(r7, a[i + 7]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                         __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
  for (; i < n; i++) res = __dadd_rn(res, a[i]);
  return res;
}

// numpy pairwise sum; iterative post-order walk of numpy's fixed recursion
// tree (split at n/2 rounded down to a multiple of 8, leaves <= 128).
template <class A>
__device__ __forceinline__ double pw_sum(A a, int64_t n) {
  if (n <= 128) return pw_leaf(a, n);
  int64_t fo[40], fl[40];
  double fleft[40];
  int fstage[40];
  int sp = 0;
  fo[0] = 0; fl[0] = n; fstage[0] = 0;
  double ret = 0.0;
  while (true) {
    if (fl[sp] <= 128) {
      ret = pw_leaf(a + fo[sp], fl[sp]);
      sp--;
    } else if (fstage[sp] == 0) {
      int64_t n2 = fl[sp] / 2; n2 -= n2 % 8;
      fstage[sp] = 1;
      fo[sp + 1] = fo[sp]; fl[sp + 1] = n2; fstage[sp + 1] = 0;
      sp++;
      continue;
    } else if (fstage[sp] == 1) {
      int64_t n2 = fl[sp] / 2; n2 -= n2 % 8;
      fleft[sp] = ret;
      fstage[sp] = 2;
      fo[sp + 1] = fo[sp] + n2; fl[sp + 1] = fl[sp] - n2; fstage[sp + 1] = 0;
      sp++;
      continue;
    } else {
      ret = __dadd_rn(fleft[sp], ret);
      sp--;
    }
    if (sp < 0) return ret;
  }
}

__device__ __forceinline__ double pw_leaf(const double* a, int64_t n) { return pw_leaf(DirectF64{a}, n); }
__device__ __forceinline__ double pw_sum(const double* a, int64_t n) { return pw_sum(DirectF64{a}, n); }

// one np.add.reduceat segment: x[0] + pairwise(x[1:])
template <class A>
__device__ __forceinline__ double seg_sum(A a, int64_t n) {
  if (n <= 0) return 0.0;
  if (n == 1) return a[0];  // x0 + pairwise([]) = x0 + (-0.0) = x0
  return __dadd_rn(a[0], pw_sum(a + 1, n - 1));
}
__device__ __forceinline__ double seg_sum(const double* a, int64_t n) { return seg_sum(DirectF64{a}, n); }

__device__ __forceinline__ uint64_t dbits(double x) { return (uint64_t)__double_as_longlong(x); }

// atomicAdd(cnt + r, delta) for every lane with r >= 0, aggregated over runs
// of equal r in consecutive lanes: histogram inputs grouped by row (sorted
// edge lists, power-law hub rows) take one atomic per run instead of one per
// item.  Returns the value the lane's own atomic would have returned in
// lane order (old + delta x rank in the run): distinct offsets per item.
// All 32 lanes of the warp must call it.
__device__ __forceinline__ int32_t run_atomic_add(int32_t* cnt, int32_t r, int32_t delta) {
  const int lane = threadIdx.x & 31;
  const int32_t prev = __shfl_up_sync(0xffffffffu, r, 1);
  const bool act = r >= 0;
  const bool head = act && (lane == 0 || prev != r);
  const unsigned heads = __ballot_sync(0xffffffffu, head);
  const unsigned stops = heads | __ballot_sync(0xffffffffu, !act);  // a run ends at the next head or inactive lane
  const unsigned upto = 0xffffffffu >> (31 - lane);                  // lanes 0..lane
  const int h = act ? 31 - __clz(heads & upto) : lane;
  int32_t old = 0;
  if (head) {
    const unsigned above = stops & ~upto;
    const int end = above ? __ffs(above) - 1 : 32;
    old = atomicAdd(cnt + r, delta * (end - lane));
  }
  old = __shfl_sync(0xffffffffu, old, h);
  return old + delta * (lane - h);
}

// Handshake votes: *pa = max(*pa, (hi, lo_a)) and *pb = max(*pb, (hi, lo_b))
// as unsigned 128-bit values (hi = cost bits, lo = ~neighbour id).  The two
// CAS loops are interleaved so both atomics are in flight together.
__device__ __forceinline__ void vote_max_pair(ulonglong2* pa, unsigned long long lo_a, ulonglong2* pb,
                                              unsigned long long lo_b, unsigned long long hi) {
  const unsigned __int128 ka = ((unsigned __int128)hi << 64) | lo_a;
  const unsigned __int128 kb = ((unsigned __int128)hi << 64) | lo_b;
  unsigned __int128 ca = 0, cb = 0;
  bool da = !(ka > ca), db = !(kb > cb);
  while (!(da && db)) {
    unsigned __int128 oa = ca, ob = cb;
    if (!da) oa = atomicCAS((unsigned __int128*)pa, ca, ka);
    if (!db) ob = atomicCAS((unsigned __int128*)pb, cb, kb);
    if (!da) {
      if (oa == ca) da = true;
      else { ca = oa; da = !(ka > ca); }
    }
    if (!db) {
      if (ob == cb) db = true;
      else { cb = ob; db = !(kb > cb); }
    }
  }
}

}  // namespace rama
