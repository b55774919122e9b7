// Generic device primitives: prefix scans, compaction, deterministic sums,
// row pointers, the caching allocator / caller workspace, and the bucket
// sort behind the positive CSR, the triplet and chord dedupe and the
// edge->slot lists (canonicalisation and contraction use the fused
// sort-reduce of sortreduce.cuh).
//
// Bucket sort = counting sort on a 32-bit row id (warp-aggregated atomic
// histogram + scan + scatter) followed by an in-row sort on a 64-bit key.
// Rows in this solver are short (grid degrees), so the in-row order comes
// from a thread-per-item rank over the row (warp-broadcast loads); rows
// longer than 64 use a shared-memory bitonic sort per block, and the rare
// huge rows (power-law hubs) CUB's segmented sort.  CUB is used only
// for generic scans/selection/segmented sorting, never for domain logic.
#include "common.cuh"
#include "sortreduce.cuh"

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <cxxabi.h>
#include <execinfo.h>

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <map>
#include <string>
#include <vector>

namespace rama {

HostStats& host_stats() {
  static thread_local HostStats hs;
  return hs;
}

namespace {
std::map<std::string, int64_t>& sync_sites() {
  static thread_local std::map<std::string, int64_t> m;
  return m;
}
bool sync_sites_on() {
  static const bool on = [] {
    const char* e = getenv("RAMA_HOST_STATS");
    return e && atoi(e) >= 2;
  }();
  return on;
}
}  // namespace

void note_sync() {
  if (!sync_sites_on()) return;
  void* bt[10];
  const int k = backtrace(bt, 10);
  char** sy = backtrace_symbols(bt, k);
  std::string key;
  for (int i = 1; i < k && i < 7; i++) {
    std::string f = sy ? sy[i] : "?";
    const size_t a = f.find('('), b = f.find('+', a == std::string::npos ? 0 : a);
    std::string name = (a != std::string::npos && b != std::string::npos && b > a + 1) ? f.substr(a + 1, b - a - 1) : "?";
    int st = 0;
    char* dm = abi::__cxa_demangle(name.c_str(), nullptr, nullptr, &st);
    if (st == 0 && dm) {
      name = dm;
      const size_t p = name.find('(');
      if (p != std::string::npos) name = name.substr(0, p);
    }
    free(dm);
    if (!key.empty()) key += " < ";
    key += name;
    if (name.find("solve") != std::string::npos) break;
  }
  free(sy);
  sync_sites()[key]++;
}

void dump_sync_sites() {
  if (!sync_sites_on()) return;
  std::vector<std::pair<int64_t, std::string>> v;
  for (auto& kv : sync_sites()) v.push_back({kv.second, kv.first});
  std::sort(v.rbegin(), v.rend());
  for (auto& x : v) fprintf(stderr, "[rama] syncs %4lld  %s\n", (long long)x.first, x.second.c_str());
  sync_sites().clear();
}

// Pinned staging blocks are recycled across calls: cudaMallocHost /
// cudaFreeHost cost milliseconds and cudaFreeHost synchronises the device.
namespace {
std::mutex g_pin_mu;
std::vector<std::pair<int64_t*, cudaEvent_t>> g_pin_free;
}  // namespace

Ctx::Ctx(cudaStream_t st) : s(st) {
  ensure_pool_configured();
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (!g_pin_free.empty()) {
      pinned = g_pin_free.back().first;
      ev = g_pin_free.back().second;
      g_pin_free.pop_back();
    }
  }
  if (!pinned) {
    RAMA_CUDA(cudaHostAlloc((void**)&pinned, kPinSlots * sizeof(int64_t), cudaHostAllocMapped | cudaHostAllocPortable));
    memset(pinned, 0, kPinSlots * sizeof(int64_t));
    RAMA_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  RAMA_CUDA(cudaHostGetDevicePointer((void**)&pinned_dev, pinned, 0));
  seq = *(volatile uint32_t*)(pinned + 63);  // a recycled block continues its sequence
}

namespace {
struct FetchArgs {
  const uint32_t* src[4];
  int words[4];
  int n;
};
// Every word travels with the call's sequence number in one 8-byte store
// (sequence << 32 | word), so the host waits for all tags instead of a flag
// published after a system-scope fence (the same self-validating 8-byte
// protocol as NCCL's LL transport): no fence round trip on the device.
__global__ void k_fetch(FetchArgs a, volatile unsigned long long* tagged, uint32_t s) {
  int o = 0;
  for (int k = 0; k < a.n; k++) {
    for (int i = threadIdx.x; i < a.words[k]; i += blockDim.x)
      tagged[o + i] = ((unsigned long long)s << 32) | (unsigned long long)__ldcg(a.src[k] + i);
    o += a.words[k];
  }
  if (o == 0 && threadIdx.x == 0) tagged[0] = (unsigned long long)s << 32;  // a pure sync point
}
}  // namespace

void* fetch(Ctx& ctx, std::initializer_list<FetchPart> parts, int at) {
  if (trace_print()) {
    fprintf(stderr, "[rama] sync\n");
    fflush(stderr);
  }
  note_sync();
  auto t0 = std::chrono::steady_clock::now();
  FetchArgs a{};
  int words = 0;
  for (const FetchPart& p : parts) {
    RAMA_REQUIRE(a.n < 4 && p.bytes % 4 == 0, "fetch: at most four word-sized parts");
    a.src[a.n] = (const uint32_t*)p.src;
    a.words[a.n] = p.bytes / 4;
    words += a.words[a.n];
    a.n++;
  }
  int piggy_at = -1;  // word offset of the piggyback value
  if (ctx.piggy && a.n < 4) {
    a.src[a.n] = (const uint32_t*)ctx.piggy;
    a.words[a.n] = 2;
    piggy_at = words;
    words += 2;
    a.n++;
  }
  RAMA_REQUIRE(at % 4 == 0 && at + 4 * words <= 63 * 8, "fetch: range exceeds the pinned block");
  const uint32_t s = ++ctx.seq;
  k_fetch<<<1, 32, 0, ctx.s>>>(a, (volatile unsigned long long*)(ctx.pinned_dev + kPinTagged), s);
  RAMA_LAUNCH_CHECK();
  volatile unsigned long long* tg = (volatile unsigned long long*)(ctx.pinned + kPinTagged);
  uint32_t* out = (uint32_t*)((char*)ctx.pinned + at);
  const int wait = words > 0 ? words : 1;
  for (int i = 0; i < wait; i++) {
    unsigned long long w;
    for (uint32_t spins = 1; (uint32_t)((w = tg[i]) >> 32) != s; spins++) {
      _mm_pause();
      if ((spins & 1023) == 0) {  // a failed kernel never publishes: surface its error
        const cudaError_t e = cudaStreamQuery(ctx.s);
        if (e != cudaSuccess && e != cudaErrorNotReady) RAMA_CUDA(e);
        if (e == cudaSuccess && (uint32_t)(tg[i] >> 32) != s) RAMA_REQUIRE(false, "read-back word not published");
      }
    }
    if (i < words) out[i] = (uint32_t)w;
  }
  *(volatile uint32_t*)(ctx.pinned + 63) = s;  // the sequence survives recycling of the block
  if (piggy_at >= 0) {
    memcpy(&ctx.piggy_val, out + piggy_at, 8);
    ctx.piggy_done = true;
    ctx.piggy = nullptr;
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  HostStats& hs = host_stats();
  hs.sync_ms += host_ms_since(t0);
  hs.syncs++;
  return (char*)ctx.pinned + at;
}

Ctx::~Ctx() {
  if (pinned) {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.emplace_back(pinned, ev);
  }
}

// ------------------------------------------------------ caching allocator

namespace {
// blocks are keyed by (device, stream, size class): the default stream's
// handle is 0 on every device, so the stream alone does not identify memory
struct CacheKey {
  int dev;
  cudaStream_t s;
  size_t bytes;  // class size
  bool operator<(const CacheKey& o) const {
    if (dev != o.dev) return dev < o.dev;
    if (s != o.s) return s < o.s;
    return bytes < o.bytes;
  }
};
std::mutex g_cache_mu;
std::map<CacheKey, std::vector<void*>> g_cache;
size_t g_cached_bytes = 0;

// classes: 256 B granules up to 64 KB, then 8 steps per power of two
inline size_t class_bytes(size_t bytes) {
  if (bytes <= 65536) return (bytes + 255) & ~(size_t)255;
  int e = 63 - __builtin_clzll((unsigned long long)(bytes - 1));  // 2^e < bytes <= 2^(e+1)
  size_t step = (size_t)1 << (e - 2);
  return (bytes + step - 1) / step * step;
}

inline int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
}  // namespace

// ------------------------------------------------- caller-owned workspace

namespace {
thread_local Arena* g_arena = nullptr;
}

Arena::Arena(void* p, size_t n) : base((char*)p), size(n) {
  const size_t skew = (256 - ((uintptr_t)base & 255)) & 255;  // first 256-byte boundary
  if (n > skew) free_[skew] = n - skew;
}

void* Arena::alloc(size_t bytes) {
  const size_t b = (bytes + 255) & ~(size_t)255;
  for (auto it = free_.begin(); it != free_.end(); ++it) {  // first fit
    if (it->second < b) continue;
    const size_t off = it->first, len = it->second;
    free_.erase(it);
    if (len > b) free_[off + b] = len - b;
    live_[off] = b;
    used += b;
    if (used > peak) peak = used;
    return base + off;
  }
  throw Error(kNoMemory, "workspace exhausted: " + std::to_string(b) + " bytes requested with " +
                             std::to_string(used) + " of " + std::to_string(size) +
                             " in use (give a larger workspace; rama_ws_bytes is an estimate)");
}

bool Arena::owns(const void* p) const { return (const char*)p >= base && (const char*)p < base + size; }

void Arena::release(void* p) {
  const size_t off = (size_t)((char*)p - base);
  auto lv = live_.find(off);
  if (lv == live_.end()) return;
  size_t len = lv->second;
  live_.erase(lv);
  used -= len;
  size_t start = off;
  auto nx = free_.lower_bound(off);
  if (nx != free_.end() && nx->first == off + len) {  // merge with the next free block
    len += nx->second;
    nx = free_.erase(nx);
  }
  if (nx != free_.begin()) {  // and with the previous one
    auto pv = std::prev(nx);
    if (pv->first + pv->second == off) {
      start = pv->first;
      len += pv->second;
      free_.erase(pv);
    }
  }
  free_[start] = len;
}

ArenaScope::ArenaScope(Arena* a) : prev(g_arena) { g_arena = a; }
ArenaScope::~ArenaScope() { g_arena = prev; }
bool arena_active() { return g_arena != nullptr; }

void* dev_alloc(size_t bytes, cudaStream_t s) {
  if (g_arena) return g_arena->alloc(bytes);  // stream-ordered: one stream per workspace call
  size_t b = class_bytes(bytes);
  const int dev = cur_device();
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find(CacheKey{dev, s, b});
    if (it != g_cache.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      g_cached_bytes -= b;
      return p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, b, s);
  if (e == cudaErrorMemoryAllocation) {  // hand the cache back to the pool, retry once
    cudaGetLastError();
    dev_release_stream(s);
    e = cudaMallocAsync(&p, b, s);
  }
  RAMA_CUDA(e);
  return p;
}

void dev_free(void* p, size_t bytes, cudaStream_t s) {
  if (g_arena && g_arena->owns(p)) {
    g_arena->release(p);
    return;
  }
  size_t b = class_bytes(bytes);
  const int dev = cur_device();
  std::lock_guard<std::mutex> lk(g_cache_mu);
  if (g_cached_bytes + b > ((size_t)48 << 30)) {  // cap what the cache holds
    cudaFreeAsync(p, s);
    return;
  }
  g_cache[CacheKey{dev, s, b}].push_back(p);
  g_cached_bytes += b;
}

void dev_release_stream(cudaStream_t s) {
  const int dev = cur_device();
  std::lock_guard<std::mutex> lk(g_cache_mu);
  for (auto it = g_cache.begin(); it != g_cache.end();) {
    if (it->first.dev != dev || it->first.s != s) {
      ++it;
      continue;
    }
    for (void* p : it->second) {
      cudaFreeAsync(p, s);
      g_cached_bytes -= it->first.bytes;
    }
    it = g_cache.erase(it);
  }
}

void dev_release_all() {
  std::vector<int> devs;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    int cur = cur_device();
    for (auto& kv : g_cache) {
      cudaSetDevice(kv.first.dev);
      for (void* p : kv.second) cudaFreeAsync(p, kv.first.s);
      devs.push_back(kv.first.dev);
    }
    g_cache.clear();
    g_cached_bytes = 0;
    cudaSetDevice(cur);
  }
  int cur = cur_device();
  for (int d : devs) {
    cudaSetDevice(d);
    cudaDeviceSynchronize();
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  }
  cudaSetDevice(cur);
}

void reserve_pool(Ctx& ctx, size_t bytes) {
  if (g_arena) return;  // scratch comes from the caller's workspace
  int dev = 0;
  RAMA_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  RAMA_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t have = 0;
  RAMA_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &have));
  if (have >= bytes) return;
  size_t free_b = 0, total_b = 0;
  RAMA_CUDA(cudaMemGetInfo(&free_b, &total_b));
  size_t want = bytes - have;
  if (want > free_b / 2) want = free_b / 2;
  void* p = nullptr;
  if (cudaMallocAsync(&p, want, ctx.s) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  RAMA_CUDA(cudaFreeAsync(p, ctx.s));
}

namespace {
constexpr int kMaxDevices = 64;
std::mutex g_pool_mu;
bool g_pool_done[kMaxDevices] = {false};
int g_sms[kMaxDevices] = {0};
}  // namespace

// per device: the stream-ordered pool keeps freed memory (release threshold
// raised), and the SM count sizes the grids of kernels launched there
void ensure_pool_configured() {
  const int dev = cur_device();
  RAMA_REQUIRE(dev >= 0 && dev < kMaxDevices, "device ordinal out of range");
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (g_pool_done[dev]) return;
  cudaMemPool_t pool;
  RAMA_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t thr = UINT64_MAX;
  RAMA_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  RAMA_CUDA(cudaDeviceGetAttribute(&g_sms[dev], cudaDevAttrMultiProcessorCount, dev));
  g_pool_done[dev] = true;
}

int num_sms() {
  const int dev = cur_device();
  return (dev >= 0 && dev < kMaxDevices && g_sms[dev] > 0) ? g_sms[dev] : 148;
}

// ------------------------------------------------------------- profiling

namespace {
struct ProfRec {
  int fam;
  cudaEvent_t a, b;
  double bytes;
};
bool g_prof = false;
std::vector<ProfRec> g_prof_recs;
double g_prof_ms[kNumFamilies] = {0};
double g_prof_bytes[kNumFamilies] = {0};
int64_t g_prof_count[kNumFamilies] = {0};

std::vector<cudaEvent_t> g_event_pool;
std::mutex g_prof_mu;  // batch solves profile from several host threads
struct KernRec {
  const char* name;
  cudaEvent_t a, b;
  double bytes;
  int fam;
};
thread_local int g_cur_fam = -1;
const char* const kFamKeys[kNumFamilies] = {"@0", "@1", "@2", "@3", "@4", "@5", "@6", "@7", "@8", "@9"};
std::vector<KernRec> g_kern_recs;
struct KernSum {
  double ms = 0, bytes = 0;
  int64_t count = 0;
};
std::map<std::string, KernSum> g_kern_sum;
thread_local double g_next_bytes = 0.0;

void kern_drain() {
  for (auto& r : g_kern_recs) {
    float ms = 0.f;
    cudaEventSynchronize(r.b);
    cudaEventElapsedTime(&ms, r.a, r.b);
    KernSum& k = g_kern_sum[r.name];
    k.ms += ms;
    k.bytes += r.bytes;
    k.count += 1;
    if (r.fam >= 0 && r.fam < kNumFamilies) {
      KernSum& f = g_kern_sum[kFamKeys[r.fam]];
      f.ms += ms;
      f.bytes += r.bytes;
      f.count += 1;
    }
    g_event_pool.push_back(r.a);
    g_event_pool.push_back(r.b);
  }
  g_kern_recs.clear();
}

void prof_drain() {
  for (auto& r : g_prof_recs) {
    float ms = 0.f;
    cudaEventSynchronize(r.b);
    cudaEventElapsedTime(&ms, r.a, r.b);
    g_prof_ms[r.fam] += ms;
    g_prof_bytes[r.fam] += r.bytes;
    g_prof_count[r.fam] += 1;
    g_event_pool.push_back(r.a);
    g_event_pool.push_back(r.b);
  }
  g_prof_recs.clear();
}
}  // namespace

cudaEvent_t prof_event() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (g_event_pool.empty()) {
    for (int i = 0; i < 256; i++) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      g_event_pool.push_back(e);
    }
  }
  cudaEvent_t e = g_event_pool.back();
  g_event_pool.pop_back();
  return e;
}

bool prof_enabled() { return g_prof; }

int prof_family_swap(int fam) {
  int old = g_cur_fam;
  g_cur_fam = fam;
  return old;
}

void prof_set_bytes(double bytes) { g_next_bytes = bytes; }

double prof_take_bytes() {
  double b = g_next_bytes;
  g_next_bytes = 0.0;
  return b;
}

void prof_kernel_push(const char* name, cudaEvent_t a, cudaEvent_t b, double bytes) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_kern_recs.push_back(KernRec{name, a, b, bytes, g_cur_fam});
  if (g_kern_recs.size() > 8192) kern_drain();
}

int64_t prof_kernels_json(char* out, int64_t cap) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  kern_drain();
  std::string js = "{";
  char buf[512];
  bool first = true;
  for (auto& kv : g_kern_sum) {
    snprintf(buf, sizeof(buf), "%s\"%s\": [%.6f, %.1f, %lld]", first ? "" : ", ", kv.first.c_str(), kv.second.ms,
             kv.second.bytes, (long long)kv.second.count);
    js += buf;
    first = false;
  }
  js += "}";
  int64_t need = (int64_t)js.size() + 1;
  if (out && cap >= need) memcpy(out, js.c_str(), need);
  return need;
}

void prof_set(bool on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  prof_drain();
  kern_drain();
  g_kern_sum.clear();
  for (int f = 0; f < kNumFamilies; f++) {
    g_prof_ms[f] = 0.0;
    g_prof_bytes[f] = 0.0;
    g_prof_count[f] = 0;
  }
  g_prof = on;
}

void prof_push(int fam, cudaEvent_t a, cudaEvent_t b, double bytes) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_recs.push_back(ProfRec{fam, a, b, bytes});
  if (g_prof_recs.size() > 4096) prof_drain();
}

void prof_read(double* ms, double* bytes, int64_t* count) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  prof_drain();
  for (int f = 0; f < kNumFamilies; f++) {
    ms[f] = g_prof_ms[f];
    bytes[f] = g_prof_bytes[f];
    count[f] = g_prof_count[f];
  }
}

static int trace_level() {
  static const int v = [] {
    const char* e = getenv("RAMA_TRACE");
    return (e && e[0] >= '1' && e[0] <= '9') ? e[0] - '0' : 0;
  }();
  return v;
}

bool trace_enabled() { return trace_level() == 1; }
bool trace_print() { return trace_level() >= 1; }

unsigned capped_grid(int64_t work, int block) {
  int64_t g = (work + block - 1) / block;
  int64_t cap = (int64_t)num_sms() * 32;  // 32 x 256 threads per SM (more loads in flight than 16)
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

// ---------------------------------------------------------------- scans


// in[i] for i < n, 0 at i == n: an exclusive scan over n + 1 items then
// leaves the total in out[n] (no separate tail kernel)
struct PadZero {
  const int32_t* in;
  int64_t n;
  __host__ __device__ int32_t operator()(int64_t i) const { return i < n ? in[i] : 0; }
};

int64_t exclusive_scan(Ctx& ctx, const int32_t* in, int32_t* out, int64_t n, bool want_total) {
  auto it = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0), PadZero{in, n});
  size_t tb = 0;
  RAMA_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, it, out, (int)(n + 1), ctx.s));
  Buf<uint8_t> tmp(tb, ctx);
  {
    KernelScope ks(ctx.s, "cub::DeviceScan", 8.0 * (double)n);
    RAMA_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, it, out, (int)(n + 1), ctx.s));
  }
  ctx.launches++;
  if (!want_total) return -1;
  return read_scalar(ctx, out + n);
}

void exclusive_scan64(Ctx& ctx, const int64_t* in, int64_t* out, int64_t n) {
  if (n <= 0) return;
  size_t tb = 0;
  RAMA_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)n, ctx.s));
  Buf<uint8_t> tmp(tb, ctx);
  {
    KernelScope ks(ctx.s, "cub::DeviceScan", 0.0);
    RAMA_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, (int)n, ctx.s));
  }
  ctx.launches++;
}

// ----------------------------------------------------------- compaction

int64_t compact_indices(Ctx& ctx, const uint8_t* flags, int64_t n, Buf<int32_t>& out) {
  out.alloc(n > 0 ? n : 1, ctx.s);
  if (n <= 0) return 0;
  Buf<int32_t> nsel(1, ctx);
  thrust::counting_iterator<int32_t> it(0);
  size_t tb = 0;
  RAMA_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, flags, out.p, nsel.p, (int)n, ctx.s));
  Buf<uint8_t> tmp(tb, ctx);
  {
    KernelScope ks(ctx.s, "cub::DeviceSelect", 1.0 * (double)n);
    RAMA_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, it, flags, out.p, nsel.p, (int)n, ctx.s));
  }
  ctx.launches++;
  return read_scalar(ctx, nsel.p);
}

void radix_sort_pairs(Ctx& ctx, const uint64_t* k_in, const int32_t* v_in, uint64_t* k_out, int32_t* v_out,
                      int64_t N, int begin_bit, int end_bit) {
  if (N <= 0) return;
  size_t tb = 0;
  RAMA_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k_in, k_out, v_in, v_out, (int)N, begin_bit, end_bit, ctx.s));
  Buf<uint8_t> tmp(tb, ctx);
  KernelScope ks(ctx.s, "cub::DeviceRadixSort", 24.0 * (double)N);
  RAMA_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, k_in, k_out, v_in, v_out, (int)N, begin_bit, end_bit, ctx.s));
  ctx.launches++;
}

// -------------------------------------------------- deterministic sum

constexpr int kSumBlocks = 592;  // 4 x 148 SMs, fixed => deterministic order

__global__ void k_partial_sum(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
  __shared__ double sh[kBlock];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc += x[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// one block, fixed tree order (deterministic)
__global__ void k_final_sum(const double* part, int np, double* out) {
  __shared__ double sh[1024];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc += part[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

void device_sum_to(Ctx& ctx, const double* x, int64_t n, double* out) {
  Buf<double> part(kSumBlocks, ctx);
  {
    KernelScope ks(ctx.s, "k_partial_sum", 8.0 * (double)n);
    k_partial_sum<<<kSumBlocks, kBlock, 0, ctx.s>>>(x, n, part.p);
  }
  RAMA_LAUNCH_CHECK();
  {
    KernelScope ks(ctx.s, "k_final_sum", 0.0);
    k_final_sum<<<1, 1024, 0, ctx.s>>>(part.p, kSumBlocks, out);
  }
  RAMA_LAUNCH_CHECK();
  ctx.launches += 2;
}

double device_sum(Ctx& ctx, const double* x, int64_t n) {
  if (n <= 0) return 0.0;
  Buf<double> part(kSumBlocks + 1, ctx);
  {
    KernelScope ks(ctx.s, "k_partial_sum", 8.0 * (double)n);
    k_partial_sum<<<kSumBlocks, kBlock, 0, ctx.s>>>(x, n, part.p);
  }
  RAMA_LAUNCH_CHECK();
  {
    KernelScope ks(ctx.s, "k_final_sum", 0.0);
    k_final_sum<<<1, 1024, 0, ctx.s>>>(part.p, kSumBlocks, part.p + kSumBlocks);
  }
  RAMA_LAUNCH_CHECK();
  ctx.launches += 2;
  return read_scalar(ctx, part.p + kSumBlocks);
}

// K independent sums in one launch pair, each in exactly device_sum's order
// (segment j = x[start[j], start[j] + len[j]) takes grid row j): the batch
// solve's per-instance objectives are bit-identical to single solves
__global__ void k_partial_sum_seg(const double* __restrict__ x, const int64_t* __restrict__ start,
                                  const int64_t* __restrict__ len, double* __restrict__ part) {
  __shared__ double sh[kBlock];
  const double* xs = x + start[blockIdx.y];
  const int64_t n = len[blockIdx.y];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc += xs[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = sh[0];
}

__global__ void k_final_sum_seg(const double* part, int np, const int64_t* __restrict__ len, double* out) {
  __shared__ double sh[1024];
  const double* ps = part + (int64_t)blockIdx.x * np;
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc += ps[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = len[blockIdx.x] > 0 ? sh[0] : 0.0;
}

void device_sums(Ctx& ctx, const double* x, const int64_t* start, const int64_t* len, int64_t K, double* out) {
  constexpr int64_t kMaxY = 65535;  // grid y limit: segments in slices
  for (int64_t k0 = 0; k0 < K; k0 += kMaxY) {
    const int64_t k = std::min<int64_t>(kMaxY, K - k0);
    Buf<double> part((size_t)k * kSumBlocks, ctx);
    {
      KernelScope ks(ctx.s, "k_partial_sum_seg", 0.0);
      k_partial_sum_seg<<<dim3(kSumBlocks, (unsigned)k), kBlock, 0, ctx.s>>>(x, start + k0, len + k0, part.p);
    }
    RAMA_LAUNCH_CHECK();
    {
      KernelScope ks(ctx.s, "k_final_sum_seg", 0.0);
      k_final_sum_seg<<<(unsigned)k, 1024, 0, ctx.s>>>(part.p, kSumBlocks, len + k0, out + k0);
    }
    RAMA_LAUNCH_CHECK();
    ctx.launches += 2;
  }
}

// ----------------------------------------------------------- row ptrs

// Row pointers of a (u, v)-sorted list: edge i opens the rows (u[i-1],
// u[i]].  Gaps of up to kShortGap rows are filled by the edge's own thread;
// longer ones (empty stretches: isolated nodes, a batch's finished
// instances) are listed and filled by whole blocks, so no thread walks a
// long gap and no row needs a binary search.  The list's length stays on
// the device.
constexpr int kShortGap = 32;
constexpr int64_t kGapPiece = 2048;

__global__ void k_row_ptr_open(const int32_t* __restrict__ u, int64_t m, int64_t n, int32_t* __restrict__ ptr,
                               int64_t* __restrict__ gaps, int32_t* __restrict__ ngaps) {
  GRID_STRIDE(i, m + 1) {
    const int64_t prev = i > 0 ? (int64_t)u[i - 1] : -1;
    const int64_t cur = i < m ? (int64_t)u[i] : n;
    if (cur - prev <= kShortGap) {
      for (int64_t x = prev + 1; x <= cur; x++) ptr[x] = (int32_t)i;
    } else {  // listed in pieces of kGapPiece rows (one block each)
      const int64_t pieces = (cur - prev + kGapPiece - 1) / kGapPiece;
      const int64_t k = atomicAdd(ngaps, (int32_t)pieces);
      for (int64_t p = 0; p < pieces; p++) {
        const int64_t lo = prev + 1 + p * kGapPiece;
        gaps[3 * (k + p)] = lo;
        gaps[3 * (k + p) + 1] = min(cur, lo + kGapPiece - 1);
        gaps[3 * (k + p) + 2] = i;
      }
    }
  }
}

__global__ void k_row_ptr_gaps(const int64_t* __restrict__ gaps, const int32_t* __restrict__ ngaps,
                               int32_t* __restrict__ ptr) {
  const int32_t ng = *ngaps;
  for (int32_t g = blockIdx.x; g < ng; g += gridDim.x) {
    const int64_t lo = gaps[3 * (int64_t)g], hi = gaps[3 * (int64_t)g + 1];
    const int32_t val = (int32_t)gaps[3 * (int64_t)g + 2];
    for (int64_t x = lo + threadIdx.x; x <= hi; x += blockDim.x) ptr[x] = val;
  }
}

void row_ptr_from_sorted(Ctx& ctx, const int32_t* u, int64_t m, int64_t n, int32_t* ptr) {
  Buf<int32_t> ng(1, ctx);
  Buf<int64_t> gaps(3 * ((n + 1) / (kShortGap + 1) + (n + 1) / kGapPiece + 2), ctx);
  ng.zero();
  RAMA_KERNEL(ctx, k_row_ptr_open, m + 1, u, m, n, ptr, gaps.p, ng.p);
  {
    KernelScope ks(ctx.s, "k_row_ptr_gaps", 0.0);
    k_row_ptr_gaps<<<(unsigned)num_sms() * 4, kBlock, 0, ctx.s>>>(gaps.p, ng.p, ptr);
  }
  RAMA_LAUNCH_CHECK();
  ctx.launches++;
}

// ---------------------------------------------------------- bucket sort

// Histogram of the rows: every item records its offset inside its row (the
// atomicAdd's old value), so the scatter pass needs no atomics.  Items with
// row < 0 are dropped (contraction's merged edges).  Plain atomics beat
// warp aggregation with __match_any_sync here (C2: 1.23 -> 0.92 ms).
__global__ void k_bucket_count(const int32_t* __restrict__ row, int64_t N, int32_t* __restrict__ cnt,
                               int32_t* __restrict__ off, int32_t* __restrict__ zero2) {
  const int lane = threadIdx.x & 31;
  if (zero2 && blockIdx.x == 0 && threadIdx.x < 2) zero2[threadIdx.x] = 0;  // the rank pass's list counters
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x - lane; i0 < N;
       i0 += (int64_t)gridDim.x * blockDim.x) {  // warp-uniform trip count
    const int64_t i = i0 + lane;
    const int32_t r = i < N ? row[i] : -1;
    const int32_t o = run_atomic_add(cnt, r, 1);
    if (r >= 0) off[i] = o;
  }
}

// scattered item: one 16-byte store per item instead of three partial-sector
// stores into separate arrays (the scatter's DRAM traffic was 4x its bytes)
struct __align__(16) BItem {
  uint64_t key;
  int32_t src;
  int32_t row;
};

__global__ void k_bucket_scatter(const int32_t* __restrict__ row, const uint64_t* __restrict__ key,
                                 const int32_t* __restrict__ off, int64_t N, const int32_t* __restrict__ ptr,
                                 BItem* __restrict__ items) {
  GRID_STRIDE(i, N) {
    int32_t r = row[i];
    if (r < 0) continue;
    int32_t p = ptr[r] + off[i];
    BItem it;
    it.key = key[i];
    it.src = (int32_t)i;
    it.row = r;
    items[p] = it;
  }
}

// Rows of at most kSmallRow items are ordered by ranking: the thread of
// slot p counts the row's keys below its own (ties by scatter slot, so the
// result is a permutation even for duplicate keys) and writes its item to
// row_start + rank.  Neighbouring threads read the same row, so the key
// loads are warp broadcasts.  Longer rows are listed for the block sort.
constexpr int kSmallRow = 256;
constexpr int kBlockRow = 4096;  // bitonic sort in shared memory: 4096 x 12 B = 48 KB

__global__ void k_rank_rows(const BItem* __restrict__ items, const int32_t* __restrict__ ptr,
                            const int32_t* __restrict__ kept, int64_t sort_rows, uint64_t* __restrict__ okey,
                            int32_t* __restrict__ osrc, int32_t* __restrict__ orow, int32_t* __restrict__ big_list,
                            int32_t* __restrict__ huge_list, int32_t* __restrict__ counters) {
  const int64_t N = *kept;  // kept items (row >= 0), on the device: no host read-back before this kernel
  GRID_STRIDE(p, N) {
    const BItem it = items[p];
    const int32_t r = it.row;
    if (orow) orow[p] = r;  // rows keep their ranges
    int32_t b = ptr[r], e = ptr[r + 1];
    if (e - b == 1 || r >= sort_rows) {
      okey[p] = it.key;
      osrc[p] = it.src;
      continue;
    }
    if (e - b > kSmallRow) {  // block bitonic (<= kBlockRow) or CUB segmented sort (hubs)
      if (p == b) {
        if (e - b > kBlockRow) huge_list[atomicAdd(counters + 1, 1)] = r;
        else big_list[atomicAdd(counters, 1)] = r;
      }
      continue;
    }
    int32_t rank = 0;
    for (int32_t q = b; q < e; q++) {
      uint64_t x = items[q].key;
      rank += (x < it.key) || (x == it.key && q < (int32_t)p);
    }
    okey[b + rank] = it.key;
    osrc[b + rank] = it.src;
  }
}

// one block per listed row: bitonic sort of (key, src) in shared memory,
// from the scatter buffers into the output; rows longer than kBlockRow go
// to the huge list (CUB segmented sort)
__global__ void __launch_bounds__(512) k_sort_rows_block(const int32_t* __restrict__ ptr,
                                                         const int32_t* __restrict__ big_list,
                                                         int32_t* __restrict__ counters,
                                                         const BItem* __restrict__ items,
                                                         uint64_t* __restrict__ key, int32_t* __restrict__ src) {
  __shared__ uint64_t sk[kBlockRow];
  __shared__ int32_t ss[kBlockRow];
  int32_t nbig = counters[0];
  for (int32_t bi = blockIdx.x; bi < nbig; bi += gridDim.x) {
    int32_t r = big_list[bi];
    int32_t b = ptr[r], len = ptr[r + 1] - b;
    int32_t P = 64;
    while (P < len) P <<= 1;
    for (int32_t i = threadIdx.x; i < P; i += blockDim.x) {
      if (i < len) { sk[i] = items[b + i].key; ss[i] = items[b + i].src; }
      else { sk[i] = ~0ULL; ss[i] = 0x7fffffff; }
    }
    __syncthreads();
    for (int32_t k = 2; k <= P; k <<= 1) {
      for (int32_t j = k >> 1; j > 0; j >>= 1) {
        for (int32_t i = threadIdx.x; i < P; i += blockDim.x) {
          int32_t ixj = i ^ j;
          if (ixj > i) {
            bool up = (i & k) == 0;
            uint64_t a = sk[i], c = sk[ixj];
            if ((a > c) == up) {
              sk[i] = c; sk[ixj] = a;
              int32_t t = ss[i]; ss[i] = ss[ixj]; ss[ixj] = t;
            }
          }
        }
        __syncthreads();
      }
    }
    for (int32_t i = threadIdx.x; i < len; i += blockDim.x) {
      key[b + i] = sk[i];
      src[b + i] = ss[i];
    }
    __syncthreads();
  }
}

__global__ void k_big_lens(const int32_t* __restrict__ rows, int64_t nb, const int32_t* __restrict__ ptr,
                           int32_t* __restrict__ len) {
  GRID_STRIDE(i, nb) len[i] = ptr[rows[i] + 1] - ptr[rows[i]];
}

// move huge rows between the row layout and a contiguous staging area
// Segmented sort of the hub rows by key, as two device-wide stable radix
// sorts: by the 64-bit key, then (stable) by the segment id -- the result
// is ordered by (segment, key).  CUB's DeviceSegmentedSort gives each long
// segment to one CTA, which serialised power-law hubs (C4: 128 ms per solve
// for rows of up to ~4e5 items); here every pass uses the whole GPU.
__global__ void k_seg_of(const int32_t* __restrict__ off, int64_t nb, int64_t tot, uint32_t* __restrict__ seg,
                         int32_t* __restrict__ idx) {
  GRID_STRIDE(p, tot) {
    int64_t lo = 0, hi = nb - 1;  // last segment whose offset <= p
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (off[mid] <= p) lo = mid; else hi = mid - 1;
    }
    seg[p] = (uint32_t)lo;
    idx[p] = (int32_t)p;
  }
}

__global__ void k_gather_seg(const uint32_t* __restrict__ seg, const int32_t* __restrict__ perm, int64_t tot,
                             uint32_t* __restrict__ out) {
  GRID_STRIDE(p, tot) out[p] = seg[perm[p]];
}

template <class V>
__global__ void k_permute_pairs(const int32_t* __restrict__ perm, int64_t tot, const uint64_t* __restrict__ k_in,
                                const V* __restrict__ v_in, uint64_t* __restrict__ k_out, V* __restrict__ v_out) {
  GRID_STRIDE(p, tot) {
    const int32_t q = perm[p];
    k_out[p] = k_in[q];
    v_out[p] = v_in[q];
  }
}

template <class V>
static void seg_sort_pairs(Ctx& ctx, const uint64_t* k1, uint64_t* k2, const V* v1, V* v2, int64_t tot, int64_t nb,
                           const int32_t* off) {
  if (tot <= 0) return;
  Buf<uint32_t> seg(tot, ctx), seg2(tot, ctx), seg3(tot, ctx);
  Buf<int32_t> idx(tot, ctx), perm1(tot, ctx), perm2(tot, ctx);
  Buf<uint64_t> ks(tot, ctx);
  RAMA_KERNEL(ctx, k_seg_of, tot, off, nb, tot, seg.p, idx.p);
  radix_sort_pairs(ctx, k1, idx.p, ks.p, perm1.p, tot, 0, 64);  // stable by key
  RAMA_KERNEL(ctx, k_gather_seg, tot, seg.p, perm1.p, tot, seg2.p);
  int bits = 1;
  while (((int64_t)1 << bits) < nb) bits++;
  size_t tb = 0;
  RAMA_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, seg2.p, seg3.p, perm1.p, perm2.p, (int)tot, 0, bits,
                                            ctx.s));
  Buf<uint8_t> tmp(tb, ctx);
  {
    KernelScope ks2(ctx.s, "cub::DeviceRadixSort", 0.0);
    RAMA_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, seg2.p, seg3.p, perm1.p, perm2.p, (int)tot, 0, bits,
                                              ctx.s));  // stable by segment: (segment, key) order
  }
  ctx.launches++;
  RAMA_KERNEL(ctx, k_permute_pairs<V>, tot, perm2.p, tot, k1, v1, k2, v2);
}

__global__ void k_big_stage(const int32_t* __restrict__ rows, int64_t nb, const int32_t* __restrict__ ptr,
                            const int32_t* __restrict__ off, const BItem* __restrict__ items,
                            uint64_t* __restrict__ key_out, int32_t* __restrict__ src_out) {
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    int32_t r = rows[b];
    int32_t base = ptr[r], len = ptr[r + 1] - base, o = off[b];
    for (int32_t j = threadIdx.x; j < len; j += blockDim.x) {
      key_out[o + j] = items[base + j].key;
      src_out[o + j] = items[base + j].src;
    }
  }
}

__global__ void k_big_unstage(const int32_t* __restrict__ rows, int64_t nb, const int32_t* __restrict__ ptr,
                              const int32_t* __restrict__ off, const uint64_t* __restrict__ key_in,
                              const int32_t* __restrict__ src_in, uint64_t* __restrict__ key_out,
                              int32_t* __restrict__ src_out) {
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    int32_t r = rows[b];
    int32_t base = ptr[r], len = ptr[r + 1] - base, o = off[b];
    for (int32_t j = threadIdx.x; j < len; j += blockDim.x) {
      key_out[base + j] = key_in[o + j];
      src_out[base + j] = src_in[o + j];
    }
  }
}

void bucket_sort(Ctx& ctx, int64_t R, int64_t N, const int32_t* row, const uint64_t* key, BucketSorted& out,
                 bool want_row, int64_t sort_rows) {
  if (sort_rows < 0 || sort_rows > R) sort_rows = R;
  out.row_ptr.alloc(R + 1, ctx.s);
  out.key.alloc(N > 0 ? N : 1, ctx.s);
  out.src.alloc(N > 0 ? N : 1, ctx.s);
  if (want_row) out.row.alloc(N > 0 ? N : 1, ctx.s);
  Buf<int32_t> cnt(R > 0 ? R : 1, ctx), off(N > 0 ? N : 1, ctx);
  cnt.zero();
  Buf<int32_t> lists(2 * sort_rows + 2, ctx);  // big list | huge list | counters (zeroed by the count pass)
  int32_t* big_list = lists.p;
  int32_t* huge_list = lists.p + sort_rows;
  int32_t* counters = lists.p + 2 * sort_rows;
  prof_set_bytes(8.0 * (double)N);
  RAMA_KERNEL(ctx, k_bucket_count, N, row, N, cnt.p, off.p, counters);
  exclusive_scan(ctx, cnt.p, out.row_ptr.p, R, false);  // row_ptr[R] = kept items (row >= 0)
  if (R == 0 || N == 0) {
    out.total = 0;
    if (!want_row) out.row.release();
    return;
  }
  // sized for all N items; the kept count stays on the device until the one
  // read-back at the end
  Buf<BItem> items(N, ctx);
  prof_set_bytes(16.0 * (double)N + 16.0 * (double)N);
  RAMA_KERNEL(ctx, k_bucket_scatter, N, row, key, off.p, N, out.row_ptr.p, items.p);
  off.release();
  cnt.release();
  prof_set_bytes(16.0 * (double)N + 12.0 * (double)N + (want_row ? 4.0 * (double)N : 0.0));
  RAMA_KERNEL(ctx, k_rank_rows, N, items.p, out.row_ptr.p, out.row_ptr.p + R, sort_rows, out.key.p, out.src.p,
              want_row ? out.row.p : (int32_t*)nullptr, big_list, huge_list, counters);
  if (!want_row) out.row.release();
  if (sort_rows > 0 && N > kSmallRow) {  // rows of kSmallRow+1..kBlockRow items: the list size is read on the device
    unsigned gb = (unsigned)std::min<int64_t>(std::max<int64_t>(N / (kSmallRow + 1), 1), 148 * 4);
    KernelScope ks_block(ctx.s, "k_sort_rows_block", 0.0);
    k_sort_rows_block<<<gb, 512, 0, ctx.s>>>(out.row_ptr.p, big_list, counters, items.p, out.key.p, out.src.p);
    RAMA_LAUNCH_CHECK();
    ctx.launches++;
  }
  // one read-back: the kept count and the number of hub rows
  const int32_t* hp = (const int32_t*)fetch(ctx, {{out.row_ptr.p + R, 4}, {counters, 8}});
  const int64_t total = hp[0];
  const int32_t nbig = hp[1], nb = hp[2];
  out.total = total;
  out.big_rows = nbig;
  if (getenv("RAMA_SORT_STATS") && (nbig || nb))
    fprintf(stderr, "[rama] bucket_sort R %lld N %lld kept %lld: %d rows > %d, %d rows > %d\n", (long long)R,
            (long long)N, (long long)total, nbig, kSmallRow, nb, kBlockRow);
  if (nb == 0) return;
  // rare (power-law hubs): CUB segmented sort of the rows > kBlockRow
  Buf<int32_t> blen(nb, ctx), boff(nb + 1, ctx);
  RAMA_KERNEL(ctx, k_big_lens, nb, huge_list, nb, out.row_ptr.p, blen.p);
  int64_t tot = exclusive_scan(ctx, blen.p, boff.p, nb, true);
  Buf<uint64_t> k1(tot, ctx), k2(tot, ctx);
  Buf<int32_t> s1(tot, ctx), s2(tot, ctx);
  unsigned g = (unsigned)std::min<int64_t>(nb, 4096);
  k_big_stage<<<g, kBlock, 0, ctx.s>>>(huge_list, nb, out.row_ptr.p, boff.p, items.p, k1.p, s1.p);
  RAMA_LAUNCH_CHECK();
  seg_sort_pairs<int32_t>(ctx, k1.p, k2.p, s1.p, s2.p, tot, nb, boff.p);
  k_big_unstage<<<g, kBlock, 0, ctx.s>>>(huge_list, nb, out.row_ptr.p, boff.p, k2.p, s2.p, out.key.p, out.src.p);
  RAMA_LAUNCH_CHECK();
  ctx.launches += 3;
}

// ------------------------------------------------ sort-reduce: huge rows

__global__ void k_sr_hlen(const int32_t* __restrict__ rows, int64_t nb, const int32_t* __restrict__ ptr,
                          int32_t* __restrict__ len) {
  GRID_STRIDE(i, nb) len[i] = ptr[rows[i] + 1] - ptr[rows[i]];
}

__global__ void k_sr_hstage(const int32_t* __restrict__ rows, int64_t nb, const int32_t* __restrict__ ptr,
                            const int32_t* __restrict__ off, const SrItem* __restrict__ items,
                            uint64_t* __restrict__ k, uint64_t* __restrict__ v) {
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const int32_t base = ptr[rows[b]], len = ptr[rows[b] + 1] - base, o = off[b];
    for (int32_t j = threadIdx.x; j < len; j += blockDim.x) {
      k[o + j] = items[base + j].key;
      v[o + j] = (uint64_t)__double_as_longlong(items[base + j].pay);
    }
  }
}

__global__ void k_sr_hunstage(const int32_t* __restrict__ rows, int64_t nb, const int32_t* __restrict__ ptr,
                              const int32_t* __restrict__ off, const uint64_t* __restrict__ k,
                              const uint64_t* __restrict__ v, SrItem* __restrict__ items) {
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const int32_t base = ptr[rows[b]], len = ptr[rows[b] + 1] - base, o = off[b];
    for (int32_t j = threadIdx.x; j < len; j += blockDim.x) {
      SrItem it;
      it.key = k[o + j];
      it.pay = __longlong_as_double((long long)v[o + j]);
      items[base + j] = it;
    }
  }
}

void sr_sort_huge(Ctx& ctx, const int32_t* rowptr, const int32_t* rows, int64_t nb, SrItem* items) {
  Buf<int32_t> blen(nb, ctx), boff(nb + 1, ctx);
  RAMA_KERNEL(ctx, k_sr_hlen, nb, rows, nb, rowptr, blen.p);
  const int64_t tot = exclusive_scan(ctx, blen.p, boff.p, nb, true);
  Buf<uint64_t> k1(tot, ctx), k2(tot, ctx), v1(tot, ctx), v2(tot, ctx);
  const unsigned g = (unsigned)std::min<int64_t>(nb, 4096);
  k_sr_hstage<<<g, kBlock, 0, ctx.s>>>(rows, nb, rowptr, boff.p, items, k1.p, v1.p);
  RAMA_LAUNCH_CHECK();
  seg_sort_pairs<uint64_t>(ctx, k1.p, k2.p, v1.p, v2.p, tot, nb, boff.p);
  k_sr_hunstage<<<g, kBlock, 0, ctx.s>>>(rows, nb, rowptr, boff.p, k2.p, v2.p, items);
  RAMA_LAUNCH_CHECK();
  ctx.launches += 3;
}

}  // namespace rama
