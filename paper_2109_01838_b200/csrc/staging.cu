// Host <-> device copies for the host-buffer entry points (rama_solve_host).
//
// A caller's numpy arrays are pageable memory: cudaMemcpy from them runs at
// ~11 GB/s on the B200 box (the driver stages through its own small pinned
// buffer, one thread), against ~55 GB/s from pinned memory.  Pinned caller
// buffers are copied directly.  Pageable ones go through a cached pinned
// staging area in 4 MiB chunks: a pool of host threads copies chunk k into
// one of four pinned slots while the DMA engine moves the previous ones, so
// the copy runs at the host's parallel memcpy rate overlapped with PCIe
// (C2 e2e: 13.9 ms of pageable cudaMemcpy -> ~5.5 ms of staging for
// 158 MB in + 8 MB out; pinned callers: 3 ms).
#include "internal.h"

#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace rama {

namespace {

// RAMA_STAGE_CHUNK_MB / RAMA_STAGE_THREADS override the chunk size and the
// memcpy threads (tuning runs)
size_t chunk_bytes() {
  static const size_t v = [] {
    const char* e = getenv("RAMA_STAGE_CHUNK_MB");
    return (size_t)(e ? atoi(e) : 4) << 20;
  }();
  return v;
}

// fixed pool of memcpy workers: parallel_for(n, f) runs f(0..n-1) on the
// pool and the calling thread, returns when all are done
class CopyPool {
 public:
  CopyPool() {
    unsigned hw = std::thread::hardware_concurrency();
    int t = hw > 2 ? (int)(hw * 3 / 8) : 1;  // 6 on the 16-core B200 host (measured best of 3-16)
    if (t > 8) t = 8;
    if (const char* e = getenv("RAMA_STAGE_THREADS")) t = atoi(e) > 0 ? atoi(e) : 1;
    for (int i = 0; i < t - 1; i++) workers_.emplace_back([this] { loop(); });
    threads_ = t;
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  int threads() const { return threads_; }
  void parallel_for(int n, const std::function<void(int)>& f) {
    std::unique_lock<std::mutex> lk(mu_);
    fn_ = &f;
    next_ = 0;
    total_ = n;
    done_ = 0;
    gen_++;
    lk.unlock();
    cv_.notify_all();
    run();
    lk.lock();
    done_cv_.wait(lk, [&] { return done_ == total_; });
    fn_ = nullptr;
  }

 private:
  void run() {
    while (true) {
      int i;
      const std::function<void(int)>* f;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (!fn_ || next_ >= total_) return;
        i = next_++;
        f = fn_;
      }
      (*f)(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (++done_ == total_) done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    while (true) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      run();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int next_ = 0, total_ = 0, done_ = 0, threads_ = 1;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

CopyPool& pool() {
  static CopyPool p;
  return p;
}

constexpr int kSlots = 4;  // pinned chunks in flight

struct Staging {
  std::mutex mu;
  void* slot[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  ~Staging() {
    // process exit: the CUDA context may already be gone; leak rather than fault
  }
};

Staging& staging() {
  static Staging s;
  return s;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

void pcopy(void* dst, const void* src, size_t bytes) {
  CopyPool& P = pool();
  const int t = P.threads();
  const size_t part = (bytes + t - 1) / t;
  P.parallel_for(t, [&](int i) {
    const size_t b = (size_t)i * part;
    if (b < bytes) memcpy((char*)dst + b, (const char*)src + b, std::min(part, bytes - b));
  });
}

}  // namespace

void copy_h2d(Ctx& ctx, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  if (is_pinned(src)) {
    RAMA_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx.s));
    return;
  }
  Staging& S = staging();
  std::lock_guard<std::mutex> lk(S.mu);
  for (int k = 0; k < kSlots; k++) {
    if (!S.slot[k]) RAMA_CUDA(cudaMallocHost(&S.slot[k], chunk_bytes()));
    if (!S.ev[k]) RAMA_CUDA(cudaEventCreateWithFlags(&S.ev[k], cudaEventDisableTiming));
  }
  size_t off = 0;
  for (int k = 0; off < bytes; k = (k + 1) % kSlots) {
    const size_t len = std::min(chunk_bytes(), bytes - off);
    RAMA_CUDA(cudaEventSynchronize(S.ev[k]));  // the slot's previous DMA is done
    pcopy(S.slot[k], (const char*)src + off, len);
    RAMA_CUDA(cudaMemcpyAsync((char*)dst + off, S.slot[k], len, cudaMemcpyHostToDevice, ctx.s));
    RAMA_CUDA(cudaEventRecord(S.ev[k], ctx.s));
    off += len;
  }
}

void copy_d2h(Ctx& ctx, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  if (is_pinned(dst)) {
    RAMA_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx.s));
    ctx.sync();
    return;
  }
  Staging& S = staging();
  std::lock_guard<std::mutex> lk(S.mu);
  for (int k = 0; k < kSlots; k++) {
    if (!S.slot[k]) RAMA_CUDA(cudaMallocHost(&S.slot[k], chunk_bytes()));
    if (!S.ev[k]) RAMA_CUDA(cudaEventCreateWithFlags(&S.ev[k], cudaEventDisableTiming));
  }
  // DMA chunk k into slot k % 2 while the host copies chunk k - 1 out
  size_t off = 0, prev_off = 0, prev_len = 0;
  int prev = -1;
  for (int k = 0; off < bytes || prev >= 0; k ^= 1) {
    int cur = -1;
    size_t len = 0;
    if (off < bytes) {
      len = std::min(chunk_bytes(), bytes - off);
      RAMA_CUDA(cudaMemcpyAsync(S.slot[k], (const char*)src + off, len, cudaMemcpyDeviceToHost, ctx.s));
      RAMA_CUDA(cudaEventRecord(S.ev[k], ctx.s));
      cur = k;
    }
    if (prev >= 0) {
      RAMA_CUDA(cudaEventSynchronize(S.ev[prev]));
      pcopy((char*)dst + prev_off, S.slot[prev], prev_len);
    }
    prev = cur;
    prev_off = off;
    prev_len = len;
    off += len;
  }
}

}  // namespace rama
