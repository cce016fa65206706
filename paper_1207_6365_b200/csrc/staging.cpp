// staging.cpp -- host <-> device copies of PAGEABLE host memory (numpy arrays,
// the reference's calling convention: sketch.py:153-165 takes ndarray / scipy
// CSR and returns a new ndarray).  The CUDA driver copies pageable memory at
// ~11 GB/s on this platform against ~55 GB/s from page-locked memory
// (tools/e2e_csr_probe.py), so skt_memcpy_staged pipelines the copy through a
// ring of page-locked chunk buffers: host threads memcpy chunk i + 1 into a
// free buffer while the DMA engine moves chunk i.  The ring (8 x 4 MB per
// device) and the worker threads are created on first use and reused.
//
//   kind 0 (H2D): returns once the source may be reused (the last DMAs are
//                 stream-ordered before later work on `stream`);
//   kind 1 (D2H): returns when dst holds the data (waits for the stream).
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include <unistd.h>

#include "common.cuh"

namespace skt {
namespace {

constexpr size_t kChunk = 4u << 20;
constexpr int kRing = 8;

// fixed pool of memcpy workers: copy() splits one memcpy into slices.  The
// workers spin briefly on the task generation before sleeping, and the caller
// spins on completion, so a chunk costs microseconds of hand-off, not a
// condition-variable wake-up per worker.
class CopyPool {
 public:
  CopyPool() : pid_(getpid()) {
    unsigned hw = std::thread::hardware_concurrency();
    nthreads_ = (int)std::max(1u, std::min(8u, hw > 1 ? hw / 2 : 1u));
    for (int i = 1; i < nthreads_; ++i) workers_.emplace_back([this, i] { run(i); });
  }
  ~CopyPool() {
    stop_.store(true);
    {
      std::lock_guard<std::mutex> g(m_);
      gen_.fetch_add(1);
    }
    cv_.notify_all();
    for (auto &t : workers_) t.join();
  }
  void copy(void *dst, const void *src, size_t bytes) {
    // a fork()ed child has none of the workers: copy on the calling thread
    if (bytes < (1u << 20) || nthreads_ == 1 || getpid() != pid_) {
      std::memcpy(dst, src, bytes);
      return;
    }
    std::lock_guard<std::mutex> call(call_m_);  // one parallel copy at a time
    dst_ = (char *)dst;
    src_ = (const char *)src;
    bytes_ = bytes;
    pending_.store(nthreads_ - 1, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> g(m_);
      gen_.fetch_add(1, std::memory_order_release);
    }
    if (sleepers_.load() > 0) cv_.notify_all();
    slice(0);
    while (pending_.load(std::memory_order_acquire) != 0) std::this_thread::yield();
  }

 private:
  void slice(int i) {
    const size_t per = ((bytes_ + nthreads_ - 1) / nthreads_ + 63) & ~(size_t)63;  // covers every byte
    const size_t b = std::min(bytes_, per * i), e = std::min(bytes_, per * (i + 1));
    if (e > b) std::memcpy(dst_ + b, src_ + b, e - b);
  }
  void run(int i) {
    uint64_t seen = 0;
    for (;;) {
      // spin ~2 ms for the next task (back-to-back calls), then sleep
      auto t0 = std::chrono::steady_clock::now();
      while (gen_.load(std::memory_order_acquire) == seen &&
             std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(2000))
        std::this_thread::yield();
      if (gen_.load(std::memory_order_acquire) == seen) {
        std::unique_lock<std::mutex> g(m_);
        sleepers_.fetch_add(1);
        cv_.wait(g, [&] { return gen_.load() != seen; });
        sleepers_.fetch_sub(1);
      }
      seen = gen_.load(std::memory_order_acquire);
      if (stop_.load()) return;
      slice(i);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  int nthreads_ = 1;
  pid_t pid_;
  std::vector<std::thread> workers_;
  std::mutex m_, call_m_;
  std::condition_variable cv_;
  std::atomic<bool> stop_{false};
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> pending_{0}, sleepers_{0};
  char *dst_ = nullptr;
  const char *src_ = nullptr;
  size_t bytes_ = 0;
};

CopyPool &pool() {
  static CopyPool p;
  return p;
}

struct Ring {
  void *buf[kRing] = {};
  cudaEvent_t ev[kRing] = {};
  std::mutex m;  // one staged copy per device at a time
};

skt_status ring_for_device(Ring **out) {
  static std::mutex m;
  static std::map<int, Ring *> rings;
  int dev = 0;
  SKT_CUDA_TRY(cudaGetDevice(&dev), "skt_memcpy_staged");
  std::lock_guard<std::mutex> g(m);
  Ring *&r = rings[dev];
  if (!r) {
    Ring *nr = new Ring;
    for (int i = 0; i < kRing; ++i) {
      if (cudaHostAlloc(&nr->buf[i], kChunk, cudaHostAllocPortable) != cudaSuccess ||
          cudaEventCreateWithFlags(&nr->ev[i], cudaEventDisableTiming) != cudaSuccess)
        return fail(SKT_ECUDA, "skt_memcpy_staged", "page-locked staging ring allocation failed");
    }
    r = nr;
  }
  *out = r;
  return SKT_OK;
}

}  // namespace
}  // namespace skt

using namespace skt;

extern "C" skt_status skt_memcpy_staged(void *dst, const void *src, size_t bytes, int32_t kind, void *stream_) {
  static const char *fn = "skt_memcpy_staged";
  if ((kind != 0 && kind != 1) || (bytes > 0 && (!dst || !src))) return fail(SKT_EINVAL, fn, "bad arguments");
  if (bytes == 0) return SKT_OK;
  cudaStream_t st = as_stream(stream_);
  Ring *r = nullptr;
  skt_status s = ring_for_device(&r);
  if (s != SKT_OK) return s;
  std::lock_guard<std::mutex> g(r->m);
  const size_t nch = (bytes + kChunk - 1) / kChunk;
  if (kind == 0) {  // host (pageable) -> device
    for (size_t i = 0; i < nch; ++i) {
      const int b = (int)(i % kRing);
      const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
      SKT_CUDA_TRY(cudaEventSynchronize(r->ev[b]), fn);  // the DMA that last read buffer b is done
      pool().copy(r->buf[b], (const char *)src + off, len);
      SKT_CUDA_TRY(cudaMemcpyAsync((char *)dst + off, r->buf[b], len, cudaMemcpyHostToDevice, st), fn);
      SKT_CUDA_TRY(cudaEventRecord(r->ev[b], st), fn);
    }
    // the caller may reuse src now; the ring buffers stay owned by the DMAs
    // until their events complete (checked before the next reuse)
    return SKT_OK;
  }
  // device -> host (pageable): chunks DMA'd ahead into the ring, drained in order
  size_t issued = 0;
  auto issue = [&](size_t i) -> skt_status {
    const int b = (int)(i % kRing);
    const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
    SKT_CUDA_TRY(cudaMemcpyAsync(r->buf[b], (const char *)src + off, len, cudaMemcpyDeviceToHost, st), fn);
    SKT_CUDA_TRY(cudaEventRecord(r->ev[b], st), fn);
    return SKT_OK;
  };
  for (; issued < nch && issued < (size_t)kRing; ++issued)
    if ((s = issue(issued)) != SKT_OK) return s;
  for (size_t i = 0; i < nch; ++i) {
    const int b = (int)(i % kRing);
    const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
    SKT_CUDA_TRY(cudaEventSynchronize(r->ev[b]), fn);
    pool().copy((char *)dst + off, r->buf[b], len);
    if (issued < nch) {
      if ((s = issue(issued)) != SKT_OK) return s;
      ++issued;
    }
  }
  return SKT_OK;
}
