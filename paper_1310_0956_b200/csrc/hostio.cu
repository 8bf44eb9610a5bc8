// hostio.cu -- host <-> device copies of caller (pageable) vectors for the
// reference-style numpy calls (geometry.py:200-215 semantics: `w @ x` copies
// x to the device and the result back before returning).
//
// H2D from pageable memory runs at ~11 GB/s through the driver's own staging,
// and cudaHostRegister of the caller's array costs more than the copy (64 MB:
// 6 ms register + 1.4 ms unregister, tools/probe_hostreg.py).  Instead the
// array is copied into a caller-provided pinned buffer by a persistent pool of
// host threads in 4 MB chunks (one thread moves ~15 GB/s, the box ~60 GB/s),
// and the calling thread issues each chunk's DMA as soon as its chunk has
// landed, so the host copies, the PCIe transfer and the issue overlap.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/wmgb200.h"

namespace {


struct Job {
  size_t chunk = 0;
  const char* src = nullptr;
  char* dst = nullptr;
  size_t bytes = 0;
  size_t nch = 0;
  std::atomic<size_t> next{0};
  std::unique_ptr<std::atomic<int>[]> done;
};

class CopyPool {
 public:
  // runs job on `helpers` pool threads plus the calling thread's idle time
  void run(Job& job, int helpers, cudaStream_t st, char* dev, cudaError_t& err) {
    std::unique_lock<std::mutex> call(call_mu_);   // one staged copy at a time
    ensure(helpers);
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &job;
      want_ = helpers;
      active_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    err = cudaSuccess;
    for (size_t i = 0; i < job.nch; ++i) {
      // help while the next chunk to issue is not there yet
      while (job.done[i].load(std::memory_order_acquire) == 0) {
        if (!copy_one(job)) std::this_thread::yield();
      }
      const size_t off = i * job.chunk, len = std::min(job.chunk, job.bytes - off);
      if (err == cudaSuccess)
        err = cudaMemcpyAsync(dev + off, job.dst + off, len, cudaMemcpyHostToDevice, st);
    }
    // helpers may still be between chunks: retire the job before it goes away
    std::unique_lock<std::mutex> lk(mu_);
    job_ = nullptr;
    idle_cv_.wait(lk, [&] { return active_ == 0; });
  }

  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }

 private:
  static bool copy_one(Job& job) {
    const size_t i = job.next.fetch_add(1, std::memory_order_relaxed);
    if (i >= job.nch) return false;
    const size_t off = i * job.chunk, len = std::min(job.chunk, job.bytes - off);
    std::memcpy(job.dst + off, job.src + off, len);
    job.done[i].store(1, std::memory_order_release);
    return true;
  }

  void ensure(int helpers) {
    const int have = (int)threads_.size();
    for (int k = have; k < helpers; ++k) threads_.emplace_back([this, k] { worker(k); });
  }

  void worker(int id) {
    unsigned long long seen = 0;
    for (;;) {
      Job* job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || (gen_ != seen && job_ != nullptr); });
        if (stop_) return;
        seen = gen_;
        if (id >= want_) continue;
        job = job_;
        ++active_;
      }
      while (copy_one(*job)) {
      }
      {
        std::lock_guard<std::mutex> lk(mu_);
        --active_;
      }
      idle_cv_.notify_all();
    }
  }

  std::mutex call_mu_, mu_;
  std::condition_variable cv_, idle_cv_;
  std::vector<std::thread> threads_;
  Job* job_ = nullptr;
  unsigned long long gen_ = 0;
  int want_ = 0, active_ = 0;
  bool stop_ = false;
};

CopyPool& pool() {
  static CopyPool p;
  return p;
}

}  // namespace

namespace wmg {

// dst (device) <- src (pageable host) through `pinned` (>= bytes), chunk DMAs
// issued on `st` as the host threads land them; returns after the last DMA is
// issued (the caller must not reuse `pinned` before `st` passes that point)
cudaError_t h2d_staged(void* dst, const void* src, size_t bytes, void* pinned, int threads,
                       cudaStream_t st) {
  if (bytes == 0) return cudaSuccess;
  Job job;
  job.src = static_cast<const char*>(src);
  job.dst = static_cast<char*>(pinned);
  job.bytes = bytes;
  const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
  const int helpers = std::max(0, std::min(threads, hw) - 1);
  // 4 MB chunks (1 MB chunks measured no better: host memory bandwidth, shared
  // by the copies and the DMA, is the limit)
  job.chunk = 4u << 20;
  job.nch = (bytes + job.chunk - 1) / job.chunk;
  job.done.reset(new std::atomic<int>[job.nch]);
  for (size_t i = 0; i < job.nch; ++i) job.done[i].store(0, std::memory_order_relaxed);
  cudaError_t e;
  pool().run(job, helpers, st, static_cast<char*>(dst), e);
  return e;
}

}  // namespace wmg
