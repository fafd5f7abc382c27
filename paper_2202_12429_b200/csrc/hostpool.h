// Host worker pool for the DMA host-link mode of the engine.
//
// Gathering prefetch rows from (and scattering written-back rows into) the
// pinned host table with CPU threads, and moving them over PCIe with the copy
// engines (cudaMemcpyAsync of contiguous staging buffers), keeps the host
// link off the SMs: zero-copy row kernels hold microsecond-latency PCIe
// accesses in the SMs' load/store queues, which stalls every co-resident
// compute kernel (measured: 1-thread kernels taking 60-90 us, the link
// kernels themselves 3x slower, while they overlap).  The pool runs inside
// cudaLaunchHostFunc callbacks on the engine's link stream, so stream order
// (and the reference's dispatch/flush order) is preserved.
#pragma once

#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace bp {

class HostPool {
 public:
  explicit HostPool(int threads) : n_(threads < 1 ? 1 : threads) {
    for (int w = 1; w < n_; ++w) workers_.emplace_back([this, w] { loop(w); });
  }

  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

  int size() const { return n_; }

  // fn(begin, end) over a static split of [0, n) into size() slices; the
  // calling thread takes slice 0.  Blocks until every slice is done.
  void parallel_for(long long n, const std::function<void(long long, long long)>& fn) {
    if (n <= 0) return;
    if (n_ == 1 || n < 256) {
      fn(0, n);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      total_ = n;
      pending_.store(n_ - 1);
      ++gen_;
    }
    cv_.notify_all();
    fn(0, slice_end(0, n));
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_.load() == 0; });
    fn_ = nullptr;
  }

 private:
  long long slice_end(int w, long long n) const { return n * (w + 1) / n_; }

  void loop(int w) {
    unsigned long long seen = 0;
    for (;;) {
      const std::function<void(long long, long long)>* fn;
      long long n;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        fn = fn_;
        n = total_;
      }
      (*fn)(n * w / n_, slice_end(w, n));
      if (pending_.fetch_sub(1) == 1) {
        std::lock_guard<std::mutex> lk(mu_);
        done_cv_.notify_one();
      }
    }
  }

  int n_;
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  unsigned long long gen_ = 0;
  bool stop_ = false;
  const std::function<void(long long, long long)>* fn_ = nullptr;
  long long total_ = 0;
  std::atomic<int> pending_{0};
};

}  // namespace bp
