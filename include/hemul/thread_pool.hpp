// hemul drop-in API (B200 build) — the reference's optional thread pool
// parameter (proj/core/include/hemul/thread_pool.hpp:17-100).
//
// The HE Mul path runs on the GPU, so the pool only exists for source
// compatibility of Scheme(params, pool) and for host-side loops that want a
// static partition; pool_for keeps the reference's semantics (results do not
// depend on the thread count).
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <thread>
#include <vector>

namespace hemul {

class ThreadPool {
 public:
  explicit ThreadPool(int threads) : threads_(std::max(1, threads)) {}
  int size() const { return threads_; }

  // fn(begin, end) on `threads` contiguous chunks of [0, total)
  void parallel_for(int64_t total, const std::function<void(int64_t, int64_t)>& fn) {
    const int64_t t = std::min<int64_t>(threads_, std::max<int64_t>(total, 1));
    if (t <= 1) {
      fn(0, total);
      return;
    }
    std::vector<std::thread> workers;
    const int64_t chunk = (total + t - 1) / t;
    for (int64_t w = 1; w < t; ++w) {
      const int64_t b = w * chunk, e = std::min(total, b + chunk);
      if (b < e) workers.emplace_back(fn, b, e);
    }
    fn(0, std::min(total, chunk));
    for (auto& th : workers) th.join();
  }

 private:
  int threads_;
};

inline void pool_for(ThreadPool* pool, int64_t total,
                     const std::function<void(int64_t, int64_t)>& fn) {
  if (pool)
    pool->parallel_for(total, fn);
  else
    fn(0, total);
}

}  // namespace hemul
