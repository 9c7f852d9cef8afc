// Persistent host worker pool (plain C++, shared by the C-ABI's host paths:
// event packing, flow widening, input validation).  run(parts, fn) calls
// fn(0..parts-1) on the pool threads and the calling thread, and returns when
// all parts are done.  One run at a time per pool.
#pragma once

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/veckm.h"

namespace vkm_host {

// host_pack.cpp: the input checks of check_event_array over rows [0, n) of
// (n, ld) f64 rows (first outside pixel relative to X), and the in-order merge
// of two consecutive ranges' results
void check_range(const double* X, int64_t n, int64_t ld, int32_t W, int32_t H, vkm_event_check& out);
// check_range and pack_events of contiguous rows in one pass
void check_pack(const double* X, int64_t n, double t0, double dt, int32_t W, int32_t H, uint32_t* out,
                vkm_event_check& res);
void merge_check(vkm_event_check& c, const vkm_event_check& q);

class HostPool {
 public:
  explicit HostPool(int n) {
    for (int i = 0; i < n; ++i) threads_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> l(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  int size() const { return int(threads_.size()) + 1; }
  void run(int parts, const std::function<void(int)>& fn) {
    {
      std::lock_guard<std::mutex> l(m_);
      task_ = &fn;
      total_ = parts;
      next_ = 0;
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> l(m_);
    done_cv_.wait(l, [&] { return done_ == total_; });
    task_ = nullptr;
  }

 private:
  void work() {
    for (;;) {
      int i;
      const std::function<void(int)>* fn;
      {
        std::lock_guard<std::mutex> l(m_);
        if (!task_ || next_ >= total_) return;
        i = next_++;
        fn = task_;
      }
      (*fn)(i);
      std::lock_guard<std::mutex> l(m_);
      if (++done_ == total_) done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> threads_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* task_ = nullptr;
  int total_ = 0, next_ = 0, done_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// Worker threads per pool (the caller is one more): VKM_HOST_THREADS, else
// hardware threads - 1, at most 15.
inline int default_pool_threads() {
  if (const char* e = std::getenv("VKM_HOST_THREADS")) return std::max(0, std::atoi(e) - 1);
  return std::max(0, std::min(15, int(std::thread::hardware_concurrency()) - 1));
}

}  // namespace vkm_host
