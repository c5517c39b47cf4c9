// A small persistent host thread pool (parallel_for) for the host side of the pipelined
// host-buffer execute: packing the referenced source rows into pinned staging memory.
#pragma once
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace sg {

class HostPool {
 public:
  explicit HostPool(int n) {
    for (int i = 0; i < n; ++i) threads_.emplace_back([this] { worker(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  int size() const { return (int)threads_.size() + 1; }
  // Runs fn(i) for i in [0, n) on the pool and the calling thread; returns when all are done.
  // Callers from several threads (in-process ranks) are serialised: one job at a time.
  void parallel_for(int n, const std::function<void(int)>& fn) {
    if (n <= 0) return;
    std::lock_guard<std::mutex> job_lock(call_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      next_.store(0);
      done_.store(0);
      ++gen_;
    }
    cv_.notify_all();
    run();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_.load() == n_; });
    fn_ = nullptr;
  }

 private:
  void run() {
    for (;;) {
      const int i = next_.fetch_add(1);
      if (i >= n_) break;
      (*fn_)(i);
      if (done_.fetch_add(1) + 1 == n_) {
        std::lock_guard<std::mutex> lk(mu_);
        done_cv_.notify_all();
      }
    }
  }
  void worker() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        if (!fn_) continue;
      }
      run();
    }
  }
  std::vector<std::thread> threads_;
  std::mutex call_mu_;  // one parallel_for at a time
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int n_ = 0;
  std::atomic<int> next_{0}, done_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
};

}  // namespace sg
