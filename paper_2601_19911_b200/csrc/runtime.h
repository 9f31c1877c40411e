// Host runtime pieces shared by the C-ABI translation units: error state,
// a small persistent worker pool (packer / gather threads), wall clock.
#pragma once
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace golp {

void set_error(const std::string& msg);
double wall_seconds();

// Fixed-size pool; run() blocks until every task index has executed. The
// calling thread takes part, so a pool of T workers runs T+1 tasks at once.
class WorkerPool {
 public:
  ~WorkerPool() { stop(); }
  void start(int workers);
  void stop();
  int size() const { return (int)threads_.size(); }
  void run(size_t ntasks, const std::function<void(size_t)>& fn);

 private:
  void loop();
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_work_, cv_done_;
  const std::function<void(size_t)>* job_ = nullptr;
  size_t total_ = 0;
  std::atomic<size_t> next_{0};
  std::atomic<int> pending_{0};
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> sleepers_{0};
  std::atomic<bool> stop_{false};
  double spin_s_ = 200e-6;  // idle workers spin this long before sleeping (GOLP_POOL_SPIN_US)
};

// memcpy split across the pool (the packer's inner loop).
void parallel_copy(WorkerPool& pool, void* dst, const void* src, size_t bytes);

// True when src[i] == src[0] + i (mod 2^32) for every i < n: a dense row-id run
// such as extract_keys's arange (pkg/src/golp/store.py:178-181). Split across
// the pool, stops at the first mismatch.
bool dense_run(WorkerPool& pool, const uint32_t* src, size_t n);

}  // namespace golp
