#include "runtime.h"

#include <cstdlib>

namespace golp {

// Per thread: threads driving different contexts (B200Device(gpus=G)) report
// their own failures.
static thread_local std::string t_err;

void set_error(const std::string& msg) { t_err = msg; }

const char* last_error_cstr() { return t_err.c_str(); }

double wall_seconds() {
  using clk = std::chrono::steady_clock;
  return std::chrono::duration<double>(clk::now().time_since_epoch()).count();
}

void WorkerPool::start(int workers) {
  stop();
  stop_ = false;
  if (const char* v = std::getenv("GOLP_POOL_SPIN_US")) spin_s_ = std::atof(v) * 1e-6;
  for (int i = 0; i < workers; ++i) threads_.emplace_back([this] { loop(); });
}

void WorkerPool::stop() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
  }
  cv_work_.notify_all();
  for (auto& t : threads_) t.join();
  threads_.clear();
}

// Idle workers spin on the job generation for spin_s_ before blocking, so the
// back-to-back jobs of one offload call (a row check or staging copy per chunk)
// do not each pay a futex wake-up; a worker that blocks counts itself in
// sleepers_ and run() only notifies when somebody sleeps.
void WorkerPool::loop() {
  uint64_t seen = 0;
  while (true) {
    const double t0 = wall_seconds();
    unsigned spins = 0;
    while (gen_.load() == seen && !stop_.load()) {
      if ((++spins & 63u) == 0 && wall_seconds() - t0 > spin_s_) {
        std::unique_lock<std::mutex> lk(mu_);
        sleepers_.fetch_add(1);
        cv_work_.wait(lk, [&] { return stop_.load() || gen_.load() != seen; });
        sleepers_.fetch_sub(1);
        break;
      }
#if defined(__x86_64__)
      __builtin_ia32_pause();
#endif
    }
    if (stop_.load()) return;
    const std::function<void(size_t)>* job;
    size_t total;
    {
      std::lock_guard<std::mutex> lk(mu_);
      seen = gen_.load();
      job = job_;
      total = total_;
    }
    for (size_t i = next_.fetch_add(1); i < total; i = next_.fetch_add(1)) (*job)(i);
    if (pending_.fetch_sub(1) == 1) {
      std::lock_guard<std::mutex> lk(mu_);
      cv_done_.notify_all();
    }
  }
}

void WorkerPool::run(size_t ntasks, const std::function<void(size_t)>& fn) {
  if (threads_.empty() || ntasks <= 1) {
    for (size_t i = 0; i < ntasks; ++i) fn(i);
    return;
  }
  {
    std::lock_guard<std::mutex> lk(mu_);
    job_ = &fn;
    total_ = ntasks;
    next_.store(0);
    pending_.store((int)threads_.size());
    gen_.fetch_add(1);
  }
  if (sleepers_.load() > 0) cv_work_.notify_all();
  for (size_t i = next_.fetch_add(1); i < ntasks; i = next_.fetch_add(1)) fn(i);
  // every worker checks in (a late one must not read the next job's state)
  const double t0 = wall_seconds();
  unsigned spins = 0;
  while (pending_.load() != 0) {
    if ((++spins & 63u) == 0 && wall_seconds() - t0 > spin_s_) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_done_.wait(lk, [&] { return pending_.load() == 0; });
      break;
    }
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
}

void parallel_copy(WorkerPool& pool, void* dst, const void* src, size_t bytes) {
  constexpr size_t kPiece = 2u << 20;
  const size_t pieces = (bytes + kPiece - 1) / kPiece;
  if (pieces <= 1 || pool.size() == 0) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t tasks = std::min(pieces, (size_t)pool.size() + 1);
  const size_t per = (bytes + tasks - 1) / tasks;
  pool.run(tasks, [&](size_t t) {
    const size_t lo = t * per;
    if (lo >= bytes) return;
    const size_t len = std::min(per, bytes - lo);
    std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, len);
  });
}

bool dense_run(WorkerPool& pool, const uint32_t* src, size_t n) {
  if (n < 2) return true;
  const uint32_t base = src[0];
  // Permuted or shifted columns fail here without touching the rest.
  if (src[1] != base + 1u || src[n - 1] != base + (uint32_t)(n - 1) || src[n / 2] != base + (uint32_t)(n / 2))
    return false;
  constexpr size_t kPiece = size_t(1) << 18;  // 1 MB of row ids per task
  const size_t tasks = (n + kPiece - 1) / kPiece;
  std::atomic<bool> ok{true};
  auto check = [&](size_t t) {
    if (!ok.load(std::memory_order_relaxed)) return;
    const size_t lo = t * kPiece, hi = std::min(n, lo + kPiece);
    uint32_t bad = 0;
    uint32_t want = base + (uint32_t)lo;
    for (size_t i = lo; i < hi; ++i, ++want) bad |= src[i] ^ want;
    if (bad) ok.store(false, std::memory_order_relaxed);
  };
  if (tasks <= 1 || pool.size() == 0) {
    for (size_t t = 0; t < tasks; ++t) check(t);
  } else {
    pool.run(tasks, check);
  }
  return ok.load();
}

}  // namespace golp

