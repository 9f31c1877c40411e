// Classical host engine: the CPU path the Risky Gate falls to when offloading
// does not pay (gate._run_query HOST branch, pkg/src/golp/gate.py:193-194,209-210).
// It is part of the product -- a designed execution path chosen per query by
// the gate -- not a fallback for the GPU path (B200Device never calls it).
//
// Outputs are identical to the reference host primitives:
//   host_topk        pkg/src/golp/host.py:133-144  (k largest, ties by row id)
//   host_hash_build  pkg/src/golp/host.py:147-165  (KeyHashTable slot layout)
//   host_hash_probe  pkg/src/golp/host.py:168-188  (probe order, then chain order)
#include <cstdlib>
#include <algorithm>
#include <memory>

#include "../../include/golp_b200.h"
#include "common.cuh"
#include "runtime.h"

using namespace golp;

namespace {

WorkerPool& host_pool() {
  static std::unique_ptr<WorkerPool> pool;
  static std::once_flag once;
  std::call_once(once, [] {
    pool.reset(new WorkerPool());
    const int hw = (int)std::thread::hardware_concurrency();
    pool->start(std::max(0, std::min(hw, 64) - 1));
  });
  return *pool;
}

struct HItem {
  uint64_t hi;  // ord(key)
  uint32_t lo;  // ~row
};
inline bool better(const HItem& a, const HItem& b) { return a.hi > b.hi || (a.hi == b.hi && a.lo > b.lo); }

std::vector<std::vector<uint32_t>> g_probe_p, g_probe_b;
uint64_t g_probe_m = 0;

int invalid(const char* msg) {
  set_error(msg);
  return GOLP_ERR_INVALID;
}

}  // namespace

extern "C" {

int golp_host_topk(const double* keys, const uint32_t* rows, uint64_t n, uint64_t k, uint32_t* out_rows,
                   int threads) {
  if (k < 1) return invalid("k must be at least 1");
  const uint64_t kk = std::min(k, n);
  if (kk == 0) return GOLP_OK;
  if (!keys || !rows || !out_rows) return invalid("null buffer");
  WorkerPool& pool = host_pool();
  uint64_t parts = threads > 0 ? (uint64_t)threads : (uint64_t)pool.size() + 1;
  parts = std::max<uint64_t>(1, std::min<uint64_t>(parts, n / 65536 + 1));
  std::vector<std::vector<HItem>> cand(parts);
  const uint64_t step = (n + parts - 1) / parts;
  pool.run(parts, [&](size_t t) {
    const uint64_t lo = t * step, hi = std::min(n, lo + step);
    if (lo >= hi) return;
    std::vector<HItem>& v = cand[t];
    if (parts == 1 && kk <= 256 && hi - lo > 8 * kk) {
      // a small input on the calling thread: a heap of the kk best (its top is
      // the worst of them) instead of an n-sized copy -- most items are
      // rejected by one compare and the caller's cache keeps its working set
      v.reserve(kk);
      uint64_t i = lo;
      for (; i < hi && v.size() < kk; ++i) {
        v.push_back(HItem{ord_key(keys[i]), ~rows[i]});
        std::push_heap(v.begin(), v.end(), better);
      }
      for (; i < hi; ++i) {
        const uint64_t h = ord_key(keys[i]);
        if (h < v.front().hi) continue;  // cannot beat the worst kept item
        const HItem it{h, ~rows[i]};
        if (!better(it, v.front())) continue;
        std::pop_heap(v.begin(), v.end(), better);
        v.back() = it;
        std::push_heap(v.begin(), v.end(), better);
      }
      return;
    }
    v.resize(hi - lo);
    for (uint64_t i = lo; i < hi; ++i) v[i - lo] = HItem{ord_key(keys[i]), ~rows[i]};
    if (v.size() > kk) {
      std::nth_element(v.begin(), v.begin() + (ptrdiff_t)kk, v.end(), better);
      v.resize(kk);
    }
  });
  std::vector<HItem> all;
  for (auto& v : cand) all.insert(all.end(), v.begin(), v.end());
  if (all.size() > kk) {
    std::nth_element(all.begin(), all.begin() + (ptrdiff_t)kk, all.end(), better);
    all.resize(kk);
  }
  std::sort(all.begin(), all.end(), better);
  for (uint64_t i = 0; i < kk; ++i) out_rows[i] = ~all[i].lo;
  return GOLP_OK;
}

int golp_host_hash_build(const double* keys, const uint32_t* rows, uint64_t n, uint64_t capacity,
                         uint64_t* slot_bits, uint32_t* slot_rows) {
  if (capacity < 1 || (capacity & (capacity - 1))) return invalid("capacity must be a positive power of two");
  if ((double)n > 0.7 * (double)capacity) {
    set_error("hash table load factor limit exceeded");
    return GOLP_ERR_CAPACITY;
  }
  if (n && (!keys || !rows || !slot_bits || !slot_rows)) return invalid("null buffer");
  const uint64_t mask = capacity - 1;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t b = canon_bits(keys[i]);
    uint64_t cur = mix64(b) & mask;
    while (slot_rows[cur] != kNoRow) cur = (cur + 1) & mask;
    slot_bits[cur] = b;
    slot_rows[cur] = rows[i];
  }
  return GOLP_OK;
}

int golp_host_hash_probe(const uint64_t* slot_bits, const uint32_t* slot_rows, uint64_t capacity,
                         const double* keys, const uint32_t* rows, uint64_t n, int threads,
                         uint64_t* out_matches) {
  if (!out_matches) return invalid("null out_matches");
  if (capacity < 1 || (capacity & (capacity - 1))) return invalid("capacity must be a positive power of two");
  if (n && (!keys || !rows || !slot_bits || !slot_rows)) return invalid("null buffer");
  WorkerPool& pool = host_pool();
  uint64_t parts = threads > 0 ? (uint64_t)threads : (uint64_t)pool.size() + 1;
  parts = std::max<uint64_t>(1, std::min<uint64_t>(parts, n / 4096 + 1));
  g_probe_p.assign(parts, {});
  g_probe_b.assign(parts, {});
  const uint64_t mask = capacity - 1;
  const uint64_t step = (n + parts - 1) / parts;
  pool.run(parts, [&](size_t t) {
    const uint64_t lo = t * step, hi = std::min(n, lo + step);
    std::vector<uint32_t>& op = g_probe_p[t];
    std::vector<uint32_t>& ob = g_probe_b[t];
    for (uint64_t i = lo; i < hi; ++i) {
      const uint64_t b = canon_bits(keys[i]);
      uint64_t cur = mix64(b) & mask;
      while (slot_rows[cur] != kNoRow) {
        if (slot_bits[cur] == b) {
          op.push_back(rows[i]);
          ob.push_back(slot_rows[cur]);
        }
        cur = (cur + 1) & mask;
      }
    }
  });
  uint64_t m = 0;
  for (auto& v : g_probe_p) m += v.size();
  g_probe_m = m;
  *out_matches = m;
  return GOLP_OK;
}

int golp_host_gather(const void* src, uint64_t row_bytes, uint64_t nrows, const uint32_t* ids, uint64_t n, void* dst,
                     int threads) {
  if (n == 0) return GOLP_OK;
  if (!src || !ids || !dst || row_bytes == 0) return invalid("null buffer");
  WorkerPool& pool = host_pool();
  uint64_t parts = threads > 0 ? (uint64_t)threads : (uint64_t)pool.size() + 1;
  parts = std::max<uint64_t>(1, std::min<uint64_t>(parts, n / 16384 + 1));
  const uint64_t step = (n + parts - 1) / parts;
  std::atomic<bool> bad{false};
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  pool.run(parts, [&](size_t t) {
    const uint64_t lo = t * step, hi = std::min(n, lo + step);
    if (row_bytes == 8) {
      const uint64_t* s8 = static_cast<const uint64_t*>(src);
      uint64_t* d8 = static_cast<uint64_t*>(dst);
      for (uint64_t i = lo; i < hi; ++i) {
        const uint32_t r = ids[i];
        if (r >= nrows) { bad = true; return; }
        d8[i] = s8[r];
      }
      return;
    }
    // Rows are random in a table far larger than the caches: prefetch the rows
    // kAhead ids ahead (every cache line of each) so that many misses overlap.
    static const uint64_t kAhead = [] {
      const char* v = std::getenv("GOLP_GATHER_PREFETCH");
      return v ? (uint64_t)std::strtoull(v, nullptr, 10) : (uint64_t)32;
    }();
    auto prefetch_row = [&](uint64_t i) {
      const uint32_t r = ids[i];
      if (r >= nrows) return;
      const char* p = s + (uint64_t)r * row_bytes;
      for (uint64_t o = 0; o < row_bytes; o += 64) __builtin_prefetch(p + o, 0, 0);
      __builtin_prefetch(p + row_bytes - 1, 0, 0);
    };
    for (uint64_t i = lo; i < std::min(hi, lo + kAhead); ++i) prefetch_row(i);
    for (uint64_t i = lo; i < hi; ++i) {
      if (kAhead && i + kAhead < hi) prefetch_row(i + kAhead);
      const uint32_t r = ids[i];
      if (r >= nrows) { bad = true; return; }
      std::memcpy(d + i * row_bytes, s + (uint64_t)r * row_bytes, row_bytes);
    }
  });
  if (bad) return invalid("row id out of range");
  return GOLP_OK;
}

// G-way merge of best-first Top-K lists (order codes u64 + rows, as
// golp_topk_codes returns them): the first k of all parts in host_topk's order
// (key descending, then row id ascending; host.py:141). Shard results of
// B200Device(gpus=G), the host side of ProxyDevice's merge (device.py:257-259).
int golp_host_merge_topk(const uint64_t* codes, const uint32_t* rows, const uint64_t* counts, int parts, uint64_t k,
                         uint32_t* out_rows, uint64_t* out_len) {
  if (parts < 0 || !out_len) return invalid("bad merge arguments");
  std::vector<uint64_t> start(parts + 1, 0), pos(parts, 0);
  for (int p = 0; p < parts; ++p) start[p + 1] = start[p] + counts[p];
  uint64_t o = 0;
  while (o < k) {
    int best = -1;
    for (int p = 0; p < parts; ++p) {
      if (pos[p] >= counts[p]) continue;
      const uint64_t i = start[p] + pos[p];
      if (best < 0) {
        best = p;
        continue;
      }
      const uint64_t j = start[best] + pos[best];
      if (codes[i] > codes[j] || (codes[i] == codes[j] && rows[i] < rows[j])) best = p;
    }
    if (best < 0) break;
    out_rows[o++] = rows[start[best] + pos[best]];
    ++pos[best];
  }
  *out_len = o;
  return GOLP_OK;
}

int golp_host_probe_copy_out(uint32_t* probe_rows, uint32_t* build_rows, uint64_t m) {
  if (m != g_probe_m) return invalid("copy_out size does not match the last host probe");
  uint64_t o = 0;
  for (size_t t = 0; t < g_probe_p.size(); ++t) {
    const size_t c = g_probe_p[t].size();
    if (c) {
      std::memcpy(probe_rows + o, g_probe_p[t].data(), c * 4);
      std::memcpy(build_rows + o, g_probe_b[t].data(), c * 4);
    }
    o += c;
  }
  g_probe_p.clear();
  g_probe_b.clear();
  g_probe_m = 0;
  return GOLP_OK;
}

}  // extern "C"
