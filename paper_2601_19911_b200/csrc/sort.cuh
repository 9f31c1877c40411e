// Full sort of (key f64, row u32) pairs on the device: the B200 counterpart of
// host_full_sort (pkg/src/golp/host.py:127-130, np.lexsort((rows, keys))): row ids
// ordered by key ascending, equal keys (-0.0 == +0.0) by ascending row id.
//
// LSD radix sort of the 96-bit composite (ord(key) << 32 | row), 8-bit digits,
// least significant first: digits 0..3 are the row bytes, 4..11 the key-code bytes.
//   1. sort_hist_kernel: one read of the input computes all 12 digit histograms
//      and whether the row column is already ascending (then the row digits are
//      skipped: a stable sort by key of row-ordered input is the lexsort order).
//      Digits whose histogram is a single bucket are skipped too.
//   2. one sort_pass_kernel per remaining digit ("onesweep"): a block claims the
//      next tile, ranks its items stably per digit (bit-plane ballots + per-warp digit
//      counters), publishes the tile's digit counts and resolves its global digit
//      offsets by decoupled look-back over earlier tiles, stages the tile in shared
//      memory in digit order and writes each digit run contiguously. One read and
//      one write of 12 B per item per pass.
#pragma once
#include "common.cuh"

namespace golp {

#ifndef GOLP_SORT_THREADS
#define GOLP_SORT_THREADS 256
#endif
#ifndef GOLP_SORT_ITEMS
#define GOLP_SORT_ITEMS 12
#endif
#ifndef GOLP_SORT_MINB
#define GOLP_SORT_MINB 4
#endif
#ifndef GOLP_SORT_LOOK_WINDOW
#define GOLP_SORT_LOOK_WINDOW 4
#endif
#ifndef GOLP_SORT_SPIN_NS
#define GOLP_SORT_SPIN_NS 0
#endif
constexpr int kSortThreads = GOLP_SORT_THREADS;
constexpr int kSortItems = GOLP_SORT_ITEMS;
constexpr uint32_t kSortTileN = (uint32_t)kSortThreads * kSortItems;  // 2048 items
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortDigits = 12;
constexpr size_t kSortSmem = (size_t)kSortTileN * (8 + 4) + (size_t)kSortWarps * 256 * 4;

// Look-back status words: flag in the top two bits, count below.
constexpr unsigned long long kStatAggregate = 1ull << 62;
constexpr unsigned long long kStatPrefix = 2ull << 62;
constexpr unsigned long long kStatValue = (1ull << 62) - 1;

__device__ __forceinline__ uint32_t sort_digit(uint64_t k, uint32_t r, int d) {
  return d < 4 ? (r >> (8 * d)) & 255u : (uint32_t)(k >> (8 * (d - 4))) & 255u;
}

// hist[d * 256 + b]: items whose digit d is b. *rows_unsorted set when some
// rows[i] < rows[i-1].
__global__ void __launch_bounds__(256) sort_hist_kernel(const double* __restrict__ keys,
                                                        const uint32_t* __restrict__ rows, uint64_t n,
                                                        unsigned long long* __restrict__ hist,
                                                        unsigned* __restrict__ rows_unsorted) {
  __shared__ unsigned s_h[kSortDigits * 256];
  for (int i = threadIdx.x; i < kSortDigits * 256; i += blockDim.x) s_h[i] = 0;
  __syncthreads();
  bool unsorted = false;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t k = ord_key(__ldg(keys + i));
    const uint32_t r = __ldg(rows + i);
    if (i > 0 && __ldg(rows + i - 1) > r) unsorted = true;
#pragma unroll
    for (int d = 0; d < kSortDigits; ++d) atomicAdd(&s_h[d * 256 + sort_digit(k, r, d)], 1u);
  }
  if (__syncthreads_or(unsorted) && threadIdx.x == 0) atomicOr(rows_unsorted, 1u);
  for (int i = threadIdx.x; i < kSortDigits * 256; i += blockDim.x)
    if (s_h[i]) atomicAdd(&hist[i], (unsigned long long)s_h[i]);
}

struct SortPassArgs {
  const double* in_f64;     // first pass: the caller's keys (converted to codes on load)
  const uint64_t* in_keys;  // later passes: key codes
  const uint32_t* in_rows;
  uint64_t* out_keys;
  uint32_t* out_rows;
  uint64_t n;
  int digit;
  const unsigned long long* digit_base;  // 256 exclusive global offsets of this digit
  unsigned long long* status;            // [tiles][256] look-back words, zeroed
  unsigned long long* tile_ctr;          // zeroed
};

__global__ void __launch_bounds__(kSortThreads, GOLP_SORT_MINB) sort_pass_kernel(SortPassArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* s_key = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* s_row = reinterpret_cast<uint32_t*>(s_key + kSortTileN);
  uint32_t* s_wh = s_row + kSortTileN;  // [warp][256] counts, then exclusive warp offsets
  __shared__ uint32_t s_start[256];     // tile-local start of each digit run
  __shared__ unsigned long long s_out[256];  // global destination of each digit run
  __shared__ unsigned long long s_w[33];
  __shared__ unsigned long long s_tile;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(a.tile_ctr, 1ull);
  for (int i = lane; i < 256; i += 32) s_wh[warp * 256 + i] = 0;
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t t0 = tile * kSortTileN;
  if (t0 >= a.n) return;
  const uint32_t cnt = (uint32_t)(a.n - t0 < kSortTileN ? a.n - t0 : kSortTileN);

  // Warp-striped positions: item j of lane l in warp w sits at w*256 + j*32 + l,
  // so visiting j in order per warp, warps in order, is tile order (stability).
  uint64_t k[kSortItems];
  uint32_t r[kSortItems], dg[kSortItems];  // dg: digit (256 = no item), then | rank << 9
  const uint32_t wbase = warp * (32 * kSortItems) + lane;
  if (cnt == kSortTileN) {  // full tile: every load in flight before any use
    if (a.in_f64) {
      double kf[kSortItems];
#pragma unroll
      for (int j = 0; j < kSortItems; ++j) kf[j] = __ldg(a.in_f64 + t0 + wbase + j * 32);
#pragma unroll
      for (int j = 0; j < kSortItems; ++j) k[j] = ord_key(kf[j]);
    } else {
#pragma unroll
      for (int j = 0; j < kSortItems; ++j) k[j] = __ldg(a.in_keys + t0 + wbase + j * 32);
    }
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) r[j] = __ldg(a.in_rows + t0 + wbase + j * 32);
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) dg[j] = sort_digit(k[j], r[j], a.digit);
  } else {
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
      const uint32_t p = wbase + j * 32;
      if (p < cnt) {
        k[j] = a.in_f64 ? ord_key(__ldg(a.in_f64 + t0 + p)) : __ldg(a.in_keys + t0 + p);
        r[j] = __ldg(a.in_rows + t0 + p);
        dg[j] = sort_digit(k[j], r[j], a.digit);
      } else {
        k[j] = 0;
        r[j] = 0;
        dg[j] = 256;  // matches no real digit
      }
    }
  }
  uint32_t* wh = s_wh + warp * 256;
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    // lanes holding the same digit: 8 bit-plane ballots (cheaper than MATCH.ANY here)
    unsigned peers = __ballot_sync(0xFFFFFFFFu, dg[j] < 256);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const unsigned bal = __ballot_sync(0xFFFFFFFFu, (dg[j] >> b) & 1u);
      peers &= ((dg[j] >> b) & 1u) ? bal : ~bal;
    }
    const unsigned below = __popc(peers & ((1u << lane) - 1u));
    const uint32_t prior = dg[j] < 256 ? wh[dg[j]] : 0u;
    __syncwarp();
    if (dg[j] < 256 && below == 0) wh[dg[j]] = prior + __popc(peers);
    __syncwarp();
    dg[j] |= (prior + below) << 9;
  }
  __syncthreads();
  // per digit: counts of the warps -> exclusive warp offsets, tile total
  uint32_t total = 0;
  if (threadIdx.x < 256) {
    const int d = threadIdx.x;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const uint32_t c = s_wh[w * 256 + d];
      s_wh[w * 256 + d] = total;
      total += c;
    }
    // publish this tile's aggregate (tile 0: already the inclusive prefix)
    volatile unsigned long long* st = a.status + tile * 256 + d;
    *st = (tile == 0 ? kStatPrefix : kStatAggregate) | total;
  }
  // tile-local digit starts (exclusive scan of the totals; 512 threads, 256 digits)
  unsigned long long tot;
  const unsigned long long e = block_excl_scan(threadIdx.x < 256 ? total : 0u, s_w, &tot);
  if (threadIdx.x < 256) s_start[threadIdx.x] = (uint32_t)e;
  __syncthreads();  // s_start ready
  // stage the tile in digit order (needs only tile-local offsets, so it overlaps
  // the look-back below)
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const uint32_t d = dg[j] & 511u;
    if (d < 256) {
      const uint32_t dst = s_start[d] + s_wh[warp * 256 + d] + (dg[j] >> 9);
      s_key[dst] = k[j];
      s_row[dst] = r[j];
    }
  }
  // decoupled look-back, one thread per digit, kLookWindow predecessors per step
  // (independent loads in flight; spin only on entries not yet published)
  if (threadIdx.x < 256) {
    const int d = threadIdx.x;
    unsigned long long excl = 0;
    if (tile > 0) {
      constexpr int kLookWindow = GOLP_SORT_LOOK_WINDOW;
      int64_t p = (int64_t)tile - 1;
      bool done = false;
      while (!done && p >= 0) {
        unsigned long long v[kLookWindow];
#pragma unroll
        for (int u = 0; u < kLookWindow; ++u)
          v[u] = p - u >= 0 ? *(const volatile unsigned long long*)(a.status + (uint64_t)(p - u) * 256 + d) : 0ull;
#pragma unroll
        for (int u = 0; u < kLookWindow; ++u) {
          if (done || p - u < 0) continue;
          while ((v[u] & ~kStatValue) == 0) {
            if (GOLP_SORT_SPIN_NS) __nanosleep(GOLP_SORT_SPIN_NS);
            v[u] = *(const volatile unsigned long long*)(a.status + (uint64_t)(p - u) * 256 + d);
          }
          excl += v[u] & kStatValue;
          if (v[u] & kStatPrefix) done = true;
        }
        p -= kLookWindow;
      }
      volatile unsigned long long* mine = a.status + tile * 256 + d;
      *mine = kStatPrefix | (excl + total);
    }
    s_out[d] = a.digit_base[d] + excl;
  }
  __syncthreads();
  // each digit run goes out contiguously
  for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
    const uint64_t kk = s_key[i];
    const uint32_t rr = s_row[i];
    const uint32_t d = sort_digit(kk, rr, a.digit);
    const uint64_t o = s_out[d] + (i - s_start[d]);
    if (a.out_keys) a.out_keys[o] = kk;  // the last pass only needs the rows
    a.out_rows[o] = rr;
  }
}

}  // namespace golp
