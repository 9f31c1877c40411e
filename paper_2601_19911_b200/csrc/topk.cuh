// Top-K selection over (key f64, row u32) pairs: the B200 replacement for the
// reference's data-parallel Top-K (ProxyDevice.topk -> _chunk_topk_candidates +
// _merge_topk_candidates, pkg/src/golp/device.py:239-259,329-380), bit-exact with
// host_topk (pkg/src/golp/host.py:133-144): the k largest keys, descending, equal
// keys by ascending row id.
//
// Order: composite item (hi = ord(key), lo = ~row), larger is better.
//
// Pipeline (one read of the key column on the common path):
//   1. threshold  : radix-select the r-th best of S stratified samples (THRESH mode
//                   of the select engine) -> conservative composite threshold T.
//   2. filter     : stream keys with 128-bit loads, keep items >= T (warp-aggregated
//                   appends), rows are gathered only for survivors.
//   3. select     : MSB radix select over the candidates (smem histograms, 8-bit
//                   digits, one grid barrier per digit) -> exact K-th item, then
//                   collect the K winners and bitonic-sort them (one block when
//                   K <= 8192, otherwise a grid-wide network with smem tiles).
// If the sampled threshold admits fewer than K or more than `cap` candidates the
// host re-runs step 3 directly over the input (exact, slower, never wrong).
#pragma once
#include <cooperative_groups.h>
#include "sortnet.cuh"

namespace golp {

namespace cg = cooperative_groups;

constexpr int kSelThreads = 1024;
constexpr uint32_t kSortTile = 8192;  // items per shared-memory sort tile (96 KB)
#ifndef GOLP_MERGE_TILE
#define GOLP_MERGE_TILE 1024
#endif
#ifndef GOLP_MERGE_PER
#define GOLP_MERGE_PER 1
#endif
constexpr uint32_t kMergeTile = GOLP_MERGE_TILE;  // winner sort: runs sorted per block before the merges
constexpr uint32_t kMergePer = GOLP_MERGE_PER;    // winner sort: outputs per thread per merge round
constexpr int kModeFull = 0;          // radix select + collect + sort + emit
constexpr int kModeThreshold = 1;     // radix select only -> ctl->thr_*

struct SelectCtl {
  unsigned int hist[12][256];
  unsigned long long cand_count;  // filter output (may exceed cap: overflow)
  unsigned long long win_count;
  unsigned long long eq_count;
  double thr_key;
  uint32_t thr_row;
  int status;  // 0 ok, 1 candidate set unusable (host falls back to direct)
  unsigned long long res_hi;
  uint32_t res_lo;
  int res_bits;
};

// ---- item sources -------------------------------------------------------------

struct SrcInput {  // the caller's (keys, rows) columns
  const double* keys;
  RowCol rows;
  __device__ __forceinline__ uint64_t hi(uint64_t i) const { return ord_key(__ldg(keys + i)); }
  __device__ __forceinline__ uint32_t lo(uint64_t i) const { return ~rows.at(i); }
};

struct SrcCand {  // encoded candidate arrays written by the filter (or a merge)
  const uint64_t* h;
  const uint32_t* l;
  __device__ __forceinline__ uint64_t hi(uint64_t i) const { return __ldcg(h + i); }
  __device__ __forceinline__ uint32_t lo(uint64_t i) const { return __ldcg(l + i); }
};

struct SrcPairs {  // encoded keys + plain row ids (all-gathered local Top-K results)
  const uint64_t* h;
  const uint32_t* rows;
  __device__ __forceinline__ uint64_t hi(uint64_t i) const { return __ldcg(h + i); }
  __device__ __forceinline__ uint32_t lo(uint64_t i) const { return ~__ldcg(rows + i); }
};

// S stratified samples of an n-item column: sample i comes from stratum
// [i*w, (i+1)*w) (w = n / S) at a hashed offset, so periodic layouts cannot
// alias. 32-bit arithmetic only (64-bit division costs ~100 instructions).
struct SrcSample {
  const double* keys;
  RowCol rows;
  uint64_t n;
  uint32_t w;  // stratum width, >= 1
  __device__ __forceinline__ uint64_t pos(uint64_t i) const {
    const uint64_t p = i * w + (hash32((uint32_t)i * 2654435761u + 12345u) % w);
    return p < n ? p : n - 1;
  }
  __device__ __forceinline__ uint64_t hi(uint64_t i) const { return ord_key(__ldg(keys + pos(i))); }
  __device__ __forceinline__ uint32_t lo(uint64_t i) const { return ~rows.at(pos(i)); }
};

template <class Src>
struct SelectArgs {
  Src src;
  uint64_t n;          // items in src (ignored when use_cand_count)
  uint64_t need;       // K' (items wanted), 1 <= need
  uint64_t cap;        // candidate capacity (use_cand_count only)
  int use_cand_count;  // n := ctl->cand_count, validated against need/cap
  int mode;
  SelectCtl* ctl;
  uint64_t* w_hi;      // winners scratch, >= 2 * need entries (the second half: merge buffer)
  uint32_t* w_lo;
  uint32_t* out_rows;  // need entries, best first
  uint64_t* out_hi;    // optional: encoded keys of the winners (for merges)
  int* host_status;    // optional mapped host word: 1 when the candidate set was unusable
  unsigned long long* host_count;  // optional mapped host word: candidate count
};

// Compare the top `bits` bits of (h, l) against the prefix: -1, 0, +1.
__device__ __forceinline__ int prefix_cmp(uint64_t h, uint32_t l, uint64_t ph, uint32_t pl, int bits) {
  if (bits <= 0) return 0;
  if (bits <= 64) {
    const int sh = 64 - bits;
    const uint64_t a = sh >= 64 ? 0 : (h >> sh), b = sh >= 64 ? 0 : (ph >> sh);
    return a > b ? 1 : (a < b ? -1 : 0);
  }
  if (h != ph) return h > ph ? 1 : -1;
  const int sh = 96 - bits;
  const uint32_t a = l >> sh, b = pl >> sh;
  return a > b ? 1 : (a < b ? -1 : 0);
}


// ---- single-block selection in shared memory -------------------------------------
// MSB radix select of the `need` best of n items held in shared memory (8-bit
// digits over the 96-bit composite, smem histogram, one warp resolves the digit).
// Leaves the resolved prefix in *pre_hi/*pre_lo/*bits and the count still to
// take from the prefix bucket in *rem (same contract as the grid engine).
// With `coarse`, stops as soon as the prefix bucket holds at most 2*need items:
// everything >= the prefix is still a superset of the best `need` (threshold use).
__device__ void block_radix_select(const uint64_t* s_hi, const uint32_t* s_lo, uint32_t n, uint64_t need,
                                   unsigned* s_hist, uint64_t* sh_pre_hi, uint32_t* sh_pre_lo, int* sh_bits,
                                   unsigned long long* sh_rem, int* sh_done, bool coarse = false) {
  if (threadIdx.x == 0) {
    *sh_pre_hi = 0;
    *sh_pre_lo = 0;
    *sh_bits = 0;
    *sh_rem = need;
    *sh_done = 0;
  }
  __syncthreads();
  for (int pass = 0; pass < 12; ++pass) {
    const uint64_t pre_hi = *sh_pre_hi;
    const uint32_t pre_lo = *sh_pre_lo;
    const int bits = *sh_bits;
    const unsigned long long rem = *sh_rem;
    for (int t = threadIdx.x; t < 256; t += blockDim.x) s_hist[t] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint64_t h = s_hi[i];
      unsigned d;
      if (bits < 64) {
        if (bits > 0 && (h >> (64 - bits)) != (pre_hi >> (64 - bits))) continue;
        d = (unsigned)(h >> (56 - bits)) & 255u;
      } else {
        if (h != pre_hi) continue;
        const uint32_t l = s_lo[i];
        if (bits > 64 && (l >> (96 - bits)) != (pre_lo >> (96 - bits))) continue;
        d = (l >> (24 - (bits - 64))) & 255u;
      }
      atomicAdd(&s_hist[d], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      unsigned c8[8];
      unsigned long long lsum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        c8[q] = s_hist[255 - 8 * lane - q];
        lsum += c8[q];
      }
      unsigned long long incl = lsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
      }
      const unsigned long long excl = incl - lsum;
      if (excl < rem && incl >= rem) {
        unsigned long long cum = excl;
        int b = -1;
        unsigned cb = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (b < 0 && cum + c8[q] >= rem) { b = 255 - 8 * lane - q; cb = c8[q]; }
          else if (b < 0) cum += c8[q];
        }
        uint64_t ph = pre_hi;
        uint32_t pl = pre_lo;
        if (bits < 64) ph |= (uint64_t)b << (56 - bits);
        else pl |= (uint32_t)b << (24 - (bits - 64));
        *sh_pre_hi = ph;
        *sh_pre_lo = pl;
        *sh_bits = bits + 8;
        *sh_rem = rem - cum;
        *sh_done = (rem - cum == cb) || (bits + 8 >= 96) || (coarse && cb <= 2 * need);
      }
    }
    __syncthreads();
    if (*sh_done) break;
  }
}

// The select engine as a device function so the fused Top-K kernel can run it
// in place (same block size and dynamic shared memory as select_kernel).
template <class Src>
__device__ void select_body(const SelectArgs<Src>& a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* s_hi = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* s_lo = reinterpret_cast<uint32_t*>(s_hi + kSortTile);
  __shared__ unsigned s_hist[256];
  __shared__ uint64_t sh_pre_hi;
  __shared__ uint32_t sh_pre_lo;
  __shared__ int sh_bits;
  __shared__ unsigned long long sh_rem;
  __shared__ int sh_done;

  const Src src = a.src;
  uint64_t n = a.n;
  if (a.use_cand_count) {
    const unsigned long long c = *(volatile unsigned long long*)&a.ctl->cand_count;
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.host_count) *(volatile unsigned long long*)a.host_count = c;
    if (c > a.cap || c < a.need) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.ctl->status = 1;
        if (a.host_status) *(volatile int*)a.host_status = 1;
        __threadfence_system();
      }
      return;  // uniform across the grid: no barrier is ever reached
    }
    n = c;
  }
  const uint64_t need = a.need < n ? a.need : n;
  const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;

  // Small lists: one block, all in shared memory. Threshold mode resolves the
  // need-th best by a smem radix select; full mode selects the best `need` the
  // same way when that beats sorting everything, then sorts only those.
  if (n <= kSortTile) {
    if (blockIdx.x != 0) return;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      s_hi[i] = src.hi(i);
      s_lo[i] = src.lo(i);
    }
    __syncthreads();
    if (a.mode == kModeThreshold || (need * 4 <= n && n > 1024)) {
      block_radix_select(s_hi, s_lo, (uint32_t)n, need, s_hist, &sh_pre_hi, &sh_pre_lo, &sh_bits, &sh_rem, &sh_done,
                         a.mode == kModeThreshold);
      const uint64_t ph = sh_pre_hi;
      const uint32_t pl = sh_pre_lo;
      const int bits = sh_bits;
      const unsigned long long rem = sh_rem;
      if (a.mode == kModeThreshold) {
        if (threadIdx.x == 0) {
          a.ctl->thr_key = key_from_ord(ph);
          a.ctl->thr_row = ~pl;
          a.ctl->res_hi = ph;
          a.ctl->res_lo = pl;
          a.ctl->res_bits = bits;
        }
        return;
      }
      // collect the winners (held in registers while the list is read), then
      // rewrite them to the front of the smem list and sort just them
      uint64_t* w_hi = s_hi;
      uint32_t* w_lo = s_lo;
      __shared__ unsigned s_cnt, s_eq;
      if (threadIdx.x == 0) { s_cnt = 0; s_eq = 0; }
      __syncthreads();
      uint64_t keep_hi[kSortTile / kSelThreads];
      uint32_t keep_lo[kSortTile / kSelThreads];
      unsigned nk = 0;
      for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint64_t h = s_hi[i];
        const uint32_t l = s_lo[i];
        const int c = prefix_cmp(h, l, ph, pl, bits);
        if (c > 0 || (c == 0 && (bits < 96 || atomicAdd(&s_eq, 1u) < rem))) {
          keep_hi[nk] = h;
          keep_lo[nk] = l;
          ++nk;
        }
      }
      __syncthreads();  // all reads of s_hi/s_lo done before the winners overwrite them
      for (unsigned q = 0; q < nk; ++q) {
        const unsigned slot = atomicAdd(&s_cnt, 1u);
        w_hi[slot] = keep_hi[q];
        w_lo[slot] = keep_lo[q];
      }
      __syncthreads();
      block_sort_desc(w_hi, w_lo, (uint32_t)need);
      for (uint32_t i = threadIdx.x; i < need; i += blockDim.x) {
        a.out_rows[i] = ~w_lo[i];
        if (a.out_hi) a.out_hi[i] = w_hi[i];
      }
      return;
    }
    block_sort_desc(s_hi, s_lo, (uint32_t)n);
    for (uint32_t i = threadIdx.x; i < need; i += blockDim.x) {
      a.out_rows[i] = ~s_lo[i];
      if (a.out_hi) a.out_hi[i] = s_hi[i];
    }
    return;
  }

  // ---- MSB radix select on the 96-bit composite, 8-bit digits ----------------
  // (grid-wide from here on: only reached under a cooperative launch)
  cg::grid_group grid = cg::this_grid();
  uint64_t pre_hi = 0;
  uint32_t pre_lo = 0;
  int bits = 0;
  uint64_t rem = need;
  for (int pass = 0; pass < 12; ++pass) {
    for (int t = threadIdx.x; t < 256; t += blockDim.x) s_hist[t] = 0;
    __syncthreads();
    for (uint64_t i = gtid; i < n; i += gstride) {
      const uint64_t h = src.hi(i);
      unsigned d;
      if (bits < 64) {
        if (bits > 0 && (h >> (64 - bits)) != (pre_hi >> (64 - bits))) continue;
        d = (unsigned)(h >> (56 - bits)) & 255u;
      } else {
        if (h != pre_hi) continue;
        const uint32_t l = src.lo(i);
        if (bits > 64 && (l >> (96 - bits)) != (pre_lo >> (96 - bits))) continue;
        d = (l >> (24 - (bits - 64))) & 255u;
      }
      atomicAdd(&s_hist[d], 1u);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 256; t += blockDim.x)
      if (s_hist[t]) atomicAdd(&a.ctl->hist[pass][t], s_hist[t]);
    grid.sync();
    // Every block resolves the digit identically from the global histogram.
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      unsigned c8[8];
      unsigned long long lsum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {  // lane covers bins 255-8*lane-q (descending)
        c8[q] = __ldcg(&a.ctl->hist[pass][255 - 8 * lane - q]);
        lsum += c8[q];
      }
      unsigned long long incl = lsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
      }
      const unsigned long long excl = incl - lsum;
      const bool mine = excl < rem && incl >= rem;
      if (mine) {
        unsigned long long cum = excl;
        int b = -1;
        unsigned cb = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (b < 0 && cum + c8[q] >= rem) { b = 255 - 8 * lane - q; cb = c8[q]; }
          else if (b < 0) cum += c8[q];
        }
        const uint64_t new_rem = rem - cum;
        uint64_t ph = pre_hi;
        uint32_t pl = pre_lo;
        if (bits < 64) ph |= (uint64_t)b << (56 - bits);
        else pl |= (uint32_t)b << (24 - (bits - 64));
        sh_pre_hi = ph;
        sh_pre_lo = pl;
        sh_bits = bits + 8;
        sh_rem = new_rem;
        sh_done = (new_rem == cb) || (bits + 8 >= 96);
      }
    }
    __syncthreads();
    pre_hi = sh_pre_hi;
    pre_lo = sh_pre_lo;
    bits = sh_bits;
    rem = sh_rem;
    const int done = sh_done;
    __syncthreads();
    if (done) break;
  }

  if (a.mode == kModeThreshold) {
    // Everything >= (pre_hi, pre_lo) (low bits zero) holds the `need` best samples.
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.ctl->thr_key = key_from_ord(pre_hi);
      a.ctl->thr_row = ~pre_lo;
      a.ctl->res_hi = pre_hi;
      a.ctl->res_lo = pre_lo;
      a.ctl->res_bits = bits;
    }
    return;
  }

  // ---- collect exactly `need` winners ----------------------------------------
  for (uint64_t wb = gtid - lane_id(); wb < n; wb += gstride) {
    const uint64_t i = wb + lane_id();
    bool take = false;
    uint64_t h = 0;
    uint32_t l = 0;
    if (i < n) {
      h = src.hi(i);
      l = (bits > 64 || h >= pre_hi) ? src.lo(i) : 0u;
      const int c = prefix_cmp(h, l, pre_hi, pre_lo, bits);
      if (c > 0) take = true;
      else if (c == 0) take = bits < 96 || atomicAdd(&a.ctl->eq_count, 1ull) < rem;
    }
    const unsigned long long slot = warp_append(&a.ctl->win_count, take);
    if (take) {
      __stcg(a.w_hi + slot, h);
      __stcg(a.w_lo + slot, l);
    }
  }
  grid.sync();

  // ---- sort the winners (best first) and emit -------------------------------
  if (need <= kSortTile) {
    if (blockIdx.x != 0) return;
    for (uint32_t i = threadIdx.x; i < need; i += blockDim.x) {
      s_hi[i] = __ldcg(a.w_hi + i);
      s_lo[i] = __ldcg(a.w_lo + i);
    }
    __syncthreads();
    block_sort_desc(s_hi, s_lo, (uint32_t)need);
    for (uint32_t i = threadIdx.x; i < need; i += blockDim.x) {
      a.out_rows[i] = ~s_lo[i];
      if (a.out_hi) a.out_hi[i] = s_hi[i];
    }
    return;
  }

  uint64_t* gh = a.w_hi;
  uint32_t* gl = a.w_lo;
  const uint64_t m = need;
  // (a) runs of kMergeTile sorted in shared memory, one block per run (small
  // runs keep every SM busy; a whole-block bitonic sort of 8192 was 120 µs)
  const uint64_t ntiles = (m + kMergeTile - 1) / kMergeTile;
#if GOLP_SEL_TIMING
  const long long ttile = clock64();
#endif
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t base = tile * kMergeTile;
    const uint32_t cnt = (uint32_t)((m - base) < kMergeTile ? (m - base) : kMergeTile);
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
      s_hi[i] = __ldcg(gh + base + i);
      s_lo[i] = __ldcg(gl + base + i);
    }
    __syncthreads();
    block_sort_desc(s_hi, s_lo, cnt);
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
      __stcg(gh + base + i, s_hi[i]);
      __stcg(gl + base + i, s_lo[i]);
    }
    __syncthreads();
  }
#if GOLP_SEL_TIMING
  if (blockIdx.x == 0 && threadIdx.x == 0) printf("tile sort %lld cycles\n", clock64() - ttile);
#endif
  grid.sync();
#if GOLP_SEL_TIMING
  const long long tsorted = clock64();
#endif
  // (b) sorted runs of kSortTile merged pairwise (merge path: every thread finds
  // where its kMergePer outputs start by a binary search on its diagonal, then
  // merges them sequentially), ping-ponging with the second half of the winners
  // scratch: ceil(log2(m / kSortTile)) rounds, one grid barrier each.
  uint64_t* sh = gh;
  uint32_t* sl = gl;
  uint64_t* dh = gh + m;
  uint32_t* dl = gl + m;
  for (uint64_t L = kMergeTile; L < m; L <<= 1) {
    const uint64_t nchunks = (m + kMergePer - 1) / kMergePer;
    for (uint64_t c = gtid; c < nchunks; c += gstride) {
      const uint64_t o0 = c * kMergePer;
      const uint64_t base = (o0 / (2 * L)) * (2 * L);
      const uint64_t la = base + L < m ? L : m - base;
      const uint64_t b0 = base + la;
      const uint64_t lb = b0 < m ? (b0 + L < m ? L : m - b0) : 0;
      const uint64_t k = o0 - base;
      // smallest i (items taken from run A among the first k) such that A[i]
      // does not go before B[k - i - 1]; A wins ties (item_gt is strict)
      uint64_t lo = k > lb ? k - lb : 0, hi = k < la ? k : la;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        const uint64_t bj = b0 + (k - mid - 1);
        if (!item_gt(__ldcg(sh + bj), __ldcg(sl + bj), __ldcg(sh + base + mid), __ldcg(sl + base + mid))) lo = mid + 1;
        else hi = mid;
      }
      uint64_t i = lo, j = k - lo;
      const uint64_t end = (o0 + kMergePer < base + la + lb) ? o0 + kMergePer : base + la + lb;
      for (uint64_t o = o0; o < end; ++o) {
        bool take_a;
        if (i >= la) take_a = false;
        else if (j >= lb) take_a = true;
        else take_a = !item_gt(__ldcg(sh + b0 + j), __ldcg(sl + b0 + j), __ldcg(sh + base + i), __ldcg(sl + base + i));
        const uint64_t src = take_a ? base + i : b0 + j;
        __stcg(dh + o, __ldcg(sh + src));
        __stcg(dl + o, __ldcg(sl + src));
        if (take_a) ++i;
        else ++j;
      }
    }
    grid.sync();
    uint64_t* th = sh;
    uint32_t* tl = sl;
    sh = dh;
    sl = dl;
    dh = th;
    dl = tl;
  }
  gh = sh;
  gl = sl;
#if GOLP_SEL_TIMING
  if (blockIdx.x == 0 && threadIdx.x == 0)
    printf("winner sort: m %llu tiles %llu cycles, merges %lld cycles\n", (unsigned long long)m,
           (unsigned long long)ntiles, clock64() - tsorted);
#endif
  for (uint64_t i = gtid; i < m; i += gstride) {
    a.out_rows[i] = ~__ldcg(gl + i);
    if (a.out_hi) a.out_hi[i] = __ldcg(gh + i);
  }
}

template <class Src>
__global__ void __launch_bounds__(kSelThreads) select_kernel(SelectArgs<Src> a) {
  select_body(a);
}

// ---- rank selection (small lists, many blocks, no grid barrier) -------------------
// For lists of at most kRankMax items every block stages the whole list in shared
// memory and its warps compute exact ranks (items strictly better, ties broken by
// index so ranks are a permutation) for a strided share of the items: O(n^2 / P)
// compares spread over the GPU, one launch, no digit passes. THRESH mode writes the
// item of rank need-1 as the threshold (and clears the candidate counter the filter
// appends to); FULL mode writes every item of rank < need to out[rank].
// Candidate lists (use_cand_count) larger than kRankMax but within the buffer set
// status 2: the host then runs the grid engine over the same candidates.
constexpr uint32_t kRankMax = 8192;
constexpr int kRankThreads = 512;
constexpr size_t kRankSmem = (size_t)kRankMax * (sizeof(uint64_t) + sizeof(uint32_t));

// Exact ranks of the m items staged in shared memory, computed for a strided
// share of the items by every warp of the grid (see above).
// Block-local MSB radix select over m staged items (96-bit composite, 8-bit
// digits): the largest prefix P (low bits zero) such that exactly `need` items
// are >= P. Every block computes the same P from the same items, so the fused
// Top-K needs no grid barrier to publish its threshold. Called by all threads.
// s_lo is filled by fill_lo() only once a pass needs row bits (a key tie at the
// threshold), so the common case stages keys alone.
template <class FillLo>
__device__ __forceinline__ void block_radix_threshold(const uint64_t* s_hi, const uint32_t* s_lo, uint32_t m,
                                                      uint64_t need, uint64_t* out_hi, uint32_t* out_lo,
                                                      FillLo fill_lo) {
  __shared__ unsigned s_h[256];
  __shared__ uint64_t sh_hi;
  __shared__ uint32_t sh_lo;
  __shared__ int sh_bits, sh_done;
  __shared__ unsigned long long sh_rem;
  uint64_t pre_hi = 0;
  uint32_t pre_lo = 0;
  int bits = 0;
  unsigned long long rem = need;
  bool lo_ready = false;
  for (int pass = 0; pass < 12; ++pass) {
    if (bits >= 64 && !lo_ready) {  // block-uniform
      fill_lo();
      lo_ready = true;
    }
    for (int t = threadIdx.x; t < 256; t += blockDim.x) s_h[t] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
      const uint64_t h = s_hi[i];
      unsigned d;
      if (bits < 64) {
        if (bits > 0 && (h >> (64 - bits)) != (pre_hi >> (64 - bits))) continue;
        d = (unsigned)(h >> (56 - bits)) & 255u;
      } else {
        if (h != pre_hi) continue;
        const uint32_t l = s_lo[i];
        if (bits > 64 && (l >> (96 - bits)) != (pre_lo >> (96 - bits))) continue;
        d = (l >> (24 - (bits - 64))) & 255u;
      }
      atomicAdd(&s_h[d], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // lane covers bins 255-8*lane-q (descending)
      const int lane = threadIdx.x;
      unsigned c8[8];
      unsigned long long lsum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        c8[q] = s_h[255 - 8 * lane - q];
        lsum += c8[q];
      }
      unsigned long long incl = lsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
      }
      const unsigned long long excl = incl - lsum;
      if (excl < rem && incl >= rem) {
        unsigned long long cum = excl;
        int b = -1;
        unsigned cb = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (b < 0 && cum + c8[q] >= rem) {
            b = 255 - 8 * lane - q;
            cb = c8[q];
          } else if (b < 0) {
            cum += c8[q];
          }
        }
        const unsigned long long nrem = rem - cum;
        uint64_t ph = pre_hi;
        uint32_t pl = pre_lo;
        if (bits < 64) ph |= (uint64_t)b << (56 - bits);
        else pl |= (uint32_t)b << (24 - (bits - 64));
        sh_hi = ph;
        sh_lo = pl;
        sh_bits = bits + 8;
        sh_rem = nrem;
        sh_done = (nrem == cb) || (bits + 8 >= 96);
      }
    }
    __syncthreads();
    pre_hi = sh_hi;
    pre_lo = sh_lo;
    bits = sh_bits;
    rem = sh_rem;
    const int done = sh_done;
    __syncthreads();
    if (done) break;
  }
  *out_hi = pre_hi;
  *out_lo = pre_lo;
}

__device__ __forceinline__ void rank_items(const uint64_t* s_hi, const uint32_t* s_lo, uint32_t m, uint64_t need,
                                           int mode, SelectCtl* ctl, uint32_t* out_rows, uint64_t* out_hi) {
  const unsigned lane = lane_id();
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < m; i += warps) {
    const uint64_t hi = s_hi[i];
    const uint32_t lo = s_lo[i];
    uint32_t better = 0, eq = 0;
    for (uint32_t j = lane; j < m; j += 32) {  // key codes only: the common case has no ties
      const uint64_t h = s_hi[j];
      better += h > hi;
      eq += h == hi;
    }
    better = __reduce_add_sync(0xFFFFFFFFu, better);
    if (__reduce_add_sync(0xFFFFFFFFu, eq) > 1) {  // equal keys: row, then index decides
      uint32_t tb = 0;
      for (uint32_t j = lane; j < m; j += 32) {
        if (s_hi[j] != hi) continue;
        const uint32_t l = s_lo[j];
        tb += (l > lo) | ((l == lo) & (j < i));
      }
      better += __reduce_add_sync(0xFFFFFFFFu, tb);
    }
    if (lane == 0) {
      if (mode == kModeThreshold) {
        if (better == need - 1) {
          ctl->thr_key = key_from_ord(hi);
          ctl->thr_row = ~lo;
          ctl->res_hi = hi;
          ctl->res_lo = lo;
          ctl->res_bits = 96;
        }
      } else if (better < need) {
        out_rows[better] = ~lo;
        if (out_hi) out_hi[better] = hi;
      }
    }
  }
}

template <class Src>
__global__ void __launch_bounds__(kRankThreads) rank_select_kernel(SelectArgs<Src> a,
                                                                   unsigned long long* clear_count) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* s_hi = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* s_lo = reinterpret_cast<uint32_t*>(s_hi + kRankMax);
  uint64_t n = a.n;
  if (a.use_cand_count) {
    const unsigned long long c = *(volatile unsigned long long*)&a.ctl->cand_count;
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.host_count) *(volatile unsigned long long*)a.host_count = c;
    if (c > a.cap || c < a.need || c > kRankMax) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        const int st = (c > a.cap || c < a.need) ? 1 : 2;
        a.ctl->status = st;
        if (a.host_status) *(volatile int*)a.host_status = st;
        __threadfence_system();
      }
      return;
    }
    n = c;
  }
  if (clear_count && blockIdx.x == 0 && threadIdx.x == 0) *clear_count = 0ull;
  const uint32_t m = (uint32_t)n;
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
    s_hi[i] = a.src.hi(i);
    s_lo[i] = a.src.lo(i);
  }
  __syncthreads();
  rank_items(s_hi, s_lo, m, a.need < n ? a.need : n, a.mode, a.ctl, a.out_rows, a.out_hi);
}

// ---- streaming filter ------------------------------------------------------------
// Keeps every item with (key, row) >= (thr_key, thr_row) in Top-K order, i.e.
// key > thr_key, or key == thr_key and row <= thr_row. Float compare gives the
// reference's -0.0 == +0.0 for free. Rows are loaded only for survivors and for
// exact threshold ties.
constexpr int kFilterThreads = 256;
constexpr int kFilterUnroll = 4;  // 4 x 16 B loads in flight per thread

__device__ __forceinline__ bool filter_keep(double k, double tk, uint32_t tr, RowCol rows, uint64_t pos) {
  if (k > tk) return true;
  if (k == tk) return rows.at(pos) <= tr;
  return false;
}

__device__ __forceinline__ void filter_body(const double* __restrict__ keys, RowCol rows,
                                            uint64_t n, double tk, uint32_t tr, unsigned long long* cand_count,
                                            uint64_t* __restrict__ cand_hi, uint32_t* __restrict__ cand_lo,
                                            uint64_t cap) {
  const uint64_t head = (((uintptr_t)keys & 15) != 0 && n > 0) ? 1 : 0;
  const uint64_t nv = (n - head) / 2;
  const uint64_t tail = head + 2 * nv;  // index of a leftover odd element (if < n)
  const double* kv = keys + head;
  const unsigned lane = lane_id();
  const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;

  if (blockIdx.x == 0 && threadIdx.x < 32) {  // scalar head / tail elements
    uint64_t pos = ~0ull;
    if (lane == 0 && head) pos = 0;
    if (lane == 1 && tail < n) pos = tail;
    bool take = false;
    if (pos != ~0ull) take = filter_keep(keys[pos], tk, tr, rows, pos);
    const unsigned long long slot = warp_append(cand_count, take);
    if (take && slot < cap) {
      cand_hi[slot] = ord_key(keys[pos]);
      cand_lo[slot] = ~rows.at(pos);
    }
  }

  for (uint64_t wb = gtid - lane; wb < nv; wb += stride * kFilterUnroll) {
    double2 v[kFilterUnroll];
#pragma unroll
    for (int u = 0; u < kFilterUnroll; ++u) {
      const uint64_t vi = wb + lane + (uint64_t)u * stride;
      if (vi < nv) v[u] = ldg_nc_d2(kv + 2 * vi);
      else v[u] = make_double2(-__longlong_as_double(0x7FF0000000000000ll), 0.0);
    }
    // keys above the threshold key are kept outright; keys equal to it (ties,
    // e.g. a Zipf head) need their row: all those row loads go out together
    unsigned flags = 0, ties = 0;
#pragma unroll
    for (int u = 0; u < kFilterUnroll; ++u) {
      const uint64_t vi = wb + lane + (uint64_t)u * stride;
      if (vi < nv) {
        if (v[u].x > tk) flags |= 1u << (2 * u);
        else if (v[u].x == tk) ties |= 1u << (2 * u);
        if (v[u].y > tk) flags |= 2u << (2 * u);
        else if (v[u].y == tk) ties |= 2u << (2 * u);
      }
    }
    if (ties) {
      uint32_t rr[2 * kFilterUnroll];
#pragma unroll
      for (int e = 0; e < 2 * kFilterUnroll; ++e)
        if ((ties >> e) & 1u) rr[e] = rows.at(head + 2 * (wb + lane + (uint64_t)(e >> 1) * stride) + (e & 1));
#pragma unroll
      for (int e = 0; e < 2 * kFilterUnroll; ++e)
        if (((ties >> e) & 1u) && rr[e] <= tr) flags |= 1u << e;
    }
    if (__any_sync(0xFFFFFFFFu, flags != 0)) {
#pragma unroll
      for (int u = 0; u < kFilterUnroll; ++u) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const bool take = (flags >> (2 * u + e)) & 1u;
          const unsigned long long slot = warp_append(cand_count, take);
          if (take && slot < cap) {
            const uint64_t p = head + 2 * (wb + lane + (uint64_t)u * stride) + e;
            cand_hi[slot] = ord_key(e ? v[u].y : v[u].x);
            cand_lo[slot] = ~rows.at(p);
          }
        }
      }
    }
  }
}


__global__ void __launch_bounds__(kFilterThreads) topk_filter_kernel(
    const double* __restrict__ keys, RowCol rows, uint64_t n, const SelectCtl* thr,
    unsigned long long* cand_count, uint64_t* __restrict__ cand_hi, uint32_t* __restrict__ cand_lo,
    uint64_t cap) {
  const double tk = *(const volatile double*)&thr->thr_key;
  const uint32_t tr = *(const volatile uint32_t*)&thr->thr_row;
  filter_body(keys, rows, n, tk, tr, cand_count, cand_hi, cand_lo, cap);
}


// ---- fused small Top-K -----------------------------------------------------------
// One cooperative launch for inputs whose sample set and expected candidate list
// fit the rank kernel (C1-sized): rank threshold over the samples | grid barrier |
// streaming filter | grid barrier | rank select over the candidates. If the
// candidate set turns out unusable it runs the grid select engine in place (over
// the candidates when they fit the buffer but not shared memory, else straight
// over the input), so the host never has to wait and decide.
struct FusedTopkArgs {
  const double* keys;
  RowCol rows;
  uint64_t n;
  uint64_t need;  // min(k, n)
  uint32_t s;     // samples (<= kRankMax)
  uint32_t need_s;
  uint32_t w;     // sample stratum width
  uint64_t cap;   // candidate buffer capacity
  uint32_t rank_max;  // largest candidate list ranked in shared memory (<= kRankMax)
  SelectCtl* ctl;  // ctl[0] threshold, ctl[1] candidates, ctl[2] direct fallback
  uint64_t* cand_hi;
  uint32_t* cand_lo;
  uint64_t* w_hi;
  uint32_t* w_lo;
  uint32_t* out_rows;
  uint64_t* out_hi;
  unsigned long long* host_count;  // optional mapped word: candidate count
  int* host_status;                // optional mapped word: 1 fell back to the direct select
};

__global__ void __launch_bounds__(kSelThreads) topk_fused_kernel(FusedTopkArgs f) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* s_hi = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* s_lo = reinterpret_cast<uint32_t*>(s_hi + kSortTile);
  static_assert(kSortTile >= kRankMax, "rank lists are staged in the select tile");
  cg::grid_group grid = cg::this_grid();
  const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // (the candidate and fallback controls, ctl[1..2], are zeroed by the launch code:
  // with no grid barrier before the filter, blocks may append candidates at once)
  const SrcSample smp{f.keys, f.rows, f.n, f.w};
  constexpr int kGather = kRankMax / kSelThreads;  // all loads of a thread in flight together
  {  // sample keys (rows only if the threshold lands in a key tie, below)
    uint64_t h[kGather];
#pragma unroll
    for (int u = 0; u < kGather; ++u) {
      const uint32_t i = threadIdx.x + u * kSelThreads;
      if (i < f.s) h[u] = smp.hi(i);
    }
#pragma unroll
    for (int u = 0; u < kGather; ++u) {
      const uint32_t i = threadIdx.x + u * kSelThreads;
      if (i < f.s) s_hi[i] = h[u];
    }
  }
  __syncthreads();
  // every block selects the same threshold from the same samples: no grid barrier
  uint64_t t_hi;
  uint32_t t_lo;
  block_radix_threshold(s_hi, s_lo, f.s, f.need_s, &t_hi, &t_lo, [&]() {
    for (uint32_t i = threadIdx.x; i < f.s; i += blockDim.x) s_lo[i] = smp.lo(i);
    __syncthreads();
  });
  const double tk = key_from_ord(t_hi);
  const uint32_t tr = ~t_lo;
  if (gtid == 0) {
    f.ctl->thr_key = tk;
    f.ctl->thr_row = tr;
  }
  filter_body(f.keys, f.rows, f.n, tk, tr, &f.ctl[1].cand_count, f.cand_hi, f.cand_lo, f.cap);
  grid.sync();
  const unsigned long long c = __ldcg(&f.ctl[1].cand_count);
  if (gtid == 0 && f.host_count) *(volatile unsigned long long*)f.host_count = c;
  if (c >= f.need && c <= f.cap) {
    if (c <= f.rank_max) {
      uint64_t h[kGather];
      uint32_t l[kGather];
#pragma unroll
      for (int u = 0; u < kGather; ++u) {
        const uint32_t i = threadIdx.x + u * kSelThreads;
        if (i < c) {
          h[u] = __ldcg(f.cand_hi + i);
          l[u] = __ldcg(f.cand_lo + i);
        }
      }
#pragma unroll
      for (int u = 0; u < kGather; ++u) {
        const uint32_t i = threadIdx.x + u * kSelThreads;
        if (i < c) {
          s_hi[i] = h[u];
          s_lo[i] = l[u];
        }
      }
      __syncthreads();
      rank_items(s_hi, s_lo, (uint32_t)c, f.need, kModeFull, nullptr, f.out_rows, f.out_hi);
      return;
    }
    SelectArgs<SrcCand> a;
    a.src = SrcCand{f.cand_hi, f.cand_lo};
    a.n = c;
    a.need = f.need;
    a.cap = 0;
    a.use_cand_count = 0;
    a.mode = kModeFull;
    a.ctl = f.ctl + 1;
    a.w_hi = f.w_hi;
    a.w_lo = f.w_lo;
    a.out_rows = f.out_rows;
    a.out_hi = f.out_hi;
    a.host_status = nullptr;
    a.host_count = nullptr;
    __syncthreads();
    select_body(a);
    return;
  }
  if (gtid == 0 && f.host_status) *(volatile int*)f.host_status = 1;
  SelectArgs<SrcInput> a;
  a.src = SrcInput{f.keys, f.rows};
  a.n = f.n;
  a.need = f.need;
  a.cap = 0;
  a.use_cand_count = 0;
  a.mode = kModeFull;
  a.ctl = f.ctl + 2;
  a.w_hi = f.w_hi;
  a.w_lo = f.w_lo;
  a.out_rows = f.out_rows;
  a.out_hi = f.out_hi;
  a.host_status = nullptr;
  a.host_count = nullptr;
  __syncthreads();
  select_body(a);
}

}  // namespace golp
