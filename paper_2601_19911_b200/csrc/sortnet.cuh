// Bitonic sorting networks in the "flip" formulation: every compare-exchange
// moves the better element to the lower index, so a virtual tail padded with
// worst-possible elements never moves and arbitrary (non power-of-two) lengths
// sort in place without padding.
//
//   for k = 2, 4, ..., P:            (P = next power of two >= n)
//     flip  : i = blk*k + off, j = blk*k + k-1-off      (off < k/2)
//     for s = k/4 ... 1 : i = 2t - (t & (s-1)), j = i + s
//   skip every pair with j >= n.
#pragma once
#include "common.cuh"

namespace golp {

__host__ __device__ __forceinline__ uint64_t next_pow2_u64(uint64_t n) {
  uint64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

__device__ __forceinline__ int ilog2_u64(uint64_t p) { return 63 - __clzll((long long)p); }

// pair index t -> (i, j) for the flip step of a k-merge
__device__ __forceinline__ void flip_pair(uint64_t t, int logk, uint64_t& i, uint64_t& j) {
  const uint64_t half = 1ull << (logk - 1);
  const uint64_t blk = t >> (logk - 1);
  const uint64_t off = t & (half - 1);
  i = (blk << logk) + off;
  j = (blk << logk) + (1ull << logk) - 1 - off;
}

// pair index t -> (i, j) for a half-cleaner step of stride s
__device__ __forceinline__ void half_pair(uint64_t t, int logs, uint64_t& i, uint64_t& j) {
  const uint64_t s = 1ull << logs;
  i = 2 * t - (t & (s - 1));
  j = i + s;
}

// ---- composite (hi, lo) items, descending ("better" first) -------------------

__device__ __forceinline__ void cx_desc(uint64_t* h, uint32_t* l, uint64_t i, uint64_t j) {
  const uint64_t hi = h[i], hj = h[j];
  const uint32_t li = l[i], lj = l[j];
  if (item_gt(hj, lj, hi, li)) {
    h[i] = hj; h[j] = hi;
    l[i] = lj; l[j] = li;
  }
}

// Full sort of `n` live items held in shared memory by one block.
__device__ void block_sort_desc(uint64_t* h, uint32_t* l, uint32_t n) {
  if (n < 2) return;
  const int logP = ilog2_u64(next_pow2_u64(n));
  const uint32_t pairs = (1u << logP) >> 1;
  for (int logk = 1; logk <= logP; ++logk) {
    for (uint32_t t = threadIdx.x; t < pairs; t += blockDim.x) {
      uint64_t i, j;
      flip_pair(t, logk, i, j);
      if (j < n) cx_desc(h, l, i, j);
    }
    __syncthreads();
    for (int logs = logk - 2; logs >= 0; --logs) {
      for (uint32_t t = threadIdx.x; t < pairs; t += blockDim.x) {
        uint64_t i, j;
        half_pair(t, logs, i, j);
        if (j < n) cx_desc(h, l, i, j);
      }
      __syncthreads();
    }
  }
}

// Half-cleaner steps s = 2^(logs_hi) ... 1 on a tile (used after global steps).
__device__ void block_half_steps_desc(uint64_t* h, uint32_t* l, uint32_t n, int logs_hi, uint32_t tile_pairs) {
  for (int logs = logs_hi; logs >= 0; --logs) {
    for (uint32_t t = threadIdx.x; t < tile_pairs; t += blockDim.x) {
      uint64_t i, j;
      half_pair(t, logs, i, j);
      if (j < n) cx_desc(h, l, i, j);
    }
    __syncthreads();
  }
}

// ---- u32 ascending (build positions inside a join group) ---------------------

__device__ __forceinline__ void cx_asc_u32(uint32_t* a, uint64_t i, uint64_t j) {
  const uint32_t x = a[i], y = a[j];
  if (y < x) { a[i] = y; a[j] = x; }
}

__device__ __forceinline__ void cx_asc_u32_cg(uint32_t* a, uint64_t i, uint64_t j) {
  const uint32_t x = __ldcg(a + i), y = __ldcg(a + j);
  if (y < x) { __stcg(a + i, y); __stcg(a + j, x); }
}

// One block sorts a[0..n) ascending. kGlobal selects L2-coherent accesses for
// arrays that live in global memory.
template <bool kGlobal>
__device__ void block_sort_asc_u32(uint32_t* a, uint64_t n) {
  if (n < 2) return;
  const int logP = ilog2_u64(next_pow2_u64(n));
  const uint64_t pairs = (1ull << logP) >> 1;
  for (int logk = 1; logk <= logP; ++logk) {
    for (uint64_t t = threadIdx.x; t < pairs; t += blockDim.x) {
      uint64_t i, j;
      flip_pair(t, logk, i, j);
      if (j < n) { if (kGlobal) cx_asc_u32_cg(a, i, j); else cx_asc_u32(a, i, j); }
    }
    __syncthreads();
    for (int logs = logk - 2; logs >= 0; --logs) {
      for (uint64_t t = threadIdx.x; t < pairs; t += blockDim.x) {
        uint64_t i, j;
        half_pair(t, logs, i, j);
        if (j < n) { if (kGlobal) cx_asc_u32_cg(a, i, j); else cx_asc_u32(a, i, j); }
      }
      __syncthreads();
    }
  }
}

}  // namespace golp
