// Shared device helpers for the B200 Top-K / hash-join path.
//
// Key semantics follow the reference exactly:
//   * keys are float64 (KeyVector coerces to <f8, reference pkg/src/golp/store.py:85);
//   * ordering is float ordering, so -0.0 ties +0.0 and the tie breaks by row id
//     (host_topk, pkg/src/golp/host.py:133-144);
//   * hash identity is key_bits = (key + 0.0).view(u64), which folds -0.0 onto +0.0
//     (pkg/src/golp/host.py:58-60), hashed with the splitmix64 finaliser mix64
//     (pkg/src/golp/host.py:63-80).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace golp {

constexpr uint64_t kSignBit = 0x8000000000000000ull;
// Slot sentinel: an all-ones bit pattern is a NaN, and KeyVector rejects NaN keys
// (pkg/src/golp/store.py:89-90), so no canonical key can ever collide with it.
constexpr uint64_t kEmptyKey = 0xFFFFFFFFFFFFFFFFull;
constexpr uint32_t kNoRow = 0xFFFFFFFFu;

__host__ __device__ __forceinline__ uint64_t canon_bits(double k) {
#ifdef __CUDA_ARCH__
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(k));
#else
  uint64_t b;
  __builtin_memcpy(&b, &k, 8);
#endif
  return b == kSignBit ? 0ull : b;  // -0.0 -> +0.0
}

// Order-preserving map of a finite double onto u64: a < b (as doubles, with
// -0 == +0) <=> ord(a) < ord(b).
__host__ __device__ __forceinline__ uint64_t ord_bits(uint64_t b) {
  return (b & kSignBit) ? ~b : (b | kSignBit);
}
__host__ __device__ __forceinline__ uint64_t ord_key(double k) { return ord_bits(canon_bits(k)); }

// Inverse of ord_key, clamped so that any u64 at or below ord(-inf) decodes to
// -inf (a prefix with zeroed low bits can otherwise land in the NaN range).
__host__ __device__ __forceinline__ double key_from_ord(uint64_t u) {
  constexpr uint64_t kOrdNegInf = 0x000FFFFFFFFFFFFFull;  // ~bits(-inf)
  uint64_t b;
  if (u <= kOrdNegInf) {
    b = 0xFFF0000000000000ull;  // -inf
  } else {
    b = (u & kSignBit) ? (u & ~kSignBit) : ~u;
  }
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(b));
#else
  double d;
  __builtin_memcpy(&d, &b, 8);
  return d;
#endif
}

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

// 32-bit integer hash for sample jitter (not part of any reference semantics).
__host__ __device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// Composite Top-K item: hi = ord(key), lo = ~row. "Better" = larger (hi, lo),
// i.e. larger key first, then smaller row id (pkg/src/golp/host.py:141).
struct Item {
  uint64_t hi;
  uint32_t lo;
};

#ifdef __CUDACC__
__device__ __forceinline__ bool item_gt(uint64_t ah, uint32_t al, uint64_t bh, uint32_t bl) {
  return ah > bh || (ah == bh && al > bl);
}

// A row-id column: the caller's array, or (rows == nullptr) the positions themselves,
// base + i -- the row ids extract_keys gives a table's key vector
// (pkg/src/golp/store.py:178-181), which then need no HBM column and no loads.
struct RowCol {
  const uint32_t* rows;
  uint32_t base;
  __device__ __forceinline__ uint32_t at(uint64_t i) const { return rows ? __ldg(rows + i) : base + (uint32_t)i; }
  // streaming (evict-first) load: a column read once
  __device__ __forceinline__ uint32_t at_cs(uint64_t i) const { return rows ? __ldcs(rows + i) : base + (uint32_t)i; }
  __host__ __device__ __forceinline__ RowCol from(uint64_t c) const {
    return rows ? RowCol{rows + c, 0} : RowCol{nullptr, base + (uint32_t)c};
  }
};

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// Warp-aggregated append: every lane with `take` gets a unique slot in [base, base+popc).
__device__ __forceinline__ unsigned long long warp_append(unsigned long long* counter, bool take) {
  const unsigned mask = __ballot_sync(0xFFFFFFFFu, take);
  if (mask == 0) return 0;
  const unsigned lane = lane_id();
  const int leader = __ffs(mask) - 1;
  unsigned long long base = 0;
  if ((int)lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(mask));
  base = __shfl_sync(0xFFFFFFFFu, base, leader);
  return base + __popc(mask & ((1u << lane) - 1u));
}

// Block-wide exclusive scan (blockDim <= 1024; every thread must call it).
__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v, unsigned long long* s_w,
                                                              unsigned long long* total) {
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  unsigned long long incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if ((int)lane >= o) incl += u;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long w = lane < (blockDim.x >> 5) ? s_w[lane] : 0ull;
    unsigned long long wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long u = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if ((int)lane >= o) wi += u;
    }
    if (lane < (blockDim.x >> 5)) s_w[lane] = wi - w;
    if (lane == 31) s_w[32] = wi;
  }
  __syncthreads();
  const unsigned long long r = s_w[warp] + incl - v;
  *total = s_w[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ double2 ldg_nc_d2(const double* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
#endif  // __CUDACC__

}  // namespace golp
