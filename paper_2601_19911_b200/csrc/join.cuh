// Hash join build + probe over (key f64, row u32) pairs: the B200 replacement for
// host_hash_build / host_hash_probe and ProxyDevice.probe
// (pkg/src/golp/host.py:147-188, pkg/src/golp/device.py:262-296,382-436).
//
// Result contract (ProbeResult, pkg/src/golp/host.py:35-55; SPEC order): pairs
// (probe_row, build_row) for bit-equal key_bits, ordered by probe position, then
// by build insertion position.
//
// Layout in HBM:
//   table  : cap x 16 B slots {u64 key_bits, u32 off, u32 cnt}, one slot per
//            DISTINCT build key. Linear probing whose start is rounded down to an
//            even slot: the probe walks 32-byte, sector-aligned slot pairs, one
//            256-bit load per pair (LDG.E.256). cap = pow2 >= 2*nb (load <= 0.5).
//   csr_row: nb x u32, the build rows of every key group in build-position order;
//            groups of one keep their row inline in slot.off (no CSR access).
// Build: insert (atomicCAS) -> group offsets (warp-aggregated cursor) -> scatter
// build positions -> per-group sort of positions (thread / block / block-global)
// -> rows. Probe: match (one lookup per probe, compacted per warp tile) -> scan
// -> emit (see below).
#pragma once
#include <cooperative_groups.h>
#include "sortnet.cuh"

namespace golp {

struct __align__(16) Slot {
  uint64_t key;
  uint32_t off;
  uint32_t cnt;
};

// First slot of a key's probe sequence: an even slot, so the walk covers whole
// 32-byte slot pairs.
__host__ __device__ __forceinline__ uint64_t home_slot(uint64_t bits, uint64_t mask) {
  return mix64(bits) & mask & ~1ull;
}

constexpr int kSmallGroup = 32;        // groups up to this size sorted by their leader thread
constexpr uint32_t kGroupTile = 16384;  // groups up to this size sorted in shared memory (64 KB)

__global__ void join_init_table_kernel(Slot* __restrict__ table, uint64_t cap) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += stride) {
    reinterpret_cast<ulonglong2*>(table)[i] = make_ulonglong2(kEmptyKey, 0ull);
  }
}

// Build kernels process tiles of kBuildThreads*kBuildItems consecutive entries;
// each thread owns kBuildItems entries strided by the block size (coalesced),
// and issues their loads / atomics together so the dependent chains overlap.
constexpr int kBuildThreads = 256;
constexpr int kBuildItems = 4;
constexpr uint64_t kBuildTile = (uint64_t)kBuildThreads * kBuildItems;

__global__ void __launch_bounds__(kBuildThreads) join_insert_kernel(const double* __restrict__ bkeys, uint64_t nb,
                                                                    Slot* table, uint64_t mask,
                                                                    uint32_t* __restrict__ bslot,
                                                                    uint32_t* __restrict__ brank) {
  for (uint64_t t0 = (uint64_t)blockIdx.x * kBuildTile; t0 < nb; t0 += (uint64_t)gridDim.x * kBuildTile) {
    uint64_t b[kBuildItems];
    uint32_t h[kBuildItems];
    unsigned pending = 0;
#pragma unroll
    for (int j = 0; j < kBuildItems; ++j) {
      const uint64_t i = t0 + (uint64_t)j * kBuildThreads + threadIdx.x;
      b[j] = i < nb ? canon_bits(__ldg(bkeys + i)) : 0ull;
      h[j] = (uint32_t)home_slot(b[j], mask);
      if (i < nb) pending |= 1u << j;
    }
    unsigned valid = pending;
    // Claim or find each key's slot: CAS issued for every pending entry at once.
    while (pending) {
      unsigned long long old[kBuildItems];
#pragma unroll
      for (int j = 0; j < kBuildItems; ++j)
        if (pending & (1u << j))
          old[j] = atomicCAS(reinterpret_cast<unsigned long long*>(&table[h[j]].key), kEmptyKey,
                             (unsigned long long)b[j]);
#pragma unroll
      for (int j = 0; j < kBuildItems; ++j) {
        if (!(pending & (1u << j))) continue;
        if (old[j] == kEmptyKey || old[j] == b[j]) pending &= ~(1u << j);
        else h[j] = (h[j] + 1) & (uint32_t)mask;
      }
    }
    uint32_t r[kBuildItems];
#pragma unroll
    for (int j = 0; j < kBuildItems; ++j)
      if (valid & (1u << j)) r[j] = atomicAdd(&table[h[j]].cnt, 1u);
#pragma unroll
    for (int j = 0; j < kBuildItems; ++j) {
      const uint64_t i = t0 + (uint64_t)j * kBuildThreads + threadIdx.x;
      if (valid & (1u << j)) {
        bslot[i] = h[j];
        brank[i] = r[j];
      }
    }
  }
}

// One leader per group (rank 0) reserves the group's CSR range; groups of one
// keep their row inline in slot.off and reserve nothing.
__global__ void __launch_bounds__(kBuildThreads) join_offsets_kernel(uint64_t nb, Slot* table,
                                                                     const uint32_t* __restrict__ bslot,
                                                                     const uint32_t* __restrict__ brank,
                                                                     const uint32_t* __restrict__ brows,
                                                                     unsigned long long* cursor, uint32_t* big_list,
                                                                     unsigned int* big_count) {
  const unsigned lane = lane_id();
  for (uint64_t t0 = (uint64_t)blockIdx.x * kBuildTile; t0 < nb; t0 += (uint64_t)gridDim.x * kBuildTile) {
    uint32_t h[kBuildItems], cnt[kBuildItems], rk[kBuildItems];
#pragma unroll
    for (int j = 0; j < kBuildItems; ++j) {
      const uint64_t i = t0 + (uint64_t)j * kBuildThreads + threadIdx.x;
      rk[j] = i < nb ? brank[i] : 1u;
      h[j] = i < nb ? bslot[i] : 0u;
    }
#pragma unroll
    for (int j = 0; j < kBuildItems; ++j) cnt[j] = rk[j] == 0 ? table[h[j]].cnt : 0u;
#pragma unroll
    for (int j = 0; j < kBuildItems; ++j) {
      const uint64_t i = t0 + (uint64_t)j * kBuildThreads + threadIdx.x;
      if (cnt[j] == 1) table[h[j]].off = __ldg(brows + i);  // singleton: inline row
      const uint32_t need = cnt[j] > 1 ? cnt[j] : 0u;
      unsigned long long incl = need;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if ((int)lane >= o) incl += v;
      }
      unsigned long long base = 0;
      if (lane == 31 && incl) base = atomicAdd(cursor, incl);
      base = __shfl_sync(0xFFFFFFFFu, base, 31);
      if (need) {
        table[h[j]].off = (uint32_t)(base + incl - need);
        if (need > (uint32_t)kSmallGroup) big_list[atomicAdd(big_count, 1u)] = h[j];
      }
    }
  }
}

// Members of multi-entry groups scatter their build positions into the group's range.
__global__ void __launch_bounds__(kBuildThreads) join_fill_kernel(uint64_t nb, const Slot* __restrict__ table,
                                                                  const uint32_t* __restrict__ bslot,
                                                                  const uint32_t* __restrict__ brank,
                                                                  uint32_t* __restrict__ csr_pos) {
  for (uint64_t t0 = (uint64_t)blockIdx.x * kBuildTile; t0 < nb; t0 += (uint64_t)gridDim.x * kBuildTile) {
    uint32_t h[kBuildItems], rk[kBuildItems];
    uint2 oc[kBuildItems];
#pragma unroll
    for (int j = 0; j < kBuildItems; ++j) {
      const uint64_t i = t0 + (uint64_t)j * kBuildThreads + threadIdx.x;
      h[j] = i < nb ? bslot[i] : 0u;
      rk[j] = i < nb ? brank[i] : 0u;
    }
#pragma unroll
    for (int j = 0; j < kBuildItems; ++j) {
      const uint64_t i = t0 + (uint64_t)j * kBuildThreads + threadIdx.x;
      oc[j] = i < nb ? *reinterpret_cast<const uint2*>(&table[h[j]].off) : make_uint2(0, 1);
    }
#pragma unroll
    for (int j = 0; j < kBuildItems; ++j) {
      const uint64_t i = t0 + (uint64_t)j * kBuildThreads + threadIdx.x;
      if (i < nb && oc[j].y > 1) csr_pos[oc[j].x + rk[j]] = (uint32_t)i;
    }
  }
}

// Groups of 2..kSmallGroup: the leader sorts the positions and writes rows.
__global__ void __launch_bounds__(kBuildThreads) join_small_groups_kernel(uint64_t nb, const Slot* __restrict__ table,
                                                                          const uint32_t* __restrict__ bslot,
                                                                          const uint32_t* __restrict__ brank,
                                                                          const uint32_t* __restrict__ csr_pos,
                                                                          const uint32_t* __restrict__ brows,
                                                                          uint32_t* __restrict__ csr_row) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += stride) {
    if (brank[i] != 0) continue;
    const uint32_t h = bslot[i];
    const uint2 oc = *reinterpret_cast<const uint2*>(&table[h].off);
    const uint32_t cnt = oc.y;
    if (cnt < 2 || cnt > (uint32_t)kSmallGroup) continue;
    const uint32_t off = oc.x;
    if (cnt == 2) {  // the common case: one compare
      const uint32_t a = csr_pos[off], b = csr_pos[off + 1];
      const uint32_t lo = a < b ? a : b, hi = a < b ? b : a;
      csr_row[off] = __ldg(brows + lo);
      csr_row[off + 1] = __ldg(brows + hi);
      continue;
    }
    uint32_t p[kSmallGroup];
    for (uint32_t m = 0; m < cnt; ++m) {
      const uint32_t v = csr_pos[off + m];
      uint32_t q = m;
      while (q > 0 && p[q - 1] > v) { p[q] = p[q - 1]; --q; }
      p[q] = v;
    }
    for (uint32_t m = 0; m < cnt; ++m) csr_row[off + m] = __ldg(brows + p[m]);
  }
}

// Groups > kSmallGroup: one block per group; shared-memory sort up to kGroupTile,
// in-place global network beyond (pathological duplicate counts only).
__global__ void __launch_bounds__(1024) join_big_groups_kernel(const Slot* __restrict__ table,
                                                               const uint32_t* __restrict__ big_list,
                                                               const unsigned int* __restrict__ big_count,
                                                               uint32_t* csr_pos, const uint32_t* __restrict__ brows,
                                                               uint32_t* __restrict__ csr_row) {
  extern __shared__ __align__(16) uint32_t s_pos[];
  const unsigned nbig = *big_count;
  for (unsigned g = blockIdx.x; g < nbig; g += gridDim.x) {
    const uint32_t h = big_list[g];
    const uint32_t cnt = table[h].cnt;
    const uint32_t off = table[h].off;
    if (cnt <= kGroupTile) {
      for (uint32_t m = threadIdx.x; m < cnt; m += blockDim.x) s_pos[m] = csr_pos[off + m];
      __syncthreads();
      block_sort_asc_u32<false>(s_pos, cnt);
      for (uint32_t m = threadIdx.x; m < cnt; m += blockDim.x) csr_row[off + m] = __ldg(brows + s_pos[m]);
    } else {
      block_sort_asc_u32<true>(csr_pos + off, cnt);
      for (uint32_t m = threadIdx.x; m < cnt; m += blockDim.x) csr_row[off + m] = __ldg(brows + __ldcg(csr_pos + off + m));
    }
    __syncthreads();
  }
}

// ---- probe ------------------------------------------------------------------------
// Bound by random table lookups: ~1 L1TEX wavefront per lookup, ~0.8/clk/SM
// from L2 (tools/microbench.cu, tools/probe_ladder.cu). Every probe key is looked
// up exactly once:
//   match : each block walks a contiguous range of warp tiles (32*kWarpItems
//           consecutive probes); a warp resolves its probes (linear probing over
//           32-byte slot pairs) and
//           compacts the hits, in probe order, into the tile's scratch segment as
//           8-byte entries {slot.off, slot.cnt << 8 | position in tile};
//           per-tile entry / pair counts and the block's pair total are written.
//   scan  : one block scans the per-block totals (+ pairs of earlier launches).
//   emit  : same block -> tile-range mapping; a block scan of the tiles' pair
//           counts gives each tile's output offset; warps expand entries to
//           (probe row, build row) pairs.
// Output order = probe position, then CSR (build insertion) order.
#ifndef GOLP_WARP_ITEMS
#define GOLP_WARP_ITEMS 2
#endif
#ifndef GOLP_PROBE_MINB
#define GOLP_PROBE_MINB 6
#endif
constexpr int kWarpItems = GOLP_WARP_ITEMS;
constexpr uint32_t kWarpTile = 32 * kWarpItems;  // probes per warp tile
static_assert(kWarpTile <= 256, "entry position is 8 bits");
constexpr int kProbeThreads = 256;
constexpr uint32_t kMaxTilesPerBlock = 4096;
constexpr uint32_t kMaxGroup = (1u << 24) - 1;  // largest key group an entry can describe

// L2 eviction policies: the table should survive the probe stream in L2, the
// streamed probe columns should not displace it.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Both slots of a 32-byte aligned pair in one 256-bit load (LDG.E.ENL2.256).
__device__ __forceinline__ ulonglong4 ldg_pair(const Slot* s, uint64_t pol) {
  ulonglong4 r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u64 {%0, %1, %2, %3}, [%4], %5;"
               : "=l"(r.x), "=l"(r.y), "=l"(r.z), "=l"(r.w)
               : "l"(s), "l"(pol));
  return r;
}
__device__ __forceinline__ double2 ldg_stream_d2(const double* p, uint64_t pol) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint4 ldg_stream_u4(const uint32_t* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

// ---- block scan helpers ----------------------------------------------------------
constexpr int kScanThreads = 1024;

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

// One block: exclusive scan of the partials, offset by *base_in; writes *total_out.
__global__ void __launch_bounds__(kScanThreads) scan_partials_kernel(unsigned long long* partial, uint32_t nparts,
                                                                     const unsigned long long* base_in,
                                                                     unsigned long long* total_out) {
  __shared__ unsigned long long s_w[33];
  unsigned long long carry = *base_in;
  for (uint32_t b0 = 0; b0 < nparts; b0 += blockDim.x) {
    const uint32_t i = b0 + threadIdx.x;
    const unsigned long long v = i < nparts ? partial[i] : 0ull;
    unsigned long long tot;
    const unsigned long long e = block_excl_scan(v, s_w, &tot);
    if (i < nparts) partial[i] = carry + e;
    carry += tot;
  }
  if (threadIdx.x == 0) *total_out = carry;
}

__device__ __forceinline__ void st_hint(uint32_t* p, uint32_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}

// Checks one slot pair: 1 = found (off/cnt set), 0 = absent, -1 = continue at h+2.
__device__ __forceinline__ int check_pair(const ulonglong4& sl, uint64_t bits, uint32_t& off, uint32_t& cnt) {
  if (sl.x == bits) { off = (uint32_t)sl.y; cnt = (uint32_t)(sl.y >> 32); return 1; }
  if (sl.x == kEmptyKey) return 0;
  if (sl.z == bits) { off = (uint32_t)sl.w; cnt = (uint32_t)(sl.w >> 32); return 1; }
  if (sl.z == kEmptyKey) return 0;
  return -1;
}

struct MatchScratch {
  uint2* entry;      // kWarpTile per warp tile: {slot.off, cnt << 8 | pos}
  uint32_t* nmatch;  // per warp tile
  uint32_t* npairs;  // per warp tile
};

__global__ void __launch_bounds__(kProbeThreads, GOLP_PROBE_MINB) join_match_kernel(
    const double* __restrict__ pkeys, uint64_t np, const Slot* __restrict__ table, uint64_t mask, MatchScratch sc,
    uint64_t nwt, uint64_t per_block, unsigned long long* __restrict__ bpart, unsigned int* __restrict__ flags) {
  __shared__ unsigned long long s_w[kProbeThreads / 32];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  constexpr unsigned kWarps = kProbeThreads / 32;
  const uint64_t pol_stream = policy_evict_first(), pol_table = policy_evict_last();
  const uint64_t lo = blockIdx.x * per_block, hi = lo + per_block < nwt ? lo + per_block : nwt;
  const uint32_t pm = (uint32_t)mask;
  unsigned long long mine = 0;
  for (uint64_t wt = lo + warp; wt < hi; wt += kWarps) {
    const uint64_t first = wt * kWarpTile + lane * kWarpItems;
    double k[kWarpItems];
    if (first + kWarpItems <= np && (((uintptr_t)(pkeys + first) & 15) == 0)) {
#pragma unroll
      for (int j = 0; j < kWarpItems; j += 2) {
        const double2 v = ldg_stream_d2(pkeys + first + j, pol_stream);
        k[j] = v.x;
        k[j + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < kWarpItems; ++j) k[j] = first + j < np ? pkeys[first + j] : 0.0;
    }
    uint64_t bits[kWarpItems];
    uint32_t h[kWarpItems], off[kWarpItems], cnt[kWarpItems];
    unsigned pending = 0;
#pragma unroll
    for (int j = 0; j < kWarpItems; ++j) {
      bits[j] = canon_bits(k[j]);
      h[j] = (uint32_t)home_slot(bits[j], mask);
      off[j] = 0;
      cnt[j] = 0;
      if (first + j < np) pending |= 1u << j;
    }
    while (pending) {
      ulonglong4 sl[kWarpItems];
#pragma unroll
      for (int j = 0; j < kWarpItems; ++j)
        if (pending & (1u << j)) sl[j] = ldg_pair(table + h[j], pol_table);
#pragma unroll
      for (int j = 0; j < kWarpItems; ++j) {
        if (!(pending & (1u << j))) continue;
        const int st = check_pair(sl[j], bits[j], off[j], cnt[j]);
        if (st >= 0) pending &= ~(1u << j);
        else h[j] = (h[j] + 2) & pm;
      }
    }
    uint32_t nm = 0, npr = 0;
#pragma unroll
    for (int j = 0; j < kWarpItems; ++j) {
      nm += cnt[j] != 0;
      npr += cnt[j];
    }
    uint32_t incl = nm;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if ((int)lane >= o) incl += v;
    }
    uint32_t pairs = npr;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pairs += __shfl_xor_sync(0xFFFFFFFFu, pairs, o);
    mine += pairs;
    if (lane == 31) {
      sc.nmatch[wt] = incl;
      sc.npairs[wt] = pairs;
    }
    uint64_t o = wt * kWarpTile + (incl - nm);
#pragma unroll
    for (int j = 0; j < kWarpItems; ++j) {
      if (cnt[j]) {
        if (cnt[j] > kMaxGroup) atomicOr(flags, 1u);  // host re-runs without the packed entry
        sc.entry[o++] = make_uint2(off[j], (cnt[j] << 8) | (lane * kWarpItems + j));
      }
    }
  }
  if (lane == 0) s_w[warp] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (unsigned w = 0; w < kWarps; ++w) t += s_w[w];
    bpart[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kProbeThreads) join_emit_kernel(MatchScratch sc, const uint32_t* __restrict__ prows,
                                                                  const uint32_t* __restrict__ csr_row, uint64_t nwt,
                                                                  uint64_t per_block,
                                                                  const unsigned long long* __restrict__ bpart,
                                                                  uint32_t* __restrict__ out_p,
                                                                  uint32_t* __restrict__ out_b, uint64_t cap) {
  __shared__ unsigned long long s_off[kMaxTilesPerBlock];
  __shared__ unsigned long long s_w[33];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  constexpr unsigned kWarps = kProbeThreads / 32;
  const uint64_t lo = blockIdx.x * per_block, hi = lo + per_block < nwt ? lo + per_block : nwt;
  if (lo >= hi) return;
  const uint32_t n = (uint32_t)(hi - lo);
  unsigned long long carry = bpart[blockIdx.x];
  for (uint32_t b0 = 0; b0 < n; b0 += kProbeThreads) {
    const uint32_t i = b0 + threadIdx.x;
    const unsigned long long v = i < n ? sc.npairs[lo + i] : 0ull;
    unsigned long long t;
    const unsigned long long e = block_excl_scan(v, s_w, &t);
    if (i < n) s_off[i] = carry + e;
    carry += t;
  }
  __syncthreads();
  const uint64_t pol_stream = policy_evict_first();
  for (uint64_t t = lo + warp; t < hi; t += kWarps) {
    const uint32_t nm = sc.nmatch[t];
    if (nm == 0) continue;
    unsigned long long run = s_off[t - lo];
    const uint64_t e0 = t * kWarpTile;
    for (uint32_t i0 = 0; i0 < nm; i0 += 32) {
      const uint32_t i = i0 + lane;
      uint32_t c = 0, pr = 0, of = 0;
      if (i < nm) {
        const uint2 en = __ldcs(sc.entry + e0 + i);
        of = en.x;
        c = en.y >> 8;
        pr = __ldg(prows + e0 + (en.y & 255u));
      }
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if ((int)lane >= o) incl += v;
      }
      const uint32_t gtot = __shfl_sync(0xFFFFFFFFu, incl, 31);
      // singletons (slot.off is the build row) land at consecutive positions;
      // the rare multi-match entries expand their CSR run serially
      unsigned long long g = run + (incl - c);
      if (c == 1) {
        if (g < cap) {
          st_hint(out_p + g, pr, pol_stream);
          st_hint(out_b + g, of, pol_stream);
        }
      } else {
        for (uint32_t m = 0; m < c; ++m, ++g)
          if (g < cap) {
            st_hint(out_p + g, pr, pol_stream);
            st_hint(out_b + g, __ldg(csr_row + of + m), pol_stream);
          }
      }
      run += gtot;
    }
  }
}

}  // namespace golp
