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
//            DISTINCT build key, linear probing on mix64(bits) & (cap-1), load <= 0.5.
//   csr_row: nb x u32, the build rows of every key group in build-position order;
//            groups of one keep their row inline in slot.off (no CSR access).
// Build: insert (atomicCAS) -> group offsets (warp-aggregated cursor) -> scatter
// build positions -> per-group sort of positions (thread / block / block-global)
// -> rows. Probe: one single-pass kernel, 2048 probes per tile: probe the table,
// block scan of match counts, decoupled look-back for the tile's output offset,
// emit pairs in probe order.
#pragma once
#include "sortnet.cuh"

namespace golp {

struct __align__(16) Slot {
  uint64_t key;
  uint32_t off;
  uint32_t cnt;
};

constexpr int kSmallGroup = 32;        // groups up to this size sorted by their leader thread
constexpr uint32_t kGroupTile = 16384;  // groups up to this size sorted in shared memory (64 KB)

__global__ void join_init_table_kernel(Slot* __restrict__ table, uint64_t cap) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += stride) {
    reinterpret_cast<ulonglong2*>(table)[i] = make_ulonglong2(kEmptyKey, 0ull);
  }
}

__global__ void join_insert_kernel(const double* __restrict__ bkeys, uint64_t nb, Slot* table, uint64_t mask,
                                   uint32_t* __restrict__ bslot, uint32_t* __restrict__ brank) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += stride) {
    const uint64_t b = canon_bits(__ldg(bkeys + i));
    uint64_t h = mix64(b) & mask;
    while (true) {
      unsigned long long* kp = reinterpret_cast<unsigned long long*>(&table[h].key);
      const unsigned long long k = *(volatile unsigned long long*)kp;
      if (k == b) break;
      if (k == kEmptyKey) {
        const unsigned long long old = atomicCAS(kp, kEmptyKey, (unsigned long long)b);
        if (old == kEmptyKey || old == b) break;
      }
      h = (h + 1) & mask;
    }
    const uint32_t r = atomicAdd(&table[h].cnt, 1u);
    bslot[i] = (uint32_t)h;
    brank[i] = r;
  }
}

// One leader per group (rank 0) reserves the group's CSR range.
__global__ void join_offsets_kernel(uint64_t nb, Slot* table, const uint32_t* __restrict__ bslot,
                                    const uint32_t* __restrict__ brank, unsigned long long* cursor,
                                    uint32_t* big_list, unsigned int* big_count) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const unsigned lane = lane_id();
  for (uint64_t wb = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x - lane; wb < nb; wb += stride) {
    const uint64_t i = wb + lane;
    uint32_t h = 0, cnt = 0;
    const bool leader = i < nb && brank[i] == 0;
    if (leader) {
      h = bslot[i];
      cnt = table[h].cnt;
    }
    unsigned long long incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if ((int)lane >= o) incl += v;
    }
    unsigned long long base = 0;
    if (lane == 31 && incl) base = atomicAdd(cursor, incl);
    base = __shfl_sync(0xFFFFFFFFu, base, 31);
    if (leader) {
      table[h].off = (uint32_t)(base + incl - cnt);
      if (cnt > (uint32_t)kSmallGroup) big_list[atomicAdd(big_count, 1u)] = h;
    }
  }
}

__global__ void join_fill_kernel(uint64_t nb, const Slot* __restrict__ table, const uint32_t* __restrict__ bslot,
                                 const uint32_t* __restrict__ brank, uint32_t* __restrict__ csr_pos) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += stride) {
    csr_pos[table[bslot[i]].off + brank[i]] = (uint32_t)i;
  }
}

// Groups of <= kSmallGroup: the leader sorts the positions and writes rows.
// Groups of one keep the row inline in slot.off.
__global__ void join_small_groups_kernel(uint64_t nb, Slot* table, const uint32_t* __restrict__ bslot,
                                         const uint32_t* __restrict__ brank, const uint32_t* __restrict__ csr_pos,
                                         const uint32_t* __restrict__ brows, uint32_t* __restrict__ csr_row) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += stride) {
    if (brank[i] != 0) continue;
    const uint32_t h = bslot[i];
    const uint32_t cnt = table[h].cnt;
    if (cnt == 1) {
      table[h].off = __ldg(brows + i);
      continue;
    }
    if (cnt > (uint32_t)kSmallGroup) continue;
    const uint32_t off = table[h].off;
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
constexpr int kProbeThreads = 256;
constexpr int kProbeItems = 8;
constexpr uint32_t kProbeTile = kProbeThreads * kProbeItems;  // 2048 probes
constexpr unsigned long long kFlagA = 1ull << 62;  // tile aggregate published
constexpr unsigned long long kFlagP = 2ull << 62;  // inclusive prefix published
constexpr unsigned long long kValMask = (1ull << 62) - 1;

struct ProbeArgs {
  const double* pkeys;
  const uint32_t* prows;
  uint64_t np;
  const Slot* table;
  uint64_t mask;
  const uint32_t* csr_row;
  uint32_t* out_p;
  uint32_t* out_b;
  uint64_t cap;
  unsigned long long* tile_status;  // ntiles entries, zeroed
  unsigned int* tile_counter;       // zeroed
  const unsigned long long* base_in;  // pairs emitted before this launch
  unsigned long long* total_out;      // base_in + pairs of this launch
  uint64_t ntiles;
};

__device__ __forceinline__ ulonglong2 ldg_slot(const Slot* s) {
  ulonglong2 r;
  asm volatile("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(s));
  return r;
}

__global__ void __launch_bounds__(kProbeThreads) join_probe_kernel(ProbeArgs a) {
  __shared__ unsigned s_tile;
  __shared__ unsigned long long s_warp[kProbeThreads / 32];
  __shared__ unsigned long long s_base;
  if (threadIdx.x == 0) s_tile = atomicAdd(a.tile_counter, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t first = tile * kProbeTile + (uint64_t)threadIdx.x * kProbeItems;

  double k[kProbeItems];
  const bool full = first + kProbeItems <= a.np && (((uintptr_t)(a.pkeys + first) & 15) == 0);
  if (full) {
#pragma unroll
    for (int j = 0; j < kProbeItems; j += 2) {
      const double2 v = ldg_nc_d2(a.pkeys + first + j);
      k[j] = v.x;
      k[j + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kProbeItems; ++j) k[j] = (first + j < a.np) ? a.pkeys[first + j] : 0.0;
  }
  uint64_t bits[kProbeItems];
  uint64_t h[kProbeItems];
  ulonglong2 s[kProbeItems];
#pragma unroll
  for (int j = 0; j < kProbeItems; ++j) {
    bits[j] = canon_bits(k[j]);
    h[j] = mix64(bits[j]) & a.mask;
  }
#pragma unroll
  for (int j = 0; j < kProbeItems; ++j) s[j] = ldg_slot(a.table + h[j]);
  uint32_t off[kProbeItems], cnt[kProbeItems];
  unsigned long long total = 0;
#pragma unroll
  for (int j = 0; j < kProbeItems; ++j) {
    cnt[j] = 0;
    off[j] = 0;
    if (first + j < a.np) {
      ulonglong2 sl = s[j];
      uint64_t hh = h[j];
      while (sl.x != bits[j] && sl.x != kEmptyKey) {
        hh = (hh + 1) & a.mask;
        sl = ldg_slot(a.table + hh);
      }
      if (sl.x == bits[j]) {
        off[j] = (uint32_t)sl.y;
        cnt[j] = (uint32_t)(sl.y >> 32);
      }
    }
    total += cnt[j];
  }

  // block-wide exclusive scan of per-thread match totals
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  unsigned long long incl = total;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if ((int)lane >= o) incl += v;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < kProbeThreads / 32 ? s_warp[lane] : 0ull;
    unsigned long long wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if ((int)lane >= o) wi += v;
    }
    if (lane < kProbeThreads / 32) s_warp[lane] = wi - w;  // exclusive warp offsets
    const unsigned long long tile_total = __shfl_sync(0xFFFFFFFFu, wi, kProbeThreads / 32 - 1);
    if (lane == 0) {
      // decoupled look-back (single-pass prefix scan over tiles)
      volatile unsigned long long* st = a.tile_status;
      unsigned long long excl;
      if (tile == 0) {
        excl = *a.base_in;
        st[0] = kFlagP | ((excl + tile_total) & kValMask);
      } else {
        st[tile] = kFlagA | (tile_total & kValMask);
        excl = 0;
        int64_t pred = (int64_t)tile - 1;
        while (true) {
          const unsigned long long v = st[pred];
          if ((v >> 62) == 0) continue;  // not yet published
          excl += v & kValMask;
          if ((v >> 62) == 2) break;
          --pred;
        }
        __threadfence();
        st[tile] = kFlagP | ((excl + tile_total) & kValMask);
      }
      if (tile == a.ntiles - 1) *a.total_out = excl + tile_total;
      s_base = excl;
    }
  }
  __syncthreads();
  unsigned long long o = s_base + s_warp[warp] + (incl - total);
#pragma unroll
  for (int j = 0; j < kProbeItems; ++j) {
    if (cnt[j] == 0) continue;
    const uint32_t pr = __ldg(a.prows + first + j);
    if (cnt[j] == 1) {
      if (o < a.cap) { a.out_p[o] = pr; a.out_b[o] = off[j]; }
      ++o;
    } else {
      for (uint32_t m = 0; m < cnt[j]; ++m, ++o) {
        if (o < a.cap) { a.out_p[o] = pr; a.out_b[o] = __ldg(a.csr_row + off[j] + m); }
      }
    }
  }
}

}  // namespace golp
