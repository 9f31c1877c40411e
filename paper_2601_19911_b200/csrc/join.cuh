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
//            256-bit load per pair (LDG.E.256). cap = pow2 >= 2*nb (load <= 0.5),
//            doubled once more while the table stays within 64 MB (L2-resident).
//   rows   : cap*kInline + nb u32: groups of 2..kInline keep their rows at
//            h*kInline, bigger groups a CSR range after that, all in build-position
//            order; groups of one keep their row inline in slot.off.
// Build: insert (atomicCAS claim, atomicAdd rank, first kInline positions into a
// slot-indexed side array) -> one pass over the slots finalizes every group ->
// overflow members and big-group sorts (rare). Probe: match (one lookup per probe, compacted per warp tile) -> scan
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
// Same for a 32-bit mask (tables are at most 2^32 slots).
__host__ __device__ __forceinline__ uint32_t home_slot32(uint64_t bits, uint32_t mask) {
  return (uint32_t)mix64(bits) & mask & ~1u;
}


// Key groups. Inserting claims an empty slot with one 16-byte CAS that writes
// {key, off = position, cnt = 1}, so a key's first member needs no second atomic
// and no side-array write; later members take rank = atomicAdd(cnt) and record
// ranks 1..kInline-1 in a slot-indexed side array (rows[h*kInline + rank]),
// higher ranks in an overflow list. One pass over the slots then finalizes each
// group:
//   cnt == 1        slot.off = the build row (probe reads no side array)
//   2..kInline      positions sorted and turned into rows at rows[h*kInline..]; slot.off = h*kInline
//   > kInline       a CSR range [off, off+cnt) after the side array; members of
//                   rank >= kInline come from the overflow list; sorted afterwards
// so no per-entry slot/rank arrays and no offset/fill/sort chain are needed for
// the common (small) groups. Probe: cnt >= 2 reads rows[off + m].

// 16-byte compare-and-swap (sm_90+): returns the slot's previous contents.
__device__ __forceinline__ ulonglong2 cas128(void* addr, ulonglong2 cmp, ulonglong2 val) {
  ulonglong2 old;
  asm volatile(
      "{\n\t.reg .b128 c, v, d;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 v, {%4, %5};\n\t"
      "atom.global.cas.b128 d, [%6], c, v;\n\t"
      "mov.b128 {%0, %1}, d;\n\t}"
      : "=l"(old.x), "=l"(old.y)
      : "l"(cmp.x), "l"(cmp.y), "l"(val.x), "l"(val.y), "l"(addr)
      : "memory");
  return old;
}

constexpr uint32_t kInline = 4;

// Home-pair overflow flag: bit 31 of the cnt word of a pair's FIRST slot is set
// when some key whose home is that pair had to be stored further on (the pair
// was full when it arrived). Keys are only ever inserted, so a probe whose key
// is not in its home pair can stop there unless the flag is set: most misses
// resolve in one lookup even when the home pair is full. Group sizes stay
// below 2^30 (join_build_impl's capacity check), so the bit is free; every
// reader of cnt masks it.
constexpr uint32_t kOverflowBit = 1u << 31;
constexpr uint32_t kCntMask = kOverflowBit - 1u;
// Two-member groups whose second row fits 30 bits live in the slot itself:
// off = first row, cnt word = kPair2Bit | second row (probe/emit read no side
// array for them; most groups have two members). Other counts stay below 2^30.
constexpr uint32_t kPair2Bit = 1u << 30;
constexpr uint32_t kPair2Row = kPair2Bit - 1u;
// Members of a slot's key from its cnt word (overflow flag already masked off).
__host__ __device__ __forceinline__ uint32_t slot_members(uint32_t cw) { return (cw & kPair2Bit) ? 2u : cw; }
constexpr uint32_t kGroupTile = 16384;  // big groups up to this size sorted in shared memory (64 KB)

// Empties the table (and the group bitmap) and settles the build row column's
// density flag *nd (0 = dense): mode 0 checks the column (*nd is 0 on entry and
// is set on a mismatch), 1 = declared dense, 2 = not dense (unchecked). The
// flag word of the next build, *nd_next, is cleared here, so no separate
// memset is needed before its check.
__device__ __forceinline__ bool rows_not_dense(const uint32_t* __restrict__ rows, uint64_t n) {
  const uint32_t b0 = rows[0];
  bool bad = false;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t n4 = ((reinterpret_cast<uintptr_t>(rows) & 15) == 0) ? n / 4 : 0;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += stride) {
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(rows) + q);
    const uint32_t e = b0 + (uint32_t)(4 * q);
    bad |= (v.x != e) | (v.y != e + 1u) | (v.z != e + 2u) | (v.w != e + 3u);
  }
  for (uint64_t i = 4 * n4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    bad |= rows[i] != b0 + (uint32_t)i;
  return bad;
}

__global__ void join_init_table_kernel(Slot* __restrict__ table, uint64_t cap, uint32_t* __restrict__ grp_bits,
                                       const uint32_t* __restrict__ rows, uint64_t n, int mode, unsigned* nd,
                                       unsigned* nd_next, unsigned long long* __restrict__ counters) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  if (blockIdx.x == 0 && threadIdx.x < 4) counters[threadIdx.x] = 0ull;  // GroupArrays::counters
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *nd_next = 0u;
    if (mode != 0) *nd = mode == 2 ? 1u : 0u;
  }
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += stride) {
    reinterpret_cast<ulonglong2*>(table)[i] = make_ulonglong2(kEmptyKey, 0ull);
    if (grp_bits && (i & 31) == 0) grp_bits[i >> 5] = 0u;
  }
  if (mode == 0 && __syncthreads_or(rows_not_dense(rows, n)) && threadIdx.x == 0) *nd = 1u;
}

// Build kernels process tiles of kBuildThreads*kBuildItems consecutive entries;
// each thread owns kBuildItems entries strided by the block size (coalesced),
// and issues their loads / atomics together so the dependent chains overlap.
#ifndef GOLP_BUILD_THREADS
#define GOLP_BUILD_THREADS 512
#endif
#ifndef GOLP_BUILD_ITEMS
#define GOLP_BUILD_ITEMS 1
#endif
constexpr int kBuildThreads = GOLP_BUILD_THREADS;
constexpr int kBuildItems = GOLP_BUILD_ITEMS;
constexpr uint64_t kBuildTile = (uint64_t)kBuildThreads * kBuildItems;

struct GroupArrays {
  uint32_t* rows;        // kInline per slot, then CSR ranges of big groups
  uint32_t* ovf_slot;    // overflow members (rank >= kInline)
  uint32_t* ovf_rank;
  uint32_t* ovf_pos;
  unsigned long long* counters;  // [0] overflow count, [1] CSR cursor, [2] big groups, [3] of them > kThreadGroup
  uint32_t* big_list;  // big groups, then (appended) the ones above kThreadGroup
  uint32_t* grp_bits;  // or null: one bit per slot, set when the slot's key gets a second member
};

// Tile schedule of kernels that walk slice-partitioned entries: with a counter,
// blocks claim tiles in order, so the tiles in flight stay consecutive (and in
// one or two table slices) however unevenly the SMs progress; without one, a
// plain grid-stride loop.
struct TileSched {
  unsigned long long* ctr;
  __device__ __forceinline__ uint64_t first(unsigned long long* s_t) const {
    return ctr ? claim(s_t) : blockIdx.x;
  }
  __device__ __forceinline__ uint64_t next(uint64_t t, unsigned long long* s_t) const {
    return ctr ? claim(s_t) : t + gridDim.x;
  }
  __device__ __forceinline__ uint64_t claim(unsigned long long* s_t) const {
    __syncthreads();  // all threads have read the previous claim
    if (threadIdx.x == 0) *s_t = atomicAdd(ctr, 1ull);
    __syncthreads();
    return *s_t;
  }
};

// bpos (optional): build position of entry i when the entries were partitioned.
// kWide (the default, GOLP_BUILD_WIDE_ALWAYS): claim slots with the 16-byte CAS,
// which saves the rank atomic of a key's first member (C4 build; C2 78 -> 75 us
// with the home-pair overflow flags). Otherwise a 64-bit key CAS plus rank =
// atomicAdd(cnt) for every member, the rank-0 member storing its position in
// slot.off.
template <bool kWide>
__global__ void __launch_bounds__(kBuildThreads) join_insert_kernel(const double* __restrict__ bkeys,
                                                                    const uint32_t* __restrict__ bpos, uint64_t nb,
                                                                    Slot* table, uint64_t mask, GroupArrays ga,
                                                                    TileSched sched) {
  __shared__ unsigned long long s_t;
  const uint64_t ntiles = (nb + kBuildTile - 1) / kBuildTile;
  for (uint64_t t = sched.first(&s_t); t < ntiles; t = sched.next(t, &s_t)) {
    const uint64_t t0 = t * kBuildTile;
    uint64_t b[kBuildItems];
    uint32_t h[kBuildItems], pos[kBuildItems], r[kBuildItems];
    unsigned pending = 0;
#pragma unroll
    for (int j = 0; j < kBuildItems; ++j) {
      const uint64_t i = t0 + (uint64_t)j * kBuildThreads + threadIdx.x;
      b[j] = i < nb ? canon_bits(__ldg(bkeys + i)) : 0ull;
      pos[j] = i < nb ? (bpos ? __ldg(bpos + i) : (uint32_t)i) : 0u;
      h[j] = (uint32_t)home_slot(b[j], mask);
      r[j] = 0;
      if (i < nb) pending |= 1u << j;
    }
    const unsigned valid = pending;
    unsigned dup = 0;  // entries whose key already owns a slot: take a rank with atomicAdd
    // Claim or find each key's slot: the CASes of all pending entries go out together.
    while (pending) {
      if constexpr (kWide) {
        ulonglong2 old[kBuildItems];
#pragma unroll
        for (int j = 0; j < kBuildItems; ++j)
          if (pending & (1u << j))
            old[j] = cas128(&table[h[j]], make_ulonglong2(kEmptyKey, 0ull),
                            make_ulonglong2(b[j], (1ull << 32) | pos[j]));
#pragma unroll
        for (int j = 0; j < kBuildItems; ++j) {
          if (!(pending & (1u << j))) continue;
          if (old[j].x == kEmptyKey) {
            pending &= ~(1u << j);  // claimed: rank 0, position stored inline
          } else if (old[j].x == b[j]) {
            pending &= ~(1u << j);
            dup |= 1u << j;
          } else {
            h[j] = (h[j] + 1) & (uint32_t)mask;
          }
        }
      } else {
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
        dup = valid;
      }
    }
#pragma unroll
    for (int j = 0; j < kBuildItems; ++j) {  // stored beyond its home pair: flag the home pair
      const uint32_t hp = (uint32_t)home_slot(b[j], mask);
      if (((valid >> j) & 1u) && (h[j] & ~1u) != hp) atomicOr(&table[hp].cnt, kOverflowBit);
    }
#pragma unroll
    for (int j = 0; j < kBuildItems; ++j)
      if (dup & (1u << j)) r[j] = atomicAdd(&table[h[j]].cnt, 1u) & kCntMask;
#pragma unroll
    for (int j = 0; j < kBuildItems; ++j)  // a key's second member marks its slot for the finalize
      if (ga.grp_bits && ((dup >> j) & 1u) && r[j] == 1) atomicOr(&ga.grp_bits[h[j] >> 5], 1u << (h[j] & 31));
    if constexpr (!kWide) {
#pragma unroll
      for (int j = 0; j < kBuildItems; ++j)
        if ((dup & (1u << j)) && r[j] == 0) table[h[j]].off = pos[j];
    }
#pragma unroll
    for (int j = 0; j < kBuildItems; ++j) {
      const bool ok = ((dup >> j) & 1u) && r[j] > 0;  // rank 0 lives in slot.off
      if (ok && r[j] < kInline) ga.rows[(uint64_t)h[j] * kInline + r[j]] = pos[j];
      const bool ovf = ok && r[j] >= kInline;
      const unsigned long long k = warp_append(&ga.counters[0], ovf);
      if (ovf) {
        ga.ovf_slot[k] = h[j];
        ga.ovf_rank[k] = r[j];
        ga.ovf_pos[k] = pos[j];
      }
    }
  }
}

// Build position -> build row. When the row column is a dense run (*dense set by
// dense_rows_check_kernel, or by the host when it regenerated the column),
// rows[p] == rows[0] + p and the gather -- a random DRAM sector per entry once
// the column outgrows L2 -- is skipped.
struct BuildRows {
  const uint32_t* rows;
  const unsigned* not_dense;  // 0: rows[i] == rows[0] + i for every i
};
struct RowMap {
  const uint32_t* rows;
  bool dense;
  uint32_t base;
  __device__ __forceinline__ explicit RowMap(const BuildRows& b)
      : rows(b.rows), dense(*b.not_dense == 0), base(dense ? b.rows[0] : 0u) {}
  __device__ __forceinline__ uint32_t operator()(uint32_t p) const { return dense ? base + p : __ldg(rows + p); }
};


__device__ __forceinline__ void cswap_u32(uint32_t& a, uint32_t& b) {
  const uint32_t lo = a < b ? a : b, hi = a < b ? b : a;
  a = lo;
  b = hi;
}

// One pass over the slots: singletons inline their row, groups of 2..kInline sort
// their recorded positions and turn them into rows, big groups reserve a CSR range.
// Dense row column: singletons keep their build POSITION in slot.off (the emit
// adds the column's first row id, *row_base): no gather and no store for them.
// Dense row column with ga.grp_bits: singletons need nothing, so lane l of a
// warp takes the 8 slots of bitmap byte wb + l and visits its flagged key
// groups one per step, instead of every slot of the table.
__global__ void __launch_bounds__(256) join_finalize_kernel(Slot* table, uint64_t cap, BuildRows br,
                                                            GroupArrays ga, uint64_t csr_base, uint32_t* row_base) {
  const unsigned lane = lane_id();
  const RowMap row(br);
  if (blockIdx.x == 0 && threadIdx.x == 0) *row_base = row.dense ? row.base : 0u;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const bool use_bits = row.dense && ga.grp_bits;
  const uint64_t nvisit = use_bits ? (cap + 7) / 8 : cap;
  const uint8_t* gbytes = reinterpret_cast<const uint8_t*>(ga.grp_bits);
  for (uint64_t wb = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x - lane; wb < nvisit; wb += stride) {
    uint32_t bits = use_bits && wb + lane < nvisit ? gbytes[wb + lane] : 0u;
    for (;;) {
    uint64_t h;
    if (use_bits) {
      if (!__any_sync(0xFFFFFFFFu, bits != 0)) break;
      h = bits ? (wb + lane) * 8 + (uint32_t)__ffs(bits) - 1 : cap;
      bits &= bits - 1;
    } else {
      h = wb + lane;
    }
    uint32_t cnt = 0, first = 0, oflag = 0;  // first: rank-0 position, stored inline by the claiming CAS
    if (h < cap) {
      const ulonglong2 sl = reinterpret_cast<const ulonglong2*>(table)[h];
      if (sl.x != kEmptyKey) {
        cnt = (uint32_t)(sl.y >> 32) & kCntMask;
        oflag = (uint32_t)(sl.y >> 32) & kOverflowBit;
        first = (uint32_t)sl.y;
      }
    }
    uint32_t* grp = ga.rows + h * kInline;
    if (cnt == 1) {
      if (!row.dense) table[h].off = row(first);
    } else if (cnt >= 2 && cnt <= kInline) {
      const uint4 v = *reinterpret_cast<const uint4*>(grp);
      uint32_t p0 = first, p1 = v.y, p2 = cnt > 2 ? v.z : 0xFFFFFFFFu, p3 = cnt > 3 ? v.w : 0xFFFFFFFFu;
      cswap_u32(p0, p1); cswap_u32(p2, p3); cswap_u32(p0, p2); cswap_u32(p1, p3); cswap_u32(p1, p2);
      uint4 o;
      o.x = row(p0);
      o.y = row(p1);
      if (cnt == 2 && o.y <= kPair2Row) {  // both rows in the slot (keeps the overflow flag)
        reinterpret_cast<unsigned long long*>(table + h)[1] =
            ((unsigned long long)(oflag | kPair2Bit | o.y) << 32) | o.x;
      } else {
        o.z = cnt > 2 ? row(p2) : 0u;
        o.w = cnt > 3 ? row(p3) : 0u;
        *reinterpret_cast<uint4*>(grp) = o;
        table[h].off = (uint32_t)(h * kInline);
      }
    }
    const uint32_t need = cnt > kInline ? cnt : 0u;  // big group: reserve its CSR range
    if (!__ballot_sync(0xFFFFFFFFu, need != 0)) {  // (almost every warp of slots)
      if (use_bits) continue;
      break;
    }
    unsigned long long incl = need;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if ((int)lane >= o) incl += v;
    }
    unsigned long long base = 0;
    if (lane == 31 && incl) base = atomicAdd(&ga.counters[1], incl);
    base = __shfl_sync(0xFFFFFFFFu, base, 31);
    if (need) {
      const uint64_t off = csr_base + base + incl - need;
      table[h].off = (uint32_t)off;
      const uint4 v = *reinterpret_cast<const uint4*>(grp);  // ranks 1..3
      ga.rows[off] = first;
      ga.rows[off + 1] = v.y;
      ga.rows[off + 2] = v.z;
      ga.rows[off + 3] = v.w;
      ga.big_list[atomicAdd(&ga.counters[2], 1ull)] = (uint32_t)h;
    }
    if (!use_bits) break;
    }
  }
}

// Overflow members (rank >= kInline) land at their rank inside their group's range.
__global__ void join_overflow_kernel(const Slot* __restrict__ table, GroupArrays ga) {
  const unsigned long long n = *(volatile unsigned long long*)&ga.counters[0];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride)
    ga.rows[table[ga.ovf_slot[k]].off + ga.ovf_rank[k]] = ga.ovf_pos[k];
}

// Big groups of up to kThreadGroup members: one thread sorts the positions
// (insertion sort) and writes rows; larger ones are queued for the block kernel.
constexpr uint32_t kThreadGroup = 32;

__global__ void join_group_sort_kernel(const Slot* __restrict__ table, GroupArrays ga, BuildRows br) {
  // one warp per group: lane m holds member m's position, its rank among the
  // group's (distinct) positions is its place in build order
  const RowMap row(br);
  const unsigned lane = lane_id();
  const unsigned nbig = (unsigned)*(volatile unsigned long long*)&ga.counters[2];
  const uint64_t wstride = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t gi = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); gi < nbig; gi += wstride) {
    const uint32_t h = ga.big_list[gi];
    const uint32_t cnt = table[h].cnt & kCntMask;
    if (cnt > kThreadGroup) {
      if (lane == 0) ga.big_list[nbig + atomicAdd(&ga.counters[3], 1ull)] = h;  // block kernel's queue
      continue;
    }
    uint32_t* seg = ga.rows + table[h].off;
    const uint32_t v = lane < cnt ? seg[lane] : 0xFFFFFFFFu;
    uint32_t rank = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const uint32_t u = __shfl_sync(0xFFFFFFFFu, v, j);
      rank += (u < v) || (u == v && j < (int)lane);
    }
    const uint32_t r = lane < cnt ? row(v) : 0u;
    __syncwarp();
    if (lane < cnt) seg[rank] = r;
  }
}

// Groups above kThreadGroup (queued by join_group_sort_kernel): one block per
// group sorts its positions (shared memory up to kGroupTile, in place in global
// memory beyond) and turns them into rows.
__global__ void __launch_bounds__(1024) join_big_groups_kernel(const Slot* __restrict__ table, GroupArrays ga,
                                                               BuildRows br) {
  const RowMap row(br);
  extern __shared__ __align__(16) uint32_t s_pos[];
  const unsigned nbig = (unsigned)*(volatile unsigned long long*)&ga.counters[2];
  const unsigned nhuge = (unsigned)*(volatile unsigned long long*)&ga.counters[3];
  for (unsigned gi = blockIdx.x; gi < nhuge; gi += gridDim.x) {
    const uint32_t h = ga.big_list[nbig + gi];
    const uint32_t cnt = table[h].cnt & kCntMask;
    uint32_t* seg = ga.rows + table[h].off;
    if (cnt <= kGroupTile) {
      for (uint32_t m = threadIdx.x; m < cnt; m += blockDim.x) s_pos[m] = seg[m];
      __syncthreads();
      block_sort_asc_u32<false>(s_pos, cnt);
      for (uint32_t m = threadIdx.x; m < cnt; m += blockDim.x) seg[m] = row(s_pos[m]);
    } else {
      block_sort_asc_u32<true>(seg, cnt);
      for (uint32_t m = threadIdx.x; m < cnt; m += blockDim.x) seg[m] = row(__ldcg(seg + m));
    }
    __syncthreads();
  }
}

// ---- probe ------------------------------------------------------------------------
// Bound by random table lookups: ~1 L1TEX wavefront per lookup, ~0.8/clk/SM
// from L2 (tools/microbench.cu, tools/probe_ladder.cu). Every probe key is looked
// up exactly once:
//   match : each warp walks a contiguous run of warp tiles (32*kWarpItems
//           consecutive probes each), resolves its probes (linear probing over
//           32-byte slot pairs) and appends the hits, in probe order, to its own
//           contiguous scratch segment {probe row, slot.off, slot.cnt}; per-warp
//           entry / pair counts and per-block pair totals are written.
//   scan  : one block scans the per-block totals (+ pairs of earlier launches).
//   emit  : same mapping; each warp streams its segment to the output at its
//           offset (block offset + pairs of the block's earlier warps).
// Output order = probe position, then CSR (build insertion) order.
#ifndef GOLP_WARP_ITEMS
#define GOLP_WARP_ITEMS 2
#endif
#ifndef GOLP_PROBE_MINB
#define GOLP_PROBE_MINB 5
#endif
constexpr int kWarpItems = GOLP_WARP_ITEMS;
static_assert(kWarpItems % 2 == 0, "keys are loaded as 16-byte pairs");
constexpr uint32_t kWarpTile = 32 * kWarpItems;  // probes per warp tile
constexpr int kProbeThreads = 256;

// L2 eviction policies: the table should survive the probe stream in L2, the
// streamed probe columns should not displace it.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
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
__device__ __forceinline__ double ldg_stream_f64(const double* p, uint64_t pol) {
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint64_t ldg_stream_u64(const uint64_t* p, uint64_t pol) {
  uint64_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(pol));
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

// One block: exclusive scan of the partials, offset by *base_in; writes *total_out.
// Each warp owns a contiguous chunk: a coalesced pass sums it, one block scan of
// the warp sums gives each chunk's base, a second coalesced pass writes the
// prefixes (warp-level scans) -- instead of one block-wide scan round (two
// barriers) per kScanThreads elements.
__global__ void __launch_bounds__(kScanThreads) scan_partials_kernel(unsigned long long* partial, uint32_t nparts,
                                                                     const unsigned long long* base_in,
                                                                     unsigned long long* total_out) {
  __shared__ unsigned long long s_w[33];
  __shared__ unsigned long long s_base[kScanThreads / 32];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  constexpr unsigned kWarps = kScanThreads / 32;
  const uint32_t per = ((nparts + kWarps - 1) / kWarps + 31) / 32 * 32;
  const uint32_t b = warp * per, e = b + per < nparts ? b + per : nparts;
  unsigned long long sum = 0;
  for (uint32_t i = b + lane; i < e; i += 32) sum += partial[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
  if (lane == 0) s_base[warp] = sum;
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the warp sums
    const unsigned long long w = lane < kWarps ? s_base[lane] : 0ull;
    unsigned long long incl = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if ((int)lane >= o) incl += u;
    }
    const unsigned long long base = base_in ? *base_in : 0ull;
    if (lane < kWarps) s_base[lane] = base + incl - w;
    if (lane == 31) s_w[0] = base + incl;
  }
  __syncthreads();
  unsigned long long run = s_base[warp];
  for (uint32_t i0 = b; i0 < e; i0 += 32) {
    const uint32_t i = i0 + lane;
    const unsigned long long v = i < e ? partial[i] : 0ull;
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if ((int)lane >= o) incl += u;
    }
    if (i < e) partial[i] = run + incl - v;
    run += __shfl_sync(0xFFFFFFFFu, incl, 31);
  }
  if (threadIdx.x == 0) *total_out = s_w[0];
}

// ---- radix partitioning (tables larger than ~L2/2) ----------------------------------
// The table is viewed as P slices of 2^slice_bits slots; a key's slice is the
// top bits of its home slot. Processing entries slice by slice keeps the part of
// the table being walked L2-resident. This is only a schedule: the walks are the
// ordinary table-wide linear probes (one that runs off the end of its slice just
// touches the next one), so the table is the same as an unpartitioned build and
// skewed keys cannot overfill a slice.
//
// Entries are grouped by slice with a count pass, a scan of the P totals and a
// scatter that sorts each tile of kPartTile entries by slice in shared memory and
// writes every slice's run of the tile contiguously at a reserved offset. The
// order inside a partition does not matter: the build inserts in any order and
// sorts key groups by position afterwards; the probe records each entry's index
// inside its tile plus the (offset, length) of every (tile, slice) run, so
// join_unpartition_kernel can put results back in probe order tile by tile with
// coalesced reads and writes (no scattered 8-byte stores).
#ifndef GOLP_PART_THREADS
#define GOLP_PART_THREADS 512
#endif
#ifndef GOLP_PART_MINB
#define GOLP_PART_MINB 2
#endif
#ifndef GOLP_PART_TILE
#define GOLP_PART_TILE 4096
#endif
constexpr uint32_t kPartTile = GOLP_PART_TILE;  // entries per partition tile (run tables, match tiles)
constexpr int kPartThreads = GOLP_PART_THREADS;
constexpr int kPartItems = (int)(kPartTile / kPartThreads);
static_assert(kPartItems * kPartThreads == (int)kPartTile && kPartItems % 2 == 0, "tile split");
constexpr uint32_t kMaxParts = 1024;
constexpr uint32_t kMaxProbeParts = 256;  // bounds the per-(tile, slice) run table
constexpr size_t kPartSmem = (size_t)kPartTile * (8 + 2 + 2) + (size_t)kMaxParts * (4 + 4 + 8);
#ifndef GOLP_PART_TMA
#define GOLP_PART_TMA 1
#endif
// + the next tile's keys, prefetched by TMA while the current tile is processed
constexpr size_t kPartScatterSmem = kPartSmem + (GOLP_PART_TMA ? (size_t)kPartTile * 8 : 0);

// ---- TMA bulk copies (cp.async.bulk, mbarrier completion) ----------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
// One thread: expect `bytes` on the barrier, then a bulk global -> shared copy
// that completes them (16-byte aligned addresses, size a multiple of 16).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar, uint64_t pol) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst), b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(d),
      "l"(src), "r"(bytes), "r"(b), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(b),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ uint32_t part_of(double k, uint32_t mask, int slice_bits) {
  return home_slot32(canon_bits(k), mask) >> slice_bits;
}

__global__ void __launch_bounds__(kPartThreads) part_count_kernel(const double* __restrict__ keys, uint64_t n,
                                                                  uint32_t mask, int slice_bits, uint32_t nparts,
                                                                  unsigned long long* __restrict__ counts) {
  __shared__ unsigned s_h[kMaxParts];
  for (uint32_t p = threadIdx.x; p < nparts; p += blockDim.x) s_h[p] = 0;
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  // 16-byte pair loads from the first 16-byte boundary on; a column that starts
  // 8 bytes off it (a view) counts its first key on its own
  const uint64_t head = (n > 0 && (reinterpret_cast<uintptr_t>(keys) & 15) != 0) ? 1 : 0;
  if (head && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&s_h[part_of(keys[0], mask, slice_bits)], 1u);
  keys += head;
  n -= head;
  const uint64_t n2 = n / 2;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n2; i += 8 * stride) {  // 8 independent 16-byte loads in flight
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = ldg_stream_d2(keys + 2 * (i + u * stride), pol);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      atomicAdd(&s_h[part_of(v[u].x, mask, slice_bits)], 1u);
      atomicAdd(&s_h[part_of(v[u].y, mask, slice_bits)], 1u);
    }
  }
  for (; i < n2; i += stride) {
    const double2 v = ldg_stream_d2(keys + 2 * i, pol);
    atomicAdd(&s_h[part_of(v.x, mask, slice_bits)], 1u);
    atomicAdd(&s_h[part_of(v.y, mask, slice_bits)], 1u);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&s_h[part_of(keys[n - 1], mask, slice_bits)], 1u);
  __syncthreads();
  for (uint32_t p = threadIdx.x; p < nparts; p += blockDim.x)
    if (s_h[p]) atomicAdd(&counts[p], (unsigned long long)s_h[p]);
}

// counts -> exclusive offsets written to cursors (one block).
__global__ void __launch_bounds__(1024) part_scan_kernel(const unsigned long long* __restrict__ counts,
                                                         unsigned long long* __restrict__ cursors, uint32_t nparts) {
  __shared__ unsigned long long s_w[33];
  unsigned long long carry = 0;
  for (uint32_t b0 = 0; b0 < nparts; b0 += blockDim.x) {
    const uint32_t i = b0 + threadIdx.x;
    const unsigned long long v = i < nparts ? counts[i] : 0ull;
    unsigned long long tot;
    const unsigned long long e = block_excl_scan(v, s_w, &tot);
    if (i < nparts) cursors[i] = carry + e;
    carry += tot;
  }
}

struct PartOut {
  double* keys;        // entries grouped by slice
  uint32_t* pos;       // build side: the entry's position (or null)
  uint16_t* idx;       // probe side: the entry's index inside its tile (or null)
  uint32_t* run_base;  // probe side: [tile * nparts + p] = offset of the tile's run of slice p
  uint16_t* run_len;   //             and its length
  // Fixed-capacity layout (capu > 0, probe side): slice p owns [p * capu, (p+1) * capu)
  // and cursors[p] counts its entries (no count pass); a run that does not fit
  // goes to the overflow area at nparts * capu (cursor *ovf). Runs are located
  // through run_base either way, so only locality suffers for skewed slices.
  uint64_t capu;
  unsigned long long* ovf;
};

// Exclusive scan of s_cnt[0..nparts) into s_start (nparts <= 2 * blockDim.x).
__device__ __forceinline__ void block_scan_parts(const unsigned* s_cnt, unsigned* s_start, uint32_t nparts,
                                                 unsigned long long* s_w) {
  const uint32_t i0 = 2 * threadIdx.x;
  const unsigned a = i0 < nparts ? s_cnt[i0] : 0u, b = i0 + 1 < nparts ? s_cnt[i0 + 1] : 0u;
  unsigned long long tot;
  const unsigned e = (unsigned)block_excl_scan((unsigned long long)(a + b), s_w, &tot);
  if (i0 < nparts) s_start[i0] = e;
  if (i0 + 1 < nparts) s_start[i0 + 1] = e + a;
  __syncthreads();
}

__global__ void __launch_bounds__(kPartThreads, GOLP_PART_MINB) part_scatter_kernel(const double* __restrict__ keys, uint64_t n,
                                                                    uint32_t mask, int slice_bits, uint32_t nparts,
                                                                    unsigned long long* __restrict__ cursors,
                                                                    PartOut out) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* s_key = reinterpret_cast<double*>(smem);
  uint16_t* s_loc = reinterpret_cast<uint16_t*>(s_key + kPartTile);
  uint16_t* s_part = s_loc + kPartTile;
  unsigned* s_cnt = reinterpret_cast<unsigned*>(s_part + kPartTile);
  unsigned* s_start = s_cnt + kMaxParts;
  unsigned long long* s_base = reinterpret_cast<unsigned long long*>(s_start + kMaxParts);
  __shared__ unsigned long long s_w[33];
  const uint64_t pol = policy_evict_first();
  const uint64_t ntiles = (n + kPartTile - 1) / kPartTile;
  // Full tiles of a 16-byte aligned key column arrive by TMA: one thread
  // issues the next tile's 32 KB bulk copy as soon as the block has read the
  // current one, so the load overlaps the ranking, scan and scatter.
  double* s_in = reinterpret_cast<double*>(smem + kPartSmem);
  __shared__ __align__(8) uint64_t s_bar;
  const bool tma = GOLP_PART_TMA && (reinterpret_cast<uintptr_t>(keys) & 15) == 0;
  auto tma_tile = [&](uint64_t t) { return tma && t < ntiles && (t + 1) * kPartTile <= n; };
  unsigned phase = 0;
  if (tma) {
    if (threadIdx.x == 0) {
      mbar_init(&s_bar, 1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0 && tma_tile(blockIdx.x))
      bulk_g2s(s_in, keys + (uint64_t)blockIdx.x * kPartTile, kPartTile * 8, &s_bar, pol);
  }
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t t0 = t * kPartTile;
    const uint32_t cnt = (uint32_t)(n - t0 < kPartTile ? n - t0 : kPartTile);
    for (uint32_t p = threadIdx.x; p < nparts; p += blockDim.x) s_cnt[p] = 0;
    double k[kPartItems];
    uint32_t pr[kPartItems];  // part << 16 | rank inside the tile's run
    if (tma_tile(t)) {
      mbar_wait(&s_bar, phase);
      phase ^= 1u;
#pragma unroll
      for (int j = 0; j < kPartItems; j += 2) {
        const double2 v = reinterpret_cast<const double2*>(s_in)[threadIdx.x + (j >> 1) * kPartThreads];
        k[j] = v.x;
        k[j + 1] = v.y;
      }
      __syncthreads();  // s_in consumed (and s_cnt cleared) before the next copy lands in it
      if (threadIdx.x == 0 && tma_tile(t + gridDim.x))
        bulk_g2s(s_in, keys + (t + gridDim.x) * kPartTile, kPartTile * 8, &s_bar, pol);
    } else if (cnt == kPartTile && ((reinterpret_cast<uintptr_t>(keys + t0) & 15) == 0)) {
      __syncthreads();
#pragma unroll
      for (int j = 0; j < kPartItems; j += 2) {
        const double2 v = ldg_stream_d2(keys + t0 + 2 * threadIdx.x + (uint64_t)j * kPartThreads, pol);
        k[j] = v.x;
        k[j + 1] = v.y;
      }
    } else {
      __syncthreads();
#pragma unroll
      for (int j = 0; j < kPartItems; j += 2) {
        const uint32_t l = 2 * threadIdx.x + j * kPartThreads;
        k[j] = l < cnt ? keys[t0 + l] : 0.0;
        k[j + 1] = l + 1 < cnt ? keys[t0 + l + 1] : 0.0;
      }
    }
#pragma unroll
    for (int j = 0; j < kPartItems; ++j) {
      const uint32_t l = 2 * threadIdx.x + (j & ~1) * kPartThreads + (j & 1);
      if (l < cnt) {
        const uint32_t p = part_of(k[j], mask, slice_bits);
        pr[j] = (p << 16) | atomicAdd(&s_cnt[p], 1u);
      }
    }
    __syncthreads();
    block_scan_parts(s_cnt, s_start, nparts, s_w);
    for (uint32_t p = threadIdx.x; p < nparts; p += blockDim.x) {
      const unsigned c = s_cnt[p];
      unsigned long long b = c ? atomicAdd(&cursors[p], (unsigned long long)c) : 0ull;
      if (out.capu && c) {
        if (b + c <= out.capu) b += p * out.capu;
        else b = (uint64_t)nparts * out.capu + atomicAdd(out.ovf, (unsigned long long)c);
      }
      s_base[p] = b;
      if (out.run_base) {
        out.run_base[t * nparts + p] = (uint32_t)b;
        out.run_len[t * nparts + p] = (uint16_t)c;
      }
    }
#pragma unroll
    for (int j = 0; j < kPartItems; ++j) {
      const uint32_t l = 2 * threadIdx.x + (j & ~1) * kPartThreads + (j & 1);
      if (l < cnt) {
        const uint32_t p = pr[j] >> 16;
        const uint32_t d = s_start[p] + (pr[j] & 0xFFFFu);
        s_key[d] = k[j];
        s_loc[d] = (uint16_t)l;
        s_part[d] = (uint16_t)p;
      }
    }
    __syncthreads();
    uint32_t o[kPartItems];  // destinations (entry counts are < 2^32)
#pragma unroll
    for (int u = 0; u < kPartItems; ++u) {  // resolve all destinations first (independent smem loads)
      const uint32_t i = threadIdx.x + u * kPartThreads;
      if (i < cnt) {
        const uint32_t p = s_part[i];
        o[u] = (uint32_t)s_base[p] + (i - s_start[p]);
      }
    }
#pragma unroll
    for (int u = 0; u < kPartItems; ++u) {
      const uint32_t i = threadIdx.x + u * kPartThreads;
      if (i < cnt) {  // streaming stores: read once, by a later kernel
        __stcs(reinterpret_cast<unsigned long long*>(out.keys) + o[u], (unsigned long long)__double_as_longlong(s_key[i]));
        if (out.pos) __stcs(out.pos + o[u], (uint32_t)(t0 + s_loc[i]));
        if (out.idx) __stcs(reinterpret_cast<unsigned short*>(out.idx) + o[u], (unsigned short)s_loc[i]);
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void st_hint(uint32_t* p, uint32_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}

// Checks one slot pair: 1 = found (off/cnt set), 0 = absent, -1 = continue at h+2.
// `home`: this is the key's home pair, whose overflow flag tells whether a key
// homed here can live further on.
__device__ __forceinline__ int check_pair(const ulonglong4& sl, uint64_t bits, uint32_t& off, uint32_t& cnt,
                                          bool home) {
  if (sl.x == bits) { off = (uint32_t)sl.y; cnt = (uint32_t)(sl.y >> 32) & kCntMask; return 1; }
  if (sl.x == kEmptyKey) return 0;
  if (sl.z == bits) { off = (uint32_t)sl.w; cnt = (uint32_t)(sl.w >> 32) & kCntMask; return 1; }
  if (sl.z == kEmptyKey) return 0;
  if (home && !((sl.y >> 32) & kOverflowBit)) return 0;
  return -1;
}

// Scratch entries are SoA {u32 probe row, u64 slot.off | slot.cnt << 32}. Each warp owns a
// contiguous run of warp tiles and appends its hits contiguously (in probe
// order) starting at its first tile's slot, so emit is a streaming copy.
struct MatchScratch {
  uint32_t* prow;
  uint64_t* oc;  // slot.off | slot.cnt << 32 (one 8-byte store / load per hit)
  uint32_t* wentries;            // per global warp: entries written
  unsigned long long* wpairs;    // per global warp: pairs produced (sum of cnt; 64-bit, big key groups)
};

constexpr unsigned kProbeWarps = kProbeThreads / 32;

// Appends one warp tile's hits (probe row, slot.off, slot.cnt) to the warp's
// scratch run in probe order; returns the tile's pair count.
// prow: the probe rows of this lane's kWarpItems probes, loaded with the keys
// (a load issued only after the lookups would add a dependent round trip).
// Returns this LANE's pair count of the tile (the warp total is reduced once,
// at the end of the warp's run).
__device__ __forceinline__ uint64_t warp_append_hits(unsigned lane, const uint32_t* off, const uint32_t* cnt,
                                                     const uint32_t* prow, const MatchScratch& sc, uint64_t& cursor) {
  uint32_t nm = 0;
  uint64_t npr = 0;
#pragma unroll
  for (int j = 0; j < kWarpItems; ++j) {  // cnt[j]: the slot's cnt word (kPair2Bit: an inline pair)
    nm += cnt[j] != 0;
    npr += slot_members(cnt[j]);
  }
  // hits of the lanes before this one, and of the tile: one ballot per hit count
  const unsigned lt = (1u << lane) - 1u;
  uint32_t excl = 0, tmatch = 0;
#pragma unroll
  for (int t = 1; t <= kWarpItems; ++t) {
    const unsigned b = __ballot_sync(0xFFFFFFFFu, nm >= (uint32_t)t);
    excl += __popc(b & lt);
    tmatch += __popc(b);
  }
  if (nm) {
    uint64_t o = cursor + excl;
#pragma unroll
    for (int j = 0; j < kWarpItems; ++j) {
      if (cnt[j]) {
        sc.prow[o] = prow[j];
        sc.oc[o] = ((uint64_t)cnt[j] << 32) | off[j];
        ++o;
      }
    }
  }
  cursor += tmatch;
  return npr;
}

// Per-warp totals -> scratch counters and the block's pair total.
__device__ __forceinline__ void finish_match_block(unsigned lane, unsigned warp, uint64_t gw, uint64_t lo,
                                                   uint64_t cursor, uint64_t pairs_total, const MatchScratch& sc,
                                                   unsigned long long* s_w, unsigned long long* __restrict__ bpart) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pairs_total += __shfl_xor_sync(0xFFFFFFFFu, pairs_total, o);  // lanes -> warp
  if (lane == 0) {
    sc.wentries[gw] = (uint32_t)(cursor - lo * kWarpTile);
    sc.wpairs[gw] = pairs_total;
    s_w[warp] = pairs_total;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (unsigned w = 0; w < kProbeWarps; ++w) t += s_w[w];
    bpart[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kProbeThreads, GOLP_PROBE_MINB) join_match_kernel(
    const double* __restrict__ pkeys, RowCol prows, uint64_t np, const Slot* __restrict__ table,
    uint64_t mask, MatchScratch sc, uint64_t nwt, uint64_t per_warp, unsigned long long* __restrict__ bpart) {
  __shared__ unsigned long long s_w[kProbeWarps];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint64_t pol_stream = policy_evict_first(), pol_table = policy_evict_last();
  const uint64_t gw = (uint64_t)blockIdx.x * kProbeWarps + warp;
  const uint64_t lo = gw * per_warp, hi = lo + per_warp < nwt ? lo + per_warp : nwt;
  uint64_t cursor = lo * kWarpTile;  // next free scratch entry of this warp
  uint64_t pairs_total = 0;
  for (uint64_t wt = lo; wt < hi; ++wt) {
    const uint64_t first = wt * kWarpTile + lane * kWarpItems;
    uint32_t off[kWarpItems], cnt[kWarpItems], prow[kWarpItems];
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
    // the probe rows go out with the keys (a load after the lookups would add a
    // dependent round trip to every tile with a hit)
#pragma unroll
    for (int j = 0; j < kWarpItems; ++j) prow[j] = first + j < np ? prows.at_cs(first + j) : 0u;
    uint64_t bits[kWarpItems];
    uint32_t h[kWarpItems];
    unsigned pending = 0;
#pragma unroll
    for (int j = 0; j < kWarpItems; ++j) {
      bits[j] = canon_bits(k[j]);
      h[j] = home_slot32(bits[j], (uint32_t)mask);
      off[j] = 0;
      cnt[j] = 0;
      if (first + j < np) pending |= 1u << j;
    }
    bool home = true;
    while (pending) {
      ulonglong4 sl[kWarpItems];
#pragma unroll
      for (int j = 0; j < kWarpItems; ++j)
        if (pending & (1u << j)) sl[j] = ldg_pair(table + h[j], pol_table);
#pragma unroll
      for (int j = 0; j < kWarpItems; ++j) {
        if (!(pending & (1u << j))) continue;
        const int st = check_pair(sl[j], bits[j], off[j], cnt[j], home);
        if (st >= 0) pending &= ~(1u << j);
        else h[j] = (h[j] + 2) & (uint32_t)mask;
      }
      home = false;
    }
    pairs_total += warp_append_hits(lane, off, cnt, prow, sc, cursor);
  }
  finish_match_block(lane, warp, gw, lo, cursor, pairs_total, sc, s_w, bpart);
}

// Radix-partitioned probe: keys arrive grouped by table slice, so consecutive
// threads walk the same L2-resident slice. res_part[i] = {off | cnt << 32} of the
// slot of keys[i] (0 when absent), in partitioned order. Blocks claim chunks of
// kPartProbeSub sub-tiles in order (TileSched); inside a chunk the keys of the
// next sub-tile are loaded while the current one's lookups are in flight.
// One lookup per thread at full occupancy (8 blocks of 256, 30 registers) beat
// 4 per thread at 3 blocks/SM (80 registers): 27.4 vs 30.3 ms for a 1.07e9-probe
// span against the C4 table (tools/part_probe_variants.py).
#ifndef GOLP_PART_PROBE_ITEMS
#define GOLP_PART_PROBE_ITEMS 1
#endif
#ifndef GOLP_PART_PROBE_MINB
#define GOLP_PART_PROBE_MINB 8
#endif
constexpr int kPartProbeItems = GOLP_PART_PROBE_ITEMS;
#ifndef GOLP_PART_PROBE_SUB
#define GOLP_PART_PROBE_SUB 16
#endif
constexpr int kPartProbeSub = GOLP_PART_PROBE_SUB;
// fixed-capacity slices are whole partition tiles: a lookup chunk must never
// straddle two of them (PartExtent::end_of)
static_assert(kPartTile % ((uint64_t)kProbeThreads * kPartProbeItems * kPartProbeSub) == 0,
              "lookup chunks must divide the partition tile");
// Deferred second rounds: a key not resolved by its home pair is queued (per
// warp, in shared memory) instead of holding its whole warp for another round
// trip; a full queue is resolved by the warp with all 32 lanes busy. res_part
// is indexed by entry, so the order in which entries resolve does not matter.
#ifndef GOLP_PART_PROBE_QUEUE
#define GOLP_PART_PROBE_QUEUE 1
#endif
#ifndef GOLP_PART_QUEUE_EVERY
#define GOLP_PART_QUEUE_EVERY 8  // > 0: also resolve a partial queue every this many sub-tiles
#endif
// Lookup results: written once, read once by match_runs much later -- streaming
// stores, so they do not push the table slice being probed out of L2.
#ifndef GOLP_RES_STREAM
#define GOLP_RES_STREAM 1
#endif
__device__ __forceinline__ void st_res(uint64_t* p, uint64_t v) {
#if GOLP_RES_STREAM
  __stcs(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
#else
  *p = v;
#endif
}
struct PartProbeQueue {
  uint64_t bits[32];
  uint32_t h[32];
  uint32_t i[32];  // entry index inside the span (< 2^32)
};

// Resolves this lane's queued key (lane < qn) to the end of its probe walk.
__device__ __forceinline__ void part_queue_drain(const PartProbeQueue& q, unsigned lane, unsigned qn,
                                                 const Slot* __restrict__ table, uint64_t mask,
                                                 uint64_t* __restrict__ res_part, uint64_t pol_table) {
  __syncwarp();
  if (lane < qn) {
    const uint64_t bits = q.bits[lane];
    uint32_t h = q.h[lane], off = 0, cnt = 0;
    for (;;) {
      const int st = check_pair(ldg_pair(table + h, pol_table), bits, off, cnt, false);
      if (st >= 0) break;
      h = (h + 2) & (uint32_t)mask;
    }
    st_res(res_part + q.i[lane], ((uint64_t)cnt << 32) | off);
  }
  __syncwarp();
}

// Fixed-capacity partitions (PartOut::capu): the valid part of each chunk.
struct PartExtent {
  uint64_t capu;                         // 0: the entries are dense in [0, n)
  uint32_t nparts;
  const unsigned long long* used;        // per slice: entries routed to it (may exceed capu)
  const unsigned long long* ovf;         // entries in the overflow area
  // end of the valid entries of the slice (or overflow area) holding position c0
  __device__ __forceinline__ uint64_t end_of(uint64_t c0, uint64_t n) const {
    if (!capu) return n;
    const uint64_t p = c0 / capu;
    if (p < nparts) {
      const unsigned long long u = __ldcg(used + p);
      return p * capu + (u < capu ? u : capu);
    }
    return (uint64_t)nparts * capu + __ldcg(ovf);
  }
};

__global__ void __launch_bounds__(kProbeThreads, GOLP_PART_PROBE_MINB) join_probe_part_kernel(const double* __restrict__ keys, uint64_t n_all,
                                                                        const Slot* __restrict__ table, uint64_t mask,
                                                                        uint64_t* __restrict__ res_part,
                                                                        int table_policy, TileSched sched,
                                                                        PartExtent ext) {
  __shared__ uint64_t s_end;
  __shared__ unsigned long long s_t;
  const uint64_t pol_table = table_policy ? policy_evict_normal() : policy_evict_last();
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t sub = (uint64_t)kProbeThreads * kPartProbeItems;
  const uint64_t chunk = sub * kPartProbeSub;
  const uint64_t nchunks = (n_all + chunk - 1) / chunk;
#if GOLP_PART_PROBE_QUEUE
  static_assert(kPartProbeItems == 1, "the deferred queue takes one entry per lane and sub-tile");
  __shared__ PartProbeQueue s_q[kProbeWarps];
  const unsigned lane = lane_id();
  PartProbeQueue& q = s_q[threadIdx.x >> 5];
  unsigned qn = 0;  // queued entries of this warp (warp-uniform)
#endif
  for (uint64_t c = sched.first(&s_t); c < nchunks; c = sched.next(c, &s_t)) {
    // valid entries end at n (chunks never straddle fixed-capacity slices)
    if (threadIdx.x == 0) s_end = ext.end_of(c * chunk, n_all);
    __syncthreads();
    const uint64_t n = s_end;
    const uint64_t c0 = c * chunk + threadIdx.x;
    double kc[kPartProbeItems];
#pragma unroll
    for (int j = 0; j < kPartProbeItems; ++j) {
      const uint64_t i = c0 + (uint64_t)j * kProbeThreads;
      kc[j] = i < n ? ldg_stream_f64(keys + i, pol_stream) : 0.0;
    }
    for (int u = 0; u < kPartProbeSub; ++u) {
      const uint64_t base = c0 + (uint64_t)u * sub;
      if (base - threadIdx.x >= n) break;
      double kn[kPartProbeItems];
#pragma unroll
      for (int j = 0; j < kPartProbeItems; ++j) {
        const uint64_t i = base + sub + (uint64_t)j * kProbeThreads;
        kn[j] = (u + 1 < kPartProbeSub && i < n) ? ldg_stream_f64(keys + i, pol_stream) : 0.0;
      }
#if GOLP_PART_PROBE_QUEUE
      {
        const uint64_t bits = canon_bits(kc[0]);
        uint32_t h = home_slot32(bits, (uint32_t)mask), off = 0, cnt = 0;
        const bool valid = base < n;
        int st = 1;
        if (valid) {
          st = check_pair(ldg_pair(table + h, pol_table), bits, off, cnt, true);
          if (st >= 0) st_res(res_part + base, ((uint64_t)cnt << 32) | off);
        }
        unsigned need = __ballot_sync(0xFFFFFFFFu, st < 0);
        while (need) {  // queue the unresolved lanes; resolve the queue whenever it fills
          const unsigned room = 32u - qn;
          const unsigned take = __popc(need) <= room ? need : need & ((1u << (__fns(need, 0, room + 1))) - 1u);
          if ((take >> lane) & 1u) {
            const unsigned pos = qn + __popc(take & ((1u << lane) - 1u));
            q.bits[pos] = bits;
            q.h[pos] = (h + 2) & (uint32_t)mask;
            q.i[pos] = (uint32_t)base;
          }
          qn += __popc(take);
          need &= ~take;
          if (qn == 32u) {
            part_queue_drain(q, lane, 32u, table, mask, res_part, pol_table);
            qn = 0;
          }
        }
#if GOLP_PART_QUEUE_EVERY > 0
        // resolve the queue every few sub-tiles even when not full: a queued
        // entry leaves a hole in its sector of res_part, which costs a DRAM
        // read-modify-write if the sector leaves L2 before the hole is filled
        if (((u + 1) % GOLP_PART_QUEUE_EVERY) == 0 && qn) {
          part_queue_drain(q, lane, qn, table, mask, res_part, pol_table);
          qn = 0;
        }
#endif
        kc[0] = kn[0];
      }
#else
      uint64_t bits[kPartProbeItems];
      uint32_t h[kPartProbeItems], off[kPartProbeItems], cnt[kPartProbeItems];
      unsigned pending = 0;
#pragma unroll
      for (int j = 0; j < kPartProbeItems; ++j) {
        bits[j] = canon_bits(kc[j]);
        h[j] = home_slot32(bits[j], (uint32_t)mask);
        off[j] = 0;
        cnt[j] = 0;
        if (base + (uint64_t)j * kProbeThreads < n) pending |= 1u << j;
      }
      bool home = true;
      while (pending) {
        ulonglong4 sl[kPartProbeItems];
#pragma unroll
        for (int j = 0; j < kPartProbeItems; ++j)
          if (pending & (1u << j)) sl[j] = ldg_pair(table + h[j], pol_table);
#pragma unroll
        for (int j = 0; j < kPartProbeItems; ++j) {
          if (!(pending & (1u << j))) continue;
          const int st = check_pair(sl[j], bits[j], off[j], cnt[j], home);
          if (st >= 0) pending &= ~(1u << j);
          else h[j] = (h[j] + 2) & (uint32_t)mask;
        }
        home = false;
      }
#pragma unroll
      for (int j = 0; j < kPartProbeItems; ++j) {
        const uint64_t i = base + (uint64_t)j * kProbeThreads;
        if (i < n) st_res(res_part + i, ((uint64_t)cnt[j] << 32) | off[j]);
        kc[j] = kn[j];
      }
#endif
    }
  }
#if GOLP_PART_PROBE_QUEUE
  if (qn) part_queue_drain(q, lane, qn, table, mask, res_part, pol_table);
#endif
}

// Match stage of the radix-partitioned probe: block b owns partition tile b
// (kPartTile probes). It gathers the tile's lookup results from its runs in
// res_part (one contiguous run per slice) into shared memory at their recorded
// in-tile indices, then its warps append hits exactly like join_match_kernel
// with per_warp = kRunWarpTiles, so scan_partials/emit are shared.
constexpr uint32_t kRunWarpTiles = kPartTile / (kProbeWarps * kWarpTile);
static_assert(kRunWarpTiles * kProbeWarps * kWarpTile == kPartTile, "partition tile must split into warp tiles");
constexpr size_t kRunSmem = (size_t)kPartTile * 8;

__global__ void __launch_bounds__(kProbeThreads) join_match_runs_kernel(
    RowCol prows, uint64_t np, const uint64_t* __restrict__ res_part,
    const uint16_t* __restrict__ idx, const uint32_t* __restrict__ run_base, const uint16_t* __restrict__ run_len,
    uint32_t nparts, MatchScratch sc, unsigned long long* __restrict__ bpart) {
  extern __shared__ __align__(16) uint64_t s_res[];  // kPartTile entries
  __shared__ unsigned s_cnt[kMaxProbeParts], s_start[kMaxProbeParts], s_base[kMaxProbeParts];
  __shared__ uint8_t s_pj[kPartTile];  // slice of the j-th entry of the tile's concatenated runs
  __shared__ unsigned long long s_w[33];
  static_assert(kMaxProbeParts <= 256, "s_pj stores slice ids as bytes");
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint64_t pol = policy_evict_first();
  const uint64_t t = blockIdx.x, t0 = t * kPartTile;
  const uint32_t tcnt = (uint32_t)(np - t0 < kPartTile ? np - t0 : kPartTile);
  for (uint32_t p = threadIdx.x; p < nparts; p += blockDim.x) {
    s_cnt[p] = run_len[t * nparts + p];
    s_base[p] = run_base[t * nparts + p];
  }
  __syncthreads();
  block_scan_parts(s_cnt, s_start, nparts, s_w);
  for (uint32_t p = threadIdx.x; p < nparts; p += blockDim.x) {  // expand runs -> slice id per entry
    const uint32_t b = s_start[p], e = b + s_cnt[p];
    for (uint32_t j = b; j < e; ++j) s_pj[j] = (uint8_t)p;
  }
  __syncthreads();
  constexpr int kBatch = 8;  // independent gathers in flight per thread
  for (uint32_t j0 = threadIdx.x; j0 < tcnt; j0 += kBatch * kProbeThreads) {
    uint64_t v[kBatch];
    uint32_t d[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const uint32_t j = j0 + u * kProbeThreads;
      if (j < tcnt) {
        const uint32_t p = s_pj[j];
        const uint64_t src = (uint64_t)s_base[p] + (j - s_start[p]);
        d[u] = idx[src];
        v[u] = ldg_stream_u64(res_part + src, pol);
      }
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (j0 + u * kProbeThreads < tcnt) s_res[d[u]] = v[u];
  }
  __syncthreads();
  const uint64_t gw = t * kProbeWarps + warp;
  const uint64_t nwt = (np + kWarpTile - 1) / kWarpTile;
  const uint64_t lo = gw * kRunWarpTiles, hi = lo + kRunWarpTiles < nwt ? lo + kRunWarpTiles : nwt;
  uint64_t cursor = lo * kWarpTile;
  uint64_t pairs_total = 0;
  uint32_t nrow[kWarpItems];  // the next warp tile's probe rows, loaded one tile ahead
#pragma unroll
  for (int j = 0; j < kWarpItems; ++j) {
    const uint64_t i = lo * kWarpTile + lane * kWarpItems + j;
    nrow[j] = lo < hi && i < np ? prows.at_cs(i) : 0u;
  }
  for (uint64_t wt = lo; wt < hi; ++wt) {
    const uint64_t first = wt * kWarpTile + lane * kWarpItems;
    uint32_t off[kWarpItems], cnt[kWarpItems], prow[kWarpItems];
#pragma unroll
    for (int j = 0; j < kWarpItems; ++j) {
      const uint64_t v = first + j < np ? s_res[first + j - t0] : 0ull;
      off[j] = (uint32_t)v;
      cnt[j] = (uint32_t)(v >> 32);
      prow[j] = nrow[j];
      const uint64_t i = first + kWarpTile + j;
      nrow[j] = wt + 1 < hi && i < np ? prows.at_cs(i) : 0u;
    }
    pairs_total += warp_append_hits(lane, off, cnt, prow, sc, cursor);
  }
  finish_match_block(lane, warp, gw, lo, cursor, pairs_total, sc, s_w, bpart);
}

// Same block/warp -> tile mapping as join_match_kernel. bpart holds the pair
// totals of the match blocks. With few blocks (kScanned = false) each emit block
// sums the totals of the blocks before it (at most a few thousand L2-resident
// words) on top of *base_in, so no separate scan launch is needed, and the last
// block writes *total_out; with many, scan_partials_kernel has already turned
// bpart into exclusive offsets. A warp's offset adds the pairs of the earlier
// warps of its block. Singletons (slot.off is the build row) are a straight
// coalesced copy; key groups expand their CSR run.
constexpr uint64_t kInlineScanBlocks = 4096;
template <bool kScanned>
__global__ void __launch_bounds__(kProbeThreads) join_emit_kernel(MatchScratch sc, const uint32_t* __restrict__ csr_row,
                                                                  uint64_t nwt, uint64_t per_warp,
                                                                  const unsigned long long* __restrict__ bpart,
                                                                  const unsigned long long* __restrict__ base_in,
                                                                  unsigned long long* __restrict__ total_out,
                                                                  uint32_t* __restrict__ out_p,
                                                                  uint32_t* __restrict__ out_b, uint64_t cap,
                                                                  const uint32_t* __restrict__ row_base) {
  __shared__ unsigned long long s_wp[kProbeWarps];
  __shared__ unsigned long long s_red[kProbeWarps];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint64_t gw = (uint64_t)blockIdx.x * kProbeWarps + warp;
  if constexpr (!kScanned) {  // exclusive offset of this block: sum of the earlier blocks' totals
    unsigned long long acc = 0;
    for (unsigned b = threadIdx.x; b < blockIdx.x; b += blockDim.x) acc += __ldcg(bpart + b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    if (lane == 0) s_red[warp] = acc;
  }
  const uint64_t lo = gw * per_warp;
  if (lane == 0) s_wp[warp] = lo < nwt ? sc.wpairs[gw] : 0ull;
  __syncthreads();
  unsigned long long run;
  if constexpr (kScanned) {
    run = bpart[blockIdx.x];
  } else {
    run = base_in ? *base_in : 0ull;
    for (unsigned w = 0; w < kProbeWarps; ++w) run += s_red[w];
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *total_out = run + __ldcg(bpart + blockIdx.x);
  }
  for (unsigned w = 0; w < warp; ++w) run += s_wp[w];
  if (lo >= nwt) return;
  const uint64_t pol_stream = policy_evict_first();
  const uint32_t rb = __ldg(row_base);
  const uint64_t e0 = lo * kWarpTile;
  const uint32_t ne = sc.wentries[gw];
#ifndef GOLP_EMIT_BATCH
#define GOLP_EMIT_BATCH 4
#endif
  constexpr int kBatch = GOLP_EMIT_BATCH;  // kBatch x 32 entries in flight per warp iteration
  for (uint32_t i0 = 0; i0 < ne; i0 += 32 * kBatch) {
    uint32_t c[kBatch], pr[kBatch], of[kBatch];
#pragma unroll
    for (int q = 0; q < kBatch; ++q) {
      const uint32_t i = i0 + q * 32 + lane;
      c[q] = 0;
      pr[q] = 0;
      of[q] = 0;
      if (i < ne) {
        const uint64_t v = __ldcs(reinterpret_cast<const unsigned long long*>(sc.oc) + e0 + i);
        c[q] = (uint32_t)(v >> 32);  // the slot's cnt word
        of[q] = (uint32_t)v;
        pr[q] = __ldcs(sc.prow + e0 + i);
      }
    }
#pragma unroll
    for (int q = 0; q < kBatch; ++q) {
      const uint32_t cw = c[q];
      c[q] = slot_members(cw);
      uint64_t incl;
      if (__any_sync(0xFFFFFFFFu, c[q] >= (1u << 26))) {  // huge key groups: 64-bit scan
        incl = c[q];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint64_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if ((int)lane >= o) incl += v;
        }
      } else {  // 32 counts below 2^26 cannot overflow a 32-bit scan
        uint32_t i32 = c[q];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, i32, o);
          if ((int)lane >= o) i32 += v;
        }
        incl = i32;
      }
      unsigned long long g = run + (incl - c[q]);
      if (c[q] == 1) {  // singleton: slot.off is its row, or its position past the first row id
        if (g < cap) {
          st_hint(out_p + g, pr[q], pol_stream);
          st_hint(out_b + g, of[q] + rb, pol_stream);
        }
      } else if (cw & kPair2Bit) {  // an inline pair: both rows came with the slot
        if (g < cap) {
          st_hint(out_p + g, pr[q], pol_stream);
          st_hint(out_b + g, of[q], pol_stream);
        }
        if (g + 1 < cap) {
          st_hint(out_p + g + 1, pr[q], pol_stream);
          st_hint(out_b + g + 1, cw & kPair2Row, pol_stream);
        }
      } else {
        // a key group: its rows are contiguous (CSR / side array); four
        // independent loads per step instead of one dependent load per member
        for (uint32_t m0 = 0; m0 < c[q]; m0 += 4) {
          uint32_t br[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) br[u] = m0 + u < c[q] ? __ldg(csr_row + of[q] + m0 + u) : 0u;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const unsigned long long gg = g + m0 + u;
            if (m0 + u < c[q] && gg < cap) {
              st_hint(out_p + gg, pr[q], pol_stream);
              st_hint(out_b + gg, br[u], pol_stream);
            }
          }
        }
      }
      run += __shfl_sync(0xFFFFFFFFu, incl, 31);
    }
  }
}

}  // namespace golp
