// Hash-join probe for tables probed directly (the table fits L2, or is not
// radix-partitioned): the B200 replacement for host_hash_probe and
// ProxyDevice._probe_chunk (pkg/src/golp/host.py:168-188,
// pkg/src/golp/device.py:262-296).
//
// Two launches, no per-hit scratch round trip through HBM:
//   join_probe_lookup_kernel : every WARP is an independent worker that claims
//       tiles of kPSpan consecutive probes in order (atomic ticket) and, per tile,
//       1. stage  : the tile's probe keys and probe rows arrive in the warp's
//                   shared-memory slice by TMA bulk copies (cp.async.bulk +
//                   mbarrier), double-buffered: the next tile's copy is issued
//                   before the current tile's lookups start;
//       2. lookup : every lane keeps kPQueue independent lookups in flight and
//                   refills a slot from its own probe list as soon as that probe
//                   resolves (hit, or an empty slot / an unflagged home pair ends
//                   the linear probe, join.cuh kOverflowBit); the packed slot
//                   {off | cnt << 32} (0 = miss) overwrites the staged key;
//       3. emit   : the tile's pair count reserves a contiguous run of a pair
//                   staging area with one atomic (no wait for earlier tiles);
//                   rows of 32 consecutive probes (lane = probe) get in-row
//                   offsets from ballots, key groups of 2..kInline members
//                   read their rows with one 16-byte load issued for all rows
//                   of the tile before the first store; consecutive hits land
//                   at consecutive positions, so the stores coalesce.
//   join_probe_place_kernel  : scans the tile pair counts into output offsets
//       (tile order = probe order, chained after *base_in; decoupled look-back
//       over blocks of tiles) and copies each tile's staged run there.
// Output order = probe position, then build insertion position (the table's
// per-key row lists are already in insertion order, join.cuh).
#pragma once
#include "join.cuh"

namespace golp {

#ifndef GOLP_PROBE_ITEMS
#define GOLP_PROBE_ITEMS 8
#endif
#ifndef GOLP_PROBE_QUEUE
#define GOLP_PROBE_QUEUE 2
#endif
#ifndef GOLP_PROBE_THREADS
#define GOLP_PROBE_THREADS 256
#endif
#ifndef GOLP_PROBE_BLOCKS
#define GOLP_PROBE_BLOCKS 4
#endif
constexpr int kPThreads = GOLP_PROBE_THREADS;
constexpr int kPWarps = kPThreads / 32;
constexpr int kPItems = GOLP_PROBE_ITEMS;  // probes per lane per tile
constexpr int kPQueue = GOLP_PROBE_QUEUE;  // lookups in flight per lane
constexpr uint32_t kPSpan = 32u * kPItems;  // probes per (warp) tile
// Group rows staged per tile (expected ~23 per 256 probes at C2's duplicate rate;
// groups beyond the cap read their rows from global memory in the emit).
constexpr uint32_t kPGroupCap = 48;
// Packed per-probe result in shared memory: off | cnt << 32 | kResStaged (rows of
// the group at S.grp[off] instead of the table's row array).
constexpr uint64_t kResStaged = 1ull << 62;
constexpr uint32_t kResCntMask = (1u << 30) - 1u;
static_assert(kPSpan * 4 % 16 == 0, "TMA copies need 16-byte multiples");

// Shared memory of one warp: two stage buffers of kPSpan keys (-> packed slots)
// and kPSpan probe rows, plus their two mbarriers.
struct __align__(16) ProbeWarpSmem {
  uint64_t key[2][kPSpan];
  uint32_t row[2][kPSpan];
  uint4 grp[kPGroupCap];  // rows of the current tile's 2..kInline-member groups
  uint64_t bar[2];
  unsigned ngrp;
};
constexpr size_t kPSmem = sizeof(ProbeWarpSmem) * kPWarps;

struct ProbeLookupArgs {
  const double* keys;
  const uint32_t* rows;
  uint64_t np;
  const Slot* table;
  uint32_t mask;
  const uint32_t* csr_row;          // group rows (side array + CSR ranges)
  const uint32_t* row_base;         // added to a singleton's slot.off (dense build rows)
  uint32_t* stage_p;                // pair staging area (stage_cap pairs)
  uint32_t* stage_b;
  uint64_t stage_cap;
  unsigned long long* bump;         // staging allocator, zeroed
  unsigned long long* ticket;       // tile counter, zeroed
  unsigned long long* tile_count;   // [ntiles] pairs of each tile
  unsigned long long* tile_stage;   // [ntiles] start of each tile's staged run
};

__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar)), "l"(pol)
      : "memory");
}

// One 16-byte row group (groups of 2..kInline members live 16-byte aligned at h*kInline).
__device__ __forceinline__ uint4 ldg_group(const uint32_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ void put_pair(uint32_t* __restrict__ out_p, uint32_t* __restrict__ out_b, uint64_t g,
                                         uint64_t cap, uint32_t pr, uint32_t br) {
  if (g < cap) {
    out_p[g] = pr;
    out_b[g] = br;
  }
}

__device__ __forceinline__ uint32_t u4_at(const uint4& v, uint32_t i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// Rows of a key group that is not staged in shared memory: lane by lane from
// the table's row array (groups above kInline members, or past the staging cap).
__device__ __forceinline__ void emit_group_global(const uint32_t* __restrict__ csr, uint32_t off, uint32_t cnt,
                                                  uint32_t pr, uint32_t* sp, uint32_t* sb) {
  for (uint32_t m0 = 0; m0 < cnt; m0 += 4) {
    uint32_t br[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) br[u] = m0 + u < cnt ? __ldg(csr + off + m0 + u) : 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (m0 + u < cnt) {
        sp[m0 + u] = pr;
        sb[m0 + u] = br[u];
      }
  }
}

// Writes one tile's pairs in probe order to sp/sb (its staged run, < 2^31 pairs):
// rows of 32 consecutive probes, lane = probe; in-row offsets from ballots plus
// the extra members of the row's key groups.
__device__ __forceinline__ void emit_tile(const ProbeLookupArgs& a, const ProbeWarpSmem& S, const uint64_t* sk,
                                          const uint32_t* sr, uint32_t wn, unsigned lane, uint32_t* sp, uint32_t* sb,
                                          uint32_t rb) {
  const unsigned lt = (1u << lane) - 1u;
  uint32_t cur = 0;
#pragma unroll 1
  for (int e = 0; e < kPItems; ++e) {
    const uint32_t j = e * 32 + lane;
    const uint64_t v = j < wn ? sk[j] : 0ull;
    const uint32_t cnt = (uint32_t)(v >> 32) & kResCntMask, off = (uint32_t)v;
    const unsigned hit = __ballot_sync(0xFFFFFFFFu, cnt != 0);
    unsigned grps = __ballot_sync(0xFFFFFFFFu, cnt > 1);
    uint32_t o = cur + __popc(hit & lt);
    cur += __popc(hit);
    while (grps) {  // extra pairs of the row's key groups
      const int src = __ffs(grps) - 1;
      grps &= grps - 1;
      const uint32_t x = __shfl_sync(0xFFFFFFFFu, cnt, src) - 1u;
      o += (src < (int)lane) ? x : 0u;
      cur += x;
    }
    const unsigned big = __ballot_sync(0xFFFFFFFFu, cnt > 32);
    const uint32_t pr = cnt ? sr[j] : 0u;
    if (cnt == 1) {
      sp[o] = pr;
      sb[o] = off + rb;
    } else if (v & kResStaged) {
      const uint4 r = S.grp[off];
      sp[o] = pr;
      sp[o + 1] = pr;
      sb[o] = r.x;
      sb[o + 1] = r.y;
      if (cnt > 2) {
        sp[o + 2] = pr;
        sb[o + 2] = r.z;
      }
      if (cnt > 3) {
        sp[o + 3] = pr;
        sb[o + 3] = r.w;
      }
    } else if (cnt > 1 && cnt <= 32) {
      emit_group_global(a.csr_row, off, cnt, pr, sp + o, sb + o);
    }
    for (unsigned bg = big; bg; bg &= bg - 1) {  // big groups: the whole warp copies each row range
      const int src = __ffs(bg) - 1;
      const uint32_t bc = __shfl_sync(0xFFFFFFFFu, cnt, src), bo = __shfl_sync(0xFFFFFFFFu, off, src);
      const uint32_t bp = __shfl_sync(0xFFFFFFFFu, pr, src), bd = __shfl_sync(0xFFFFFFFFu, o, src);
      for (uint32_t m = lane; m < bc; m += 32) {
        sp[bd + m] = bp;
        sb[bd + m] = __ldg(a.csr_row + bo + m);
      }
    }
  }
}

// Same for a run of 2^31 or more pairs (huge key groups): 64-bit offsets, lane-serial.
__device__ __forceinline__ void emit_tile_wide(const ProbeLookupArgs& a, const ProbeWarpSmem& S, const uint64_t* sk,
                                            const uint32_t* sr, uint32_t wn, unsigned lane, uint64_t run, uint32_t rb) {
  uint64_t cur = run;
  for (int e = 0; e < kPItems; ++e) {
    const uint32_t j = e * 32 + lane;
    const uint64_t v = j < wn ? sk[j] : 0ull;
    const uint64_t cnt = (v >> 32) & kResCntMask;
    uint64_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if ((int)lane >= o) incl += u;
    }
    const uint64_t g = cur + incl - cnt;
    const uint32_t off = (uint32_t)v, pr = cnt ? sr[j] : 0u;
    for (uint64_t m = 0; m < cnt; ++m) {
      a.stage_p[g + m] = pr;
      uint32_t br;
      if (cnt == 1) br = off + rb;
      else if (v & kResStaged) br = u4_at(S.grp[off], (uint32_t)m);
      else br = __ldg(a.csr_row + off + m);
      a.stage_b[g + m] = br;
    }
    cur += __shfl_sync(0xFFFFFFFFu, incl, 31);
  }
}

__global__ void __launch_bounds__(kPThreads, GOLP_PROBE_BLOCKS) join_probe_lookup_kernel(ProbeLookupArgs a) {
  extern __shared__ __align__(16) unsigned char p_smem[];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  ProbeWarpSmem& S = reinterpret_cast<ProbeWarpSmem*>(p_smem)[warp];
  const uint64_t pol_stream = policy_evict_first(), pol_table = policy_evict_last();
  const uint64_t ntiles = (a.np + kPSpan - 1) / kPSpan;
  const uint32_t rb = __ldg(a.row_base);
  // TMA needs 16-byte aligned sources: row tiles start at multiples of
  // kPSpan*4 bytes, key tiles at kPSpan*8, so aligned bases suffice.
#ifdef GOLP_PROBE_NO_TMA  // tuning knob: plain staging loads
  const bool tma = false;
#else
  const bool tma = ((reinterpret_cast<uintptr_t>(a.keys) | reinterpret_cast<uintptr_t>(a.rows)) & 15) == 0;
#endif
  if (lane == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned phase = 0;  // bit b: parity of the next completion of bar[b]

#ifdef GOLP_PROBE_STATIC_TILES  // tuning knob: grid-stride tile order instead of a ticket
  uint64_t next_static = (uint64_t)blockIdx.x * kPWarps + warp;
  const uint64_t stride_static = (uint64_t)gridDim.x * kPWarps;
  auto claim = [&]() -> uint64_t {
    const uint64_t t = next_static;
    next_static += stride_static;
    return t;
  };
#else
  auto claim = [&]() -> uint64_t {
    uint64_t t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1ull);
    return __shfl_sync(0xFFFFFFFFu, t, 0);
  };
#endif
  auto full_tile = [&](uint64_t t) { return tma && (t + 1) * kPSpan <= a.np; };
  auto stage = [&](uint64_t t, int b) {  // full tiles: bulk copies issued by lane 0
    if (t >= ntiles || !full_tile(t)) return;
    if (lane == 0) {
      mbar_expect(&S.bar[b], kPSpan * 12);
      bulk_copy(S.key[b], a.keys + t * kPSpan, kPSpan * 8, &S.bar[b], pol_stream);
      bulk_copy(S.row[b], a.rows + t * kPSpan, kPSpan * 4, &S.bar[b], pol_stream);
    }
  };

  uint64_t t = claim();
  stage(t, 0);
  int b = 0;
  while (t < ntiles) {
    const uint64_t tn = claim();  // next tile: its copy overlaps this tile's lookups
    stage(tn, b ^ 1);
    const uint64_t w0 = t * kPSpan;
    const uint32_t wn = a.np - w0 < kPSpan ? (uint32_t)(a.np - w0) : kPSpan;
    uint64_t* sk = S.key[b];
    uint32_t* sr = S.row[b];
    if (full_tile(t)) {
      mbar_wait(&S.bar[b], (phase >> b) & 1u);
      phase ^= 1u << b;
    } else {  // partial or unaligned tile: plain loads
#pragma unroll
      for (int e = 0; e < kPItems; ++e) {
        const uint32_t j = e * 32 + lane;
        if (j < wn) {
          sk[j] = __double_as_longlong(ldg_stream_f64(a.keys + w0 + j, pol_stream));
          sr[j] = __ldcs(a.rows + w0 + j);
        }
      }
      __syncwarp();
    }

    // lookups: kPQueue in flight per lane, refilled in probe order. A hit on a
    // group of 2..kInline members re-arms its slot once more to fetch the
    // group's rows (one 16-byte load) into the warp's group area.
    if (lane == 0) S.ngrp = 0;
    __syncwarp();
    uint32_t nxt = 0;
    uint32_t idx[kPQueue], h[kPQueue];  // probe index (lookup) / group-area index (fetch); slot / row offset
    uint64_t bits[kPQueue];
    unsigned act = 0, home = 0, fetch = 0;  // per slot q: active / at its home pair / fetching group rows
    auto start = [&](int q) {
      const uint32_t j = nxt * 32 + lane;
      if (nxt < (uint32_t)kPItems && j < wn) {
        bits[q] = canon_bits(__longlong_as_double((long long)sk[j]));
        h[q] = home_slot32(bits[q], a.mask);
        idx[q] = j;
        act |= 1u << q;
        home |= 1u << q;
        ++nxt;
      } else {
        act &= ~(1u << q);
      }
    };
#pragma unroll
    for (int q = 0; q < kPQueue; ++q) start(q);
    while (__any_sync(0xFFFFFFFFu, act != 0)) {
      ulonglong4 sl[kPQueue];
#pragma unroll
      for (int q = 0; q < kPQueue; ++q) {
        if (!(act & (1u << q))) continue;
        if (fetch & (1u << q)) {
          const uint4 r = ldg_group(a.csr_row + h[q]);
          sl[q].x = ((uint64_t)r.y << 32) | r.x;
          sl[q].y = ((uint64_t)r.w << 32) | r.z;
        } else {
          sl[q] = ldg_pair(a.table + h[q], pol_table);
        }
      }
#pragma unroll
      for (int q = 0; q < kPQueue; ++q) {
        if (!(act & (1u << q))) continue;
        if (fetch & (1u << q)) {
          S.grp[idx[q]] = make_uint4((uint32_t)sl[q].x, (uint32_t)(sl[q].x >> 32), (uint32_t)sl[q].y,
                                     (uint32_t)(sl[q].y >> 32));
          fetch &= ~(1u << q);
          start(q);
          continue;
        }
        uint32_t off = 0, cnt = 0;
        const int st = check_pair(sl[q], bits[q], off, cnt, (home >> q) & 1u);
        if (st < 0) {
          h[q] = (h[q] + 2) & a.mask;
          home &= ~(1u << q);
          continue;
        }
        uint64_t res = st ? (((uint64_t)cnt << 32) | off) : 0ull;
        const uint32_t j = idx[q];
#ifdef GOLP_PROBE_NO_GROUP_FETCH  // tuning knob: group rows read in the emit
        if (false) {
#else
        if (st && cnt >= 2 && cnt <= kInline) {
#endif
          const unsigned gi = atomicAdd(&S.ngrp, 1u);
          if (gi < kPGroupCap) {
            res = ((uint64_t)cnt << 32) | kResStaged | gi;
            fetch |= 1u << q;
            h[q] = off;
            idx[q] = gi;
          }
        }
        sk[j] = res;
        if (!(fetch & (1u << q))) start(q);
      }
    }
    __syncwarp();

    // pair count -> a contiguous staged run (one atomic, no wait on other tiles)
    uint64_t agg = 0;
#pragma unroll
    for (int e = 0; e < kPItems; ++e) {
      const uint32_t j = e * 32 + lane;
      agg += j < wn ? ((sk[j] >> 32) & kResCntMask) : 0ull;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) agg += __shfl_xor_sync(0xFFFFFFFFu, agg, o);
    uint64_t run = 0;
    if (lane == 0) {
      run = atomicAdd(a.bump, (unsigned long long)agg);
      a.tile_count[t] = agg;
      a.tile_stage[t] = run;
    }
    run = __shfl_sync(0xFFFFFFFFu, run, 0);
    // a run that does not fit the staging area is not written (M > cap: the
    // caller re-probes with larger buffers); runs of 2^31+ pairs take 64-bit offsets
#ifdef GOLP_PROBE_DIAG_NO_EMIT  // diagnostic only: lookups without pair writes
    if (false)
#else
    if (run + agg <= a.stage_cap && agg < (1ull << 31))
#endif
      emit_tile(a, S, sk, sr, wn, lane, a.stage_p + run, a.stage_b + run, rb);
    else if (run + agg <= a.stage_cap)
      emit_tile_wide(a, S, sk, sr, wn, lane, run, rb);
    __syncwarp();  // buffer b is restaged two tiles from now
    t = tn;
    b ^= 1;
  }
}

// Tile status words of the placement's look-back: flag in the top two bits,
// pair count below.
constexpr uint64_t kStatAgg = 1ull << 62;
constexpr uint64_t kStatInc = 2ull << 62;
constexpr uint64_t kStatVal = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_relaxed_u64(const unsigned long long* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Exclusive prefix of block-group q (warp-wide look-back over the preceding
// groups' published aggregates / inclusive prefixes; every lane returns it).
__device__ __forceinline__ uint64_t lookback(unsigned long long* status, uint64_t q, unsigned lane) {
  uint64_t excl = 0;
  int64_t p = (int64_t)q - 1;
  while (true) {
    const int64_t r = p - (int64_t)lane;
    uint64_t v = kStatInc;  // (never reached: group 0 always publishes an inclusive prefix)
    if (r >= 0) {
      do {
        v = ld_relaxed_u64(status + r);
      } while ((v >> 62) == 0);
    }
    const unsigned inc = __ballot_sync(0xFFFFFFFFu, (v >> 62) == 2);
    const unsigned take = inc ? ((inc & (0u - inc)) << 1) - 1u : 0xFFFFFFFFu;  // up to the nearest inclusive one
    uint64_t x = ((take >> lane) & 1u) ? (v & kStatVal) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
    excl += x;
    if (inc) return excl;
    p -= 32;
  }
}

// Places the staged pairs: block q takes kPlaceTiles (= 32) consecutive tiles;
// warp 0 scans their pair counts and gets the pairs of all earlier tiles by
// decoupled look-back over the blocks before it (+ *base_in); then every warp
// copies some of the tiles' staged runs to their output offsets. The last
// block writes *total_out.
constexpr int kPlaceTiles = 32;
constexpr int kPlaceThreads = 256;
__global__ void __launch_bounds__(kPlaceThreads) join_probe_place_kernel(
    const uint32_t* __restrict__ stage_p, const uint32_t* __restrict__ stage_b, uint64_t stage_cap,
    const unsigned long long* __restrict__ tile_count, const unsigned long long* __restrict__ tile_stage,
    uint64_t ntiles, unsigned long long* status, const unsigned long long* __restrict__ base_in,
    unsigned long long* __restrict__ total_out, uint32_t* __restrict__ out_p, uint32_t* __restrict__ out_b,
    uint64_t cap) {
  __shared__ unsigned long long s_dst[kPlaceTiles], s_n[kPlaceTiles], s_src[kPlaceTiles];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint64_t q = blockIdx.x, t0 = q * kPlaceTiles;
  if (warp == 0) {
    const uint64_t t = t0 + lane;
    const uint64_t c = t < ntiles ? tile_count[t] : 0ull;
    uint64_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if ((int)lane >= o) incl += u;
    }
    const uint64_t agg = __shfl_sync(0xFFFFFFFFu, incl, 31);
    uint64_t excl;
    if (q == 0) {
      excl = *base_in;
      if (lane == 0) st_relaxed_u64(status, kStatInc | (excl + agg));
    } else {
      if (lane == 0) st_relaxed_u64(status + q, kStatAgg | agg);
      excl = lookback(status, q, lane);
      if (lane == 0) st_relaxed_u64(status + q, kStatInc | (excl + agg));
    }
    if (lane == 0 && q == gridDim.x - 1) *total_out = excl + agg;
    s_dst[lane] = excl + incl - c;
    s_n[lane] = c;
    s_src[lane] = t < ntiles ? tile_stage[t] : 0ull;
  }
  __syncthreads();
  for (unsigned k = warp; k < (unsigned)kPlaceTiles; k += kPlaceThreads / 32) {
    const uint64_t dst = s_dst[k], n = s_n[k], src = s_src[k];
    for (uint64_t i = lane; i < n; i += 32) {
      if (src + i >= stage_cap || dst + i >= cap) break;
      out_p[dst + i] = __ldcs(stage_p + src + i);
      out_b[dst + i] = __ldcs(stage_b + src + i);
    }
  }
}

}  // namespace golp
