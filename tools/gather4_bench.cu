// Random 32-byte row lookups from an L2-resident table: LSU loads (one
// LDG.256 per lookup, the probe kernels' way) against TMA tile::gather4 (one
// cp.async.bulk.tensor per 4 rows, the TMA unit instead of L1TEX request
// slots). Table = C2's 2^21 16-B slots viewed as 2^20 rows of 32 B; 1e7 lookups.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/gather4_bench tools/gather4_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e = (x);                                                      \
    if (e != cudaSuccess) {                                                   \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 27; z *= 0x94D049BB133111EBull; z ^= z >> 31; return z;
}

// (a) one 256-bit LDG per lookup, W lookups in flight per thread
template <int W>
__global__ void ldg_lookups(const ulonglong4* __restrict__ rows, uint32_t mask, uint64_t n, unsigned long long* out) {
  unsigned long long acc = 0;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, st = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = tid * W; i < n; i += st * W) {
    ulonglong4 v[W];
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const ulonglong4* p = rows + (mix64(i + j) & mask);
      asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(v[j].x), "=l"(v[j].y), "=l"(v[j].z), "=l"(v[j].w) : "l"(p));
    }
#pragma unroll
    for (int j = 0; j < W; ++j) acc += v[j].x == 5;
  }
  if (acc == 0x123456) *out = acc;
}

// (b) TMA gather4: each lane issues one gather of 4 random rows (128 B) into
// its shared-memory slot; the warp waits on one mbarrier per round (32 x 128 B).
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(b),
               "r"(phase) : "memory");
}

template <int ROUNDS_IN_FLIGHT>
__global__ void __launch_bounds__(256) tma_gather_lookups(const __grid_constant__ CUtensorMap tmap, uint32_t mask,
                                                           uint64_t n, unsigned long long* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr unsigned kBytes = 32 * 128;  // one round: 32 lanes x 4 rows x 32 B
  unsigned char* wbuf = smem + (size_t)warp * ROUNDS_IN_FLIGHT * kBytes;  // 128-byte aligned slots
  __shared__ __align__(8) uint64_t s_bars[8 * ROUNDS_IN_FLIGHT];
  uint64_t* bars = s_bars + warp * ROUNDS_IN_FLIGHT;
  if (lane == 0)
    for (int r = 0; r < ROUNDS_IN_FLIGHT; ++r) mbar_init(&bars[r], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  unsigned long long acc = 0;
  const uint64_t wid = blockIdx.x * (uint64_t)(blockDim.x >> 5) + warp, nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t per_round = 32 * 4;
  uint64_t r = 0;
  unsigned phase = 0;
  auto issue = [&](uint64_t base, int slot) {
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bars[slot])),
                   "r"(kBytes) : "memory");
    }
    __syncwarp();
    const uint64_t i = base + lane * 4;
    const int r0 = (int)(mix64(i) & mask), r1 = (int)(mix64(i + 1) & mask), r2 = (int)(mix64(i + 2) & mask),
              r3 = (int)(mix64(i + 3) & mask);
    const unsigned dst = (unsigned)__cvta_generic_to_shared(wbuf + slot * kBytes + lane * 128);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(&tmap), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"((unsigned)__cvta_generic_to_shared(&bars[slot]))
        : "memory");
  };
  const uint64_t rounds = (n + per_round - 1) / per_round;
  // keep ROUNDS_IN_FLIGHT rounds of this warp in flight
  uint64_t next = wid;
  for (int s = 0; s < ROUNDS_IN_FLIGHT; ++s, next += nw)
    if (next < rounds) issue(next * per_round, s);
  for (uint64_t t = wid; t < rounds; t += nw, ++r) {
    const int slot = (int)(r % ROUNDS_IN_FLIGHT);
    mbar_wait(&bars[slot], (phase >> slot) & 1u);
    phase ^= 1u << slot;
    const uint64_t* v = reinterpret_cast<const uint64_t*>(wbuf + slot * kBytes + lane * 128);
    acc += (v[0] == 5) + (v[4] == 5) + (v[8] == 5) + (v[12] == 5);
    __syncwarp();
    if (next < rounds) issue(next * per_round, slot);
    next += nw;
  }
  if (acc == 0x123456) *out = acc;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const uint64_t rows = 1u << 20, n = 10'000'000;
  ulonglong4* table;
  unsigned long long* out;
  CK(cudaMalloc(&table, rows * 32));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(table, 1, rows * 32));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  auto timeit = [&](const char* name, auto launch) {
    float best = 1e9f;
    for (int rep = 0; rep < 10; ++rep) {
      CK(cudaEventRecord(a));
      launch();
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      if (rep) best = ms < best ? ms : best;
    }
    printf("%-44s %8.1f us  %6.1f G lookups/s  (%s)\n", name, best * 1e3, n / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  timeit("LDG.256 W4, 592x256", [&] { ldg_lookups<4><<<sms * 4, 256>>>(table, rows - 1, n, out); });
  timeit("LDG.256 W8, 592x256", [&] { ldg_lookups<8><<<sms * 4, 256>>>(table, rows - 1, n, out); });

  EncodeTiled encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q));
  CUtensorMap tmap;
  const cuuint64_t dims[2] = {4, rows};         // 4 u64 per row, rows
  const cuuint64_t strides[1] = {32};           // bytes between rows
  const cuuint32_t box[2] = {4, 1};             // gather4: one row per index
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, table, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("tensor map encode: %d\n", (int)cr);
  for (int per_sm : {1, 2, 4}) {
    constexpr int R = 4;
    const size_t smem = 8 * R * (32 * 128);
    CK(cudaFuncSetAttribute(tma_gather_lookups<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    char name[64];
    snprintf(name, 64, "TMA gather4, 4 rounds/warp, %dx256", sms * per_sm);
    timeit(name, [&] { tma_gather_lookups<R><<<sms * per_sm, 256, smem>>>(tmap, rows - 1, n, out); });
  }
  {
    constexpr int R = 8;
    const size_t smem = 8 * R * (32 * 128);
    CK(cudaFuncSetAttribute(tma_gather_lookups<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    timeit("TMA gather4, 8 rounds/warp, 148x256", [&] { tma_gather_lookups<R><<<sms, 256, smem>>>(tmap, rows - 1, n, out); });
  }
  return 0;
}
