// Memory-system microbenchmarks used to size the join probe (tools/, not product).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 27; z *= 0x94D049BB133111EBull; z ^= z >> 31; return z;
}

__global__ void stream_sum(const double2* __restrict__ a, uint64_t n2, double* out) {
  double s = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n2; i += (uint64_t)gridDim.x * blockDim.x) {
    double2 v = __ldg(a + i); s += v.x + v.y;
  }
  if (s == 12345.678) *out = s;
}

// random 32-byte (256-bit) loads: each thread does `per` independent lookups
template <int W>
__global__ void rand_read(const ulonglong4* __restrict__ t, uint64_t mask, uint64_t n, uint64_t* out) {
  uint64_t acc = 0;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, st = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = tid * W; i < n; i += st * W) {
    ulonglong4 v[W];
#pragma unroll
    for (int j = 0; j < W; ++j) {
      uint64_t h = mix64(i + j) & mask;
      asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(v[j].x), "=l"(v[j].y), "=l"(v[j].z), "=l"(v[j].w) : "l"(t + h));
    }
#pragma unroll
    for (int j = 0; j < W; ++j) acc += v[j].x ^ v[j].w;
  }
  if (acc == 0x1234567) *out = acc;
}

template <int W>
__global__ void rand_read16(const ulonglong2* __restrict__ t, uint64_t mask, uint64_t n, uint64_t* out) {
  uint64_t acc = 0;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, st = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = tid * W; i < n; i += st * W) {
    ulonglong2 v[W];
#pragma unroll
    for (int j = 0; j < W; ++j) v[j] = __ldg(t + (mix64(i + j) & mask));
#pragma unroll
    for (int j = 0; j < W; ++j) acc += v[j].x ^ v[j].y;
  }
  if (acc == 0x1234567) *out = acc;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  uint64_t* out; CK(cudaMalloc(&out, 8));
  void* flush; CK(cudaMalloc(&flush, 512 << 20));
  auto time_it = [&](const char* name, double bytes, auto fn) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaMemset(flush, r, 512 << 20);
      cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("%-44s %9.1f us  %8.1f GB/s (%s)\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  const uint64_t n = 10000000;
  double* keys; CK(cudaMalloc(&keys, n * 8)); cudaMemset(keys, 0, n * 8);
  time_it("stream 80 MB (double2, grid sms*8x256)", n * 8.0, [&] { stream_sum<<<sms * 8, 256>>>((double2*)keys, n / 2, (double*)out); });
  for (uint64_t tb : {uint64_t(16) << 20, uint64_t(64) << 20, uint64_t(1) << 30}) {
    void* t; CK(cudaMalloc(&t, tb)); cudaMemset(t, 1, tb);
    uint64_t m32 = tb / 32 - 1, m16 = tb / 16 - 1;
    char nm[128];
    // warm table into L2 where it fits: first launch after memset, measured best-of
    snprintf(nm, 128, "rand32B x1e7 table %llu MB W=4", (unsigned long long)(tb >> 20));
    time_it(nm, n * 32.0, [&] { rand_read<4><<<sms * 8, 256>>>((ulonglong4*)t, m32, n, out); });
    snprintf(nm, 128, "rand32B x1e7 table %llu MB W=8", (unsigned long long)(tb >> 20));
    time_it(nm, n * 32.0, [&] { rand_read<8><<<sms * 8, 256>>>((ulonglong4*)t, m32, n, out); });
    snprintf(nm, 128, "rand16B x1e7 table %llu MB W=8", (unsigned long long)(tb >> 20));
    time_it(nm, n * 16.0, [&] { rand_read16<8><<<sms * 8, 256>>>((ulonglong2*)t, m16, n, out); });
    // warm (no flush between)
    float ms; cudaEventRecord(a); rand_read<4><<<sms * 8, 256>>>((ulonglong4*)t, m32, n, out); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventRecord(a); rand_read<4><<<sms * 8, 256>>>((ulonglong4*)t, m32, n, out); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("  warm (no flush) rand32B W=4: %9.1f us\n", ms * 1e3);
    cudaFree(t);
  }
  return 0;
}
