// Random-address atomic throughput on B200 (tools/): 1e6 ops on an L2-resident
// 32 MB table and on a 4 GB table; with/without returned values; CAS then add.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 27; z *= 0x94D049BB133111EBull; z ^= z >> 31; return z;
}
template <int MODE, int W>
__global__ void k(unsigned long long* t, uint64_t mask, uint64_t n, unsigned long long* out) {
  unsigned long long acc = 0;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, st = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = tid * W; i < n; i += st * W) {
    unsigned long long r[W];
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const uint64_t h = (mix64(i + j) & mask) * 2;  // 16-byte slots: key at 2h, cnt at 2h+1
      if (MODE == 0) atomicAdd(t + h + 1, 1ull);                       // RED, no return
      if (MODE == 1) r[j] = atomicAdd(t + h + 1, 1ull);                // ATOM with return
      if (MODE == 2) r[j] = atomicCAS(t + h, ~0ull, i + j);             // CAS
    }
    if (MODE == 3) {
#pragma unroll
      for (int j = 0; j < W; ++j) r[j] = atomicCAS(t + (mix64(i + j) & mask) * 2, ~0ull, i + j);
#pragma unroll
      for (int j = 0; j < W; ++j) r[j] += atomicAdd(t + (mix64(i + j) & mask) * 2 + 1, 1ull);
    }
    if (MODE > 0)
#pragma unroll
      for (int j = 0; j < W; ++j) acc += r[j];
  }
  if (acc == 0x1234567) *out = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* out; cudaMalloc(&out, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (size_t slots : {size_t(1) << 21, size_t(1) << 28}) {
    unsigned long long* t; cudaMalloc(&t, slots * 16);
    const uint64_t mask = slots - 1, n = 1000000;
    auto run = [&](const char* nm, auto fn) {
      float best = 1e9;
      for (int r = 0; r < 5; ++r) {
        cudaMemset(t, 0xFF, slots * 16);
        cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
      }
      printf("table %5zu MB  %-28s 1e6 ops: %7.1f us  (%5.1f G ops/s) %s\n", (slots * 16) >> 20, nm, best * 1e3,
             n / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    run("RED add (no return) W4", [&] { k<0, 4><<<sms * 8, 256>>>(t, mask, n, out); });
    run("ATOM add (return) W4", [&] { k<1, 4><<<sms * 8, 256>>>(t, mask, n, out); });
    run("CAS u64 (return) W4", [&] { k<2, 4><<<sms * 8, 256>>>(t, mask, n, out); });
    run("CAS then add W4", [&] { k<3, 4><<<sms * 8, 256>>>(t, mask, n, out); });
    run("ATOM add (return) W1", [&] { k<1, 1><<<sms * 8, 256>>>(t, mask, n, out); });
    cudaFree(t);
  }
  return 0;
}
