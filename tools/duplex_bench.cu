// Do H2D and D2H copies on different streams overlap on this box? And how fast
// do SM stores into mapped pinned host memory run (zero-copy D2H)? (tools/)
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
__global__ void store_host(uint4* dst, const uint4* src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) dst[i] = src[i];
}
int main() {
  const size_t up = size_t(132) << 20, down = size_t(40) << 20;
  void *hu, *hd, *du, *dd;
  cudaHostAlloc(&hu, up, 0); cudaHostAlloc(&hd, down, cudaHostAllocMapped);
  cudaMalloc(&du, up); cudaMalloc(&dd, down);
  cudaStream_t a, b; cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  for (int rep = 0; rep < 3; ++rep) {
    double t0 = now(); cudaMemcpyAsync(du, hu, up, cudaMemcpyHostToDevice, a); cudaStreamSynchronize(a); double t1 = now();
    cudaMemcpyAsync(hd, dd, down, cudaMemcpyDeviceToHost, b); cudaStreamSynchronize(b); double t2 = now();
    cudaMemcpyAsync(du, hu, up, cudaMemcpyHostToDevice, a); cudaMemcpyAsync(hd, dd, down, cudaMemcpyDeviceToHost, b);
    cudaStreamSynchronize(a); double t3 = now(); cudaStreamSynchronize(b); double t4 = now();
    printf("H2D alone %.3f ms | D2H alone %.3f ms | together: H2D done %.3f ms, D2H done %.3f ms\n",
           (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t4 - t2) * 1e3);
  }
  uint4* hdp; cudaHostGetDevicePointer((void**)&hdp, hd, 0);
  for (int rep = 0; rep < 3; ++rep) {
    double t0 = now(); store_host<<<148 * 4, 256, 0, b>>>(hdp, (uint4*)dd, down / 16); cudaStreamSynchronize(b); double t1 = now();
    cudaMemcpyAsync(du, hu, up, cudaMemcpyHostToDevice, a); store_host<<<148 * 4, 256, 0, b>>>(hdp, (uint4*)dd, down / 16);
    cudaStreamSynchronize(b); double t2 = now(); cudaStreamSynchronize(a); double t3 = now();
    printf("zero-copy kernel store 40MB alone %.3f ms | with concurrent H2D: kernel %.3f ms, H2D %.3f ms\n",
           (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t1) * 1e3);
  }
  return 0;
}
