// H2D from cudaHostRegister'ed malloc memory vs cudaHostAlloc, as the offload
// path issues it (two async copies on a non-blocking stream, event sync).
//   nvcc -O3 -std=c++17 -o tools/reg_bench tools/reg_bench.cu
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sys/mman.h>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
  const size_t a = 8u << 20, b = 4u << 20;
  void *d;
  cudaMalloc(&d, a + b);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  auto run = [&](const char* tag, char* pa, char* pb) {
    double best = 1e9, sum = 0;
    for (int r = 0; r < 30; ++r) {
      double t0 = now();
      cudaMemcpyAsync(d, pa, a, cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync((char*)d + a, pb, b, cudaMemcpyHostToDevice, s);
      cudaEventRecord(ev, s);
      cudaEventSynchronize(ev);
      double t = now() - t0;
      if (r >= 5) { best = t < best ? t : best; sum += t; }
    }
    printf("%-40s best %.3f ms  mean %.3f ms\n", tag, best * 1e3, sum / 25 * 1e3);
  };
  char *ha, *hb;
  cudaHostAlloc((void**)&ha, a, 0);
  cudaHostAlloc((void**)&hb, b, 0);
  memset(ha, 1, a); memset(hb, 1, b);
  run("cudaHostAlloc", ha, hb);
  for (unsigned flags : {cudaHostRegisterDefault, cudaHostRegisterReadOnly, cudaHostRegisterPortable}) {
    char* ma = (char*)malloc(a + 100);
    char* mb = (char*)malloc(b + 100);
    memset(ma, 2, a + 100); memset(mb, 2, b + 100);
    char* pa = ma + 16; char* pb = mb + 16;
    cudaError_t e1 = cudaHostRegister(pa, a, flags), e2 = cudaHostRegister(pb, b, flags);
    char tag[64];
    snprintf(tag, 64, "malloc registered flags=%u (%d %d)", flags, (int)e1, (int)e2);
    run(tag, pa, pb);
    cudaHostUnregister(pa); cudaHostUnregister(pb);
    free(ma); free(mb);
  }
  {
    char* ma = (char*)aligned_alloc(2 << 20, a);
    char* mb = (char*)aligned_alloc(2 << 20, b);
    madvise(ma, a, 14); madvise(mb, b, 14);  // MADV_HUGEPAGE
    memset(ma, 3, a); memset(mb, 3, b);
    cudaHostRegister(ma, a, cudaHostRegisterReadOnly); cudaHostRegister(mb, b, cudaHostRegisterReadOnly);
    run("2MB-aligned MADV_HUGEPAGE registered", ma, mb);
  }
  return 0;
}
