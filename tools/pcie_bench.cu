// Host<->device transfer characteristics of the GPU box (tools/, not product):
// pinned vs pageable copies, host memcpy bandwidth by thread count, and the
// cost of cudaHostRegister (page-locking a caller's buffer in place).
//   nvcc -O3 -std=c++17 -o tools/pcie_bench tools/pcie_bench.cu -lpthread
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
  const size_t sizes[] = {size_t(4) << 20, size_t(8) << 20, size_t(12) << 20, size_t(132) << 20};
  void* dev;
  cudaMalloc(&dev, size_t(1) << 30);
  printf("host threads: %u\n", std::thread::hardware_concurrency());
  for (size_t n : sizes) {
    void* pin;
    cudaHostAlloc(&pin, n, cudaHostAllocDefault);
    memset(pin, 1, n);
    char* pg = (char*)aligned_alloc(4096, n);
    memset(pg, 2, n);
    auto bw = [&](const char* what, auto fn) {
      double best = 1e9;
      for (int r = 0; r < 5; ++r) {
        double t0 = now();
        fn();
        double t = now() - t0;
        best = t < best ? t : best;
      }
      printf("  %-42s %8.3f ms  %7.1f GB/s\n", what, best * 1e3, n / best / 1e9);
    };
    printf("size %zu MB\n", n >> 20);
    bw("H2D pinned cudaMemcpy", [&] { cudaMemcpy(dev, pin, n, cudaMemcpyHostToDevice); });
    bw("D2H pinned cudaMemcpy", [&] { cudaMemcpy(pin, dev, n, cudaMemcpyDeviceToHost); });
    bw("H2D pageable cudaMemcpy", [&] { cudaMemcpy(dev, pg, n, cudaMemcpyHostToDevice); });
    bw("D2H pageable cudaMemcpy", [&] { cudaMemcpy(pg, dev, n, cudaMemcpyDeviceToHost); });
    for (int th : {1, 4, 8, 16}) {
      char nm[64];
      snprintf(nm, 64, "host memcpy pageable->pinned %2d threads", th);
      bw(nm, [&] {
        std::vector<std::thread> ts;
        size_t per = (n + th - 1) / th;
        for (int t = 0; t < th; ++t)
          ts.emplace_back([&, t] {
            size_t lo = t * per, len = lo < n ? std::min(per, n - lo) : 0;
            if (len) memcpy((char*)pin + lo, pg + lo, len);
          });
        for (auto& x : ts) x.join();
      });
    }
    bw("cudaHostRegister + H2D + Unregister", [&] {
      cudaHostRegister(pg, n, cudaHostRegisterDefault);
      cudaMemcpy(dev, pg, n, cudaMemcpyHostToDevice);
      cudaHostUnregister(pg);
    });
    bw("cudaHostRegister + Unregister only", [&] {
      cudaHostRegister(pg, n, cudaHostRegisterDefault);
      cudaHostUnregister(pg);
    });
    cudaError_t e = cudaHostRegister(pg, n, cudaHostRegisterReadOnly);
    printf("  register readonly: %s\n", cudaGetErrorString(e));
    if (e == cudaSuccess) {
      bw("H2D from registered pageable", [&] { cudaMemcpy(dev, pg, n, cudaMemcpyHostToDevice); });
      cudaHostUnregister(pg);
    }
    cudaFreeHost(pin);
    free(pg);
  }
  return 0;
}
