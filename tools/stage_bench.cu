// Staging-loop experiments (tools/, not product): pageable -> pinned ring -> device
// with a worker pool, the way api.cu's stage_h2d does it, to find what limits the
// E2E upload.
//   nvcc -O3 -std=c++17 -o tools/stage_bench tools/stage_bench.cu ../paper_2601_19911_b200/csrc/runtime.cpp -lpthread
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2601_19911_b200/csrc/runtime.h"

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }


int main(int argc, char** argv) {
  const size_t total = size_t(132) << 20;
  char* src = (char*)aligned_alloc(4096, total);
  memset(src, 3, total);
  void* dev;
  cudaMalloc(&dev, total);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int threads : {2, 3, 4, 6}) {
    golp::WorkerPool pool;
    pool.start(threads);
    for (size_t chunk_mb : {8, 12, 16, 24}) {
      const size_t chunk = chunk_mb << 20;
      for (int slots : {2, 3}) {
        std::vector<void*> pin(slots);
        std::vector<cudaEvent_t> ev(slots);
        std::vector<bool> busy(slots, false);
        for (int i = 0; i < slots; ++i) {
          cudaHostAlloc(&pin[i], chunk, cudaHostAllocDefault);
          cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
        }
        double best = 1e9, tcopy_best = 0, twait_best = 0;
        for (int rep = 0; rep < 9; ++rep) {
          double tcopy = 0, twait = 0;
          double t0 = now();
          int next = 0;
          for (size_t done = 0; done < total;) {
            const int slot = next;
            next = (next + 1) % slots;
            double a = now();
            if (busy[slot]) cudaEventSynchronize(ev[slot]);
            double b = now();
            const size_t len = std::min(chunk, total - done);
            golp::parallel_copy(pool, pin[slot], src + done, len);
            double c = now();
            cudaMemcpyAsync((char*)dev + done, pin[slot], len, cudaMemcpyHostToDevice, s);
            cudaEventRecord(ev[slot], s);
            busy[slot] = true;
            done += len;
            twait += b - a;
            tcopy += c - b;
          }
          cudaStreamSynchronize(s);
          for (auto&& x : busy) x = false;
          double t = now() - t0;
          if (t < best) { best = t; tcopy_best = tcopy; twait_best = twait; }
        }
        printf("threads %2d chunk %2zu MB slots %d: %7.2f ms  %5.1f GB/s  (copy %6.2f ms, wait %6.2f ms)\n", threads,
               chunk_mb, slots, best * 1e3, total / best / 1e9, tcopy_best * 1e3, twait_best * 1e3);
        for (int i = 0; i < slots; ++i) {
          cudaFreeHost(pin[i]);
          cudaEventDestroy(ev[i]);
        }
      }
    }
    pool.stop();
  }
  return 0;
}
