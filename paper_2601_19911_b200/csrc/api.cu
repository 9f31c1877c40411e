// C ABI of libgolp_b200.so (declared in include/golp_b200.h): device context,
// HBM workspace, pinned staging ring, stream/event orchestration and ledgers.
//
// Boundary being replaced: the reference's device protocol topk()/probe()
// (ProxyDevice, pkg/src/golp/device.py:299-436), whose ledgers feed the gate
// (pkg/src/golp/gate.py:185-213) and calibrate_profile (device.py:490-554).
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <sys/mman.h>
#include <unistd.h>

#include <map>
#include <set>
#include <string>

#include "../../include/golp_b200.h"
#include "join.cuh"
#include "runtime.h"
#include "sort.cuh"
#include "topk.cuh"

namespace golp {
const char* last_error_cstr();
}

using namespace golp;

namespace {

std::atomic<uint64_t> g_launches{0};

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      set_error(std::string(#x) + " failed: " + cudaGetErrorString(e_));                   \
      return GOLP_ERR_CUDA;                                                                \
    }                                                                                      \
  } while (0)
#define CKL() CK(cudaGetLastError())
#define RET(x)                   \
  do {                           \
    int r_ = (x);                \
    if (r_ != GOLP_OK) return r_; \
  } while (0)

int invalid(const std::string& msg) {
  set_error(msg);
  return GOLP_ERR_INVALID;
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    const size_t alloc = std::max<size_t>(want + want / 8, 256);
    cudaError_t e = cudaMalloc(&p, alloc);
    if (e == cudaSuccess) bytes = alloc;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

// Small pinned rings stay resident in the host's last-level cache, so the DMA
// engine reads/writes them there instead of DRAM (tools/stage_bench.cu: 2 x 16 MB
// slots with 4 copy threads beat 8 slots or more threads on the GPU box).
constexpr int kSlots = 2;     // H2D pinned ring
constexpr int kD2HSlots = 2;  // D2H pinned ring
constexpr int kNumCtl = 3;  // 0: threshold select, 1: candidate select (+filter count), 2: fallback

struct Ctx {
  bool ready = false;
  int device = 0;
  int sms = 148;
  cudaStream_t s_main = nullptr, s_h2d = nullptr, s_d2h = nullptr;
  size_t chunk = 16u << 20;
  void* pin[kSlots] = {};
  cudaEvent_t pin_ev[kSlots] = {};
  bool pin_busy[kSlots] = {};
  int next_slot = 0;
  void* dpin[kD2HSlots] = {};
  cudaEvent_t dpin_ev[kD2HSlots] = {};
  uint64_t d2h_seq = 0;
  struct D2HPiece {
    int slot;
    char* dst;
    size_t len;
  };
  std::vector<D2HPiece> d2h_q;  // FIFO (front = index d2h_head)
  size_t d2h_head = 0;
  bool d2h_direct = false;  // direct (pinned-destination) copies pending on s_d2h
  std::vector<cudaEvent_t> chunk_ev, h2d_ev;
  uint64_t* mirror = nullptr;  // mapped pinned copy of per-chunk pair totals
  uint64_t* mirror_dev = nullptr;
  size_t mirror_n = 0;
  void* pin_small = nullptr;  // samples, counters, small outputs
  size_t pin_small_bytes = 16u << 20;
  WorkerPool pool;
  cudaEvent_t ev[8] = {};
  cudaEvent_t ev_rows = nullptr;  // a copied row column of a chunked upload has landed

  DevBuf ctl, cand_hi, cand_lo, w_hi, w_lo, out_rows, out_hi, samples;
  DevBuf table, rows_arr, ovf, big_list, grp_bits, jcount, wcount, partial, totals, totals2;
  DevBuf sc_prow, sc_oc;
  DevBuf part_keys, part_pos, part_cnt, part_cur, run_base, run_len, res_part, work_ctr;
  DevBuf pairs_p, pairs_b;
  DevBuf rows_flag;  // two words: the build row column is NOT a dense run (alternate builds, join_build_impl)
  DevBuf row_base;   // what the emit adds to a singleton's slot.off (rows[0] for a dense column, else 0)
  DevBuf srt_hist, srt_k0, srt_k1, srt_r0, srt_r1, srt_status, srt_base;
  DevBuf in_keys, in_rows, in_bkeys, in_brows, in_payload;
  uint64_t jcap = 0, jmask = 0, jnb = 0;
  uint32_t jparts = 1;  // table slices of the radix-partitioned join (1 = not partitioned)
  int jslice_bits = 0;
  uint64_t last_m = 0;
  bool last_probe_valid = false;
  // Bytes the copy engines actually moved for the current / last host-buffer
  // call (the ledger keeps the reference's shape formulas instead).
  uint64_t moved_h2d = 0, moved_d2h = 0;
  bool dense_rows = true;  // GOLP_DENSE_ROWS=0 ships every row-id column
  bool rows_hint = false;
  unsigned build_parity = 0;  // which rows_flag word the next build uses
  int prof_last = -1, probe_start_ev = 6;  // prof_record: last event recorded, probe start event
  cudaStream_t prof_last_stream = nullptr;
  uint64_t prof_last_launches = 0;  // golp_hint_dense_rows: the next call's row columns are positions

  char* status_host = nullptr;  // mapped pinned words: select status + candidate count
  char* status_dev = nullptr;
  bool prof = false;
  bool build_timed = false;
  bool prof_build_start = true;  // golp_set_profiling(2) drops the build-start event
  bool probe_timed = false;
  bool topk_pending = false;  // fused Top-K in flight: candidates/fallback read on demand
  bool topk_timed = false;
  golp_kernel_times kt{};
  // Per-context launch caches: kernels whose dynamic shared memory limit was
  // raised on this device, and occupancy-derived grid sizes.
  std::set<const void*> smem_set;
  std::map<std::pair<const void*, int>, int> per_sm;
  std::vector<cudaEvent_t> trace_ev;  // GOLP_TRACE upload markers (golp_probe)
  std::vector<cudaEvent_t> kspan_ev;  // profiling: (start, end) pairs around each kernel group of a call
  size_t kspan_n = 0;
};

// One context per (device, handle): streams, pinned staging rings, HBM
// workspace and launch caches. A thread works on one context at a time
// (golp_init / golp_use_device / golp_context_use select it); calls stay
// externally synchronous per context, and threads on different contexts run
// concurrently (B200Device(gpus=G) drives G of them from G host threads).
constexpr int kMaxContexts = 64;
std::mutex g_ctx_mu;
Ctx* g_ctx[kMaxContexts] = {};
int g_default_ctx[kMaxContexts];  // device -> handle of its default context (-1: none)
bool g_default_init = false;
thread_local Ctx* t_cur = nullptr;
std::atomic<bool> g_any_ready{false};  // some context initialized the CUDA runtime

int device_of_thread() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) {
    cudaGetLastError();
    d = 0;
  }
  return d;
}

// Handle of the default context of `device`, created (not yet initialized) on first use.
int default_handle(int device) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  if (!g_default_init) {
    for (int& h : g_default_ctx) h = -1;
    g_default_init = true;
  }
  if (device < 0 || device >= kMaxContexts) return -1;
  if (g_default_ctx[device] >= 0) return g_default_ctx[device];
  for (int h = 0; h < kMaxContexts; ++h)
    if (!g_ctx[h]) {
      g_ctx[h] = new Ctx();
      g_ctx[h]->device = device;
      g_default_ctx[device] = h;
      return h;
    }
  return -1;
}

// The calling thread's context (the current CUDA device's default one when the
// thread has not selected any); initialized by ensure_init().
Ctx& cur() {
  if (!t_cur) {
    const int h = default_handle(device_of_thread());
    // no context slot left (or a device index past kMaxContexts): an unusable
    // context whose initialization reports the error
    static Ctx unusable;
    unusable.device = kMaxContexts;
    t_cur = h >= 0 ? g_ctx[h] : &unusable;
  }
  return *t_cur;
}

int do_init(Ctx& g, int device, uint64_t chunk_bytes, int host_threads) {
  if (g.ready) {
    if (device >= 0 && device != g.device) {
      set_error("context is bound to device " + std::to_string(g.device) + ", not " + std::to_string(device));
      return GOLP_ERR_INVALID;
    }
    CK(cudaSetDevice(g.device));
    return GOLP_OK;
  }
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev <= 0) {
    set_error("no CUDA device visible");
    return GOLP_ERR_CUDA;
  }
  if (device < 0) device = g.device;
  if (device < 0 || device >= ndev) {
    set_error("CUDA device " + std::to_string(device) + " is not visible (" + std::to_string(ndev) + " devices)");
    return GOLP_ERR_INVALID;
  }
  CK(cudaSetDevice(device));
  g.device = device;
  CK(cudaDeviceGetAttribute(&g.sms, cudaDevAttrMultiProcessorCount, device));
  CK(cudaStreamCreateWithFlags(&g.s_main, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&g.s_h2d, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&g.s_d2h, cudaStreamNonBlocking));
  if (chunk_bytes) g.chunk = (size_t)chunk_bytes;
  for (int i = 0; i < kSlots; ++i) {
    CK(cudaHostAlloc(&g.pin[i], g.chunk, cudaHostAllocDefault));
    CK(cudaEventCreateWithFlags(&g.pin_ev[i], cudaEventDisableTiming));
    g.pin_busy[i] = false;
  }
  for (int i = 0; i < kD2HSlots; ++i) {
    CK(cudaHostAlloc(&g.dpin[i], g.chunk, cudaHostAllocDefault));
    CK(cudaEventCreateWithFlags(&g.dpin_ev[i], cudaEventDisableTiming));
  }
  CK(cudaHostAlloc(&g.pin_small, g.pin_small_bytes, cudaHostAllocDefault));
  for (auto& e : g.ev) CK(cudaEventCreate(&e));
  CK(cudaEventCreateWithFlags(&g.ev_rows, cudaEventDisableTiming));
  int hw = (int)std::thread::hardware_concurrency();
  if (host_threads <= 0) host_threads = std::max(1, std::min(4, hw - 1));
  g.pool.start(host_threads);
  if (const char* v = getenv("GOLP_DENSE_ROWS")) g.dense_rows = std::atoi(v) != 0;
  CK(g.ctl.ensure(sizeof(SelectCtl) * kNumCtl));
  g.ready = true;
  g_any_ready = true;
  return GOLP_OK;
}

// Initializes the calling thread's context on first use and makes its device
// current on this thread.
int ensure_init() {
  Ctx& g = cur();
  if (!g.ready) return do_init(g, -1, 0, 0);
  int d = -1;
  if (cudaGetDevice(&d) != cudaSuccess || d != g.device) CK(cudaSetDevice(g.device));
  return GOLP_OK;
}

// A device pointer handed to a resident entry point must live on the context's
// device (a tensor on another GPU would be a foreign pointer to this context).
int check_device_ptr(const void* p) {
  if (!p) return GOLP_OK;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return GOLP_OK;  // not a CUDA allocation the runtime knows: let the kernel fault report it
  }
  const int dev = cur().device;
  if ((at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) && at.device != dev) {
    set_error("device pointer is on CUDA device " + std::to_string(at.device) + " but the golp context is on " +
              std::to_string(dev));
    return GOLP_ERR_INVALID;
  }
  return GOLP_OK;
}

// Raises `fn`'s dynamic shared memory limit once per context (per device).
template <typename K>
int smem_attr(K fn, size_t smem) {
  Ctx& g = cur();
  const void* key = reinterpret_cast<const void*>(fn);
  if (smem == 0 || g.smem_set.count(key)) return GOLP_OK;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  g.smem_set.insert(key);
  return GOLP_OK;
}

// Resident blocks per SM of `fn` at (threads, smem), cached per context; 0 if it cannot run.
template <typename K>
int blocks_per_sm(K fn, int threads, size_t smem) {
  Ctx& g = cur();
  const auto key = std::make_pair(reinterpret_cast<const void*>(fn), threads * 1024 + (int)(smem >> 10));
  auto it = g.per_sm.find(key);
  if (it != g.per_sm.end()) return it->second;
  if (smem_attr(fn, smem) != GOLP_OK) return 0;
  int per = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    per = 0;
  }
  g.per_sm[key] = per;
  return per;
}

SelectCtl* ctl(int i) { return cur().ctl.as<SelectCtl>() + i; }

// Integer tuning knob from the environment (default when unset or malformed).
uint64_t env_u64(const char* name, uint64_t dflt) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  char* end = nullptr;
  const unsigned long long x = strtoull(v, &end, 0);
  return (end && *end == 0) ? (uint64_t)x : dflt;
}

// Page-locked host ranges this library knows about: the pinned result arena's
// regions and the caller buffers golp_host_register page-locked. A transfer
// takes the direct-DMA path only when its WHOLE range lies in one of them
// (a registered prefix view says nothing about the bytes after it); any other
// buffer goes through the staging ring.
std::mutex g_pin_mu;
std::map<uintptr_t, size_t> g_pinned;  // base -> bytes

void pinned_add(const void* p, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pinned[reinterpret_cast<uintptr_t>(p)] = bytes;
}
void pinned_remove(const void* p) {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pinned.erase(reinterpret_cast<uintptr_t>(p));
}
bool is_pinned(const void* p, size_t bytes) {
  if (!p) return false;
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  std::lock_guard<std::mutex> lk(g_pin_mu);
  auto it = g_pinned.upper_bound(a);
  if (it == g_pinned.begin()) return false;
  --it;
  return a >= it->first && a + std::max<size_t>(bytes, 1) <= it->first + it->second;
}

// ---- pinned staging ring ----------------------------------------------------------
// Host -> device copy of an arbitrary pageable buffer: the pool packs chunk i+1
// into a pinned slot while the DMA engine drains chunk i.
int stage_h2d(void* dst, const void* src, size_t bytes) {
  Ctx& g = cur();
  g.moved_h2d += bytes;
  if (bytes && is_pinned(src, bytes)) {  // page-locked source: no host copy
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, g.s_h2d));
    return GOLP_OK;
  }
  size_t done = 0;
  while (done < bytes) {
    const int slot = g.next_slot;
    g.next_slot = (g.next_slot + 1) % kSlots;
    if (g.pin_busy[slot]) CK(cudaEventSynchronize(g.pin_ev[slot]));
    const size_t len = std::min(g.chunk, bytes - done);
    parallel_copy(g.pool, g.pin[slot], static_cast<const char*>(src) + done, len);
    CK(cudaMemcpyAsync(static_cast<char*>(dst) + done, g.pin[slot], len, cudaMemcpyHostToDevice, g.s_h2d));
    CK(cudaEventRecord(g.pin_ev[slot], g.s_h2d));
    g.pin_busy[slot] = true;
    done += len;
  }
  return GOLP_OK;
}

__global__ void fill_dense_rows_kernel(uint32_t* __restrict__ dst, uint32_t base, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = base + (uint32_t)i;
}

// Row-id column upload. A dense run (rows[i] == rows[0] + i, which is what
// extract_keys produces, pkg/src/golp/store.py:178-181) does not cross PCIe:
// the pool verifies it on the host while the key column queued just before it
// is in flight, and a fill kernel writes it in HBM on the main stream, where
// every consumer of the column runs (on the copy stream it would hold back the
// next upload until it finished). Any other column is copied as is. The
// device therefore sees exactly the caller's row ids either way. A consumer that
// reads rows only through a RowCol (the Top-K kernels) passes `as_rows`: a dense
// run then becomes positions (RowCol{nullptr, rows[0]}) and nothing is written.
int upload_rows(uint32_t* dst, const uint32_t* src, uint64_t n, bool* copied = nullptr, RowCol* as_rows = nullptr) {
  Ctx& g = cur();
  if (copied) *copied = false;
  if (as_rows) *as_rows = RowCol{dst, 0};
  if (!n) return GOLP_OK;
  const double tv = wall_seconds();
  // A caller-declared dense column (golp_hint_dense_rows: the table's own
  // positions, extract_keys) skips the scan; its end points are still checked.
  const bool hinted = g.rows_hint && src[n - 1] == src[0] + (uint32_t)(n - 1);
  const bool dense = g.dense_rows && (hinted || dense_run(g.pool, src, n));
  if (std::getenv("GOLP_TRACE"))
    std::fprintf(stderr, "[golp] rows [%llu] verified in %.3f ms: %s\n", (unsigned long long)n, (wall_seconds() - tv) * 1e3,
                 dense ? "dense" : "copied");
  if (dense && as_rows) {
    *as_rows = RowCol{nullptr, src[0]};
    return GOLP_OK;
  }
  if (dense) {
    const int grid = (int)std::min<uint64_t>((n + 1023) / 1024, (uint64_t)g.sms * 8);
    fill_dense_rows_kernel<<<grid, 256, 0, g.s_main>>>(dst, src[0], n);
    CKL();
    ++g_launches;
    return GOLP_OK;
  }
  if (copied) *copied = true;
  return stage_h2d(dst, src, n * 4);
}

// Full-row mode ships payload bytes the device never reads: stream a pinned slot
// (contents irrelevant) into a device scratch chunk, repeatedly.
int stage_dummy_h2d(size_t bytes) {
  Ctx& g = cur();
  if (!bytes) return GOLP_OK;
  g.moved_h2d += bytes;
  CK(g.in_payload.ensure(g.chunk));
  size_t done = 0;
  while (done < bytes) {
    const int slot = g.next_slot;
    g.next_slot = (g.next_slot + 1) % kSlots;
    if (g.pin_busy[slot]) CK(cudaEventSynchronize(g.pin_ev[slot]));
    const size_t len = std::min(g.chunk, bytes - done);
    CK(cudaMemcpyAsync(g.in_payload.p, g.pin[slot], len, cudaMemcpyHostToDevice, g.s_h2d));
    CK(cudaEventRecord(g.pin_ev[slot], g.s_h2d));
    g.pin_busy[slot] = true;
    done += len;
  }
  return GOLP_OK;
}

// Device -> host copies into pageable memory through a separate pinned ring:
// pieces are DMA'd on s_d2h and unpacked (pool memcpy) in FIFO order, either
// opportunistically (d2h_poll) or when a slot is needed / at the end (d2h_flush).
int d2h_complete_one() {
  Ctx& g = cur();
  Ctx::D2HPiece pc = g.d2h_q[g.d2h_head++];
  CK(cudaEventSynchronize(g.dpin_ev[pc.slot]));
  parallel_copy(g.pool, pc.dst, g.dpin[pc.slot], pc.len);
  if (g.d2h_head == g.d2h_q.size()) {
    g.d2h_q.clear();
    g.d2h_head = 0;
  }
  return GOLP_OK;
}

int d2h_enqueue(void* dst, const void* src, size_t bytes) {
  Ctx& g = cur();
  g.moved_d2h += bytes;
  if (bytes && is_pinned(dst, bytes)) {  // page-locked destination (result arena): no host copy
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, g.s_d2h));
    g.d2h_direct = true;
    return GOLP_OK;
  }
  size_t done = 0;
  while (done < bytes) {
    while (g.d2h_q.size() - g.d2h_head >= (size_t)kD2HSlots) RET(d2h_complete_one());
    const int slot = (int)(g.d2h_seq++ % kD2HSlots);
    const size_t len = std::min(g.chunk, bytes - done);
    CK(cudaMemcpyAsync(g.dpin[slot], static_cast<const char*>(src) + done, len, cudaMemcpyDeviceToHost, g.s_d2h));
    CK(cudaEventRecord(g.dpin_ev[slot], g.s_d2h));
    g.d2h_q.push_back(Ctx::D2HPiece{slot, static_cast<char*>(dst) + done, len});
    done += len;
  }
  return GOLP_OK;
}

int d2h_poll() {
  Ctx& g = cur();
  while (g.d2h_head < g.d2h_q.size()) {
    const cudaError_t e = cudaEventQuery(g.dpin_ev[g.d2h_q[g.d2h_head].slot]);
    if (e == cudaErrorNotReady) return GOLP_OK;
    CK(e);
    RET(d2h_complete_one());
  }
  return GOLP_OK;
}

int d2h_flush() {
  Ctx& g = cur();
  while (g.d2h_head < g.d2h_q.size()) RET(d2h_complete_one());
  if (g.d2h_direct) {
    CK(cudaStreamSynchronize(g.s_d2h));
    g.d2h_direct = false;
  }
  return GOLP_OK;
}

int stage_d2h(void* dst, const void* src, size_t bytes) {
  RET(d2h_enqueue(dst, src, bytes));
  return d2h_flush();
}

int sync_ring() {
  Ctx& g = cur();
  for (int i = 0; i < kSlots; ++i) {
    if (g.pin_busy[i]) CK(cudaEventSynchronize(g.pin_ev[i]));
    g.pin_busy[i] = false;
  }
  return d2h_flush();
}

int ensure_chunk_events(size_t n) {
  Ctx& g = cur();
  while (g.chunk_ev.size() < n) {
    cudaEvent_t e, f;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&f, cudaEventDisableTiming));
    g.chunk_ev.push_back(e);
    g.h2d_ev.push_back(f);
  }
  if (g.mirror_n < n + 1) {
    if (g.mirror) cudaFreeHost(g.mirror);
    g.mirror = nullptr;
    g.mirror_n = 0;
    CK(cudaHostAlloc(reinterpret_cast<void**>(&g.mirror), (n + 2) * 8, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&g.mirror_dev), g.mirror, 0));
    g.mirror_n = n + 1;
  }
  return GOLP_OK;
}

// Publishes a device counter to mapped pinned host memory with a one-thread
// kernel: a memcpy here would sit in the D2H copy queue ahead of the pair
// downloads and block them (head-of-line) until its stream dependency clears.
__global__ void publish_u64_kernel(volatile unsigned long long* host_dst, const unsigned long long* src) {
  *host_dst = *src;
  __threadfence_system();
}

// ---- pinned result arena ---------------------------------------------------------
// Result arrays handed to Python live here: page-locked, so pairs DMA straight
// into them. First-fit over 2 MB-granular blocks, coalescing frees; regions are
// added on demand up to arena_max(), beyond that golp_host_alloc falls back to mmap.
constexpr size_t kArenaRegion = size_t(256) << 20;
// Cap on page-locked result memory: a quarter of host RAM (pinned pages cannot
// be swapped or reclaimed), at least 4 GiB.
size_t arena_max() {
  static size_t cap = 0;
  if (!cap) {
    const long pages = sysconf(_SC_PHYS_PAGES), psz = sysconf(_SC_PAGESIZE);
    const size_t ram = (pages > 0 && psz > 0) ? (size_t)pages * (size_t)psz : (size_t(16) << 30);
    cap = std::max(ram / 4, size_t(4) << 30);
  }
  return cap;
}
constexpr size_t kArenaGrain = size_t(2) << 20;
struct ArenaRegion {
  char* base;
  size_t size;
  std::map<size_t, size_t> free_;  // offset -> length
};
std::mutex g_arena_mu;
std::vector<ArenaRegion> g_arena;
std::map<const void*, std::pair<size_t, size_t>> g_arena_live;  // ptr -> (region, length)
size_t g_arena_total = 0;

void* arena_alloc(size_t bytes) {
  const size_t len = (bytes + kArenaGrain - 1) / kArenaGrain * kArenaGrain;
  std::lock_guard<std::mutex> lk(g_arena_mu);
  for (int attempt = 0; attempt < 2; ++attempt) {
    for (size_t r = 0; r < g_arena.size(); ++r) {
      auto& fl = g_arena[r].free_;
      for (auto it = fl.begin(); it != fl.end(); ++it) {
        if (it->second < len) continue;
        const size_t off = it->first, rest = it->second - len;
        fl.erase(it);
        if (rest) fl[off + len] = rest;
        char* p = g_arena[r].base + off;
        g_arena_live[p] = {r, len};
        return p;
      }
    }
    const size_t want = std::max(kArenaRegion, len);
    if (g_arena_total + want > arena_max() || !g_any_ready.load()) return nullptr;
    void* base = nullptr;
    // portable: result arrays of every context (device) DMA straight into it
    if (cudaHostAlloc(&base, want, cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    ArenaRegion reg{static_cast<char*>(base), want, {}};
    reg.free_[0] = want;
    pinned_add(base, want);
    g_arena.push_back(std::move(reg));
    g_arena_total += want;
  }
  return nullptr;
}

bool arena_free(const void* p) {
  std::lock_guard<std::mutex> lk(g_arena_mu);
  auto it = g_arena_live.find(p);
  if (it == g_arena_live.end()) return false;
  const size_t r = it->second.first, len = it->second.second;
  g_arena_live.erase(it);
  auto& fl = g_arena[r].free_;
  size_t off = static_cast<const char*>(p) - g_arena[r].base, l = len;
  auto nx = fl.lower_bound(off);
  if (nx != fl.end() && off + l == nx->first) {
    l += nx->second;
    nx = fl.erase(nx);
  }
  if (nx != fl.begin()) {
    auto pv = std::prev(nx);
    if (pv->first + pv->second == off) {
      off = pv->first;
      l += pv->second;
      fl.erase(pv);
    }
  }
  fl[off] = l;
  return true;
}

// ---- Top-K planning ---------------------------------------------------------------
struct TopkPlan {
  bool direct;      // select straight over the input (no sampled threshold)
  uint64_t s;       // samples
  uint64_t need_s;  // rank of the threshold sample (1-based)
  uint64_t cap;     // candidate capacity
  uint64_t expect;  // expected candidates
};

// With S stratified samples and K' = min(k, n), the number X of samples that
// fall in the true top K' is ~Binomial(S, K'/n). Taking the threshold at sample
// rank r = lam + 6 sqrt(lam) + 7 (lam = S K'/n) makes P(X >= r), the only way the
// filter can keep fewer than K' items, negligible; expected survivors ~ r n / S.
TopkPlan plan_topk(uint64_t n, uint64_t kk) {
  TopkPlan p{true, 0, 0, 0, 0};
  if (n <= kSortTile) return p;
  uint64_t s = n / 256;
  s = std::max<uint64_t>(2048, std::min<uint64_t>(s, 262144));
  const double lam = (double)s * (double)kk / (double)n;
  const uint64_t need_s = (uint64_t)std::ceil(lam + 6.0 * std::sqrt(lam) + 7.0);
  if (need_s * 4 >= s) return p;
  const uint64_t expect = (uint64_t)std::ceil((double)need_s * (double)n / (double)s);
  p.direct = false;
  p.s = s;
  p.need_s = need_s;
  p.cap = std::min<uint64_t>(n, std::max<uint64_t>(4 * expect + 65536, 1u << 20));
  p.expect = expect;
  return p;
}

template <class Src>
int launch_select(const SelectArgs<Src>& a, cudaStream_t s) {
  Ctx& g = cur();
  const size_t smem = (size_t)kSortTile * (sizeof(uint64_t) + sizeof(uint32_t));
  RET(smem_attr(select_kernel<Src>, smem));
  if (!a.use_cand_count && a.n <= kSortTile) {  // one block, shared memory only: plain launch
    select_kernel<Src><<<1, kSelThreads, smem, s>>>(a);
    CKL();
    ++g_launches;
    return GOLP_OK;
  }
  const int per = blocks_per_sm(select_kernel<Src>, kSelThreads, smem);
  if (per < 1) {
    set_error("select_kernel cannot be co-resident");
    return GOLP_ERR_CUDA;
  }
  const int blocks = per * g.sms;
  void* args[] = {const_cast<SelectArgs<Src>*>(&a)};
  CK(cudaLaunchCooperativeKernel((const void*)select_kernel<Src>, dim3(blocks), dim3(kSelThreads), args, smem, s));
  ++g_launches;
  return GOLP_OK;
}

template <class Src>
SelectArgs<Src> make_args(Src src, uint64_t n, uint64_t need, int mode, int c, uint32_t* out_rows,
                          uint64_t* out_hi) {
  Ctx& g = cur();
  SelectArgs<Src> a;
  a.src = src;
  a.n = n;
  a.need = need;
  a.cap = 0;
  a.use_cand_count = 0;
  a.mode = mode;
  a.ctl = ctl(c);
  a.w_hi = g.w_hi.as<uint64_t>();
  a.w_lo = g.w_lo.as<uint32_t>();
  a.out_rows = out_rows;
  a.out_hi = out_hi;
  a.host_status = nullptr;
  a.host_count = nullptr;
  return a;
}

template <class Src>
int launch_rank(const SelectArgs<Src>& a, unsigned long long* clear_count, cudaStream_t s) {
  Ctx& g = cur();
  RET(smem_attr(rank_select_kernel<Src>, kRankSmem));
  const int blocks = std::max(1, blocks_per_sm(rank_select_kernel<Src>, kRankThreads, kRankSmem)) * g.sms;
  rank_select_kernel<Src><<<blocks, kRankThreads, kRankSmem, s>>>(a, clear_count);
  CKL();
  ++g_launches;
  return GOLP_OK;
}

int ensure_topk_ws(uint64_t kk, uint64_t cap) {
  Ctx& g = cur();
  CK(g.w_hi.ensure(std::max<uint64_t>(kk, 1) * 16));  // winners + merge buffer
  CK(g.w_lo.ensure(std::max<uint64_t>(kk, 1) * 8));
  if (cap) {
    CK(g.cand_hi.ensure(cap * 8));
    CK(g.cand_lo.ensure(cap * 4));
  }
  return GOLP_OK;
}

int launch_filter(const double* keys, RowCol rows, uint64_t n, uint64_t cap, cudaStream_t s) {
  Ctx& g = cur();
  if (n == 0) return GOLP_OK;
  const uint64_t vec = n / 2 + 1;
  uint64_t blocks = (vec + (uint64_t)kFilterThreads * kFilterUnroll - 1) / ((uint64_t)kFilterThreads * kFilterUnroll);
  blocks = std::max<uint64_t>(1, std::min<uint64_t>(blocks, (uint64_t)g.sms * 8));
  topk_filter_kernel<<<(unsigned)blocks, kFilterThreads, 0, s>>>(keys, rows, n, ctl(0), &ctl(1)->cand_count,
                                                                  g.cand_hi.as<uint64_t>(), g.cand_lo.as<uint32_t>(),
                                                                  cap);
  CKL();
  ++g_launches;
  return GOLP_OK;
}

void prof_record(int idx, cudaStream_t s) {
  Ctx& g = cur();
  if (!g.prof) return;
  // A probe that starts right where the build ended (same stream, no launch in
  // between) reuses the build's end event: one event node less per graph step.
  if (idx == 6 && g.prof_last == 5 && g.prof_last_stream == s && g.prof_last_launches == g_launches) {
    g.probe_start_ev = 5;
    return;
  }
  if (idx == 6) g.probe_start_ev = 6;
  g.prof_last = idx;
  g.prof_last_stream = s;
  g.prof_last_launches = g_launches;
  // Inside a CUDA-graph capture the record must be an external event node, or
  // the event cannot be synchronized / timed after a replay.
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(g.ev[idx], s, cudaEventRecordExternal);
  else
    cudaEventRecord(g.ev[idx], s);
}
double prof_ms(int a, int b) {
  Ctx& g = cur();
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, g.ev[a], g.ev[b]) != cudaSuccess) return 0.0;
  return (double)ms;
}

// Device time of the kernels of one host-buffer call (golp_set_profiling on):
// timing events around each group of kernels a call enqueues on its main
// stream (a chunk's filter or probe, the build, the final select), summed when
// the call has finished. Upload waits between the groups are not counted, so
// this is the kernel term of C_gpu (device.py:154-181) for calibration.
void kspan_reset() { cur().kspan_n = 0; }
int kspan_mark(cudaStream_t s) {
  Ctx& g = cur();
  if (!g.prof) return GOLP_OK;
  if (g.kspan_ev.size() <= g.kspan_n) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    g.kspan_ev.push_back(e);
  }
  CK(cudaEventRecord(g.kspan_ev[g.kspan_n++], s));
  return GOLP_OK;
}
int kspan_finish() {
  Ctx& g = cur();
  double ms = 0.0;
  if (g.prof && g.kspan_n >= 2) {
    CK(cudaEventSynchronize(g.kspan_ev[g.kspan_n - 1]));
    for (size_t i = 0; i + 1 < g.kspan_n; i += 2) {
      float x = 0.f;
      CK(cudaEventElapsedTime(&x, g.kspan_ev[i], g.kspan_ev[i + 1]));
      ms += x;
    }
  }
  g.kt.call_kernel_ms = ms;
  return GOLP_OK;
}

// Status / candidate count of a sampled run: the select kernel stores them into
// mapped pinned words, so one stream sync replaces a D2H copy + sync.
int ensure_status_words() {
  Ctx& g = cur();
  if (!g.status_host) {
    CK(cudaHostAlloc(reinterpret_cast<void**>(&g.status_host), 64, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&g.status_dev), g.status_host, 0));
  }
  return GOLP_OK;
}

// status: 0 ok, 1 candidate set unusable (direct fallback), 2 too many
// candidates for the rank kernel (grid engine over the same candidates).
int read_topk_status(cudaStream_t s, int* status, uint64_t* cands) {
  Ctx& g = cur();
  CK(cudaStreamSynchronize(s));
  *status = *reinterpret_cast<volatile int*>(g.status_host);
  *cands = *reinterpret_cast<volatile unsigned long long*>(g.status_host + 8);
  return GOLP_OK;
}

SelectArgs<SrcCand> cand_args(uint64_t kk, uint64_t cap, uint32_t* out_rows, uint64_t* out_hi) {
  Ctx& g = cur();
  SelectArgs<SrcCand> a = make_args(SrcCand{g.cand_hi.as<uint64_t>(), g.cand_lo.as<uint32_t>()}, 0, kk, kModeFull, 1,
                                    out_rows, out_hi);
  a.use_cand_count = 1;
  a.cap = cap;
  *reinterpret_cast<volatile int*>(g.status_host) = 0;
  a.host_status = reinterpret_cast<int*>(g.status_dev);
  a.host_count = reinterpret_cast<unsigned long long*>(g.status_dev + 8);
  return a;
}

// Exact fallback: radix select straight over the device-resident input.
int topk_direct(const double* keys, RowCol rows, uint64_t n, uint64_t kk, uint32_t* out_rows,
                uint64_t* out_hi, cudaStream_t s) {
  CK(cudaMemsetAsync(ctl(2), 0, sizeof(SelectCtl), s));
  RET(launch_select(make_args(SrcInput{keys, rows}, n, kk, kModeFull, 2, out_rows, out_hi), s));
  return GOLP_OK;
}

// Top-K over device-resident columns (sampling on the device).
int topk_device_impl(const double* keys, RowCol rows, uint64_t n, uint64_t k, uint32_t* out_rows,
                     uint64_t* out_hi, cudaStream_t s) {
  Ctx& g = cur();
  const uint64_t kk = std::min(k, n);
  if (kk == 0) return GOLP_OK;
  const TopkPlan p = plan_topk(n, kk);
  RET(ensure_topk_ws(kk, p.direct ? 0 : p.cap));
  g.kt.topk_fallback = 0;
  g.kt.topk_candidates = 0;
  g.topk_pending = false;
  g.topk_timed = false;
  prof_record(0, s);
  if (p.direct) {
    RET(topk_direct(keys, rows, n, kk, out_rows, out_hi, s));
    prof_record(1, s);
    prof_record(2, s);
    prof_record(3, s);
    CK(cudaStreamSynchronize(s));
  } else {
    // Small sample sets / candidate lists use the one-launch rank kernel; the
    // radix engines (which need zeroed histograms) handle the rest.
    const bool rank_thr = p.s <= kRankMax;
    const bool rank_sel = p.expect <= kRankMax / 2 && kk <= kRankMax;
    if (rank_thr && rank_sel && env_u64("GOLP_TOPK_FUSED", 1)) {
      // everything in one cooperative launch, no host round trip (stream-ordered)
      RET(ensure_status_words());
      *reinterpret_cast<volatile int*>(g.status_host) = 0;
      FusedTopkArgs f;
      f.keys = keys;
      f.rows = rows;
      f.n = n;
      f.need = kk;
      f.s = (uint32_t)p.s;
      f.need_s = (uint32_t)p.need_s;
      f.w = (uint32_t)std::max<uint64_t>(1, n / p.s);
      // test knobs: shrink the candidate buffer / rank limit to exercise the in-kernel fallbacks
      f.cap = std::min<uint64_t>(p.cap, env_u64("GOLP_TOPK_CAP", p.cap));
      f.rank_max = (uint32_t)std::min<uint64_t>(kRankMax, env_u64("GOLP_TOPK_RANK_MAX", kRankMax));
      f.ctl = ctl(0);
      f.cand_hi = g.cand_hi.as<uint64_t>();
      f.cand_lo = g.cand_lo.as<uint32_t>();
      f.w_hi = g.w_hi.as<uint64_t>();
      f.w_lo = g.w_lo.as<uint32_t>();
      f.out_rows = out_rows;
      f.out_hi = out_hi;
      f.host_count = reinterpret_cast<unsigned long long*>(g.status_dev + 8);
      f.host_status = reinterpret_cast<int*>(g.status_dev);
      const size_t smem = (size_t)kSortTile * (sizeof(uint64_t) + sizeof(uint32_t));
      int per = blocks_per_sm(topk_fused_kernel, kSelThreads, smem);
      if (per < 1) {
        set_error("topk_fused_kernel cannot be co-resident");
        return GOLP_ERR_CUDA;
      }
      // blocks per SM (test / tuning knob GOLP_TOPK_FUSED_PER_SM; default: all that fit)
      per = (int)std::min<uint64_t>((uint64_t)per, std::max<uint64_t>(1, env_u64("GOLP_TOPK_FUSED_PER_SM", per)));
      const int blocks = per * g.sms;
      CK(cudaMemsetAsync(ctl(1), 0, 2 * sizeof(SelectCtl), s));  // candidate + fallback controls
      void* args[] = {&f};
      CK(cudaLaunchCooperativeKernel((void*)topk_fused_kernel, blocks, kSelThreads, args, smem, s));
      ++g_launches;
      prof_record(3, s);  // one kernel: select time = events 0 -> 3 (no graph nodes for 1, 2)
      g.topk_pending = true;  // candidate count / fallback resolved lazily
      if (g.prof) {
        g.kt.topk_threshold_ms = g.kt.topk_filter_ms = 0.0;
        g.topk_timed = true;
      }
      return GOLP_OK;
    }
    if (!(rank_thr && rank_sel)) CK(cudaMemsetAsync(ctl(0), 0, sizeof(SelectCtl) * 2, s));
    const SrcSample smp{keys, rows, n, (uint32_t)std::max<uint64_t>(1, n / p.s)};
    if (rank_thr)
      RET(launch_rank(make_args(smp, p.s, p.need_s, kModeThreshold, 0, nullptr, nullptr), &ctl(1)->cand_count, s));
    else
      RET(launch_select(make_args(smp, p.s, p.need_s, kModeThreshold, 0, nullptr, nullptr), s));
    prof_record(1, s);
    RET(launch_filter(keys, rows, n, p.cap, s));
    prof_record(2, s);
    RET(ensure_status_words());
    if (rank_sel) RET(launch_rank(cand_args(kk, p.cap, out_rows, out_hi), nullptr, s));
    else RET(launch_select(cand_args(kk, p.cap, out_rows, out_hi), s));
    prof_record(3, s);
    int status = 0;
    uint64_t cands = 0;
    RET(read_topk_status(s, &status, &cands));
    g.kt.topk_candidates = cands;
    if (status == 2) {  // more candidates than the rank kernel holds: grid engine
      char* c1 = reinterpret_cast<char*>(ctl(1));
      CK(cudaMemsetAsync(c1, 0, offsetof(SelectCtl, cand_count), s));  // histograms
      CK(cudaMemsetAsync(c1 + offsetof(SelectCtl, win_count), 0, sizeof(SelectCtl) - offsetof(SelectCtl, win_count),
                         s));
      RET(launch_select(cand_args(kk, p.cap, out_rows, out_hi), s));
      prof_record(3, s);
      RET(read_topk_status(s, &status, &cands));
    }
    if (status != 0) {
      g.kt.topk_fallback = 1;
      RET(topk_direct(keys, rows, n, kk, out_rows, out_hi, s));
      prof_record(3, s);
      CK(cudaStreamSynchronize(s));
    }
  }
  if (g.prof) {
    g.kt.topk_threshold_ms = prof_ms(0, 1);
    g.kt.topk_filter_ms = prof_ms(1, 2);
    g.kt.topk_select_ms = prof_ms(2, 3);
  }
  return GOLP_OK;
}

// ---- join -------------------------------------------------------------------------
int grid_for(uint64_t n, int threads, int per_sm) {
  Ctx& g = cur();
  uint64_t b = (n + threads - 1) / threads;
  b = std::max<uint64_t>(1, std::min<uint64_t>(b, (uint64_t)g.sms * per_sm));
  return (int)b;
}

// Radix partitioning of the join (see join.cuh): slices of GOLP_JOIN_SLICE_BYTES
// (default 32 MiB of slots) once the table exceeds two slices, at most
// kMaxProbeParts slices.

void plan_partitions(uint64_t cap) {
  Ctx& g = cur();
  const uint64_t slice_bytes = std::max<uint64_t>(64, env_u64("GOLP_JOIN_SLICE_BYTES", 32ull << 20));
  uint64_t parts = 1;
  if (cap * sizeof(Slot) > 2 * slice_bytes) {
    while (parts < kMaxProbeParts && cap * sizeof(Slot) / parts > slice_bytes) parts <<= 1;
  }
  while (parts > 1 && cap / parts < 2) parts >>= 1;
  int cap_bits = 0;
  while ((1ull << cap_bits) < cap) ++cap_bits;
  int part_bits = 0;
  while ((1ull << part_bits) < parts) ++part_bits;
  g.jparts = (uint32_t)parts;
  g.jslice_bits = cap_bits - part_bits;
}

// Blocks of `kernel` that fit on the GPU at once: grid-stride kernels that
// walk partitioned data must not have blocks queued behind the resident ones
// (a queued block would start its walk far behind the others).
template <typename K>
int resident_grid(K kernel, int threads, size_t smem) {
  return std::max(1, blocks_per_sm(kernel, threads, smem)) * cur().sms;
}

// Groups the entries of [keys, keys+n) by table slice into g.part_keys, with
// positions (build) or in-tile indices + (tile, slice) runs (probe). 3 launches.
#ifndef GOLP_PART_CAP
#define GOLP_PART_CAP 1  // probe side: fixed-capacity slices + overflow area instead of a count pass
#endif
// Fixed slice capacity for n probe entries over P slices: the expected share
// + 1/32 + one tile, in whole partition tiles (the lookup kernel's chunks
// never straddle two slices); 0 = exact layout (count pass + scan).
uint64_t probe_slice_capacity(uint64_t n, uint32_t P) {
  if (!GOLP_PART_CAP || !env_u64("GOLP_PART_CAP", 1) || P < 2) return 0;
  const uint64_t share = (n + P - 1) / P;
  return (share + share / 32 + 2 * kPartTile) / kPartTile * kPartTile;
}

// Entries the partitioned probe buffers hold for n probes (slices + overflow area).
uint64_t probe_part_entries(uint64_t n, uint32_t P) {
  const uint64_t capu = probe_slice_capacity(n, P);
  return capu ? (uint64_t)P * capu + n : n;
}

int partition_entries(const double* keys, uint64_t n, bool probe_side, cudaStream_t s) {
  Ctx& g = cur();
  const uint32_t P = g.jparts;
  const uint64_t ntiles = (n + kPartTile - 1) / kPartTile;
  const uint64_t capu = probe_side ? probe_slice_capacity(n, P) : 0;
  const uint64_t nall = probe_side ? probe_part_entries(n, P) : n;
  CK(g.part_keys.ensure(std::max<uint64_t>(nall, 1) * 8));
  CK(g.part_pos.ensure(std::max<uint64_t>(nall, 1) * (probe_side ? 2 : 4)));
  CK(g.part_cnt.ensure(P * 8));
  CK(g.part_cur.ensure((P + 1) * 8));
  PartOut o{g.part_keys.as<double>(), nullptr, nullptr, nullptr, nullptr, 0, nullptr};
  if (probe_side) {
    CK(g.run_base.ensure(std::max<uint64_t>(ntiles * P, 1) * 4));
    CK(g.run_len.ensure(std::max<uint64_t>(ntiles * P, 1) * 2));
    o.idx = g.part_pos.as<uint16_t>();
    o.run_base = g.run_base.as<uint32_t>();
    o.run_len = g.run_len.as<uint16_t>();
  } else {
    o.pos = g.part_pos.as<uint32_t>();
  }
  unsigned long long* cnt = g.part_cnt.as<unsigned long long>();
  unsigned long long* cursors = g.part_cur.as<unsigned long long>();
  if (capu) {  // slice cursors count from each slice's fixed base; cursors[P] = overflow area
    CK(cudaMemsetAsync(cursors, 0, (P + 1) * 8, s));
    o.capu = capu;
    o.ovf = cursors + P;
  } else {
    CK(cudaMemsetAsync(cnt, 0, P * 8, s));
    part_count_kernel<<<g.sms * 4, kPartThreads, 0, s>>>(keys, n, (uint32_t)g.jmask, g.jslice_bits, P, cnt);
    CKL();
    part_scan_kernel<<<1, 1024, 0, s>>>(cnt, cursors, P);
    CKL();
    g_launches += 2;
  }
  RET(smem_attr(part_scatter_kernel, kPartScatterSmem));
  const int gsmax = resident_grid(part_scatter_kernel, kPartThreads, kPartScatterSmem);
  const int gs = (int)std::max<uint64_t>(1, std::min<uint64_t>(ntiles, (uint64_t)gsmax));
  part_scatter_kernel<<<gs, kPartThreads, kPartScatterSmem, s>>>(keys, n, (uint32_t)g.jmask, g.jslice_bits, P, cursors, o);
  CKL();
  g_launches += 1;
  return GOLP_OK;
}

// Slice-ordered lookups of [pkeys, pkeys+n): partition by table slice, then
// g.res_part[i] = packed slot of g.part_keys[i] (4 launches).
int probe_partitioned(const double* pkeys, uint64_t n, cudaStream_t s) {
  Ctx& g = cur();
  RET(partition_entries(pkeys, n, true, s));
  const uint64_t nall = probe_part_entries(n, g.jparts);
  CK(g.res_part.ensure(nall * 8));
  const int grid = resident_grid(join_probe_part_kernel, kProbeThreads, 0);
  const int policy = (int)env_u64("GOLP_JOIN_PART_POLICY", 0);
  const uint64_t items = (uint64_t)kProbeThreads * kPartProbeItems;
  const int gp = (int)std::max<uint64_t>(1, std::min<uint64_t>((nall + items - 1) / items, (uint64_t)grid));
  CK(g.work_ctr.ensure(8));
  CK(cudaMemsetAsync(g.work_ctr.p, 0, 8, s));
  const unsigned long long* cursors = g.part_cur.as<unsigned long long>();
  const PartExtent ext{probe_slice_capacity(n, g.jparts), g.jparts, cursors, cursors + g.jparts};
  join_probe_part_kernel<<<gp, kProbeThreads, 0, s>>>(g.part_keys.as<double>(), nall, g.table.as<Slot>(), g.jmask,
                                                      g.res_part.as<uint64_t>(), policy,
                                                      TileSched{g.work_ctr.as<unsigned long long>()}, ext);
  CKL();
  ++g_launches;
  return GOLP_OK;
}

// rows_dense: 1 when the caller knows the build row column is a dense run (the
// host regenerated it, upload_rows), 0 when unknown -- then a check kernel decides
// on the device for columns beyond kDenseCheckMin entries (below that the check
// would cost more than it saves). With a dense column singletons keep their
// position (the emit adds rows[0]): the finalize neither gathers nor stores them.
constexpr uint64_t kDenseCheckMin = 256u << 10;

#ifndef GOLP_GROUP_BITS_MIN_CAP
#define GOLP_GROUP_BITS_MIN_CAP (1ull << 20)
#endif
int join_build_impl(const double* bkeys, const uint32_t* brows, uint64_t nb, cudaStream_t s, int rows_dense = 0) {
  Ctx& g = cur();
  uint64_t cap = 1024;
  while (cap < 2 * nb && cap < (1ull << 32)) cap <<= 1;
#ifndef GOLP_SMALL_TABLE_SPREAD
#define GOLP_SMALL_TABLE_SPREAD 2
#endif
  // tables that stay in L2 either way get extra room: fewer CAS collisions in the
  // build and fewer second lookups in the probe
  {
    const uint64_t spread = env_u64("GOLP_SMALL_TABLE_SPREAD", GOLP_SMALL_TABLE_SPREAD);
    const uint64_t l2cap = env_u64("GOLP_SMALL_TABLE_BYTES", 64ull << 20) / sizeof(Slot);
    while (spread > 1 && cap * 2 <= l2cap && cap < 2 * spread * nb && cap < (1ull << 32)) cap <<= 1;
  }
  if (cap < 2 * nb || cap * kInline + nb > (1ull << 32)) {
    set_error("join build side too large for 32-bit slot / row indices");
    return GOLP_ERR_CAPACITY;
  }
  const uint64_t nbb = std::max<uint64_t>(nb, 1);
  CK(g.table.ensure(cap * sizeof(Slot)));
  CK(g.rows_arr.ensure((cap * kInline + nbb) * 4));
  CK(g.ovf.ensure(nbb * 12));
  CK(g.big_list.ensure((nbb / (kInline + 1) * 2 + 2) * 4));
  CK(g.jcount.ensure(32));
  CK(g.row_base.ensure(4));
  g.jcap = cap;
  g.jmask = cap - 1;
  g.jnb = nb;
  plan_partitions(cap);
  g.kt.join_capacity = cap;
  g.kt.join_slices = g.jparts;
  Slot* table = g.table.as<Slot>();
  // two "not dense" words, used by alternate builds (see join_init_table_kernel)
  if (!g.rows_flag.p) {
    CK(g.rows_flag.ensure(8));
    CK(cudaMemsetAsync(g.rows_flag.p, 0, 8, s));
  }
  unsigned* dflag = g.rows_flag.as<unsigned>() + g.build_parity;
  unsigned* dflag_next = g.rows_flag.as<unsigned>() + (g.build_parity ^ 1);
  g.build_parity ^= 1;
  const bool check = !rows_dense && nb >= kDenseCheckMin;
  // (the check itself runs inside join_init_table_kernel)
  const BuildRows br{brows, dflag};
  GroupArrays ga;
  ga.rows = g.rows_arr.as<uint32_t>();
  ga.ovf_slot = g.ovf.as<uint32_t>();
  ga.ovf_rank = ga.ovf_slot + nbb;
  ga.ovf_pos = ga.ovf_rank + nbb;
  ga.counters = g.jcount.as<unsigned long long>();
  ga.big_list = g.big_list.as<uint32_t>();
  // key groups flagged in a slot bitmap: a dense build's finalize visits only them
  ga.grp_bits = nullptr;
  if (cap >= env_u64("GOLP_GROUP_BITS_MIN_CAP", GOLP_GROUP_BITS_MIN_CAP)) {
    CK(g.grp_bits.ensure((cap + 31) / 32 * 4));
    ga.grp_bits = g.grp_bits.as<uint32_t>();
  }
  if (g.prof_build_start) prof_record(4, s);
  join_init_table_kernel<<<grid_for(cap, 256, 8), 256, 0, s>>>(table, cap, ga.grp_bits, brows, nb,
                                                                check ? 0 : (rows_dense ? 1 : 2), dflag, dflag_next,
                                                                ga.counters);
  CKL();
  ++g_launches;
  if (nb == 0) {
    prof_record(5, s);
    return GOLP_OK;
  }
  const double* ikeys = bkeys;
  const uint32_t* ipos = nullptr;
  if (g.jparts > 1) {
    RET(partition_entries(bkeys, nb, false, s));
    ikeys = g.part_keys.as<double>();
    ipos = g.part_pos.as<uint32_t>();
  }
#ifndef GOLP_BUILD_PER_SM
#define GOLP_BUILD_PER_SM 4
#endif
  int gb = grid_for((nb + kBuildItems - 1) / kBuildItems, kBuildThreads, GOLP_BUILD_PER_SM);
  TileSched sched{nullptr};
  if (ipos) {  // partitioned order: blocks claim tiles in order (see TileSched)
    const int grid = resident_grid(join_insert_kernel<true>, kBuildThreads, 0);
    gb = std::min(gb, grid);
    CK(g.work_ctr.ensure(8));
    CK(cudaMemsetAsync(g.work_ctr.p, 0, 8, s));
    sched.ctr = g.work_ctr.as<unsigned long long>();
  }
#ifndef GOLP_BUILD_WIDE_ALWAYS
#define GOLP_BUILD_WIDE_ALWAYS 1  // 16-byte claim CAS for L2-resident tables too (C2 build 78 -> 73 us)
#endif
  if (g.jparts > 1 || GOLP_BUILD_WIDE_ALWAYS)  // table in HBM: one 16-byte CAS per new key
    join_insert_kernel<true><<<gb, kBuildThreads, 0, s>>>(ikeys, ipos, nb, table, g.jmask, ga, sched);
  else
    join_insert_kernel<false><<<gb, kBuildThreads, 0, s>>>(ikeys, ipos, nb, table, g.jmask, ga, sched);
  CKL();
  join_finalize_kernel<<<grid_for(cap, 256, 8), 256, 0, s>>>(table, cap, br, ga, cap * kInline,
                                                               g.row_base.as<uint32_t>());
  CKL();
  join_overflow_kernel<<<g.sms, 256, 0, s>>>(table, ga);
  CKL();
  join_group_sort_kernel<<<g.sms, 256, 0, s>>>(table, ga, br);
  CKL();
  const size_t smem = kGroupTile * sizeof(uint32_t);
  RET(smem_attr(join_big_groups_kernel, smem));
  join_big_groups_kernel<<<std::max(1, g.sms / 4), 1024, smem, s>>>(table, ga, br);
  CKL();
  g_launches += 5;
  prof_record(5, s);
  return GOLP_OK;
}

// One probe over [pkeys, pkeys+np): match -> scan of block totals -> emit, per
// sub-chunk (the sub-chunk bounds the scratch); radix-partitioned probes
// (C4-sized tables) first partition each span and look its keys up slice by
// slice. Pair offsets continue from *base_in; *total_out = *base_in + pairs of
// this call.
int launch_probe(const double* pkeys, RowCol prows, uint64_t np, uint32_t* out_p, uint32_t* out_b,
                 uint64_t cap, const unsigned long long* base_in, unsigned long long* total_out, cudaStream_t s) {
  Ctx& g = cur();
  if (np == 0 || g.jnb == 0) {  // base_in null: no pairs before this probe
    if (base_in) CK(cudaMemcpyAsync(total_out, base_in, 8, cudaMemcpyDeviceToDevice, s));
    else CK(cudaMemsetAsync(total_out, 0, 8, s));
    return GOLP_OK;
  }
  // Partition the probe side (in spans of kSpan probes) when a span reuses each
  // table slice several times: span * 32 B of slot-pair reads >= 2x the table.
  // (GOLP_JOIN_SPAN shrinks the span so tests cover several spans on small inputs.)
  const uint64_t kSpan = std::max<uint64_t>(kPartTile, env_u64("GOLP_JOIN_SPAN", 1ull << 30) / kPartTile * kPartTile);
  const uint64_t force = env_u64("GOLP_JOIN_PART_PROBE", 2);
  const bool part_probe =
      g.jparts > 1 && (force == 1 || (force == 2 && std::min(np, kSpan) >= g.jcap));
  constexpr uint64_t kSub = 1ull << 27;  // probes per sub-chunk (scratch <= 1.5 GiB)
  const uint64_t sub = std::min(np, kSub);
  const uint64_t nwt_max = (sub + kWarpTile - 1) / kWarpTile;
  const uint64_t nwarps_max = (uint64_t)g.sms * GOLP_PROBE_MINB * kProbeWarps;
  CK(g.sc_prow.ensure(nwt_max * kWarpTile * 4));
  CK(g.sc_oc.ensure(nwt_max * kWarpTile * 8));
  CK(g.wcount.ensure((std::max(nwt_max, nwarps_max) + kProbeWarps) * 12));
  CK(g.totals2.ensure(16));
  MatchScratch sc;
  sc.prow = g.sc_prow.as<uint32_t>();
  sc.oc = g.sc_oc.as<uint64_t>();
  unsigned long long* tmp = g.totals2.as<unsigned long long>();
  const uint64_t span = part_probe ? kSpan : np;
  uint64_t ci = 0;  // running sub-chunk index (pair-offset chaining)
  for (uint64_t s0 = 0; s0 < np; s0 += span) {
    const uint64_t sn = std::min(span, np - s0);
    if (part_probe) RET(probe_partitioned(pkeys + s0, sn, s));
    for (uint64_t c0 = s0; c0 < s0 + sn; c0 += kSub) {
      const uint64_t cn = std::min(kSub, s0 + sn - c0);
      const uint64_t nwt = (cn + kWarpTile - 1) / kWarpTile;
      // one contiguous run of tiles per warp; enough warps to fill the GPU
      const uint64_t want_warps = std::min<uint64_t>(nwarps_max, nwt);
      // the partitioned path runs one block per partition tile (kRunWarpTiles per warp)
      const uint64_t per_warp = part_probe ? kRunWarpTiles : (nwt + want_warps - 1) / want_warps;
      const uint64_t warps = (nwt + per_warp - 1) / per_warp;
      const uint64_t blocks = (warps + kProbeWarps - 1) / kProbeWarps;
      sc.wpairs = g.wcount.as<unsigned long long>();
      sc.wentries = reinterpret_cast<uint32_t*>(sc.wpairs + blocks * kProbeWarps);
      CK(g.partial.ensure(blocks * 8));
      unsigned long long* part = g.partial.as<unsigned long long>();
      if (part_probe) {
        const uint64_t tile0 = (c0 - s0) / kPartTile;  // sub-chunks start on partition tiles
        RET(smem_attr(join_match_runs_kernel, kRunSmem));
        join_match_runs_kernel<<<(unsigned)blocks, kProbeThreads, kRunSmem, s>>>(
            prows.from(c0), cn, g.res_part.as<uint64_t>(), g.part_pos.as<uint16_t>(),
            g.run_base.as<uint32_t>() + tile0 * g.jparts, g.run_len.as<uint16_t>() + tile0 * g.jparts, g.jparts, sc,
            part);
      } else {
        join_match_kernel<<<(unsigned)blocks, kProbeThreads, 0, s>>>(pkeys + c0, prows.from(c0), cn, g.table.as<Slot>(),
                                                                     g.jmask, sc, nwt, per_warp, part);
      }
      CKL();
      const bool last = c0 + cn >= np;
      const unsigned long long* bin = ci == 0 ? base_in : tmp + (ci & 1);
      unsigned long long* bout = last ? total_out : tmp + ((ci + 1) & 1);
      ++ci;
      if (blocks <= kInlineScanBlocks) {  // emit blocks add up the earlier blocks' totals themselves
        join_emit_kernel<false><<<(unsigned)blocks, kProbeThreads, 0, s>>>(
            sc, g.rows_arr.as<uint32_t>(), nwt, per_warp, part, bin, bout, out_p, out_b, cap,
            g.row_base.as<uint32_t>());
      } else {
        scan_partials_kernel<<<1, kScanThreads, 0, s>>>(part, (uint32_t)blocks, bin, bout);
        CKL();
        ++g_launches;
        join_emit_kernel<true><<<(unsigned)blocks, kProbeThreads, 0, s>>>(
            sc, g.rows_arr.as<uint32_t>(), nwt, per_warp, part, bin, bout, out_p, out_b, cap,
            g.row_base.as<uint32_t>());
      }
      CKL();
      g_launches += 2;
    }
  }
  return GOLP_OK;
}

int read_u64(const void* dptr, uint64_t* out, cudaStream_t s) {
  Ctx& g = cur();
  uint64_t* h = static_cast<uint64_t*>(g.pin_small);
  CK(cudaMemcpyAsync(h, dptr, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *out = *h;
  return GOLP_OK;
}

// Match count of a finished probe (one sync).
int read_probe_total(const void* dptr, uint64_t* out, cudaStream_t s) { return read_u64(dptr, out, s); }

int join_probe_impl(const double* pkeys, RowCol prows, uint64_t np, uint32_t* out_p, uint32_t* out_b,
                    uint64_t cap, uint64_t* out_m, cudaStream_t s) {
  Ctx& g = cur();
  CK(g.totals.ensure(16));
  unsigned long long* totals = g.totals.as<unsigned long long>();
  prof_record(6, s);
  RET(launch_probe(pkeys, prows, np, out_p, out_b, cap, nullptr, totals + 1, s));
  prof_record(7, s);
  RET(read_probe_total(totals + 1, out_m, s));
  if (g.prof) g.kt.join_probe_ms = prof_ms(g.probe_start_ev, 7);
  return GOLP_OK;
}

cudaStream_t as_stream(void* p) { return p ? static_cast<cudaStream_t>(p) : (cudaStream_t)0; }

int check_mode(int mode, uint32_t payload_bytes, uint64_t* entry) {
  if (mode == GOLP_KEY_ONLY) {
    *entry = 12;
    return GOLP_OK;
  }
  if (mode == GOLP_FULL_ROW) {
    if (payload_bytes < 1) return invalid("full_row transfers need a positive payload_bytes");
    *entry = 8 + (uint64_t)payload_bytes;
    return GOLP_OK;
  }
  return invalid("unknown transfer mode");
}


// ---- full sort ----------------------------------------------------------------------
// host_full_sort on the device (sort.cuh): histogram pass, host picks the digits
// that need a pass (row digits only when the rows are not ascending; no
// single-bucket digits), then one onesweep pass per digit. The last pass writes
// only the rows, straight into out_rows.
int full_sort_impl(const double* keys, const uint32_t* rows, uint64_t n, uint32_t* out_rows, cudaStream_t s) {
  Ctx& g = cur();
  g.kt.full_sort_passes = 0;
  if (n == 0) return GOLP_OK;
  prof_record(0, s);
  CK(g.srt_hist.ensure(kSortDigits * 256 * 8 + 8));
  unsigned long long* hist = g.srt_hist.as<unsigned long long>();
  unsigned* unsorted = reinterpret_cast<unsigned*>(hist + kSortDigits * 256);
  CK(cudaMemsetAsync(hist, 0, kSortDigits * 256 * 8 + 8, s));
  sort_hist_kernel<<<grid_for(n, 256, 4), 256, 0, s>>>(keys, rows, n, hist, unsorted);
  CKL();
  ++g_launches;
  unsigned long long* hh = static_cast<unsigned long long*>(g.pin_small);
  CK(cudaMemcpyAsync(hh, hist, kSortDigits * 256 * 8 + 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const bool rows_sorted = *reinterpret_cast<const unsigned*>(hh + kSortDigits * 256) == 0;
  int digits[kSortDigits];
  int nd = 0;
  for (int d = 0; d < kSortDigits; ++d) {
    if (d < 4 && rows_sorted) continue;
    bool trivial = false;
    for (int b = 0; b < 256; ++b) trivial |= hh[d * 256 + b] == n;
    if (!trivial) digits[nd++] = d;
  }
  g.kt.full_sort_passes = (uint64_t)nd;
  if (nd == 0) {  // every item has the same code and the rows are in order already
    CK(cudaMemcpyAsync(out_rows, rows, n * 4, cudaMemcpyDeviceToDevice, s));
    prof_record(1, s);
    return GOLP_OK;
  }
  // exclusive global offsets of every digit that gets a pass
  unsigned long long* base = hh + kSortDigits * 256 + 8;
  for (int i = 0; i < nd; ++i) {
    unsigned long long run = 0;
    for (int b = 0; b < 256; ++b) {
      base[i * 256 + b] = run;
      run += hh[digits[i] * 256 + b];
    }
  }
  CK(g.srt_base.ensure((size_t)nd * 256 * 8));
  CK(cudaMemcpyAsync(g.srt_base.p, base, (size_t)nd * 256 * 8, cudaMemcpyHostToDevice, s));
  const uint64_t ntiles = (n + kSortTileN - 1) / kSortTileN;
  CK(g.srt_status.ensure(ntiles * 256 * 8 + 8));
  if (nd > 1) {
    CK(g.srt_k0.ensure(n * 8));
    CK(g.srt_r0.ensure(n * 4));
  }
  if (nd > 2) {
    CK(g.srt_k1.ensure(n * 8));
    CK(g.srt_r1.ensure(n * 4));
  }
  RET(smem_attr(sort_pass_kernel, kSortSmem));
  unsigned long long* status = g.srt_status.as<unsigned long long>();
  unsigned long long* ctr = status + ntiles * 256;
  const uint64_t* in_k = nullptr;
  const uint32_t* in_r = rows;
  for (int i = 0; i < nd; ++i) {
    const bool last = i + 1 == nd;
    uint64_t* ok = last ? nullptr : (i % 2 == 0 ? g.srt_k0.as<uint64_t>() : g.srt_k1.as<uint64_t>());
    uint32_t* orow = last ? out_rows : (i % 2 == 0 ? g.srt_r0.as<uint32_t>() : g.srt_r1.as<uint32_t>());
    CK(cudaMemsetAsync(status, 0, ntiles * 256 * 8 + 8, s));
    SortPassArgs a;
    a.in_f64 = i == 0 ? keys : nullptr;
    a.in_keys = in_k;
    a.in_rows = in_r;
    a.out_keys = ok;
    a.out_rows = orow;
    a.n = n;
    a.digit = digits[i];
    a.digit_base = g.srt_base.as<unsigned long long>() + (size_t)i * 256;
    a.status = status;
    a.tile_ctr = ctr;
    sort_pass_kernel<<<(unsigned)ntiles, kSortThreads, kSortSmem, s>>>(a);
    CKL();
    ++g_launches;
    in_k = ok;
    in_r = orow;
  }
  prof_record(1, s);
  return GOLP_OK;
}
}  // namespace

// Frees a context's streams, pinned staging and HBM workspace (the pinned
// result arena outlives it: result arrays may still be alive).
void release_context(Ctx& g) {
  if (!g.ready) return;
  cudaSetDevice(g.device);
  for (cudaStream_t st : {g.s_main, g.s_h2d, g.s_d2h}) cudaStreamSynchronize(st);
  g.pool.stop();
  DevBuf* bufs[] = {&g.ctl, &g.cand_hi, &g.cand_lo, &g.w_hi, &g.w_lo, &g.out_rows, &g.out_hi, &g.samples,
                    &g.table, &g.rows_arr, &g.ovf, &g.big_list, &g.grp_bits, &g.jcount,
                    &g.wcount, &g.partial, &g.totals, &g.totals2, &g.sc_prow, &g.sc_oc, &g.part_keys, &g.part_pos, &g.part_cnt, &g.part_cur, &g.run_base, &g.run_len, &g.res_part, &g.work_ctr, &g.pairs_p, &g.pairs_b, &g.srt_hist, &g.srt_k0, &g.srt_k1, &g.srt_r0, &g.srt_r1, &g.srt_status, &g.srt_base, &g.in_keys, &g.in_rows,
                    &g.in_bkeys, &g.in_brows, &g.in_payload, &g.rows_flag, &g.row_base};
  for (DevBuf* b : bufs) b->release();
  for (int i = 0; i < kSlots; ++i) {
    if (g.pin[i]) cudaFreeHost(g.pin[i]);
    if (g.pin_ev[i]) cudaEventDestroy(g.pin_ev[i]);
    g.pin[i] = nullptr;
    g.pin_ev[i] = nullptr;
    g.pin_busy[i] = false;
  }
  if (g.pin_small) cudaFreeHost(g.pin_small);
  g.pin_small = nullptr;
  if (g.status_host) cudaFreeHost(g.status_host);
  g.status_host = g.status_dev = nullptr;
  for (int i = 0; i < kD2HSlots; ++i) {
    if (g.dpin[i]) cudaFreeHost(g.dpin[i]);
    if (g.dpin_ev[i]) cudaEventDestroy(g.dpin_ev[i]);
    g.dpin[i] = nullptr;
    g.dpin_ev[i] = nullptr;
  }
  g.d2h_q.clear();
  g.d2h_head = 0;
  g.d2h_direct = false;
  for (cudaEvent_t e : g.chunk_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : g.h2d_ev) cudaEventDestroy(e);
  g.chunk_ev.clear();
  g.h2d_ev.clear();
  if (g.mirror) cudaFreeHost(g.mirror);
  g.mirror = nullptr;
  g.mirror_dev = nullptr;
  g.mirror_n = 0;
  for (auto& e : g.ev) {
    if (e) cudaEventDestroy(e);
    e = nullptr;
  }
  if (g.ev_rows) cudaEventDestroy(g.ev_rows);
  g.ev_rows = nullptr;
  cudaStreamDestroy(g.s_main);
  cudaStreamDestroy(g.s_h2d);
  cudaStreamDestroy(g.s_d2h);
  g.jcap = g.jmask = g.jnb = 0;
  g.last_probe_valid = false;
  g.smem_set.clear();
  g.per_sm.clear();
  for (cudaEvent_t e : g.trace_ev) cudaEventDestroy(e);
  g.trace_ev.clear();
  for (cudaEvent_t e : g.kspan_ev) cudaEventDestroy(e);
  g.kspan_ev.clear();
  g.kspan_n = 0;
  g.ready = false;
}

// =====================================================================================
extern "C" {

const char* golp_last_error(void) { return last_error_cstr(); }
int golp_version(void) { return 1; }

int golp_init(int device, uint64_t pinned_chunk_bytes, int host_threads) {
  if (device < 0) device = device_of_thread();
  const int h = default_handle(device);
  if (h < 0) return invalid("device index out of range");
  t_cur = g_ctx[h];
  return do_init(*t_cur, device, pinned_chunk_bytes, host_threads);
}

int golp_use_device(int device) { return golp_init(device, 0, 0); }

int golp_current_device(int* device) {
  if (!device) return invalid("null output");
  RET(ensure_init());
  *device = cur().device;
  return GOLP_OK;
}

int golp_context_open(int device, uint64_t pinned_chunk_bytes, int host_threads, int* handle) {
  if (!handle) return invalid("null handle");
  if (device < 0) device = device_of_thread();
  int h = -1;
  {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    for (int i = 0; i < kMaxContexts; ++i)
      if (!g_ctx[i]) {
        g_ctx[i] = new Ctx();
        g_ctx[i]->device = device;
        h = i;
        break;
      }
  }
  if (h < 0) return invalid("too many golp contexts");
  t_cur = g_ctx[h];
  RET(do_init(*t_cur, device, pinned_chunk_bytes, host_threads));
  *handle = h;
  return GOLP_OK;
}

int golp_context_use(int handle) {
  if (handle < 0 || handle >= kMaxContexts || !g_ctx[handle]) return invalid("unknown golp context");
  t_cur = g_ctx[handle];
  return ensure_init();
}

int golp_context_close(int handle) {
  if (handle < 0 || handle >= kMaxContexts || !g_ctx[handle]) return invalid("unknown golp context");
  release_context(*g_ctx[handle]);
  return GOLP_OK;
}

// Releases every context (process-wide). Context objects stay allocated, so a
// thread that still has one selected re-initializes it on its next call.
int golp_shutdown(void) {
  for (int h = 0; h < kMaxContexts; ++h)
    if (g_ctx[h]) release_context(*g_ctx[h]);
  return GOLP_OK;
}

uint64_t golp_launch_count(void) { return g_launches.load(); }

int golp_set_dense_rows(int on) {
  Ctx& g = cur();
  RET(ensure_init());
  g.dense_rows = on != 0;
  return GOLP_OK;
}

int golp_last_transfer(uint64_t* h2d_bytes, uint64_t* d2h_bytes) {
  Ctx& g = cur();
  if (!h2d_bytes || !d2h_bytes) return invalid("null output pointer");
  *h2d_bytes = g.moved_h2d;
  *d2h_bytes = g.moved_d2h;
  return GOLP_OK;
}

int golp_hint_dense_rows(void) {
  RET(ensure_init());
  cur().rows_hint = true;
  return GOLP_OK;
}

int golp_set_profiling(int on) {
  Ctx& g = cur();
  RET(ensure_init());
  g.prof = on != 0;
  g.prof_build_start = on != 2;
  g.build_timed = g.probe_timed = g.topk_timed = false;
  return GOLP_OK;
}

// The timing flags stay set while profiling is on, so a CUDA graph that captured
// the event records can be replayed and read again after every replay.
int golp_last_kernel_times(golp_kernel_times* out) {
  Ctx& g = cur();
  if (!out) return invalid("null output");
  if (g.topk_pending) {
    CK(cudaDeviceSynchronize());
    g.kt.topk_candidates = *reinterpret_cast<volatile unsigned long long*>(g.status_host + 8);
    g.kt.topk_fallback = *reinterpret_cast<volatile int*>(g.status_host) != 0;
  }
  if (g.topk_timed) {
    CK(cudaEventSynchronize(g.ev[3]));
    g.kt.topk_select_ms = prof_ms(0, 3);
  }
  if (g.build_timed) {
    CK(cudaEventSynchronize(g.ev[5]));
    g.kt.join_build_ms = prof_ms(4, 5);
  }
  if (g.probe_timed) {
    CK(cudaEventSynchronize(g.ev[7]));
    g.kt.join_probe_ms = prof_ms(g.probe_start_ev, 7);
  }
  *out = g.kt;
  return GOLP_OK;
}

// ---- device-resident ------------------------------------------------------------------
int golp_topk_device(const double* d_keys, const uint32_t* d_rows, uint64_t n, uint64_t k, uint32_t* d_out_rows,
                     uint64_t* d_out_keys, void* stream) {
  if (k < 1) return invalid("k must be at least 1");
  RET(ensure_init());
  if (n > 0 && (!d_keys || !d_rows || !d_out_rows)) return invalid("null device pointer");
  RET(check_device_ptr(d_keys));
  return topk_device_impl(d_keys, RowCol{d_rows, 0}, n, k, d_out_rows, d_out_keys, as_stream(stream));
}

int golp_topk_device_positions(const double* d_keys, uint64_t n, uint32_t row_base, uint64_t k,
                               uint32_t* d_out_rows, uint64_t* d_out_keys, void* stream) {
  if (k < 1) return invalid("k must be at least 1");
  if (n > 0 && (uint64_t)row_base + n - 1 > 0xFFFFFFFFull) return invalid("row ids row_base + i exceed u32");
  RET(ensure_init());
  if (n > 0 && (!d_keys || !d_out_rows)) return invalid("null device pointer");
  RET(check_device_ptr(d_keys));
  return topk_device_impl(d_keys, RowCol{nullptr, row_base}, n, k, d_out_rows, d_out_keys, as_stream(stream));
}

int golp_full_sort_device(const double* d_keys, const uint32_t* d_rows, uint64_t n, uint32_t* d_out_rows,
                          void* stream) {
  Ctx& g = cur();
  RET(ensure_init());
  if (n > 0 && (!d_keys || !d_rows || !d_out_rows)) return invalid("null device pointer");
  RET(check_device_ptr(d_keys));
  cudaStream_t s = as_stream(stream);
  RET(full_sort_impl(d_keys, d_rows, n, d_out_rows, s));
  if (g.prof) {
    CK(cudaStreamSynchronize(s));
    g.kt.full_sort_ms = prof_ms(0, 1);
  }
  return GOLP_OK;
}

int golp_full_sort(const double* keys, const uint32_t* rows, uint64_t n, int mode, uint32_t payload_bytes,
                   uint32_t* out_rows, golp_ledger* led) {
  Ctx& g = cur();
  uint64_t entry = 0;
  RET(check_mode(mode, payload_bytes, &entry));
  if (!led) return invalid("null ledger");
  RET(ensure_init());
  g.moved_h2d = g.moved_d2h = 0;
  kspan_reset();
  struct HintReset {  // the row-id hint covers this one call
    Ctx& c;
    ~HintReset() { c.rows_hint = false; }
  } hint_reset{g};
  const double t0 = wall_seconds();
  *led = golp_ledger{entry * n, 4 * n, 0.0, 0.0, 0.0, 0.0};
  if (n == 0) return GOLP_OK;
  if (!keys || !rows || !out_rows) return invalid("null buffer");
  cudaStream_t s = g.s_main;
  CK(g.in_keys.ensure(n * 8));
  CK(g.in_rows.ensure(n * 4));
  CK(g.out_rows.ensure(n * 4));
  RET(stage_h2d(g.in_keys.p, keys, n * 8));
  RET(upload_rows(g.in_rows.as<uint32_t>(), rows, n));
  if (mode == GOLP_FULL_ROW) RET(stage_dummy_h2d(n * (size_t)payload_bytes));
  cudaEvent_t ev_up = g.ev[2];
  CK(cudaEventRecord(ev_up, g.s_h2d));
  CK(cudaEventSynchronize(ev_up));
  g.next_slot = 0;
  for (bool& b : g.pin_busy) b = false;
  const double t1 = wall_seconds();
  CK(cudaStreamWaitEvent(s, ev_up, 0));
  RET(kspan_mark(s));
  RET(full_sort_impl(g.in_keys.as<double>(), g.in_rows.as<uint32_t>(), n, g.out_rows.as<uint32_t>(), s));
  RET(kspan_mark(s));
  CK(cudaStreamSynchronize(s));
  if (g.prof) g.kt.full_sort_ms = prof_ms(0, 1);
  const double t2 = wall_seconds();
  if (is_pinned(out_rows, n * 4)) {
    CK(cudaMemcpyAsync(out_rows, g.out_rows.p, n * 4, cudaMemcpyDeviceToHost, g.s_d2h));
    g.moved_d2h += n * 4;
    CK(cudaStreamSynchronize(g.s_d2h));
  } else {
    RET(stage_d2h(out_rows, g.out_rows.p, n * 4));
  }
  led->t_h2d = t1 - t0;
  led->t_kernel = t2 - t1;
  led->t_d2h = wall_seconds() - t2;
  return kspan_finish();
}

int golp_topk_merge_device(const uint64_t* d_key_codes, const uint32_t* d_rows, uint64_t n, uint64_t k,
                           uint32_t* d_out_rows, uint64_t* d_out_keys, void* stream) {
  if (k < 1) return invalid("k must be at least 1");
  RET(ensure_init());
  const uint64_t kk = std::min(k, n);
  if (kk == 0) return GOLP_OK;
  RET(check_device_ptr(d_key_codes));
  cudaStream_t s = as_stream(stream);
  RET(ensure_topk_ws(kk, 0));
  CK(cudaMemsetAsync(ctl(2), 0, sizeof(SelectCtl), s));
  RET(launch_select(make_args(SrcPairs{d_key_codes, d_rows}, n, kk, kModeFull, 2, d_out_rows, d_out_keys), s));
  CK(cudaStreamSynchronize(s));
  return GOLP_OK;
}

int golp_join_build_device(const double* d_build_keys, const uint32_t* d_build_rows, uint64_t nb, void* stream) {
  Ctx& g = cur();
  RET(ensure_init());
  RET(check_device_ptr(d_build_keys));
  cudaStream_t s = as_stream(stream);
  RET(join_build_impl(d_build_keys, d_build_rows, nb, s));
  g.build_timed = g.prof && g.prof_build_start;  // resolved lazily by golp_last_kernel_times (no sync here)
  if (g.prof && !g.prof_build_start) g.kt.join_build_ms = 0.0;
  return GOLP_OK;
}

namespace {
int probe_device_async(const double* d_probe_keys, RowCol prows, uint64_t np, uint32_t* d_out_probe_rows,
                       uint32_t* d_out_build_rows, uint64_t cap, uint64_t* d_out_matches, void* stream) {
  Ctx& g = cur();
  RET(ensure_init());
  if (!d_out_matches) return invalid("null d_out_matches");
  RET(check_device_ptr(d_probe_keys));
  cudaStream_t s = as_stream(stream);
  prof_record(6, s);
  RET(launch_probe(d_probe_keys, prows, np, d_out_probe_rows, d_out_build_rows, cap, nullptr,
                   reinterpret_cast<unsigned long long*>(d_out_matches), s));
  prof_record(7, s);
  g.probe_timed = g.prof;  // resolved lazily by golp_last_kernel_times
  return GOLP_OK;
}

int probe_device(const double* d_probe_keys, RowCol prows, uint64_t np, uint32_t* d_out_probe_rows,
                 uint32_t* d_out_build_rows, uint64_t cap, uint64_t* out_matches, void* stream) {
  RET(ensure_init());
  if (!out_matches) return invalid("null out_matches");
  RET(check_device_ptr(d_probe_keys));
  cudaStream_t s = as_stream(stream);
  RET(join_probe_impl(d_probe_keys, prows, np, d_out_probe_rows, d_out_build_rows, cap, out_matches, s));
  if (*out_matches > cap) {
    set_error("probe output exceeds the supplied capacity");
    return GOLP_ERR_CAPACITY;
  }
  return GOLP_OK;
}

int check_positions(uint64_t n, uint32_t row_base) {
  if (n > 0 && (uint64_t)row_base + n - 1 > 0xFFFFFFFFull) return invalid("row ids row_base + i exceed u32");
  return GOLP_OK;
}
}  // namespace

int golp_join_probe_device_async(const double* d_probe_keys, const uint32_t* d_probe_rows, uint64_t np,
                                 uint32_t* d_out_probe_rows, uint32_t* d_out_build_rows, uint64_t cap,
                                 uint64_t* d_out_matches, void* stream) {
  if (np > 0 && !d_probe_rows) return invalid("null device pointer");
  return probe_device_async(d_probe_keys, RowCol{d_probe_rows, 0}, np, d_out_probe_rows, d_out_build_rows, cap,
                            d_out_matches, stream);
}

int golp_join_probe_device(const double* d_probe_keys, const uint32_t* d_probe_rows, uint64_t np,
                           uint32_t* d_out_probe_rows, uint32_t* d_out_build_rows, uint64_t cap,
                           uint64_t* out_matches, void* stream) {
  if (np > 0 && !d_probe_rows) return invalid("null device pointer");
  return probe_device(d_probe_keys, RowCol{d_probe_rows, 0}, np, d_out_probe_rows, d_out_build_rows, cap, out_matches,
                      stream);
}

int golp_join_probe_device_positions_async(const double* d_probe_keys, uint64_t np, uint32_t row_base,
                                           uint32_t* d_out_probe_rows, uint32_t* d_out_build_rows, uint64_t cap,
                                           uint64_t* d_out_matches, void* stream) {
  RET(check_positions(np, row_base));
  return probe_device_async(d_probe_keys, RowCol{nullptr, row_base}, np, d_out_probe_rows, d_out_build_rows, cap,
                            d_out_matches, stream);
}

int golp_join_probe_device_positions(const double* d_probe_keys, uint64_t np, uint32_t row_base,
                                     uint32_t* d_out_probe_rows, uint32_t* d_out_build_rows, uint64_t cap,
                                     uint64_t* out_matches, void* stream) {
  RET(check_positions(np, row_base));
  return probe_device(d_probe_keys, RowCol{nullptr, row_base}, np, d_out_probe_rows, d_out_build_rows, cap,
                      out_matches, stream);
}

// ---- host buffers (E2E) -----------------------------------------------------------------
int golp_topk(const double* keys, const uint32_t* rows, uint64_t n, uint64_t k, int mode, uint32_t payload_bytes,
              uint32_t* out_rows, uint64_t* out_len, golp_ledger* led) {
  return golp_topk_codes(keys, rows, n, k, mode, payload_bytes, out_rows, nullptr, out_len, led);
}

int golp_topk_codes(const double* keys, const uint32_t* rows, uint64_t n, uint64_t k, int mode,
                    uint32_t payload_bytes, uint32_t* out_rows, uint64_t* out_codes, uint64_t* out_len,
                    golp_ledger* led) {
  Ctx& g = cur();
  if (k < 1) return invalid("k must be at least 1");
  uint64_t entry = 0;
  RET(check_mode(mode, payload_bytes, &entry));
  if (!out_len || !led) return invalid("null output pointer");
  RET(ensure_init());
  g.moved_h2d = g.moved_d2h = 0;
  kspan_reset();
  struct HintReset {  // the row-id hint covers this one call
    Ctx& c;
    ~HintReset() { c.rows_hint = false; }
  } hint_reset{g};
  const double t0 = wall_seconds();
  const uint64_t kk = std::min(k, n);
  *out_len = kk;
  *led = golp_ledger{entry * n, 4 * kk, 0.0, 0.0, 0.0, 0.0};
  if (n == 0) return GOLP_OK;
  if (!keys || !rows || !out_rows) return invalid("null buffer");
  cudaStream_t s = g.s_main;
  CK(g.in_keys.ensure(n * 8));
  CK(g.in_rows.ensure(n * 4));
  CK(g.out_rows.ensure(kk * 4));
  if (out_codes) CK(g.out_hi.ensure(kk * 8));
  uint64_t* d_hi = out_codes ? g.out_hi.as<uint64_t>() : nullptr;  // winners' order codes (cross-shard merges)
  double* dk = g.in_keys.as<double>();
  uint32_t* dr = g.in_rows.as<uint32_t>();
  const TopkPlan p = plan_topk(n, kk);
  RET(ensure_topk_ws(kk, p.direct ? 0 : p.cap));
  g.kt.topk_fallback = 0;
  g.kt.topk_candidates = 0;

  cudaEvent_t ev_chunk = g.ev[0];
  const uint64_t per_chunk = std::max<uint64_t>(g.chunk / 8, 1);
  if (n <= per_chunk) {
    // One chunk: upload both columns, then the device-resident pipeline (the
    // samples are drawn on the device; nothing to overlap with).
    const bool trace = std::getenv("GOLP_TRACE") != nullptr;
    RET(stage_h2d(dk, keys, n * 8));
    if (trace) std::fprintf(stderr, "[golp] topk %.3f ms keys queued\n", (wall_seconds() - t0) * 1e3);
    RowCol rc{dr, 0};
    RET(upload_rows(dr, rows, n, nullptr, &rc));
    if (mode == GOLP_FULL_ROW) RET(stage_dummy_h2d(n * (size_t)payload_bytes));
    CK(cudaEventRecord(ev_chunk, g.s_h2d));
    if (trace) std::fprintf(stderr, "[golp] topk %.3f ms rows queued\n", (wall_seconds() - t0) * 1e3);
    CK(cudaEventSynchronize(ev_chunk));
    g.next_slot = 0;
    for (bool& b : g.pin_busy) b = false;
    const double t1 = wall_seconds();
    if (trace) std::fprintf(stderr, "[golp] topk %.3f ms uploads done\n", (t1 - t0) * 1e3);
    CK(cudaStreamWaitEvent(s, ev_chunk, 0));
    uint32_t* d_out = g.out_rows.as<uint32_t>();
    RET(kspan_mark(s));
    RET(topk_device_impl(dk, rc, n, kk, d_out, d_hi, s));
    RET(kspan_mark(s));
    CK(cudaStreamSynchronize(s));  // the fused path is stream-ordered: charge its time to t_kernel
    const double t2 = wall_seconds();
    uint32_t* hbuf = static_cast<uint32_t*>(g.pin_small);
    if (kk * 4 <= g.pin_small_bytes) {
      CK(cudaMemcpyAsync(hbuf, d_out, kk * 4, cudaMemcpyDeviceToHost, s));
      g.moved_d2h += kk * 4;
      CK(cudaStreamSynchronize(s));
      std::memcpy(out_rows, hbuf, kk * 4);
    } else {
      RET(stage_d2h(out_rows, d_out, kk * 4));
    }
    if (out_codes) RET(stage_d2h(out_codes, d_hi, kk * 8));
    led->t_h2d = t1 - t0;
    led->t_kernel = t2 - t1;
    led->t_d2h = wall_seconds() - t2;
    return kspan_finish();
  }
  if (!p.direct) {
    // Stratified samples gathered on the host (same strata as SrcSample).
    double* hs = static_cast<double*>(g.pin_small);
    uint32_t* hr = reinterpret_cast<uint32_t*>(hs + p.s);
    const uint32_t w = (uint32_t)std::max<uint64_t>(1, n / p.s);
    for (uint64_t i = 0; i < p.s; ++i) {
      uint64_t pos = i * w + (hash32((uint32_t)i * 2654435761u + 12345u) % w);
      if (pos >= n) pos = n - 1;
      hs[i] = keys[pos];
      hr[i] = rows[pos];
    }
    CK(g.samples.ensure(p.s * 12));
    double* ds = g.samples.as<double>();
    uint32_t* dsr = reinterpret_cast<uint32_t*>(ds + p.s);
    CK(cudaMemcpyAsync(ds, hs, p.s * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dsr, hr, p.s * 4, cudaMemcpyHostToDevice, s));
    g.moved_h2d += p.s * 12;
    CK(cudaMemsetAsync(ctl(0), 0, sizeof(SelectCtl) * 2, s));
    RET(launch_select(make_args(SrcInput{ds, RowCol{dsr, 0}}, p.s, p.need_s, kModeThreshold, 0, nullptr, nullptr), s));
  }
  // Stream the columns chunk by chunk; filter each chunk as soon as it lands.
  // The rows of chunk c are verified (or copied) after the keys of chunk c+1
  // are queued, so the copy engine has the next upload while the pool reads.
  // h2d_ev[c] fires when the keys of chunk c have landed; a copied row column
  // (or full-row payload) adds a second event after the next chunk's keys.
  const uint64_t nchunks = (n + per_chunk - 1) / per_chunk;
  RET(ensure_chunk_events(nchunks));
  auto finish_chunk = [&](uint64_t c) -> int {
    const uint64_t c0 = c * per_chunk, cn = std::min(per_chunk, n - c0);
    bool copied = false;
    RET(upload_rows(dr + c0, rows + c0, cn, &copied));
    if (mode == GOLP_FULL_ROW) RET(stage_dummy_h2d(cn * (size_t)payload_bytes));
    if (!p.direct) {
      CK(cudaStreamWaitEvent(s, g.h2d_ev[c], 0));
      if (copied || mode == GOLP_FULL_ROW) {
        CK(cudaEventRecord(ev_chunk, g.s_h2d));
        CK(cudaStreamWaitEvent(s, ev_chunk, 0));
      }
      RET(kspan_mark(s));
      RET(launch_filter(dk + c0, RowCol{dr + c0, 0}, cn, p.cap, s));
      RET(kspan_mark(s));
    }
    return GOLP_OK;
  };
  for (uint64_t c = 0; c < nchunks; ++c) {
    const uint64_t c0 = c * per_chunk;
    RET(stage_h2d(dk + c0, keys + c0, std::min(per_chunk, n - c0) * 8));
    CK(cudaEventRecord(g.h2d_ev[c], g.s_h2d));
    if (c) RET(finish_chunk(c - 1));
  }
  RET(finish_chunk(nchunks - 1));
  CK(cudaEventRecord(ev_chunk, g.s_h2d));
  CK(cudaEventSynchronize(ev_chunk));
  g.next_slot = 0;
  for (bool& b : g.pin_busy) b = false;
  const double t1 = wall_seconds();
  CK(cudaStreamWaitEvent(s, ev_chunk, 0));
  uint32_t* d_out = g.out_rows.as<uint32_t>();
  RET(kspan_mark(s));
  if (p.direct) {
    RET(topk_direct(dk, RowCol{dr, 0}, n, kk, d_out, d_hi, s));
    CK(cudaStreamSynchronize(s));
  } else {
    RET(ensure_status_words());
    RET(launch_select(cand_args(kk, p.cap, d_out, d_hi), s));
    int bad = 0;
    uint64_t cands = 0;
    RET(read_topk_status(s, &bad, &cands));
    g.kt.topk_candidates = cands;
    if (bad) {
      g.kt.topk_fallback = 1;
      RET(topk_direct(dk, RowCol{dr, 0}, n, kk, d_out, d_hi, s));
      CK(cudaStreamSynchronize(s));
    }
  }
  RET(kspan_mark(s));
  const double t2 = wall_seconds();
  uint32_t* hbuf = static_cast<uint32_t*>(g.pin_small);
  if (kk * 4 <= g.pin_small_bytes) {
    CK(cudaMemcpyAsync(hbuf, d_out, kk * 4, cudaMemcpyDeviceToHost, s));
    g.moved_d2h += kk * 4;
    CK(cudaStreamSynchronize(s));
    std::memcpy(out_rows, hbuf, kk * 4);
  } else {
    CK(cudaStreamSynchronize(s));
    RET(stage_d2h(out_rows, d_out, kk * 4));
  }
  if (out_codes) RET(stage_d2h(out_codes, d_hi, kk * 8));
  const double t3 = wall_seconds();
  led->t_h2d = t1 - t0;
  led->t_kernel = t2 - t1;
  led->t_d2h = t3 - t2;
  return kspan_finish();
}

#ifndef GOLP_TAIL_SPLIT
#define GOLP_TAIL_SPLIT 4
#endif
#ifndef GOLP_H2D_AHEAD
#define GOLP_H2D_AHEAD 2
#endif
int golp_probe(const double* build_keys, const uint32_t* build_rows, uint64_t nb, const double* probe_keys,
               const uint32_t* probe_rows, uint64_t np, int mode, uint32_t payload_bytes, uint32_t* out_probe_rows,
               uint32_t* out_build_rows, uint64_t out_cap, uint64_t* out_matches, golp_ledger* led) {
  Ctx& g = cur();
  uint64_t entry = 0;
  RET(check_mode(mode, payload_bytes, &entry));
  if (!out_matches || !led) return invalid("null output pointer");
  if (out_cap && (!out_probe_rows || !out_build_rows)) return invalid("null output arrays");
  RET(ensure_init());
  g.last_probe_valid = false;
  g.moved_h2d = g.moved_d2h = 0;
  kspan_reset();
  struct HintReset {  // the row-id hint covers this one call
    Ctx& c;
    ~HintReset() { c.rows_hint = false; }
  } hint_reset{g};
  const double t0 = wall_seconds();
  *led = golp_ledger{entry * (nb + np), 0, 0.0, 0.0, 0.0, 0.0};
  *out_matches = 0;
  if ((nb && (!build_keys || !build_rows)) || (np && (!probe_keys || !probe_rows))) return invalid("null buffer");
  cudaStream_t s = g.s_main;
  CK(g.in_bkeys.ensure(std::max<uint64_t>(nb, 1) * 8));
  CK(g.in_brows.ensure(std::max<uint64_t>(nb, 1) * 4));
  CK(g.in_keys.ensure(std::max<uint64_t>(np, 1) * 8));
  CK(g.in_rows.ensure(std::max<uint64_t>(np, 1) * 4));
  double* dbk = g.in_bkeys.as<double>();
  uint32_t* dbr = g.in_brows.as<uint32_t>();
  double* dpk = g.in_keys.as<double>();
  uint32_t* dpr = g.in_rows.as<uint32_t>();

  // GOLP_TRACE: per-upload host queue times and device completion times
  const bool trace = std::getenv("GOLP_TRACE") != nullptr;
  std::vector<cudaEvent_t>& tr_ev = g.trace_ev;
  std::vector<double> tr_q;
  auto tr_mark = [&]() -> int {
    if (!trace) return GOLP_OK;
    if (tr_ev.size() <= tr_q.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      tr_ev.push_back(e);
    }
    CK(cudaEventRecord(tr_ev[tr_q.size()], g.s_h2d));
    tr_q.push_back((wall_seconds() - t0) * 1e3);
    return GOLP_OK;
  };
  RET(tr_mark());
  // build side first, then the probe side in chunks that are probed as they land
  RET(stage_h2d(dbk, build_keys, nb * 8));
  bool brows_copied = true;
  RET(upload_rows(dbr, build_rows, nb, &brows_copied));
  RET(tr_mark());
  if (mode == GOLP_FULL_ROW) RET(stage_dummy_h2d(nb * (size_t)payload_bytes));
  cudaEvent_t ev_chunk = g.ev[0];
  CK(cudaEventRecord(ev_chunk, g.s_h2d));
  CK(cudaStreamWaitEvent(s, ev_chunk, 0));
  RET(kspan_mark(s));
  RET(join_build_impl(dbk, dbr, nb, s, (nb > 0 && !brows_copied) ? 1 : 0));
  RET(kspan_mark(s));

  uint64_t per_chunk = std::max<uint64_t>(g.chunk / 8, kWarpTile);
  per_chunk = (per_chunk / kWarpTile) * kWarpTile;
  // Chunk bounds: full staging chunks, then the last chunk's worth of probes in
  // kTailSplit pieces, so the work left after the final upload (its probe and
  // its pairs' download) is a fraction of a chunk.
  constexpr uint64_t kTailSplit = GOLP_TAIL_SPLIT;
  std::vector<uint64_t> cb{0};
  while (cb.back() < np) {
    const uint64_t left = np - cb.back();
    uint64_t len = per_chunk;
    if (left <= per_chunk) {
      len = std::max<uint64_t>(((per_chunk / kTailSplit) / kWarpTile) * kWarpTile, kWarpTile);
      if (left < 2 * len) len = left;
    }
    cb.push_back(cb.back() + std::min(len, left));
  }
  const uint64_t nchunks = cb.size() - 1;
  // each chunk's probe row ids: its slice of the device column, or positions when dense
  std::vector<RowCol> crows(nchunks, RowCol{nullptr, 0});
  for (uint64_t c = 0; c < nchunks; ++c) crows[c] = RowCol{dpr + cb[c], 0};
  CK(g.totals.ensure((nchunks + 1) * 8));
  CK(cudaMemsetAsync(g.totals.p, 0, (nchunks + 1) * 8, s));
  RET(ensure_chunk_events(nchunks));
  g.mirror[0] = 0;
  // Pairs land in HBM and stream back through the D2H engine chunk by chunk.
  // (A zero-copy variant -- the emit kernel storing pairs into the pinned arena
  // over PCIe -- measured 3x slower at C2: 4-byte scattered stores make poor
  // PCIe transactions.)
  // At least the caller's capacity: M > dcap then implies M > out_cap (copy_out path).
  uint64_t dcap = std::max<uint64_t>(g.pairs_p.bytes / 4, std::max<uint64_t>(std::max<uint64_t>(np, out_cap), 1024));
  CK(g.pairs_p.ensure(dcap * 4));
  CK(g.pairs_b.ensure(dcap * 4));
  dcap = std::min(g.pairs_p.bytes, g.pairs_b.bytes) / 4;
  uint32_t* dev_p = g.pairs_p.as<uint32_t>();
  uint32_t* dev_b = g.pairs_b.as<uint32_t>();
  unsigned long long* totals = g.totals.as<unsigned long long>();
  // Pairs of chunk c stream back (DMA + unpack into the caller's arrays) while
  // later chunks upload; a chunk is ready once its probe event has fired.
  uint64_t streamed = 0;     // chunks whose pairs are queued for D2H
  bool streaming = out_cap > 0;
  auto stream_ready = [&](bool block) -> int {
    while (streaming && streamed < nchunks) {
      cudaEvent_t e = g.chunk_ev[streamed];
      if (block) {
        CK(cudaEventSynchronize(e));
      } else {
        const cudaError_t q = cudaEventQuery(e);
        if (q == cudaErrorNotReady) break;
        CK(q);
      }
      const uint64_t lo = g.mirror[streamed], hi = g.mirror[streamed + 1];
      if (trace) std::fprintf(stderr, "[golp] %.3f ms chunk %llu probed, pairs [%llu, %llu)\n", (wall_seconds() - t0) * 1e3,
                              (unsigned long long)streamed, (unsigned long long)lo, (unsigned long long)hi);
      if (hi > out_cap || hi > dcap) {
        streaming = false;  // caller's arrays (or the device buffer) too small: copy_out path
        break;
      }
      if (hi > lo) {
        RET(d2h_enqueue(out_probe_rows + lo, dev_p + lo, (hi - lo) * 4));
        RET(d2h_enqueue(out_build_rows + lo, dev_b + lo, (hi - lo) * 4));
      }
      ++streamed;
    }
    return d2h_poll();
  };
  // The rows of chunk c are verified (or copied) after the keys of chunk c+1
  // are queued, so the copy engine has the next upload while the pool reads.
  // h2d_ev[c] fires when the keys of chunk c have landed; a copied row column
  // (or full-row payload) adds a second event after the next chunk's keys.
  auto finish_upload = [&](uint64_t c) -> int {
    const uint64_t c0 = cb[c], cn = cb[c + 1] - c0;
    bool copied = false;
    RET(upload_rows(dpr + c0, probe_rows + c0, cn, &copied, &crows[c]));
    if (mode == GOLP_FULL_ROW) RET(stage_dummy_h2d(cn * (size_t)payload_bytes));
    CK(cudaStreamWaitEvent(s, g.h2d_ev[c], 0));
    if (copied || mode == GOLP_FULL_ROW) {
      CK(cudaEventRecord(g.ev_rows, g.s_h2d));
      CK(cudaStreamWaitEvent(s, g.ev_rows, 0));
    }
    return GOLP_OK;
  };
  auto probe_chunk = [&](uint64_t c, uint32_t* op, uint32_t* ob, uint64_t cap_) -> int {
    const uint64_t c0 = cb[c], cn = cb[c + 1] - c0;
    RET(kspan_mark(s));
    RET(launch_probe(dpk + c0, crows[c], cn, op, ob, cap_, totals + c, totals + c + 1, s));
    RET(kspan_mark(s));
    publish_u64_kernel<<<1, 1, 0, s>>>(reinterpret_cast<volatile unsigned long long*>(g.mirror_dev + c + 1),
                                       totals + c + 1);
    CKL();
    ++g_launches;
    CK(cudaEventRecord(g.chunk_ev[c], s));
    return GOLP_OK;
  };
  auto run_chunks = [&](bool with_h2d, uint32_t* op, uint32_t* ob, uint64_t cap_) -> int {
    if (!with_h2d) {
      for (uint64_t c = 0; c < nchunks; ++c) RET(probe_chunk(c, op, ob, cap_));
      return GOLP_OK;
    }
    for (uint64_t c = 0; c < nchunks; ++c) {
      // Keep at most GOLP_H2D_AHEAD chunks of uploads in flight: copies are
      // serviced in submission order, so pair downloads queued in between can
      // overlap them.
      if (c >= GOLP_H2D_AHEAD) {
        while (true) {
          const cudaError_t q = cudaEventQuery(g.h2d_ev[c - GOLP_H2D_AHEAD]);
          if (q == cudaSuccess) break;
          if (q != cudaErrorNotReady) CK(q);
          RET(stream_ready(false));
          std::this_thread::yield();
        }
      }
      RET(stage_h2d(dpk + cb[c], probe_keys + cb[c], (cb[c + 1] - cb[c]) * 8));
      RET(tr_mark());
      CK(cudaEventRecord(g.h2d_ev[c], g.s_h2d));
      if (c > 0) {
        RET(finish_upload(c - 1));
        RET(probe_chunk(c - 1, op, ob, cap_));
        RET(stream_ready(false));
      }
    }
    if (nchunks) {
      RET(finish_upload(nchunks - 1));
      RET(probe_chunk(nchunks - 1, op, ob, cap_));
      RET(stream_ready(false));
    }
    return GOLP_OK;
  };
  RET(run_chunks(true, dev_p, dev_b, dcap));
  if (trace) std::fprintf(stderr, "[golp] %.3f ms all chunks queued\n", (wall_seconds() - t0) * 1e3);
  CK(cudaEventRecord(ev_chunk, g.s_h2d));
  // Wait for the last upload while still handing finished chunks' pairs to the
  // D2H engine, so downloads overlap the remaining uploads.
  while (true) {
    const cudaError_t q = cudaEventQuery(ev_chunk);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) CK(q);
    RET(stream_ready(false));
    std::this_thread::yield();
  }
  g.next_slot = 0;
  for (bool& b : g.pin_busy) b = false;
  const double t1 = wall_seconds();
  if (trace) std::fprintf(stderr, "[golp] %.3f ms uploads done\n", (t1 - t0) * 1e3);
  auto finished_total = [&](uint64_t* m_out) -> int {  // totals via the mapped mirror (no copy engine)
    if (nchunks) {
      CK(cudaEventSynchronize(g.chunk_ev[nchunks - 1]));
      *m_out = g.mirror[nchunks];
    } else {
      CK(cudaStreamSynchronize(s));
      *m_out = 0;
    }
    return GOLP_OK;
  };
  while (streaming && streamed < nchunks) {  // keep streaming while the last chunks finish
    const cudaError_t q = cudaEventQuery(g.chunk_ev[nchunks - 1]);
    if (q != cudaErrorNotReady) {
      CK(q);
      break;
    }
    RET(stream_ready(false));
    std::this_thread::yield();
  }
  uint64_t m = 0;
  RET(finished_total(&m));
  const double t2 = wall_seconds();
  if (trace) std::fprintf(stderr, "[golp] %.3f ms last chunk probed, M=%llu\n", (t2 - t0) * 1e3, (unsigned long long)m);
  if (m > dcap) {  // rare: more pairs than the output capacity; re-probe the resident input into HBM
    streaming = false;
    RET(d2h_flush());
    CK(g.pairs_p.ensure(m * 4));
    CK(g.pairs_b.ensure(m * 4));
    dcap = std::min(g.pairs_p.bytes, g.pairs_b.bytes) / 4;
    CK(cudaMemsetAsync(g.totals.p, 0, (nchunks + 1) * 8, s));
    RET(run_chunks(false, g.pairs_p.as<uint32_t>(), g.pairs_b.as<uint32_t>(), dcap));
    RET(finished_total(&m));
    dev_p = g.pairs_p.as<uint32_t>();
    dev_b = g.pairs_b.as<uint32_t>();
  }
  RET(stream_ready(true));
  RET(d2h_flush());
  const double t3 = wall_seconds();
  if (trace) {
    std::fprintf(stderr, "[golp] %.3f ms pairs landed\n", (t3 - t0) * 1e3);
    for (size_t i = 1; i < tr_q.size(); ++i) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, tr_ev[0], tr_ev[i]));
      std::fprintf(stderr, "[golp]   upload %zu: queued at %.3f ms, landed %.3f ms after the first queue\n", i - 1, tr_q[i], ms);
    }
  }
  *out_matches = m;
  g.last_m = m;
  g.last_probe_valid = true;  // copy_out reads the device pair buffers
  bool delivered = streaming && m <= out_cap && streamed == nchunks;
  if (!delivered && m <= out_cap) {
    // Streaming stopped early (a re-probe into larger device buffers): the
    // pairs still fit the caller's arrays, so deliver all of them here.
    if (m) {
      RET(stage_d2h(out_probe_rows, dev_p, m * 4));
      RET(stage_d2h(out_build_rows, dev_b, m * 4));
    }
    delivered = true;
  }
  led->t_h2d = t1 - t0;
  led->t_kernel = t2 - t1;
  if (delivered) {
    led->t_d2h = wall_seconds() - t2;
    led->d2h_bytes = 8 * m;
  } else {
    led->t_kernel += t3 - t2;  // copy_out adds the D2H phase
  }
  return kspan_finish();
}

int golp_probe_copy_out(uint32_t* probe_rows, uint32_t* build_rows, uint64_t m, golp_ledger* led) {
  Ctx& g = cur();
  if (!g.last_probe_valid) return invalid("no probe result to copy out");
  if (m != g.last_m) return invalid("copy_out size does not match the last probe's match count");
  const double t0 = wall_seconds();
  if (m) {
    if (!probe_rows || !build_rows) return invalid("null buffer");
    RET(stage_d2h(probe_rows, g.pairs_p.p, m * 4));
    RET(stage_d2h(build_rows, g.pairs_b.p, m * 4));
  }
  RET(sync_ring());
  if (led) {
    led->d2h_bytes = 8 * m;
    led->t_d2h = wall_seconds() - t0;
  }
  return GOLP_OK;
}

// ---- host result allocator: pinned arena, mmap fallback ----------------------------
void* golp_host_alloc(uint64_t bytes) {
  if (bytes == 0) bytes = 1;
  if (void* p = arena_alloc(bytes)) return p;  // page-locked: results DMA straight in
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) {
    set_error("mmap failed for a host result buffer");
    return nullptr;
  }
  madvise(p, bytes, MADV_HUGEPAGE);
  return p;
}

int golp_host_free(void* p, uint64_t bytes) {
  if (!p) return GOLP_OK;
  if (arena_free(p)) return GOLP_OK;
  if (bytes == 0) bytes = 1;
  return munmap(p, bytes) == 0 ? GOLP_OK : GOLP_ERR_INVALID;
}

int golp_host_is_pinned(const void* p) { return is_pinned(p, 1) ? 1 : 0; }
int golp_host_is_pinned_range(const void* p, uint64_t bytes) { return is_pinned(p, bytes) ? 1 : 0; }

// Page-lock a caller buffer in place (read-only) so repeated transfers of it skip
// the staging copy. Slow (~5 GB/s): worth it only for buffers reused across calls.
int golp_host_register(const void* p, uint64_t bytes) {
  RET(ensure_init());
  if (!p || !bytes) return invalid("empty range");
  // DMA from registered memory runs at ~half the PCIe rate when the range is
  // backed by 4 KB pages (measured: 12 MB in 0.45 ms vs 0.23 ms from huge
  // pages). Ask the kernel to collapse the 2 MB-aligned interior into huge pages
  // first (MADV_COLLAPSE, Linux >= 6.1; best effort, errors ignored).
#ifndef MADV_COLLAPSE
#define MADV_COLLAPSE 25
#endif
  {
    constexpr uintptr_t kHuge = uintptr_t(2) << 20;
    const uintptr_t a = (reinterpret_cast<uintptr_t>(p) + kHuge - 1) & ~(kHuge - 1);
    const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes) & ~(kHuge - 1);
    if (e > a) {
      madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);
      const int rc = madvise(reinterpret_cast<void*>(a), e - a, MADV_COLLAPSE);
      if (std::getenv("GOLP_TRACE"))
        std::fprintf(stderr, "[golp] register %p +%llu: collapse %llu bytes rc=%d errno=%d\n", p,
                     (unsigned long long)bytes, (unsigned long long)(e - a), rc, rc ? errno : 0);
    }
  }
  CK(cudaHostRegister(const_cast<void*>(p), bytes, cudaHostRegisterReadOnly | cudaHostRegisterPortable));
  pinned_add(p, bytes);
  return GOLP_OK;
}

int golp_host_unregister(const void* p) {
  if (!p) return GOLP_OK;
  pinned_remove(p);
  CK(cudaHostUnregister(const_cast<void*>(p)));
  return GOLP_OK;
}

}  // extern "C"
