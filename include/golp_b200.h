/*
 * golp_b200.h -- C ABI of libgolp_b200.so, the B200 offload path for the
 * reference `golp` package (arXiv 2601.19911, /root/reference/pkg/src/golp).
 *
 * The reference's plug-in boundary is the duck-typed device protocol
 * {name, topk(), probe(), close()} that gate._run_query calls
 * (pkg/src/golp/gate.py:185-213) and make_device() constructs
 * (pkg/src/golp/device.py:439-445). Each entry point below replaces one step of
 * that protocol; see INTEGRATION.md for the ctypes binding a golp maintainer adds.
 *
 * Conventions
 *   - plain pointers and sizes; no torch / CUDA types in signatures
 *     (streams are passed as an opaque `void*` = cudaStream_t, NULL = default);
 *   - every function returns a golp_status; golp_last_error() describes the
 *     last failure of the calling process;
 *   - work runs on a CONTEXT bound to one CUDA device (streams, pinned staging,
 *     HBM workspace). Each host thread has a current context: golp_init /
 *     golp_use_device select a device's default context, golp_context_open
 *     creates an independent one; a thread that selected none uses the default
 *     context of its current CUDA device. Calls are externally synchronous per
 *     context, exactly like the reference's ProxyDevice ("one call, one
 *     ledger"); threads on different contexts run concurrently
 *     (the G-GPU sharding of B200Device(gpus=G), ProxyDevice's chunk workers
 *     at device.py:308-327 with GPUs as the workers);
 *   - the library never writes to input buffers and never retains input
 *     pointers after a call returns. (Page-locking a caller buffer for reuse
 *     is an explicit request, golp_host_register; the Python B200Device's
 *     PinCache makes it for columns it sees repeatedly -- pin_inputs=False
 *     turns that off.)
 */
#ifndef GOLP_B200_H
#define GOLP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum golp_status {
  GOLP_OK = 0,
  GOLP_ERR_INVALID = 1,  /* -> ValueError (device.py:336-337, device.py:144-151) */
  GOLP_ERR_CAPACITY = 2, /* -> CapacityError (host.py:155-159)                  */
  GOLP_ERR_CUDA = 3      /* -> RuntimeError                                     */
} golp_status;

typedef enum golp_mode {
  GOLP_KEY_ONLY = 0, /* 12 B per entry: f64 key + u32 row id (store.py:23-26) */
  GOLP_FULL_ROW = 1  /* 8 + payload_bytes per row (device.py:144-151)         */
} golp_mode;

/* Mirrors TransferLedger (pkg/src/golp/device.py:98-126). Byte counts follow
 * the reference's shape formulas (device.py:372-379, 428-435), never measured;
 * phase times are seconds on the critical path, so their sum is the wall time
 * of the call. */
typedef struct golp_ledger {
  uint64_t h2d_bytes;
  uint64_t d2h_bytes;
  double t_h2d;
  double t_kernel;
  double t_d2h;
  double t_post;
} golp_ledger;

/* Device-time breakdown of the last call (CUDA events on the launching stream;
 * filled only while golp_set_profiling(1) is active). Milliseconds. */
typedef struct golp_kernel_times {
  double topk_threshold_ms;
  double topk_filter_ms;
  double topk_select_ms;
  double join_build_ms;
  double join_probe_ms;
  uint64_t topk_candidates; /* survivors of the streaming filter          */
  uint64_t topk_fallback;   /* 1 if the exact direct path had to run       */
  uint64_t join_groups;     /* distinct build keys                         */
  uint64_t join_capacity;   /* hash-table slots                            */
  uint64_t join_slices;     /* table slices of a radix-partitioned join (1 = not partitioned) */
  double full_sort_ms;      /* device time of the last full sort                     */
  uint64_t full_sort_passes;/* digit passes it needed (of 12)                         */
  double call_kernel_ms;    /* device time of the kernels of the last host-buffer call
                               (golp_topk / golp_probe / golp_full_sort), summed over its
                               kernel groups; upload waits excluded (C_gpu's kernel term) */
} golp_kernel_times;

/* ---- lifecycle ---------------------------------------------------------------- */
const char* golp_last_error(void);
int golp_version(void);
/* Make the default context of `device` (-1: the calling thread's current CUDA
 * device) current on this thread, creating it with a pinned staging ring of
 * pinned_chunk_bytes per slot and host_threads packer threads (0 = defaults)
 * on first use. Replaces ProxyDevice.__init__ (device.py:308-310). Implicit on
 * first use. */
int golp_init(int device, uint64_t pinned_chunk_bytes, int host_threads);
/* golp_init(device, 0, 0): select device's default context on this thread. */
int golp_use_device(int device);
/* Device of the calling thread's current context (initializing it if needed). */
int golp_current_device(int* device);
/* An independent context on `device` (its own streams, staging and workspace),
 * made current on this thread; *handle names it for golp_context_use/close. */
int golp_context_open(int device, uint64_t pinned_chunk_bytes, int host_threads, int* handle);
int golp_context_use(int handle);
int golp_context_close(int handle);
/* Frees every context's device buffers, pinned staging and streams. Replaces
 * ProxyDevice.close (device.py:312-315). A context used again afterwards is
 * re-initialized on its device. */
int golp_shutdown(void);
/* Number of CUDA kernels this library has launched (process lifetime). */
uint64_t golp_launch_count(void);
/* Bytes the copy engines actually moved during the last host-buffer call
 * (golp_topk / golp_probe [+ golp_probe_copy_out] / golp_full_sort). The
 * ledger's h2d_bytes / d2h_bytes keep the reference's shape formulas
 * (device.py:372-379, 428-435); these can be lower, because a dense row-id
 * column (rows[i] == rows[0] + i, extract_keys's arange, store.py:178-181) is
 * verified on the host and regenerated on the device instead of copied. */
int golp_last_transfer(uint64_t* h2d_bytes, uint64_t* d2h_bytes);
/* 1 (default; env GOLP_DENSE_ROWS=0 turns it off): dense row-id columns are
 * regenerated on the device; 0: every row-id column is copied. */
int golp_set_dense_rows(int on);
/* Declares that the row-id columns of the NEXT host-buffer call on this
 * context are dense runs (rows[i] == rows[0] + i), e.g. a table's own
 * positions as extract_keys passes them (store.py:178-181): the host-side scan
 * that verifies this is skipped (the end points are still checked). */
int golp_hint_dense_rows(void);
/* 0: off; 1: timing events around each kernel group of every call; 2: the same
 * without the event at a join build's start (join_build_ms stays 0), which
 * saves one event node per CUDA-graph step when only the probe is timed. */
int golp_set_profiling(int on);
int golp_last_kernel_times(golp_kernel_times* out);

/* ---- host-buffer entry points: ProxyDevice.topk / ProxyDevice.probe ------------ */
/* Replaces ProxyDevice.topk (pkg/src/golp/device.py:329-380). keys/rows are the
 * KeyVector columns (store.py:75-112). Writes min(k, n) row ids, best first:
 * keys descending, equal keys by ascending row id (host.py:133-144).
 * k < 1 -> GOLP_ERR_INVALID. FULL_ROW additionally ships n*payload_bytes bytes. */
int golp_topk(const double* keys, const uint32_t* rows, uint64_t n, uint64_t k, int mode,
              uint32_t payload_bytes, uint32_t* out_rows, uint64_t* out_len, golp_ledger* led);

/* golp_topk plus the winners' order-preserving u64 key codes (out_codes, min(k,
 * n) entries, may be NULL): the input of golp_host_merge_topk when a key column
 * is sharded over several contexts (B200Device(gpus=G)). */
int golp_topk_codes(const double* keys, const uint32_t* rows, uint64_t n, uint64_t k, int mode,
                    uint32_t payload_bytes, uint32_t* out_rows, uint64_t* out_codes, uint64_t* out_len,
                    golp_ledger* led);

/* Replaces ProxyDevice.probe (pkg/src/golp/device.py:382-436). Ships both sides
 * (build first, then the probe side in chunks that are probed as they land),
 * builds, probes, and sets *out_matches = M. When M <= out_cap the pairs are
 * streamed back into out_probe_rows / out_build_rows during the call (chunk c's
 * pairs download while chunk c+1 uploads), in reference order: probe position,
 * then build insertion position (host.py:168-188). When M > out_cap the pairs
 * stay in library memory for golp_probe_copy_out. */
int golp_probe(const double* build_keys, const uint32_t* build_rows, uint64_t nb,
               const double* probe_keys, const uint32_t* probe_rows, uint64_t np, int mode,
               uint32_t payload_bytes, uint32_t* out_probe_rows, uint32_t* out_build_rows,
               uint64_t out_cap, uint64_t* out_matches, golp_ledger* led);
/* Copy the M pairs of the last golp_probe into caller arrays of m = M entries
 * (the M > out_cap case). Adds t_d2h and d2h_bytes = 8*M to *led. */
int golp_probe_copy_out(uint32_t* probe_rows, uint32_t* build_rows, uint64_t m, golp_ledger* led);
/* Full sort from host buffers (the fig3 full_sort baseline, harness.py:247-270,
 * offloaded): out_rows gets all n row ids in host_full_sort order. Ledger as the
 * device protocol: H2D = entry bytes * n, D2H = 4 * n. */
int golp_full_sort(const double* keys, const uint32_t* rows, uint64_t n, int mode, uint32_t payload_bytes,
                   uint32_t* out_rows, golp_ledger* led);
/* Host memory for result arrays: a page-locked arena (so results are DMA'd
 * straight in), falling back to mmap + transparent huge pages. Owned by the
 * caller's result object, released with golp_host_free(ptr, bytes). */
void* golp_host_alloc(uint64_t bytes);
int golp_host_free(void* ptr, uint64_t bytes);
/* Page-lock a caller buffer in place (read-only) so that transfers of it skip
 * the staging copy; for columns reused across calls (registration is slow). */
int golp_host_register(const void* ptr, uint64_t bytes);
/* 1 when ptr lies in page-locked host memory this library allocated
 * (golp_host_alloc) or registered (golp_host_register). */
int golp_host_is_pinned(const void* ptr);
/* 1 when all of [ptr, ptr+bytes) lies in ONE such range: only then does a
 * transfer of it skip the staging ring. */
int golp_host_is_pinned_range(const void* ptr, uint64_t bytes);
int golp_host_unregister(const void* ptr);

/* ---- device-resident entry points (inputs already in HBM) ---------------------- */
/* Device-resident entry points run on the calling thread's context and fail
 * with GOLP_ERR_INVALID when the first input pointer lives on another device. */
/* Top-K of n device-resident items. d_out_rows gets min(k, n) rows best first;
 * d_out_keys (optional, may be NULL) gets their order-preserving u64 key codes
 * (for cross-GPU merges via golp_topk_merge_device). */
int golp_topk_device(const double* d_keys, const uint32_t* d_rows, uint64_t n, uint64_t k,
                     uint32_t* d_out_rows, uint64_t* d_out_keys, void* stream);
/* golp_topk_device whose row ids are the positions themselves, row_base + i:
 * the key vector extract_keys makes of a table (pkg/src/golp/store.py:178-181,
 * rows = arange) needs no row column in HBM, and no row loads for threshold
 * ties (a Zipf head). Same output contract; GOLP_ERR_INVALID when
 * row_base + n - 1 exceeds 2^32 - 1. */
int golp_topk_device_positions(const double* d_keys, uint64_t n, uint32_t row_base, uint64_t k,
                               uint32_t* d_out_rows, uint64_t* d_out_keys, void* stream);
/* Exact Top-K of n already-encoded candidates (u64 key code, u32 row), e.g. the
 * all-gathered local results of G GPUs. Same output contract as above. */
int golp_topk_merge_device(const uint64_t* d_key_codes, const uint32_t* d_rows, uint64_t n, uint64_t k,
                           uint32_t* d_out_rows, uint64_t* d_out_keys, void* stream);
/* Build the library's join table from nb device-resident build entries
 * (host_hash_build, host.py:147-165; insertion order = position order). */
int golp_join_build_device(const double* d_build_keys, const uint32_t* d_build_rows, uint64_t nb,
                           void* stream);
/* Probe the table built last. Writes min(M, cap) pairs and sets *out_matches = M;
 * returns GOLP_ERR_CAPACITY (pairs truncated) when M > cap. */
int golp_join_probe_device(const double* d_probe_keys, const uint32_t* d_probe_rows, uint64_t np,
                           uint32_t* d_out_probe_rows, uint32_t* d_out_build_rows, uint64_t cap,
                           uint64_t* out_matches, void* stream);

/* Asynchronous probe: enqueues the probe on `stream` and writes M to the device
 * word d_out_matches; pairs beyond cap are dropped (the caller compares M with
 * cap after synchronizing and re-probes with a larger buffer if needed). */
int golp_join_probe_device_async(const double* d_probe_keys, const uint32_t* d_probe_rows, uint64_t np,
                                 uint32_t* d_out_probe_rows, uint32_t* d_out_build_rows, uint64_t cap,
                                 uint64_t* d_out_matches, void* stream);
/* The two probes above for a probe key vector whose row ids are its positions,
 * row_base + i (extract_keys, pkg/src/golp/store.py:178-181): the match kernels
 * compute the probe row ids instead of reading a u32 column. GOLP_ERR_INVALID
 * when row_base + np - 1 exceeds 2^32 - 1. */
int golp_join_probe_device_positions(const double* d_probe_keys, uint64_t np, uint32_t row_base,
                                     uint32_t* d_out_probe_rows, uint32_t* d_out_build_rows, uint64_t cap,
                                     uint64_t* out_matches, void* stream);
int golp_join_probe_device_positions_async(const double* d_probe_keys, uint64_t np, uint32_t row_base,
                                           uint32_t* d_out_probe_rows, uint32_t* d_out_build_rows, uint64_t cap,
                                           uint64_t* d_out_matches, void* stream);

/* Full sort on the device: host_full_sort (host.py:127-130, np.lexsort((rows,
 * keys))) -- d_out_rows gets the n row ids ordered by key ascending (-0.0 ==
 * +0.0), equal keys by ascending row id. Stream-ordered (synchronizes once
 * after its histogram pass to plan the digit passes). */
int golp_full_sort_device(const double* d_keys, const uint32_t* d_rows, uint64_t n, uint32_t* d_out_rows,
                          void* stream);

/* ---- classical host engine (the gate's HOST path, gate.py:193-194,209-210) ------ */
/* Multi-threaded CPU Top-K with host_topk's exact output (host.py:133-144). */
int golp_host_topk(const double* keys, const uint32_t* rows, uint64_t n, uint64_t k, uint32_t* out_rows,
                   int threads);
/* KeyHashTable build with the reference's slot layout (host.py:83-165):
 * capacity = smallest power of two >= 8 with capacity*0.7 >= n; serial
 * insertion in position order; linear probing on mix64(key_bits). The caller
 * passes zeroed slot_bits and ROW_EMPTY-filled slot_rows of `capacity` entries. */
int golp_host_hash_build(const double* keys, const uint32_t* rows, uint64_t n, uint64_t capacity,
                         uint64_t* slot_bits, uint32_t* slot_rows);
/* host_hash_probe (host.py:168-188) on such a table, chunk-parallel over the
 * probe side. Phase 1 of 2: sets *out_matches = M and keeps the pairs. */
int golp_host_hash_probe(const uint64_t* slot_bits, const uint32_t* slot_rows, uint64_t capacity,
                         const double* keys, const uint32_t* rows, uint64_t n, int threads,
                         uint64_t* out_matches);
/* Phase 2: copy the M pairs of the last golp_host_hash_probe, reference order. */
int golp_host_probe_copy_out(uint32_t* probe_rows, uint32_t* build_rows, uint64_t m);
/* Merge of `parts` best-first (codes, rows) lists of counts[p] entries each,
 * stored back to back: the first k in host_topk's order (key descending, row id
 * ascending, host.py:133-144) -> out_rows, *out_len = min(k, total). The merge
 * step of ProxyDevice.topk (device.py:257-259) over per-GPU shard results. */
int golp_host_merge_topk(const uint64_t* codes, const uint32_t* rows, const uint64_t* counts, int parts, uint64_t k,
                         uint32_t* out_rows, uint64_t* out_len);
/* Late materialization (store.materialize, store.py:184-201, and its join
 * counterpart): dst[i] = src row ids[i] (row_bytes each), multi-threaded;
 * an id >= nrows -> GOLP_ERR_INVALID. */
int golp_host_gather(const void* src, uint64_t row_bytes, uint64_t nrows, const uint32_t* ids, uint64_t n, void* dst,
                     int threads);

#ifdef __cplusplus
}
#endif
#endif /* GOLP_B200_H */
