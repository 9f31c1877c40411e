/*
 * TEST INFRASTRUCTURE ONLY -- never linked into or called by the product path.
 *
 * CPU restatement of the reference algorithms on the offload path of
 * arXiv 2601.19911's `golp` package (/root/reference/pkg/src/golp), used as the
 * parity checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs. Pinned against golden vectors produced by the reference
 * itself (tests/golden/make_golden.py -> tests/golden/*.npz, checked in
 * tests/test_oracle.py).
 *
 *   oracle_topk        host_topk        host.py:133-144  heapq.nlargest(take, zip(keys, -rows))
 *   oracle_hash_build  host_hash_build  host.py:147-165  + KeyHashTable.insert host.py:103-112
 *   oracle_hash_probe  host_hash_probe  host.py:168-188
 *   key_bits / mix64                    host.py:58-80
 *   oracle_proxy_topk  ProxyDevice.topk device.py:329-380 (chunk top-k + merge), threaded
 *   oracle_proxy_probe ProxyDevice.probe device.py:382-436 (serial build, chunk-parallel probe)
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ROW_EMPTY 0xFFFFFFFFu

/* key_bits: (key + 0.0).view(u64) folds -0.0 onto +0.0 (host.py:58-60) */
static uint64_t key_bits(double k) {
  double z = k + 0.0;
  uint64_t b;
  memcpy(&b, &z, 8);
  return b;
}

/* mix64 (host.py:72-80) */
uint64_t oracle_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

/* heapq.nlargest orders tuples (key, -row): larger key first, then larger -row,
 * i.e. smaller row. Python float compare: -0.0 == 0.0. */
static int better(double ka, uint32_t ra, double kb, uint32_t rb) {
  if (ka > kb) return 1;
  if (ka < kb) return 0;
  return ra < rb;
}

typedef struct {
  double k;
  uint32_t r;
} ent;

/* min-heap on `better` (root = worst kept entry) */
static void sift_down(ent* h, uint64_t n, uint64_t i) {
  for (;;) {
    uint64_t l = 2 * i + 1, m = i;
    if (l < n && better(h[m].k, h[m].r, h[l].k, h[l].r)) m = l;
    if (l + 1 < n && better(h[m].k, h[m].r, h[l + 1].k, h[l + 1].r)) m = l + 1;
    if (m == i) return;
    ent t = h[i];
    h[i] = h[m];
    h[m] = t;
    i = m;
  }
}

static int cmp_desc(const void* a, const void* b) {
  const ent* x = (const ent*)a;
  const ent* y = (const ent*)b;
  if (better(x->k, x->r, y->k, y->r)) return -1;
  if (better(y->k, y->r, x->k, x->r)) return 1;
  return 0;
}

/* Bounded heap of size take over the input, then sort descending. */
static uint64_t topk_into(const double* keys, const uint32_t* rows, uint64_t n, uint64_t k, ent* h) {
  const uint64_t take = k < n ? k : n;
  uint64_t sz = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (sz < take) {
      h[sz].k = keys[i];
      h[sz].r = rows[i];
      ++sz;
      if (sz == take)
        for (uint64_t j = take / 2 + 1; j-- > 0;) sift_down(h, sz, j);
    } else if (take && better(keys[i], rows[i], h[0].k, h[0].r)) {
      h[0].k = keys[i];
      h[0].r = rows[i];
      sift_down(h, sz, 0);
    }
  }
  qsort(h, sz, sizeof(ent), cmp_desc);
  return sz;
}

/* host_topk: returns min(k, n) rows; k < 1 -> -1 (ValueError in the reference) */
int64_t oracle_topk(const double* keys, const uint32_t* rows, uint64_t n, uint64_t k, uint32_t* out) {
  if (k < 1) return -1;
  const uint64_t take = k < n ? k : n;
  ent* h = (ent*)malloc((take ? take : 1) * sizeof(ent));
  if (!h) return -2;
  const uint64_t sz = topk_into(keys, rows, n, k, h);
  for (uint64_t i = 0; i < sz; ++i) out[i] = h[i].r;
  free(h);
  return (int64_t)sz;
}

/* capacity = smallest power of two >= 8 with capacity * 0.7 >= n (host.py:151-153) */
uint64_t oracle_table_capacity(uint64_t n) {
  uint64_t c = 8;
  while ((double)c * 0.7 < (double)n) c *= 2;
  return c;
}

/* KeyHashTable.insert in position order; slot_bits zeroed, slot_rows = ROW_EMPTY */
int oracle_hash_build(const double* keys, const uint32_t* rows, uint64_t n, uint64_t cap, uint64_t* slot_bits,
                      uint32_t* slot_rows) {
  const uint64_t mask = cap - 1;
  for (uint64_t i = 0; i < n; ++i) {
    if ((double)(i + 1) > 0.7 * (double)cap) return -1; /* CapacityError */
    const uint64_t b = key_bits(keys[i]);
    uint64_t cur = oracle_mix64(b) & mask;
    while (slot_rows[cur] != ROW_EMPTY) cur = (cur + 1) & mask;
    slot_bits[cur] = b;
    slot_rows[cur] = rows[i];
  }
  return 0;
}

/* host_hash_probe: probe order, then chain (insertion) order. Writes at most
 * out_cap pairs; returns the total match count. */
uint64_t oracle_hash_probe(const uint64_t* slot_bits, const uint32_t* slot_rows, uint64_t cap, const double* keys,
                           const uint32_t* rows, uint64_t n, uint32_t* out_p, uint32_t* out_b, uint64_t out_cap) {
  const uint64_t mask = cap - 1;
  uint64_t m = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t b = key_bits(keys[i]);
    uint64_t cur = oracle_mix64(b) & mask;
    while (slot_rows[cur] != ROW_EMPTY) {
      if (slot_bits[cur] == b) {
        if (m < out_cap) {
          out_p[m] = rows[i];
          out_b[m] = slot_rows[cur];
        }
        ++m;
      }
      cur = (cur + 1) & mask;
    }
  }
  return m;
}

/* ---- threaded ports of ProxyDevice (CPU baseline) ------------------------------- */

typedef struct {
  const double* keys;
  const uint32_t* rows;
  uint64_t lo, hi, k;
  ent* cand;
  uint64_t ncand;
} topk_job;

static void* topk_worker(void* p) {
  topk_job* j = (topk_job*)p;
  j->ncand = topk_into(j->keys + j->lo, j->rows + j->lo, j->hi - j->lo, j->k, j->cand);
  return NULL;
}

/* _chunk_bounds (device.py:317-322) with floor max(4k, 4096), chunk top-k, merge. */
int64_t oracle_proxy_topk(const double* keys, const uint32_t* rows, uint64_t n, uint64_t k, uint32_t* out,
                          int workers) {
  if (k < 1) return -1;
  if (workers < 1) workers = 1;
  const uint64_t floor_ = (4 * k > 4096) ? 4 * k : 4096;
  uint64_t chunks = n / floor_;
  if (chunks < 1) chunks = 1;
  if (chunks > (uint64_t)workers) chunks = (uint64_t)workers;
  const uint64_t step = (n + chunks - 1) / (chunks ? chunks : 1);
  topk_job* jobs = (topk_job*)calloc(chunks, sizeof(topk_job));
  pthread_t* th = (pthread_t*)calloc(chunks, sizeof(pthread_t));
  const uint64_t per = k < step ? k : step;
  ent* cand = (ent*)malloc((chunks * per + 1) * sizeof(ent));
  uint64_t nj = 0;
  for (uint64_t lo = 0; lo < n || (n == 0 && nj == 0); lo += step) {
    jobs[nj].keys = keys;
    jobs[nj].rows = rows;
    jobs[nj].lo = lo;
    jobs[nj].hi = lo + step < n ? lo + step : n;
    jobs[nj].k = k;
    jobs[nj].cand = cand + nj * per;
    ++nj;
    if (n == 0) break;
  }
  for (uint64_t i = 1; i < nj; ++i) pthread_create(&th[i], NULL, topk_worker, &jobs[i]);
  topk_worker(&jobs[0]);
  for (uint64_t i = 1; i < nj; ++i) pthread_join(th[i], NULL);
  /* _merge_topk_candidates: lexsort by (-key, row) over all candidates */
  uint64_t total = 0;
  for (uint64_t i = 0; i < nj; ++i) {
    memmove(cand + total, jobs[i].cand, jobs[i].ncand * sizeof(ent));
    total += jobs[i].ncand;
  }
  qsort(cand, total, sizeof(ent), cmp_desc);
  const uint64_t take = k < total ? k : total;
  for (uint64_t i = 0; i < take; ++i) out[i] = cand[i].r;
  free(cand);
  free(th);
  free(jobs);
  return (int64_t)take;
}

typedef struct {
  const uint64_t* slot_bits;
  const uint32_t* slot_rows;
  uint64_t cap;
  const double* keys;
  const uint32_t* rows;
  uint64_t lo, hi;
  uint32_t* p;
  uint32_t* b;
  uint64_t m, mcap;
} probe_job;

static void* probe_worker(void* arg) {
  probe_job* j = (probe_job*)arg;
  const uint64_t mask = j->cap - 1;
  uint64_t cap = (j->hi - j->lo) + 16, m = 0;
  j->p = (uint32_t*)malloc(cap * 4);
  j->b = (uint32_t*)malloc(cap * 4);
  for (uint64_t i = j->lo; i < j->hi; ++i) { /* one pass, growable output (host.py:168-188) */
    const uint64_t b = key_bits(j->keys[i]);
    uint64_t cur = oracle_mix64(b) & mask;
    while (j->slot_rows[cur] != ROW_EMPTY) {
      if (j->slot_bits[cur] == b) {
        if (m == cap) {
          cap *= 2;
          j->p = (uint32_t*)realloc(j->p, cap * 4);
          j->b = (uint32_t*)realloc(j->b, cap * 4);
        }
        j->p[m] = j->rows[i];
        j->b[m] = j->slot_rows[cur];
        ++m;
      }
      cur = (cur + 1) & mask;
    }
  }
  j->m = m;
  return NULL;
}

/* Chunk-parallel probe of a built table (ProxyDevice's _probe_chunk fan-out,
 * chunks >= 4096 probes); pairs concatenated in chunk order. Returns M. */
uint64_t oracle_proxy_probe(const uint64_t* slot_bits, const uint32_t* slot_rows, uint64_t cap, const double* keys,
                            const uint32_t* rows, uint64_t n, uint32_t* out_p, uint32_t* out_b, uint64_t out_cap,
                            int workers) {
  if (workers < 1) workers = 1;
  uint64_t chunks = n / 4096;
  if (chunks < 1) chunks = 1;
  if (chunks > (uint64_t)workers) chunks = (uint64_t)workers;
  const uint64_t step = (n + chunks - 1) / chunks;
  probe_job* jobs = (probe_job*)calloc(chunks, sizeof(probe_job));
  pthread_t* th = (pthread_t*)calloc(chunks, sizeof(pthread_t));
  uint64_t nj = 0;
  for (uint64_t lo = 0; lo < n; lo += step) {
    probe_job* j = &jobs[nj++];
    j->slot_bits = slot_bits;
    j->slot_rows = slot_rows;
    j->cap = cap;
    j->keys = keys;
    j->rows = rows;
    j->lo = lo;
    j->hi = lo + step < n ? lo + step : n;
  }
  for (uint64_t i = 1; i < nj; ++i) pthread_create(&th[i], NULL, probe_worker, &jobs[i]);
  if (nj) probe_worker(&jobs[0]);
  for (uint64_t i = 1; i < nj; ++i) pthread_join(th[i], NULL);
  uint64_t m = 0;
  for (uint64_t i = 0; i < nj; ++i) {
    for (uint64_t t = 0; t < jobs[i].m; ++t, ++m) {
      if (m < out_cap) {
        out_p[m] = jobs[i].p[t];
        out_b[m] = jobs[i].b[t];
      }
    }
    free(jobs[i].p);
    free(jobs[i].b);
  }
  free(th);
  free(jobs);
  return m;
}
