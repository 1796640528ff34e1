/*
 * flycoo_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port" kind).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path
 * (paper_2309_09131_b200) never links, imports or calls it.
 *
 * What it restates (reference = /root/reference/pkg/src/modecycle):
 *   orc_morton          morton.py:15-44   (key_widths + interleave)
 *   orc_mode_worker     _kernels.py:38-88 (per-worker fused MTTKRP + remap)
 *   orc_mode_pass       engine.py:214-245 (fan-out of workers over threads,
 *                                          join = end-of-mode barrier)
 *   orc_reference_mttkrp coo.py:406-426   (sequential oracle)
 *
 * Data layout is the reference's own: sids/idxs (nnz, N) int64 row-major,
 * vals (nnz,) float64, factors stacked row-wise (engine.py:153-160).
 * Build with -O2 -ffp-contract=off so every multiply and add rounds exactly
 * like numba/numpy do (no FMA contraction), which is what makes the oracle
 * bit-identical to the reference on the golden fixtures.
 */
#include <immintrin.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- morton */

static int bit_length_u64(uint64_t x) {
  int b = 0;
  while (x) { b++; x >>= 1; }
  return b;
}

/* morton.py:15-17 width = bit_length(count-1); morton.py:20-44 LSB-first
 * interleave, mode 0 least significant inside each bit level, spill past
 * bit 63 into hi.  Returns -1 when the key would exceed 128 bits. */
int orc_morton(const int64_t *coords, int64_t n, int nmodes,
               const int64_t *counts, uint64_t *hi, uint64_t *lo) {
  int widths[64];
  int total = 0, maxw = 0;
  if (nmodes > 64) return -2;
  for (int w = 0; w < nmodes; ++w) {
    int64_t c = counts[w] - 1;
    widths[w] = c > 0 ? bit_length_u64((uint64_t)c) : 0;
    total += widths[w];
    if (widths[w] > maxw) maxw = widths[w];
  }
  if (total > 128) return -1;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t h = 0, l = 0;
    int pos = 0;
    const int64_t *c = coords + i * nmodes;
    for (int b = 0; b < maxw; ++b) {
      for (int w = 0; w < nmodes; ++w) {
        if (b >= widths[w]) continue;
        uint64_t bit = ((uint64_t)c[w] >> b) & 1u;
        if (pos < 64) l |= bit << pos;
        else h |= bit << (pos - 64);
        ++pos;
      }
    }
    hi[i] = h;
    lo[i] = l;
  }
  return 0;
}

/* ----------------------------------------------------------- mode worker */

typedef struct {
  const int64_t *sids, *idxs;
  const double *vals;
  int64_t *dst_sids, *dst_idxs;
  double *dst_vals;
  const double *fstack;
  const int64_t *foffs;
  double *out;
  int64_t rank;
  int nmodes, mode, next_mode;
  const int64_t *starts, *ends; /* this worker's super-shard element ranges */
  int64_t nranges;
  const int64_t *dest_base;     /* next-mode shard offsets */
  _Atomic int64_t *cursors;     /* next-mode shard fill counters */
  const int64_t *dest_slots;    /* precomputed slots */
  int use_cursor, do_compute, do_remap;
  _Atomic int64_t *errflag;
  int64_t processed;
} orc_worker_t;

/* _kernels.py:38-88, statement for statement (fields hoisted into locals so
 * the compiler can keep them in registers across the element loop). */
static void *orc_worker_run(void *arg) {
  orc_worker_t *a = (orc_worker_t *)arg;
  const int64_t R = a->rank, N = a->nmodes;
  const int mode = a->mode, next_mode = a->next_mode;
  const int64_t *restrict sids = a->sids;
  const int64_t *restrict idxs = a->idxs;
  const double *restrict vals = a->vals;
  int64_t *restrict dst_sids = a->dst_sids;
  int64_t *restrict dst_idxs = a->dst_idxs;
  double *restrict dst_vals = a->dst_vals;
  const double *restrict fstack = a->fstack;
  const int64_t *restrict foffs = a->foffs;
  double *restrict out = a->out;
  const int64_t *restrict dest_slots = a->dest_slots;
  const int64_t *restrict dest_base = a->dest_base;
  const int use_cursor = a->use_cursor, do_compute = a->do_compute, do_remap = a->do_remap;
  double *restrict ell = (double *)malloc(sizeof(double) * (size_t)(R > 0 ? R : 1));
  int64_t processed = 0;
  for (int64_t s = 0; s < a->nranges; ++s) {
    const int64_t e0 = a->starts[s], e1 = a->ends[s];
    for (int64_t i = e0; i < e1; ++i) {
      if (do_compute) {
        for (int64_t r = 0; r < R; ++r) ell[r] = 1.0;
        for (int64_t w = 0; w < N; ++w) {
          if (w == mode) continue;
          const double *restrict row = fstack + (foffs[w] + idxs[i * N + w]) * R;
          for (int64_t r = 0; r < R; ++r) ell[r] *= row[r];
        }
        const double v = vals[i];
        double *restrict orow = out + idxs[i * N + mode] * R;
        for (int64_t r = 0; r < R; ++r) orow[r] += v * ell[r];
      }
      if (do_remap) {
        int64_t slot;
        if (use_cursor) {
          const int64_t b = sids[i * N + next_mode];
          slot = dest_base[b] + atomic_fetch_add_explicit(&a->cursors[b], 1,
                                                          memory_order_relaxed);
          if (slot >= dest_base[b + 1]) {
            atomic_store(a->errflag, b + 1);
            processed += 1;
            continue;
          }
        } else {
          slot = dest_slots[i];
        }
        for (int64_t w = 0; w < N; ++w) {
          dst_sids[slot * N + w] = sids[i * N + w];
          dst_idxs[slot * N + w] = idxs[i * N + w];
        }
        dst_vals[slot] = vals[i];
      }
      processed += 1;
    }
  }
  a->processed = processed;
  free(ell);
  return NULL;
}

/* engine.py:214-253: one call = one pass (compute and/or remap) over every
 * worker's ranges; worker w owns ranges [range_offs[w], range_offs[w+1]).
 * Returns total processed elements; *errflag_out = overflowed shard + 1. */
int64_t orc_mode_pass(const int64_t *sids, const int64_t *idxs, const double *vals,
                      int64_t *dst_sids, int64_t *dst_idxs, double *dst_vals,
                      const double *fstack, const int64_t *foffs, int64_t rank,
                      double *out, int nmodes, int mode, int next_mode,
                      const int64_t *starts, const int64_t *ends,
                      const int64_t *range_offs, int workers,
                      const int64_t *dest_base, int64_t *cursors,
                      const int64_t *dest_slots, int use_cursor, int do_compute,
                      int do_remap, int64_t *errflag_out) {
  if (workers < 1) return -1;
  orc_worker_t *ws = (orc_worker_t *)calloc((size_t)workers, sizeof(orc_worker_t));
  pthread_t *th = (pthread_t *)calloc((size_t)workers, sizeof(pthread_t));
  _Atomic int64_t err = 0;
  for (int w = 0; w < workers; ++w) {
    orc_worker_t *a = &ws[w];
    a->sids = sids; a->idxs = idxs; a->vals = vals;
    a->dst_sids = dst_sids; a->dst_idxs = dst_idxs; a->dst_vals = dst_vals;
    a->fstack = fstack; a->foffs = foffs; a->out = out; a->rank = rank;
    a->nmodes = nmodes; a->mode = mode; a->next_mode = next_mode;
    a->starts = starts + range_offs[w];
    a->ends = ends + range_offs[w];
    a->nranges = range_offs[w + 1] - range_offs[w];
    a->dest_base = dest_base;
    a->cursors = (_Atomic int64_t *)cursors;
    a->dest_slots = dest_slots;
    a->use_cursor = use_cursor; a->do_compute = do_compute; a->do_remap = do_remap;
    a->errflag = &err;
  }
  if (workers == 1) {
    orc_worker_run(&ws[0]);
  } else {
    for (int w = 0; w < workers; ++w) pthread_create(&th[w], NULL, orc_worker_run, &ws[w]);
    for (int w = 0; w < workers; ++w) pthread_join(th[w], NULL); /* mode barrier */
  }
  int64_t total = 0;
  for (int w = 0; w < workers; ++w) total += ws[w].processed;
  if (errflag_out) *errflag_out = atomic_load(&err);
  free(ws);
  free(th);
  return total;
}

/* ------------------------------------------------------ reference mttkrp */

/* coo.py:406-426: ell = 1; ell *= F_w[subs[:, w]] for w != mode ascending;
 * ell *= vals; np.add.at(out, subs[:, mode], ell) -- i.e. sequential
 * accumulation in nonzero storage order. */
void orc_reference_mttkrp(const int64_t *subs, const double *vals, int64_t nnz,
                          int nmodes, const double *const *factors, int64_t rank,
                          int mode, double *out) {
  double *ell = (double *)malloc(sizeof(double) * (size_t)(rank > 0 ? rank : 1));
  for (int64_t i = 0; i < nnz; ++i) {
    for (int64_t r = 0; r < rank; ++r) ell[r] = 1.0;
    for (int w = 0; w < nmodes; ++w) {
      if (w == mode) continue;
      const double *row = factors[w] + subs[i * nmodes + w] * rank;
      for (int64_t r = 0; r < rank; ++r) ell[r] *= row[r];
    }
    double *orow = out + subs[i * nmodes + mode] * rank;
    for (int64_t r = 0; r < rank; ++r) orow[r] += ell[r] * vals[i];
  }
  free(ell);
}

/* ------------------------------------------------------------ stable sort */

/* Stable LSD radix sort of `keys` on bits [0, bits): order[r] = index of the
 * r-th smallest key, equal keys in index order -- i.e. np.lexsort((seq, key))
 * for a composite key.  canonical_build uses it for the per-mode orders
 * lexsort((seq, lo, hi, iv_n)) of layout.py:484 when (iv_n, hi, lo) packs into
 * 64 bits, which turns the 76.9M-element c2 build from minutes into seconds.
 * Returns 0, or -1 when out of memory. */
int orc_stable_sort_u64(const uint64_t *keys, int64_t n, int bits, int64_t *order) {
  enum { D = 11, B = 1 << D };
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  if (n < 2 || bits <= 0) return 0;
  int64_t *tmp = (int64_t *)malloc((size_t)n * sizeof(int64_t));
  uint64_t *kc = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
  uint64_t *kt = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
  if (!tmp || !kc || !kt) {
    free(tmp); free(kc); free(kt);
    return -1;
  }
  memcpy(kc, keys, (size_t)n * sizeof(uint64_t));
  int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (B + 1));
  for (int shift = 0; shift < bits; shift += D) {
    memset(cnt, 0, sizeof(int64_t) * (B + 1));
    for (int64_t i = 0; i < n; ++i) cnt[((kc[i] >> shift) & (B - 1)) + 1]++;
    for (int d = 0; d < B; ++d) cnt[d + 1] += cnt[d];
    for (int64_t i = 0; i < n; ++i) {
      const int64_t dst = cnt[(kc[i] >> shift) & (B - 1)]++;
      tmp[dst] = order[i];
      kt[dst] = kc[i];
    }
    memcpy(order, tmp, (size_t)n * sizeof(int64_t));
    uint64_t *sw = kc; kc = kt; kt = sw;
  }
  free(cnt); free(tmp); free(kc); free(kt);
  return 0;
}

/* --------------------------------------------------- streaming shard hashes */

/* Per-shard order-independent digests of the reference's canonical layout
 * for tensors too large for canonical_build (c3-c5).  For mode
 * n: super-shard s = c_n / m_n (layout.py:474-476); inside s the canonical
 * order is (Morton(hi, lo) of every mode's interval coordinate, input
 * position) (layout.py:477-484, morton.py:20-44); element r of s belongs to
 * shard first[s] + r / g (layout.py:491-492).  Every element contributes
 * orc_elem_hash(coords, value bits) to its shard's wrapping 64-bit sum and 1
 * to its count -- a multiset digest the GPU side recomputes from its buffer.
 *
 * coords: int32 rows of stride cs (>= N; the 16-B device records work
 * directly), vbits: uint32 values of stride vs.  Memory: nnz uint32 ids +
 * per-thread (key, id) radix scratch of the largest super-shard.  Morton
 * keys must fit 64 bits (every BASELINE config does).  Returns 0, -1 when out
 * of memory, -2 when the key needs more than 64 bits. */

static inline uint64_t orc_mix64(uint64_t x) {
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27; x *= 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

uint64_t orc_elem_hash(const int32_t *c, int nmodes, uint32_t vbits) {
  uint64_t h = 0x9E3779B97F4A7C15ull;
  for (int w = 0; w < nmodes; ++w) h = orc_mix64(h ^ (uint64_t)(uint32_t)c[w]);
  return orc_mix64(h ^ ((uint64_t)vbits << 32 | 0x5bd1e995u));
}

typedef struct {
  const int32_t *coords; int64_t cs;
  const uint32_t *vbits; int64_t vs;
  int nmodes, mode;
  const int64_t *m;
  int widths[16], maxw, total;
  uint64_t deposit[16];             /* key bit positions of every mode (morton.py:20-44) */
  const uint32_t *ids; const int64_t *ss_off; const int64_t *first; int64_t g;
  int64_t nss;
  _Atomic int64_t *next;            /* work queue over super-shards (largest first) */
  const int64_t *queue;
  uint64_t *hash; int64_t *count;   /* per shard */
  int err;
} orc_hash_job_t;

/* the same key as orc_morton: bit b of mode w goes to the position the
 * level-major interleave gives it, here one bit-deposit per mode */
static uint64_t orc_morton_row(const orc_hash_job_t *J, const int32_t *c) {
  uint64_t l = 0;
  for (int w = 0; w < J->nmodes; ++w)
    l |= _pdep_u64((uint64_t)(c[w] / J->m[w]), J->deposit[w]);
  return l;
}

static void *orc_hash_run(void *arg) {
  orc_hash_job_t *J = (orc_hash_job_t *)arg;
  /* scratch grows to the largest super-shard this thread draws: the queue is
   * largest-first, so the threads together hold about the sizes of the
   * `threads` largest super-shards */
  uint64_t *k0 = NULL, *k1 = NULL;
  uint32_t *i0 = NULL, *i1 = NULL;
  int64_t cap = 0;
  int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * 2049);
  if (!cnt) { J->err = -1; return NULL; }
  for (;;) {
    const int64_t q = atomic_fetch_add(J->next, 1);
    if (q >= J->nss) break;
    const int64_t s = J->queue[q];
    const int64_t lo = J->ss_off[s], n = J->ss_off[s + 1] - lo;
    if (n == 0) continue;
    if (n > cap) {
      free(k0); free(k1); free(i0); free(i1);
      k0 = (uint64_t *)malloc((size_t)n * 8); k1 = (uint64_t *)malloc((size_t)n * 8);
      i0 = (uint32_t *)malloc((size_t)n * 4); i1 = (uint32_t *)malloc((size_t)n * 4);
      cap = n;
      if (!k0 || !k1 || !i0 || !i1) { J->err = -1; break; }
    }
    for (int64_t r = 0; r < n; ++r) {
      const uint32_t id = J->ids[lo + r];
      i0[r] = id;
      k0[r] = orc_morton_row(J, J->coords + (int64_t)id * J->cs);
    }
    /* stable LSD radix on the Morton key; ids enter in input order */
    uint64_t *ka = k0, *kb = k1;
    uint32_t *ia = i0, *ib = i1;
    for (int sh = 0; sh < J->total; sh += 11) {
      memset(cnt, 0, sizeof(int64_t) * 2049);
      for (int64_t r = 0; r < n; ++r) cnt[((ka[r] >> sh) & 2047) + 1]++;
      for (int d = 0; d < 2048; ++d) cnt[d + 1] += cnt[d];
      for (int64_t r = 0; r < n; ++r) {
        const int64_t t = cnt[(ka[r] >> sh) & 2047]++;
        kb[t] = ka[r];
        ib[t] = ia[r];
      }
      uint64_t *tk = ka; ka = kb; kb = tk;
      uint32_t *ti = ia; ia = ib; ib = ti;
    }
    for (int64_t r = 0; r < n; ++r) {
      const int64_t id = ia[r];
      const int64_t sh = J->first[s] + r / J->g;
      J->hash[sh] += orc_elem_hash(J->coords + id * J->cs, J->nmodes, J->vbits[id * J->vs]);
      J->count[sh] += 1;
    }
  }
  free(k0); free(k1); free(i0); free(i1); free(cnt);
  return NULL;
}

/* (count, id) pairs: count descending, id ascending */
static int orc_cmp_desc(const void *a, const void *b) {
  const int64_t *x = (const int64_t *)a, *y = (const int64_t *)b;
  if (x[0] != y[0]) return x[0] > y[0] ? -1 : 1;
  return (x[1] > y[1]) - (x[1] < y[1]);
}

/* One big super-shard processed by all threads: Morton keys, a parallel
 * stable LSD radix sort (per-thread digit histograms, thread-ordered
 * offsets, in-order scatter), then per-shard digests with atomic wrapping
 * adds (sums commute, so the digests are deterministic). */
typedef struct {
  const orc_hash_job_t *J;
  int64_t lo, n;                     /* super-shard s: elements ids[lo, lo + n) */
  int64_t s;
  uint64_t *k0, *k1;
  uint32_t *i0, *i1;
  int64_t *hist;                     /* [threads][2048] */
  pthread_barrier_t *bar;
  int t, T;
} orc_big_t;

static void *orc_big_run(void *arg) {
  orc_big_t *B = (orc_big_t *)arg;
  const orc_hash_job_t *J = B->J;
  const int64_t a = B->n * B->t / B->T, b = B->n * (B->t + 1) / B->T;
  for (int64_t r = a; r < b; ++r) {
    const uint32_t id = J->ids[B->lo + r];
    B->i0[r] = id;
    B->k0[r] = orc_morton_row(J, J->coords + (int64_t)id * J->cs);
  }
  uint64_t *ka = B->k0, *kb = B->k1;
  uint32_t *ia = B->i0, *ib = B->i1;
  int64_t *h = B->hist + (int64_t)B->t * 2048;
  for (int sh = 0; sh < J->total; sh += 11) {
    pthread_barrier_wait(B->bar);
    memset(h, 0, sizeof(int64_t) * 2048);
    for (int64_t r = a; r < b; ++r) h[(ka[r] >> sh) & 2047]++;
    pthread_barrier_wait(B->bar);
    if (B->t == 0) {                 /* offsets: digit-major, thread order inside a digit */
      int64_t run = 0;
      for (int d = 0; d < 2048; ++d)
        for (int t = 0; t < B->T; ++t) {
          int64_t *c = B->hist + (int64_t)t * 2048 + d;
          const int64_t x = *c;
          *c = run;
          run += x;
        }
    }
    pthread_barrier_wait(B->bar);
    for (int64_t r = a; r < b; ++r) {
      const int64_t t = h[(ka[r] >> sh) & 2047]++;
      kb[t] = ka[r];
      ib[t] = ia[r];
    }
    uint64_t *tk = ka; ka = kb; kb = tk;
    uint32_t *ti = ia; ia = ib; ib = ti;
  }
  pthread_barrier_wait(B->bar);
  for (int64_t r = a; r < b; ++r) {
    const int64_t id = ia[r];
    const int64_t sh = J->first[B->s] + r / J->g;
    __atomic_fetch_add(&J->hash[sh], orc_elem_hash(J->coords + id * J->cs, J->nmodes,
                                                    J->vbits[id * J->vs]), __ATOMIC_RELAXED);
    __atomic_fetch_add(&J->count[sh], 1, __ATOMIC_RELAXED);
  }
  return NULL;
}

static int orc_big_super_shard(const orc_hash_job_t *J, int64_t s, int T) {
  const int64_t lo = J->ss_off[s], n = J->ss_off[s + 1] - lo;
  uint64_t *k0 = (uint64_t *)malloc((size_t)n * 8), *k1 = (uint64_t *)malloc((size_t)n * 8);
  uint32_t *i0 = (uint32_t *)malloc((size_t)n * 4), *i1 = (uint32_t *)malloc((size_t)n * 4);
  int64_t *hist = (int64_t *)malloc(sizeof(int64_t) * 2048 * T);
  pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * T);
  orc_big_t *B = (orc_big_t *)malloc(sizeof(orc_big_t) * T);
  int rc = 0;
  if (!k0 || !k1 || !i0 || !i1 || !hist || !tid || !B) {
    rc = -1;
  } else {
    pthread_barrier_t bar;
    pthread_barrier_init(&bar, NULL, (unsigned)T);
    for (int t = 0; t < T; ++t) {
      B[t] = (orc_big_t){J, lo, n, s, k0, k1, i0, i1, hist, &bar, t, T};
      pthread_create(&tid[t], NULL, orc_big_run, &B[t]);
    }
    for (int t = 0; t < T; ++t) pthread_join(tid[t], NULL);
    pthread_barrier_destroy(&bar);
  }
  free(k0); free(k1); free(i0); free(i1); free(hist); free(tid); free(B);
  return rc;
}

/* Memory-lean variant for Morton keys of <= 32 bits (c2, c5): every element
 * of the super-shard is one word (key << 32 | input position); the words
 * enter in position order, so a stable LSD radix sort on the key bits alone
 * gives the canonical (key, position) order.  16 bytes of scratch per
 * element instead of 24 (c5's first mode-0 super-shard holds 2.5B). */
typedef struct {
  const orc_hash_job_t *J;
  uint64_t *P, *Q;
  int64_t lo, n, s;
  int64_t *hist;                     /* [threads][2048] */
  pthread_barrier_t *bar;
  int t, T;
} orc_pk_t;

static void *orc_pk_run(void *arg) {
  orc_pk_t *W = (orc_pk_t *)arg;
  const orc_hash_job_t *J = W->J;
  const int64_t a = W->n * W->t / W->T, b = W->n * (W->t + 1) / W->T;
  for (int64_t r = a; r < b; ++r) {
    const uint32_t id = J->ids[W->lo + r];
    W->P[r] = orc_morton_row(J, J->coords + (int64_t)id * J->cs) << 32 | id;
  }
  uint64_t *pa = W->P, *pb = W->Q;
  int64_t *h = W->hist + (int64_t)W->t * 2048;
  for (int sh = 32; sh < 32 + J->total; sh += 11) {
    pthread_barrier_wait(W->bar);
    memset(h, 0, sizeof(int64_t) * 2048);
    for (int64_t r = a; r < b; ++r) h[(pa[r] >> sh) & 2047]++;
    pthread_barrier_wait(W->bar);
    if (W->t == 0) {
      int64_t run = 0;
      for (int d = 0; d < 2048; ++d)
        for (int t = 0; t < W->T; ++t) {
          int64_t *c = W->hist + (int64_t)t * 2048 + d;
          const int64_t x = *c;
          *c = run;
          run += x;
        }
    }
    pthread_barrier_wait(W->bar);
    for (int64_t r = a; r < b; ++r) pb[h[(pa[r] >> sh) & 2047]++] = pa[r];
    uint64_t *tp = pa; pa = pb; pb = tp;
  }
  pthread_barrier_wait(W->bar);
  for (int64_t r = a; r < b; ++r) {
    const int64_t id = (int64_t)(pa[r] & 0xFFFFFFFFull);
    const int64_t sh = J->first[W->s] + r / J->g;
    __atomic_fetch_add(&J->hash[sh], orc_elem_hash(J->coords + id * J->cs, J->nmodes,
                                                    J->vbits[id * J->vs]), __ATOMIC_RELAXED);
    __atomic_fetch_add(&J->count[sh], 1, __ATOMIC_RELAXED);
  }
  return NULL;
}

static int orc_big_packed(const orc_hash_job_t *J, int64_t s, int T) {
  const int64_t lo = J->ss_off[s], n = J->ss_off[s + 1] - lo;
  uint64_t *P = (uint64_t *)malloc((size_t)n * 8), *Q = (uint64_t *)malloc((size_t)n * 8);
  int64_t *hist = (int64_t *)malloc(sizeof(int64_t) * 2048 * T);
  pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * T);
  orc_pk_t *W = (orc_pk_t *)malloc(sizeof(orc_pk_t) * T);
  int rc = 0;
  if (!P || !Q || !hist || !tid || !W) {
    rc = -1;
  } else {
    pthread_barrier_t bar;
    pthread_barrier_init(&bar, NULL, (unsigned)T);
    for (int t = 0; t < T; ++t) {
      W[t] = (orc_pk_t){J, P, Q, lo, n, s, hist, &bar, t, T};
      pthread_create(&tid[t], NULL, orc_pk_run, &W[t]);
    }
    for (int t = 0; t < T; ++t) pthread_join(tid[t], NULL);
    pthread_barrier_destroy(&bar);
  }
  free(P); free(Q); free(hist); free(tid); free(W);
  return rc;
}

/* Stable counting sort of element ids by super-shard, by all threads:
 * per-thread counts over contiguous id ranges, thread-ordered offsets,
 * in-order scatter -- ids ascending inside every super-shard. */
typedef struct {
  const int32_t *coords; int64_t cs; int mode; int64_t m;
  int64_t nnz, K;
  int64_t *cnt;                      /* [threads][K] counts, then offsets */
  uint32_t *ids;
  pthread_barrier_t *bar;
  int t, T;
} orc_cs_t;

static void *orc_cs_run(void *arg) {
  orc_cs_t *C = (orc_cs_t *)arg;
  const int64_t a = C->nnz * C->t / C->T, b = C->nnz * (C->t + 1) / C->T;
  int64_t *c = C->cnt + (int64_t)C->t * C->K;
  for (int64_t i = a; i < b; ++i) c[C->coords[i * C->cs + C->mode] / C->m]++;
  pthread_barrier_wait(C->bar);
  if (C->t == 0) {
    int64_t run = 0;
    for (int64_t s = 0; s < C->K; ++s)
      for (int t = 0; t < C->T; ++t) {
        int64_t *x = C->cnt + (int64_t)t * C->K + s;
        const int64_t v = *x;
        *x = run;
        run += v;
      }
  }
  pthread_barrier_wait(C->bar);
  for (int64_t i = a; i < b; ++i) C->ids[c[C->coords[i * C->cs + C->mode] / C->m]++] = (uint32_t)i;
  return NULL;
}

static int orc_counting_sort(const int32_t *coords, int64_t cs, int mode, int64_t m, int64_t nnz,
                             int64_t K, int T, uint32_t *ids) {
  if ((int64_t)T * K > (1ll << 28)) T = 1;   /* per-thread counts must stay small */
  int64_t *cnt = (int64_t *)calloc((size_t)T * (size_t)K, sizeof(int64_t));
  pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * T);
  orc_cs_t *C = (orc_cs_t *)malloc(sizeof(orc_cs_t) * T);
  if (!cnt || !tid || !C) {
    free(cnt); free(tid); free(C);
    return -1;
  }
  pthread_barrier_t bar;
  pthread_barrier_init(&bar, NULL, (unsigned)T);
  for (int t = 0; t < T; ++t) {
    C[t] = (orc_cs_t){coords, cs, mode, m, nnz, K, cnt, ids, &bar, t, T};
    pthread_create(&tid[t], NULL, orc_cs_run, &C[t]);
  }
  for (int t = 0; t < T; ++t) pthread_join(tid[t], NULL);
  pthread_barrier_destroy(&bar);
  free(cnt); free(tid); free(C);
  return 0;
}

int orc_shard_hashes(const int32_t *coords, int64_t cs, const uint32_t *vbits, int64_t vs,
                     int64_t nnz, int nmodes, int mode, const int64_t *m, const int64_t *k,
                     int64_t g, int threads, int64_t *ss_counts, uint64_t *hash,
                     int64_t *count) {
  if (nmodes > 16 || threads < 1) return -3;
  orc_hash_job_t J;
  memset(&J, 0, sizeof(J));
  J.coords = coords; J.cs = cs; J.vbits = vbits; J.vs = vs;
  J.nmodes = nmodes; J.mode = mode; J.m = m; J.g = g;
  for (int w = 0; w < nmodes; ++w) {
    J.widths[w] = k[w] > 1 ? bit_length_u64((uint64_t)(k[w] - 1)) : 0;
    J.total += J.widths[w];
    if (J.widths[w] > J.maxw) J.maxw = J.widths[w];
  }
  if (J.total > 64) return -2;
  {
    int pos = 0;
    for (int b = 0; b < J.maxw; ++b)
      for (int w = 0; w < nmodes; ++w)
        if (b < J.widths[w]) J.deposit[w] |= 1ull << pos++;
  }
  const int64_t K = k[mode];
  /* super-shard of every element, counts (layout.py:487) */
  memset(ss_counts, 0, sizeof(int64_t) * K);
  for (int64_t i = 0; i < nnz; ++i) ss_counts[coords[i * cs + mode] / m[mode]]++;
  int64_t *off = (int64_t *)malloc(sizeof(int64_t) * (K + 1));
  int64_t *first = (int64_t *)malloc(sizeof(int64_t) * (K + 1));
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * K);
  int64_t *queue = (int64_t *)malloc(sizeof(int64_t) * K);
  uint32_t *ids = (uint32_t *)malloc((size_t)nnz * 4);
  if (!off || !first || !fill || !queue || !ids) {
    free(off); free(first); free(fill); free(queue); free(ids);
    return -1;
  }
  off[0] = first[0] = 0;
  int64_t big = 0;
  for (int64_t s = 0; s < K; ++s) {
    off[s + 1] = off[s] + ss_counts[s];
    first[s + 1] = first[s] + (ss_counts[s] + g - 1) / g;
    fill[s] = off[s];
    queue[s] = s;
    if (ss_counts[s] > big) big = ss_counts[s];
  }
  /* stable counting sort of element ids by super-shard (ids ascending) */
  if (orc_counting_sort(coords, cs, mode, m[mode], nnz, K, threads, ids) != 0) {
    free(off); free(first); free(fill); free(queue); free(ids);
    return -1;
  }
  {
    int64_t *pairs = (int64_t *)malloc(sizeof(int64_t) * 2 * (K > 0 ? K : 1));
    if (!pairs) {
      free(off); free(first); free(fill); free(queue); free(ids);
      return -1;
    }
    for (int64_t s = 0; s < K; ++s) { pairs[2 * s] = ss_counts[s]; pairs[2 * s + 1] = s; }
    qsort(pairs, (size_t)K, 2 * sizeof(int64_t), orc_cmp_desc);
    for (int64_t s = 0; s < K; ++s) queue[s] = pairs[2 * s + 1];
    free(pairs);
  }
  memset(hash, 0, sizeof(uint64_t) * first[K]);
  memset(count, 0, sizeof(int64_t) * first[K]);
  _Atomic int64_t next = 0;
  J.ids = ids; J.ss_off = off; J.first = first; J.nss = K; J.next = &next; J.queue = queue;
  J.hash = hash; J.count = count;
  /* super-shards holding more than 1/(2 threads) of the elements (Zipf
   * heads: c4's first super-shard) are sorted by all threads together */
  int64_t nbig = 0;
  while (threads > 1 && nbig < K && ss_counts[queue[nbig]] * 2 * threads > nnz) {
    const int rc = J.total <= 32 ? orc_big_packed(&J, queue[nbig], threads)
                                 : orc_big_super_shard(&J, queue[nbig], threads);
    if (rc != 0) {
      free(off); free(first); free(fill); free(queue); free(ids);
      return -1;
    }
    ++nbig;
  }
  next = nbig;
  /* the largest super-shards go first: one thread holds the largest scratch,
   * the others the size of the (threads)-th largest */
  if (threads > K) threads = (int)(K > 0 ? K : 1);
  (void)big;
  pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * threads);
  orc_hash_job_t *jobs = (orc_hash_job_t *)malloc(sizeof(orc_hash_job_t) * threads);
  for (int t = 0; t < threads; ++t) {
    jobs[t] = J;
    pthread_create(&tid[t], NULL, orc_hash_run, &jobs[t]);
  }
  int err = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(tid[t], NULL);
    if (jobs[t].err) err = jobs[t].err;
  }
  free(tid); free(jobs); free(off); free(first); free(fill); free(queue); free(ids);
  return err;
}
