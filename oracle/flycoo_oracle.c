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
