/*
 * flycoo.h -- C ABI of the B200 FLYCOO all-mode spMTTKRP + dynamic-remap path.
 *
 * Every entry point is plain C: device pointers, host arrays of device
 * pointers, sizes and a cudaStream_t passed as void*.  No torch types.  All
 * calls are stream-ordered, allocate nothing (the caller passes workspace)
 * and return 0 on success or a negative FC_ERR_* code; fc_last_error()
 * describes the last failure.  Device-detected layout violations are
 * reported through a caller-provided device flag word (see FC_FLAG_*), which
 * the host shim turns into the reference's exceptions.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/modecycle):
 *   fc_mode_worker      <- _kernels.mode_worker            _kernels.py:38-88
 *                          fanned out by engine.mttkrp_mode engine.py:214-245
 *   fc_remap_cursor     <- _kernels.mode_worker cursor path _kernels.py:73-82
 *                          (+ _atomic_fetch_add             _kernels.py:18-35)
 *   fc_build_*          <- layout.build_sharded             layout.py:462-531
 *                          + morton.interleave              morton.py:20-44
 *   fc_synth_*          <- coo.synth_tensor (measurement inputs only;
 *                          bounded Zipf, not the reference's power law)
 *                                                           coo.py:323-399
 */
#ifndef FLYCOO_H_
#define FLYCOO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FC_OK 0
#define FC_ERR_ARG (-1)          /* bad argument (null pointer, size)       */
#define FC_ERR_UNSUPPORTED (-2)  /* shape outside what the kernels handle   */
#define FC_ERR_CUDA (-3)         /* a CUDA launch / runtime call failed     */

/* Bits of the device flag word (int32) written by fc_mode_worker /
 * fc_remap_cursor.  The host shim raises ShardOverflowError for
 * FC_FLAG_SLOT_RANGE / FC_FLAG_SHARD_OVERFLOW and BufferOrderError for
 * FC_FLAG_ROW_OUTSIDE_SS (engine.py:41-46, 255-263). */
#define FC_FLAG_SLOT_RANGE 1      /* a destination slot >= nnz              */
#define FC_FLAG_ROW_OUTSIDE_SS 2  /* element's output row not in its chunk's
                                     super-shard: buffer not ordered for mode */
#define FC_FLAG_SHARD_OVERFLOW 4  /* cursor strategy: shard fill exceeded   */
#define FC_FLAG_INDEX_CHECK 8     /* checked build (FC_DEVICE_CHECKS) only: a
                                     shared/global index outside its tile  */

/* Element record layout in HBM ("crd" words are int32, 16-B aligned rows):
 *   N <= 3 : 4 words  {c0, c1, c2, bits(value)}   (N = 2: word 2 is 0)
 *   N == 4 : 4 words  {c0..c3} + separate float value array
 *   5..7   : 8 words  {c0..c_{N-1}, 0.., bits(value) in word 7}
 *   N == 8 : 8 words  {c0..c7} + separate float value array            */
int fc_crd_words(int nmodes);        /* 4 or 8; <0 when N unsupported   */
int fc_value_embedded(int nmodes);   /* 1 if the value lives in word CW-1 */

/* Library introspection. */
int fc_version(void);
const char *fc_last_error(void);
/* Largest super-shard row count whose rank-R accumulator tile is kept in
 * shared memory; larger intervals accumulate in global memory (out rows). */
int64_t fc_smem_acc_rows_max(int rank);
int fc_tile_elems(void);             /* elements per CTA tile (fixed)     */
/* Kernel variant for A/B runs (default 1, 1; the environment variables
 * FLYCOO_PACK=0 / FLYCOO_PACK_WIDE=0 set it once when the library loads):
 * pack = 8-byte sorted records for 3-mode tensors whose input coordinates
 * fit 32 bits, pack_wide = the {c_w1, c_w2} + value variant otherwise. */
int fc_set_kernel_variant(int pack, int pack_wide);
/* Row capacity of a "direct" chunk merging consecutive small super-shards
 * (fast path only; returns m when merging is not supported). */
int64_t fc_chunk_rows_max(int nmodes, int rank, int64_t m);

/* ------------------------------------------------------------------ K1/K2
 * One mode pass: for every element i of the active buffer (ordered for
 * `mode`), y[c_mode,:] += v * prod_{w != mode} F_w[c_w,:] and, if do_remap,
 * dst[dest_slots[i]] = src[i].
 *
 * Work plan (host-built, static per tensor and mode; see layout.py):
 *   chunk c covers elements [chunk_start[c], chunk_start[c+1]) of one
 *   super-shard chunk_ss[c]; chunk_part[c] == -1 means the chunk is the only
 *   one of its super-shard and owns its output rows, otherwise it writes its
 *   partial rows to part_ws slot chunk_part[c] (m_mode x rank floats).
 *   chunk_rows (optional, fast path): a chunk may cover several whole
 *   consecutive super-shards starting at chunk_ss[c]; it then owns
 *   chunk_rows[c] rows (<= tile_rows <= fc_chunk_rows_max) and chunk_part[c]
 *   is -1; or, with chunk_part[c] == -2 ("direct"), at most one tile
 *   (fc_tile_elems) of nonzeros and chunk_rows[c] <= hist_rows <= 256 rows,
 *   stored straight to `out` without an accumulator tile.
 *   Deterministic two-level reduce of the partials (K2): red1 holds nred1
 *   tasks {ss, p0, p1, dst}: rows of super-shard ss = sum of partials
 *   [p0, p1) in chunk order, written to `out` (dst < 0) or to part_ws2 slot
 *   dst; red2 holds nred2 tasks {ss, q0, q1} summing part_ws2 slots [q0, q1)
 *   into `out`.  Empty super-shards appear as {ss, 0, 0, -1} (zero rows).
 *   acc_in_smem must be 1 iff m_mode <= fc_smem_acc_rows_max(rank); with
 *   acc_in_smem == 0 every chunk must own its super-shard and `out` must be
 *   zero on entry.
 * Slots must be < nnz, the destination capacity (on one GPU the buffer
 * size; multi-GPU: local part + send region, see dist.py).
 * `dims` (optional) lets 3-mode tensors whose two input coordinates fit 32
 * bits use 8-byte sorted records (same results, less shared traffic).
 * counters[0] += elements processed (the engine.py:247-250 check).        */
int fc_mode_worker(const void *src_crd, const float *src_val,
                   void *dst_crd, float *dst_val,
                   const float *const *factors, /* host array, N device ptrs */
                   const int64_t *dims,         /* host array, N (may be NULL) */
                   float *out, int nmodes, int mode, int rank,
                   int64_t out_rows, int64_t m_mode,
                   const int64_t *chunk_start, const int32_t *chunk_ss,
                   const int32_t *chunk_part, const int32_t *chunk_rows,
                   int64_t tile_rows, int64_t hist_rows, int64_t nchunks,
                   const int64_t *red1, int64_t nred1, const int64_t *red2, int64_t nred2,
                   float *part_ws, float *part_ws2, const uint32_t *dest_slots, int64_t nnz,
                   int do_compute, int do_remap, int acc_in_smem,
                   int32_t *flags, unsigned long long *counters, void *stream);

/* Tile plan.  The layout is static, so every 2048-element tile of a mode's
 * buffer is sorted by output row the same way in every sweep (the stable
 * counting sort in front of the row-segmented reduction; the reference's
 * per-element loop _kernels.py:58-72 has no such step).  fc_tile_plan_emit
 * runs that ranking once over the buffer that is active for `mode` and
 * writes, per element, its position in the sorted tile (tile_perm: 2048
 * uint16 per tile key, the 8 elements of a thread adjacent) and, per tile,
 * the bin starts (tile_bins, hist_rows uint16 per tile key;
 * fc_tile_plan_keys(nnz, nchunks) keys; hist_rows = the work plan's, or
 * m_mode when chunk_rows is NULL).  fc_mode_worker_planned is
 * fc_mode_worker (do_compute = 1, shared-memory accumulation) reading that
 * plan instead of ranking: same sorted order, hence bitwise the same sums.
 * Both return FC_ERR_UNSUPPORTED outside the kernels that take a plan
 * (3-mode tensors at R = 32 or 16, 4-mode tensors at R = 32); callers then
 * use fc_mode_worker.
 * The plan is valid for the work plan (chunk arrays) it was emitted with and
 * for the canonical (slot-remapped) order only. */
int fc_tile_plan_emit(const void *src_crd, const float *src_val,
                      const float *const *factors, const int64_t *dims,
                      int nmodes, int mode, int rank, int64_t out_rows, int64_t m_mode,
                      const int64_t *chunk_start, const int32_t *chunk_ss,
                      const int32_t *chunk_part, const int32_t *chunk_rows,
                      int64_t tile_rows, int64_t hist_rows, int64_t nchunks, int64_t nnz,
                      int32_t *flags, unsigned long long *counters,
                      uint16_t *tile_perm, uint16_t *tile_bins, void *stream);
int64_t fc_tile_plan_keys(int64_t nnz, int64_t nchunks);
int fc_mode_worker_planned(const void *src_crd, const float *src_val,
                           void *dst_crd, float *dst_val,
                           const float *const *factors, const int64_t *dims,
                           float *out, int nmodes, int mode, int rank,
                           int64_t out_rows, int64_t m_mode,
                           const int64_t *chunk_start, const int32_t *chunk_ss,
                           const int32_t *chunk_part, const int32_t *chunk_rows,
                           int64_t tile_rows, int64_t hist_rows, int64_t nchunks,
                           const int64_t *red1, int64_t nred1, const int64_t *red2, int64_t nred2,
                           float *part_ws, float *part_ws2, const uint32_t *dest_slots,
                           int64_t nnz, int do_remap, int32_t *flags,
                           unsigned long long *counters, const uint16_t *tile_perm,
                           const uint16_t *tile_bins, void *stream);

/* Multi-GPU mode pass with the remap fused with the exchange (dist.py,
 * exchange "p2p"): same work plan and arguments as fc_mode_worker, but
 * dest_slots hold GLOBAL mode-(n+1) positions and every record is stored
 * straight into the back buffer of the GPU that owns its slot -- GPU q owns
 * [peer_base[q], peer_base[q+1]) and its buffer is peer_crd[q] (peer_val[q]
 * for N = 4 / N >= 5 separate values), an NVLink peer mapping from
 * fc_ipc_open (or this GPU's own buffer).  Replaces the send-region pass,
 * the NCCL all-to-all and fc_scatter_records.  npeers <= 8; nnz = local
 * element count (remap-only pass); the caller orders the passes of all GPUs
 * (barrier between modes).  Heavy super-shards may be split across GPUs at
 * chunk granularity: `chunk_owner[c]` names the GPU that owns chunk c's
 * super-shard and the partial tile goes to its workspace peer_part_ws[owner]
 * (partial ids are global); pass nred1 = nred2 = 0 and reduce on the owner
 * with fc_reduce_partials after a barrier.  chunk_owner may be NULL (every
 * chunk local). */
int fc_mode_worker_peers(const void *src_crd, const float *src_val,
                         const float *const *factors, const int64_t *dims,
                         float *out, int nmodes, int mode, int rank,
                         int64_t out_rows, int64_t m_mode,
                         const int64_t *chunk_start, const int32_t *chunk_ss,
                         const int32_t *chunk_part, const int32_t *chunk_rows,
                         int64_t tile_rows, int64_t hist_rows, int64_t nchunks,
                         const int64_t *red1, int64_t nred1, const int64_t *red2,
                         int64_t nred2, float *part_ws, float *part_ws2,
                         const uint32_t *dest_slots, int64_t nnz, int do_compute,
                         int acc_in_smem, int32_t *flags, unsigned long long *counters,
                         int npeers, void *const *peer_crd, float *const *peer_val,
                         const int64_t *peer_base, float *const *peer_part_ws,
                         const int32_t *chunk_owner, void *stream);
/* fc_mode_worker_peers reading a tile plan emitted on this GPU's slice
 * (fc_tile_plan_emit with the same shifted pointers and chunk range; keys
 * t0 / 2048 + local chunk index, t0 the global element index); tile_perm
 * NULL: rank in the kernel. */
int fc_mode_worker_peers_planned(const void *src_crd, const float *src_val,
                         const float *const *factors, const int64_t *dims,
                         float *out, int nmodes, int mode, int rank,
                         int64_t out_rows, int64_t m_mode,
                         const int64_t *chunk_start, const int32_t *chunk_ss,
                         const int32_t *chunk_part, const int32_t *chunk_rows,
                         int64_t tile_rows, int64_t hist_rows, int64_t nchunks,
                         const int64_t *red1, int64_t nred1, const int64_t *red2,
                         int64_t nred2, float *part_ws, float *part_ws2,
                         const uint32_t *dest_slots, int64_t nnz, int do_compute,
                         int acc_in_smem, int32_t *flags, unsigned long long *counters,
                         int npeers, void *const *peer_crd, float *const *peer_val,
                         const int64_t *peer_base, float *const *peer_part_ws,
                         const int32_t *chunk_owner, const uint16_t *tile_perm, const uint16_t *tile_bins,
                         void *stream);

/* K2 alone (the second half of fc_mode_worker): the deterministic two-level
 * reduce of partial tiles into `out`.  Multi-GPU: the owner of super-shards
 * whose chunks ran on several GPUs reduces the partials the peers wrote into
 * its workspace, after a barrier. */
int fc_reduce_partials(const int64_t *red1, int64_t nred1, const int64_t *red2, int64_t nred2,
                       const float *part_ws, float *part_ws2, float *out, int64_t out_rows,
                       int64_t m_mode, int rank, void *stream);

/* Peer-memory plumbing for the fused exchange (no reference counterpart:
 * the reference is single-node shared memory).  IPC-shareable cudaMalloc
 * allocations, their fc_ipc_handle_bytes()-byte handles, peer mappings and
 * stream-ordered copies (cudaMemcpyDefault: local or peer). */
int fc_ipc_handle_bytes(void);
int fc_ipc_alloc(int64_t bytes, void **ptr);
int fc_ipc_free(void *ptr);
int fc_ipc_handle(const void *ptr, void *handle);
int fc_ipc_open(const void *handle, void **ptr);
int fc_ipc_close(void *ptr);
int fc_copy_async(void *dst, const void *src, int64_t bytes, void *stream);
/* Factor-row all-gather of the fused exchange in one launch: rows
 * [row_lo[q], row_lo[q+1]) of peer_src[q] (GPU q's output, peer-mapped) are
 * copied into dst for every q != self; rows are row_floats fp32 wide. */
int fc_gather_peer_rows(float *dst, const float *const *peer_src, const int64_t *row_lo,
                        int npeers, int self, int64_t row_floats, void *stream);
/* Cross-GPU ordering on the stream, without the host: the GPU's front end
 * writes `value` to a (peer-mapped) 32-bit flag after fencing the stream's
 * prior memory operations, or waits until (int32)(*flag - value) >= 0
 * (cuStreamWriteValue32 / cuStreamWaitValue32; no SM spins). */
int fc_stream_signal(void *flag, uint32_t value, void *stream);
/* 1 if fc_stream_wait flushes peers' remote writes on the current device
 * (CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES), 0 if not, <0 on error. */
int fc_stream_wait_flush_supported(void);
int fc_stream_wait(const void *flag, uint32_t value, void *stream);

/* Cursor remap strategy (_kernels.py:73-80): b = src_sid[i, next_mode];
 * slot = dest_base[b] + fetch_add(cursors[b]); dst[slot] = src[i] together
 * with the element's N shard ids (the reference carries sids in every
 * element, layout.py:395).  Order inside a shard is nondeterministic;
 * cursors must be zero on entry. */
int fc_remap_cursor(const void *src_crd, const float *src_val, void *dst_crd,
                    float *dst_val, const uint32_t *src_sid, uint32_t *dst_sid,
                    int nmodes, int next_mode, int64_t nnz, const int64_t *dest_base,
                    unsigned long long *cursors, int32_t *flags, void *stream);

/* Receiver-side unpack of the multi-GPU remap: dst[slots[k]] = src[k] for
 * k < n, slots < dst_capacity; counters[0] += n. */
int fc_scatter_records(const void *src_crd, const float *src_val, int64_t n,
                       void *dst_crd, float *dst_val, int64_t dst_capacity,
                       const uint32_t *slots, int nmodes, int32_t *flags,
                       unsigned long long *counters, void *stream);

/* ---------------------------------------------------------------- K5 build
 * Layout build (layout.py:462-531) in device passes; the host shim
 * (paper_2309_09131_b200/layout.py) sequences them.  `coords` is (nnz, N)
 * int32 in input order (seq), `ids` / `keys` are scratch of nnz entries. */
/* Morton (hi, lo) of interval coordinates iv_w = coords[:, w] / m[w]
 * (morton.py:20-44); m/k are host arrays; hi may be NULL when the key fits
 * 64 bits.  Returns FC_ERR_UNSUPPORTED if the key needs more than 128 bits. */
int fc_build_morton(const int32_t *coords, int64_t nnz, int nmodes,
                    const int64_t *m, const int64_t *k,
                    uint64_t *hi, uint64_t *lo, void *stream);
/* Temp-storage bytes for fc_build_sort_pairs on nnz items. */
int64_t fc_build_sort_temp_bytes(int64_t nnz);
/* Stable LSD radix sort of (key, id) pairs on bits [0, end_bit); keys_out /
 * ids_out receive the sorted sequence. */
int fc_build_sort_pairs(const uint64_t *keys_in, uint64_t *keys_out,
                        const uint32_t *ids_in, uint32_t *ids_out, int64_t nnz,
                        int end_bit, void *temp, int64_t temp_bytes, void *stream);
/* keys[p] = f(ids[p]) for the sort passes of one mode's canonical order:
 *   what = 0: lo[id];  1: hi[id];  2: iv_mode[id] = coords[id, mode] / m
 *   what = 3: (iv_mode[id] << shift) | lo[id]   (single-pass key)        */
int fc_build_gather_key(const uint32_t *ids, int64_t nnz, int what,
                        const uint64_t *hi, const uint64_t *lo,
                        const int32_t *coords, int nmodes, int mode, int64_t m,
                        int shift, uint64_t *keys, void *stream);
/* Histogram of iv_mode over k bins (super-shard fills, layout.py:487). */
int fc_build_ss_hist(const int32_t *coords, int64_t nnz, int nmodes, int mode,
                     int64_t m, int64_t k, unsigned long long *hist, void *stream);
/* From the canonical order of one mode: sid[id] = first[iv] + (p - offs[iv]) / g
 * (layout.py:491-492).  first/offs are device arrays of k+1 int64. */
int fc_build_shard_ids(const uint32_t *order, int64_t nnz, const int32_t *coords,
                       int nmodes, int mode, int64_t m, const int64_t *ss_offs,
                       const int64_t *ss_first, int64_t g, uint32_t *sid, void *stream);
/* keys[p] = (sid_mode[ids[p]] << 32) | sid_prev[ids[p]]: the B200 intra-shard
 * order key (Layout). */
int fc_build_device_key(const uint32_t *ids, int64_t nnz, const uint32_t *sid_mode,
                        const uint32_t *sid_prev, uint64_t *keys, void *stream);
/* pos[order[p]] = p */
int fc_build_invert(const uint32_t *order, int64_t nnz, uint32_t *pos, void *stream);
/* slot[p] = pos_next[order[p]]  (layout.py:516-519 slot maps) */
int fc_build_slots(const uint32_t *order, const uint32_t *pos_next, int64_t nnz,
                   uint32_t *slot, void *stream);
/* Memory-lean forms used by the build: slot[pos_n[id]] = pos_next[id], and
 * records scattered to their positions crd[pos[id]] = (coords[id], vals[id]). */
int fc_build_slots_scatter(const uint32_t *pos_n, const uint32_t *pos_next, int64_t nnz,
                           uint32_t *slot, void *stream);
int fc_build_records_scatter(const uint32_t *pos, int64_t nnz, int nmodes,
                             const int32_t *coords, const float *vals, void *crd,
                             float *val_out, void *stream);
/* Records of the active buffer in `order`: crd/val per the record layout. */
int fc_build_records(const uint32_t *order, int64_t nnz, int nmodes,
                     const int32_t *coords, const float *vals, void *crd,
                     float *val_out, void *stream);

/* Lean build (layout.build_device_sharded_lean): the same orders with 32-bit
 * sort keys, coordinates read in place from 16-B records (cstride = ints per
 * record), so that a tensor whose layout fills most of HBM (config 5:
 * 3.6B nonzeros) builds inside the memory of its own final buffers.
 *   iota: out[i] = i;  morton32: Morton key of <= 32 bits (else UNSUPPORTED);
 *   sort_pairs32: stable LSD radix sort of (uint32 key, id) on [0, end_bit);
 *   iv_key32: keys[p] = crd[ids[p]*cstride + mode] / m;
 *   gather_u32: dst[p] = src[ids[p]];
 *   scatter_rec16: dst[pos[i]] = src[i] (16-B records). */
int fc_build_iota(uint32_t *out, int64_t n, void *stream);
int fc_build_morton32(const int32_t *crd, int64_t nnz, int nmodes, int cstride,
                      const int64_t *m, const int64_t *k, uint32_t *key, void *stream);
int64_t fc_build_sort32_temp_bytes(int64_t nnz);
int fc_build_sort_pairs32(const uint32_t *keys_in, uint32_t *keys_out,
                          const uint32_t *ids_in, uint32_t *ids_out, int64_t nnz,
                          int end_bit, void *temp, int64_t temp_bytes, void *stream);
int fc_build_iv_key32(const uint32_t *ids, int64_t n, const int32_t *crd, int cstride,
                      int mode, int64_t m, uint32_t *keys, void *stream);
int fc_build_gather_u32(const uint32_t *ids, int64_t n, const uint32_t *src,
                        uint32_t *dst, void *stream);
int fc_build_scatter_rec16(const uint32_t *pos, int64_t n, const void *src, void *dst,
                           void *stream);

/* ---------------------------------------------------------------- K6 synth
 * Measurement-input generator (bench / tests; not the product path).
 * Draw j, mode w: u = philox(seed, w, j) in [0,1); index = smallest i with
 * u < cdf_w[i] (bounded Zipf inverse CDF, cdf_w has dims[w] entries ending
 * in 1.0), or floor(u * dims[w]) when cdf_w is NULL (uniform). */
int fc_synth_draw(uint64_t seed, int64_t ndraws, int nmodes, const int64_t *dims,
                  const double *const *cdfs, const int64_t *cdf_len,
                  int32_t *coords, void *stream);
/* Linearised keys (mixed radix over dims, 128-bit as hi/lo) of drawn coords. */
int fc_synth_keys(const int32_t *coords, int64_t n, int nmodes, const int64_t *dims,
                  uint64_t *hi, uint64_t *lo, void *stream);
/* keep[ids[p]] = (p == 0 || keys differ from p-1) over a key-sorted run. */
int fc_synth_mark_first(const uint64_t *hi_sorted, const uint64_t *lo_sorted,
                        const uint32_t *ids_sorted, int64_t n, uint8_t *keep,
                        void *stream);
/* Coordinates of modes [mode_lo, mode_hi) of the draws js[i] (same law as
 * fc_synth_draw): out[i*cstride + w - mode_lo].  Used by the bucketed
 * generator of the tensors too large for one dedup sort (synth.py). */
int fc_synth_draw_at(uint64_t seed, const int64_t *js, int64_t n, int nmodes,
                     const int64_t *dims, const double *const *cdfs,
                     const int64_t *cdf_len, int mode_lo, int mode_hi,
                     int32_t *out, int cstride, void *stream);
/* fp32 values in (0, 1]: vals[i] = philox(seed, stream, i). */
int fc_synth_uniform(uint64_t seed, uint32_t stream_id, int64_t n, float *out,
                     int open_low, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FLYCOO_H_ */
