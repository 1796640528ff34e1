// K1 / K2: one FLYCOO mode pass on sm_100a -- sparse MTTKRP for `mode` fused
// with the dynamic remap of every element into its next-mode slot.
//
// Replaces the reference's per-thread numba kernel _kernels.mode_worker
// (/root/reference/pkg/src/modecycle/_kernels.py:38-88) and the thread
// fan-out / join of engine.mttkrp_mode (engine.py:214-245).
//
// Work decomposition: one CTA per chunk, a chunk being a
// contiguous run of elements inside ONE super-shard, so the CTA owns (or
// holds a private partial of) that super-shard's m output rows -- the
// reference's row-ownership argument (PAPER §4, SPEC "lock-free row
// ownership") with CTAs in place of CPU threads.  Per tile of kTile
// elements:
//   A  stream the records in (16-B vector loads, L1 no-allocate), scatter
//      each one to dst[slot] (the remap; slots are the build-time
//      permutation, so writes are disjoint and deterministic), stage the
//      tile in shared memory and form its local output-row key;
//   B  stable block radix sort of (row, tile index) -- deterministic order;
//   C  groups of LPG lanes (VEC columns per lane: one 128-B factor row per
//      8 lanes at R=32) walk fixed pieces of the sorted tile, gather the N-1
//      factor rows with read-only 16-B loads, form the Hadamard product in
//      registers and reduce each equal-row segment in registers; segments
//      that stay inside a piece are added to the accumulator tile directly
//      (exclusive rows), boundary segments go to a small side buffer;
//   D  one warp folds the boundary segments in piece order.
// No global atomics on data; every sum has a fixed order, so a sweep is
// bitwise reproducible.  Rows of super-shards split over several chunks
// are summed by K2 in chunk order.
#include <cub/block/block_radix_sort.cuh>
#include <stdlib.h>
#include <string.h>

#include "mode_args.cuh"

namespace fc {
namespace {

constexpr int kRadixBits = 6;
using BlockSort = cub::BlockRadixSort<uint32_t, kBlock, kIPT, uint16_t, kRadixBits>;

// Shared-memory plan of one CTA (dynamic smem, carved in this order).
template <int CW4, bool EMB>
struct SmemPlan {
  static constexpr size_t rec_bytes = sizeof(int4) * CW4 * kTile;
  static constexpr size_t val_bytes = EMB ? 0 : sizeof(float) * kTile;
  static constexpr size_t keyidx_bytes = (sizeof(uint32_t) + sizeof(uint16_t)) * kTile;
  static constexpr size_t sort_bytes =
      sizeof(typename BlockSort::TempStorage) > keyidx_bytes ? sizeof(typename BlockSort::TempStorage)
                                                             : keyidx_bytes;
  static constexpr size_t fixed_bytes = rec_bytes + val_bytes + ((sort_bytes + 15) / 16) * 16 + 16;
  static size_t total(int groups, int rank, int64_t acc_rows) {
    return fixed_bytes + (size_t)2 * groups * sizeof(int) + (size_t)2 * groups * rank * sizeof(float) +
           (size_t)acc_rows * rank * sizeof(float) + 64;
  }
};

// NM_T: number of modes (0 = runtime, up to 8).  VEC/LPG: columns per lane /
// lanes per element group.  MAXIT: column blocks of LPG*VEC per group.
template <int NM_T, int VEC, int LPG, int MAXIT, bool SMEM_ACC>
__global__ void __launch_bounds__(kBlock) mode_pass_kernel(const __grid_constant__ ModeArgs a) {
  constexpr int NMAX = NM_T > 0 ? NM_T : 8;
  constexpr int CW4 = NM_T > 0 ? crd_words(NM_T) / 4 : 2;  // runtime NM: room for 8 words
  constexpr bool EMB_T = NM_T > 0 ? value_embedded(NM_T) : false;
  constexpr int G = kBlock / LPG;
  constexpr int P = kTile / G;
  constexpr int U = NM_T > 0 ? 4 : 1;  // elements in flight per group
  constexpr int COLS = MAXIT * LPG * VEC;
  constexpr int RC = (COLS + 31) / 32;
  using SP = SmemPlan<CW4, EMB_T>;

  const int nm = NM_T > 0 ? NM_T : a.nmodes;
  const int cw4 = NM_T > 0 ? CW4 : crd_words(a.nmodes) / 4;
  const bool emb = NM_T > 0 ? EMB_T : value_embedded(a.nmodes);
  const int mode = a.mode;
  const int R = a.rank;

  extern __shared__ __align__(16) unsigned char smem[];
  int4 *s_rec = reinterpret_cast<int4 *>(smem);
  float *s_val = reinterpret_cast<float *>(smem + SP::rec_bytes);
  unsigned char *s_union = smem + SP::rec_bytes + SP::val_bytes;
  auto &sort_tmp = *reinterpret_cast<typename BlockSort::TempStorage *>(s_union);
  uint32_t *s_key = reinterpret_cast<uint32_t *>(s_union);
  uint16_t *s_idx = reinterpret_cast<uint16_t *>(s_union + sizeof(uint32_t) * kTile);
  int *s_nv = reinterpret_cast<int *>(smem + SP::fixed_bytes - 16);
  int *s_bnd_row = reinterpret_cast<int *>(smem + SP::fixed_bytes);
  float *s_bnd = reinterpret_cast<float *>(smem + SP::fixed_bytes + 2 * G * sizeof(int));
  float *s_acc = reinterpret_cast<float *>(smem + SP::fixed_bytes + 2 * G * sizeof(int) +
                                           (size_t)2 * G * R * sizeof(float));

  const int tid = threadIdx.x;
  const int64_t chunk = blockIdx.x;
  const int64_t start = a.chunk_start[chunk];
  const int64_t end = a.chunk_start[chunk + 1];
  const int64_t ss = a.chunk_ss[chunk];
  const int part = a.chunk_part[chunk];
  const int64_t row0 = ss * a.m;
  const int rows = chunk_row_count(a, chunk, row0);
  const int key_bits = bit_length_u64((uint64_t)rows);  // room for the sentinel `rows`

  float *acc_base;
  if constexpr (SMEM_ACC) {
    acc_base = s_acc;
    for (int i = tid; i < rows * R; i += kBlock) s_acc[i] = 0.f;
  } else {
    acc_base = a.out + row0 * R;
  }
  if (tid < 2) s_nv[tid] = 0;
  __syncthreads();

  const int gi = tid / LPG;
  const int lg = tid % LPG;
  const int warp = tid >> 5, lane = tid & 31;

  int tile_no = 0;
  for (int64_t t0 = start; t0 < end; t0 += kTile, ++tile_no) {
    const int cnt = (int)min64(kTile, end - t0);
    // ---------------------------------------------------------------- A
    uint32_t keys[kIPT];
    uint16_t vals16[kIPT];
    int4 r0[kIPT], r1[kIPT];
    float rv[kIPT];
    uint32_t slot[kIPT];
#pragma unroll
    for (int j = 0; j < kIPT; ++j) {
      const int e = j * kBlock + tid;
      if (e < cnt) {
        const int64_t i = t0 + e;
        r0[j] = ld_stream_v4(a.src + i * cw4);
        if (CW4 == 2 && cw4 == 2) r1[j] = ld_stream_v4(a.src + i * cw4 + 1);
        else r1[j] = make_int4(0, 0, 0, 0);
        rv[j] = emb ? 0.f : ld_stream_f32(a.src_val + i);
        if (a.do_remap) slot[j] = ld_stream_u32(a.slots + i);
      }
    }
    int nvalid_local = 0;
#pragma unroll
    for (int j = 0; j < kIPT; ++j) {
      const int e = j * kBlock + tid;
      keys[j] = (uint32_t)rows;
      vals16[j] = (uint16_t)e;
      if (e < cnt) {
        if (a.do_remap) {
          // general kernel (N >= 5, R > 64): peer test at run time
          const bool two = CW4 == 2 && cw4 == 2;
          if (a.peers.n > 0) {
            if (two && emb) remap_store<2, true, true>(a, slot[j], r0[j], r1[j], 0.f);
            else if (two) remap_store<2, false, true>(a, slot[j], r0[j], r1[j], rv[j]);
            else if (emb) remap_store<1, true, true>(a, slot[j], r0[j], r1[j], 0.f);
            else remap_store<1, false, true>(a, slot[j], r0[j], r1[j], rv[j]);
          } else {
            if (two && emb) remap_store<2, true>(a, slot[j], r0[j], r1[j], 0.f);
            else if (two) remap_store<2, false>(a, slot[j], r0[j], r1[j], rv[j]);
            else if (emb) remap_store<1, true>(a, slot[j], r0[j], r1[j], 0.f);
            else remap_store<1, false>(a, slot[j], r0[j], r1[j], rv[j]);
          }
        }
        s_rec[e * CW4] = r0[j];
        if (CW4 == 2) s_rec[e * CW4 + 1] = r1[j];
        if (!EMB_T) s_val[e] = rv[j];
        const int64_t lr = (int64_t)word_of(r0[j], r1[j], mode) - row0;
        if (lr >= 0 && lr < rows) {
          keys[j] = (uint32_t)lr;
          ++nvalid_local;
        } else {
          atomicOr(a.flags, FC_FLAG_ROW_OUTSIDE_SS);
        }
      }
    }
    if (nvalid_local) atomicAdd(&s_nv[tile_no & 1], nvalid_local);
    // ---------------------------------------------------------------- B
    BlockSort(sort_tmp).Sort(keys, vals16, 0, key_bits);
    __syncthreads();  // sort temp storage aliases s_key / s_idx
#pragma unroll
    for (int j = 0; j < kIPT; ++j) {
      s_key[tid * kIPT + j] = keys[j];
      s_idx[tid * kIPT + j] = vals16[j];
    }
    __syncthreads();
    const int nvalid = s_nv[tile_no & 1];
    // ---------------------------------------------------------------- C
    if (lg == 0) {
      s_bnd_row[2 * gi] = -1;
      s_bnd_row[2 * gi + 1] = -1;
    }
    if (tid == 0) s_nv[(tile_no + 1) & 1] = 0;
    const int pb = gi * P;
    const int pe = min(pb + P, nvalid);
    if (pb < nvalid) {
      int cur = (int)s_key[pb];
      bool head = pb > 0 && (int)s_key[pb - 1] == cur;
      float acc[MAXIT][VEC];
#pragma unroll
      for (int it = 0; it < MAXIT; ++it)
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[it][v] = 0.f;

      auto flush = [&](int row, bool as_head) {
        if (as_head) {
          if (lg == 0) s_bnd_row[2 * gi] = row;
#pragma unroll
          for (int it = 0; it < MAXIT; ++it) {
            const int col = it * LPG * VEC + lg * VEC;
            if (col < R) VecT<VEC>::store(s_bnd + (2 * gi) * R + col, acc[it]);
          }
        } else {
#pragma unroll
          for (int it = 0; it < MAXIT; ++it) {
            const int col = it * LPG * VEC + lg * VEC;
            if (col < R) {
              float *p = acc_base + (int64_t)row * R + col;
              float o[VEC];
              VecT<VEC>::load(p, o);
#pragma unroll
              for (int v = 0; v < VEC; ++v) o[v] += acc[it][v];
              VecT<VEC>::store(p, o);
            }
          }
        }
      };

      for (int p = pb; p < pe; p += U) {
        int rowu[U];
        float vu[U];
        int cu[U][NMAX];
        bool oku[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int pp = p + u;
          oku[u] = pp < pe;
          const int e = s_idx[oku[u] ? pp : pb];
          rowu[u] = oku[u] ? (int)s_key[pp] : -1;
          const int4 q0 = s_rec[e * CW4];
          const int4 q1 = CW4 == 2 ? s_rec[e * CW4 + 1] : make_int4(0, 0, 0, 0);
#pragma unroll
          for (int w = 0; w < NMAX; ++w) cu[u][w] = word_of(q0, q1, w);
          vu[u] = emb ? __int_as_float(word_of(q0, q1, cw4 * 4 - 1)) : s_val[e];
        }
        float pr[U][MAXIT][VEC];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int it = 0; it < MAXIT; ++it)
#pragma unroll
            for (int v = 0; v < VEC; ++v) pr[u][it][v] = 1.f;
#pragma unroll
        for (int w = 0; w < NMAX; ++w) {
          if (w >= nm || w == mode) continue;
          const float *F = a.fac[w];
#pragma unroll
          for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int it = 0; it < MAXIT; ++it) {
              const int col = it * LPG * VEC + lg * VEC;
              if (oku[u] && col < R) {
                float f[VEC];
                VecT<VEC>::load_ro(F + (int64_t)cu[u][w] * R + col, f);
#pragma unroll
                for (int v = 0; v < VEC; ++v) pr[u][it][v] *= f[v];
              }
            }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (!oku[u]) break;
          if (rowu[u] != cur) {
            flush(cur, head);
            head = false;
            cur = rowu[u];
#pragma unroll
            for (int it = 0; it < MAXIT; ++it)
#pragma unroll
              for (int v = 0; v < VEC; ++v) acc[it][v] = 0.f;
          }
#pragma unroll
          for (int it = 0; it < MAXIT; ++it)
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[it][v] += vu[u] * pr[u][it][v];
        }
      }
      const bool tail = pe < nvalid && (int)s_key[pe] == cur;
      if (tail && !head) {
        if (lg == 0) s_bnd_row[2 * gi + 1] = cur;
#pragma unroll
        for (int it = 0; it < MAXIT; ++it) {
          const int col = it * LPG * VEC + lg * VEC;
          if (col < R) VecT<VEC>::store(s_bnd + (2 * gi + 1) * R + col, acc[it]);
        }
      } else {
        flush(cur, head);
      }
    }
    __syncthreads();
    // ---------------------------------------------------------------- D
    if (warp == 0) {
      float run[RC];
#pragma unroll
      for (int q = 0; q < RC; ++q) run[q] = 0.f;
      int curr = -1;
      for (int ent = 0; ent < 2 * G; ++ent) {
        const int row = s_bnd_row[ent];
        if (row < 0) continue;
        if (row != curr) {
          if (curr >= 0) {
#pragma unroll
            for (int q = 0; q < RC; ++q) {
              const int col = q * 32 + lane;
              if (col < R) acc_base[(int64_t)curr * R + col] += run[q];
              run[q] = 0.f;
            }
          }
          curr = row;
        }
#pragma unroll
        for (int q = 0; q < RC; ++q) {
          const int col = q * 32 + lane;
          if (col < R) run[q] += s_bnd[ent * R + col];
        }
      }
      if (curr >= 0) {
#pragma unroll
        for (int q = 0; q < RC; ++q) {
          const int col = q * 32 + lane;
          if (col < R) acc_base[(int64_t)curr * R + col] += run[q];
        }
      }
    }
  }
  __syncthreads();
  if constexpr (SMEM_ACC) {
    float *dstp = part < 0 ? a.out + row0 * R : partial_ws(a, chunk) + (int64_t)part * a.m * R;
    const int n = rows * R;
    if ((R & 3) == 0) {
      const float4 *s4 = reinterpret_cast<const float4 *>(s_acc);
      float4 *d4 = reinterpret_cast<float4 *>(dstp);
      for (int i = tid; i < n / 4; i += kBlock) d4[i] = s4[i];
    } else {
      for (int i = tid; i < n; i += kBlock) dstp[i] = s_acc[i];
    }
  }
  if (tid == 0) atomicAdd(a.counters, (unsigned long long)(end - start));
}


// K2: deterministic two-level reduce of partial tiles.  Level 1: task t
// sums partials [p0, p1) of super-shard ss (<= kReduceFan of them) in chunk
// order into out rows (dst < 0) or level-2 slot dst; level 2 sums a
// super-shard's level-1 slots in order into out.  Thread per (row, column).
__global__ void __launch_bounds__(256) reduce_level_kernel(const int64_t *tasks, int stride,
                                                           const float *src, float *slots,
                                                           float *out, int64_t out_rows, int64_t m,
                                                           int rank) {
  const int64_t t = blockIdx.x;
  const int64_t ss = tasks[t * stride];
  const int64_t p0 = tasks[t * stride + 1], p1 = tasks[t * stride + 2];
  const int64_t dst = stride > 3 ? tasks[t * stride + 3] : -1;
  const int64_t row0 = ss * m;
  const int64_t rows = min64(m, out_rows - row0);
  const int64_t idx = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  if (idx >= rows * rank) return;
  const int64_t cells = m * rank;
  const float *p = src + p0 * cells + idx;
  float s = 0.f;
  int64_t q = p0;
  for (; q + 4 <= p1; q += 4, p += 4 * cells) {
    const float x0 = p[0], x1 = p[cells], x2 = p[2 * cells], x3 = p[3 * cells];
    s += x0;
    s += x1;
    s += x2;
    s += x3;
  }
  for (; q < p1; ++q, p += cells) s += *p;
  if (dst < 0) out[row0 * rank + idx] = s;
  else slots[dst * cells + idx] = s;
}

// Remap-only pass (split_remap second pass, engine.py:224) of n elements;
// also the receiver unpack of the NCCL exchange (fc_scatter_records).
template <int CW4, bool EMB>
__global__ void __launch_bounds__(256) remap_only_kernel(const __grid_constant__ ModeArgs a, int64_t n) {
  unsigned done = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t s = ld_stream_u32(a.slots + i);
    const int4 r0 = ld_stream_v4(a.src + i * CW4);
    const int4 r1 = CW4 == 2 ? ld_stream_v4(a.src + i * CW4 + 1) : r0;
    const float v = EMB ? 0.f : ld_stream_f32(a.src_val + i);
    if (a.peers.n > 0) remap_store<CW4, EMB, true>(a, s, r0, r1, v);
    else remap_store<CW4, EMB>(a, s, r0, r1, v);
    ++done;
  }
  done = __reduce_add_sync(0xffffffffu, done);
  if ((threadIdx.x & 31) == 0 && done) atomicAdd(a.counters, (unsigned long long)done);
}

// Cursor strategy (_kernels.py:73-80).
template <int CW4, bool EMB>
__global__ void __launch_bounds__(256) remap_cursor_kernel(const int4 *src, const float *src_val,
                                                           int4 *dst, float *dst_val,
                                                           const uint32_t *src_sid,
                                                           uint32_t *dst_sid, int nmodes,
                                                           int next_mode,
                                                           const int64_t *dest_base,
                                                           unsigned long long *cursors,
                                                           int64_t nnz, int32_t *flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t b = src_sid[i * nmodes + next_mode];
    const int64_t slot = dest_base[b] + (int64_t)atomicAdd(cursors + b, 1ull);
    if (slot >= dest_base[b + 1]) {
      atomicOr(flags, FC_FLAG_SHARD_OVERFLOW);
      continue;
    }
#pragma unroll
    for (int q = 0; q < CW4; ++q) dst[slot * CW4 + q] = src[i * CW4 + q];
    if (!EMB) dst_val[slot] = src_val[i];
    for (int q = 0; q < nmodes; ++q) dst_sid[slot * nmodes + q] = src_sid[i * nmodes + q];
  }
}

template <int NM_T, int VEC, int LPG, int MAXIT, bool SMEM_ACC>
int launch_mode_pass(const ModeArgs &a, int64_t nchunks, cudaStream_t st) {
  constexpr int CW4 = NM_T > 0 ? crd_words(NM_T) / 4 : 2;
  constexpr bool EMB_T = NM_T > 0 ? value_embedded(NM_T) : false;
  constexpr int G = kBlock / LPG;
  const int64_t acc_rows = SMEM_ACC ? a.m : 0;
  const size_t smem = SmemPlan<CW4, EMB_T>::total(G, a.rank, acc_rows);
  auto kern = mode_pass_kernel<NM_T, VEC, LPG, MAXIT, SMEM_ACC>;
  static size_t configured = 0;
  if (smem > configured) {
    FC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  if (nchunks > 0) {
    kern<<<(unsigned)nchunks, kBlock, smem, st>>>(a);
    FC_LAUNCH_CHECK();
  }
  return FC_OK;
}

// Fast path when the accumulator tile is in shared memory, m <= 256,
// N <= 4 and R % 4 == 0, R <= 64; the general kernel otherwise.
bool fast_ok(const ModeArgs &a, bool smem_acc) {
  return smem_acc && a.hist_rows <= kMaxBins && a.nmodes >= 2 && a.nmodes <= 4 && a.rank % 4 == 0 &&
         a.rank <= 64;
}

template <bool SMEM_ACC>
int dispatch(const ModeArgs &a, int64_t nchunks, cudaStream_t st) {
  const int R = a.rank;
  const int N = a.nmodes;
  if (fast_ok(a, SMEM_ACC)) {
    if (a.peers.n > 0) {
      if (N == 3) return fast_dispatch_peer_n3(a, nchunks, st);
      if (N == 4) return fast_dispatch_peer_n4(a, nchunks, st);
      return fast_dispatch_peer_n2(a, nchunks, st);
    }
    if (N == 3) return fast_dispatch_n3(a, nchunks, st);
    if (N == 4) return fast_dispatch_n4(a, nchunks, st);
    return fast_dispatch_n2(a, nchunks, st);
  }
  if (R % 4 == 0 && R <= 32 && N == 3) {
    if (R <= 16) return launch_mode_pass<3, 4, 4, 1, SMEM_ACC>(a, nchunks, st);
    return launch_mode_pass<3, 4, 8, 1, SMEM_ACC>(a, nchunks, st);
  }
  if (R % 4 == 0 && R <= 32 && R > 16 && N == 4) return launch_mode_pass<4, 4, 8, 1, SMEM_ACC>(a, nchunks, st);
  return launch_mode_pass<0, 1, 32, 8, SMEM_ACC>(a, nchunks, st);
}

}  // namespace

int64_t smem_acc_rows_max(int rank) { return rank > 0 ? kSmemAccBytes / (4 * (int64_t)rank) : 0; }

// read once, when the library is loaded (dispatch.cuh)
static KernelVariant variant_from_env() {
  KernelVariant v;
  const char *p = getenv("FLYCOO_PACK");
  const char *w = getenv("FLYCOO_PACK_WIDE");
  v.pack = !(p && strcmp(p, "0") == 0);
  v.pack_wide = !(w && strcmp(w, "0") == 0);
  return v;
}
static KernelVariant g_variant = variant_from_env();
KernelVariant &kernel_variant() { return g_variant; }

}  // namespace fc

using namespace fc;

extern "C" {

int64_t fc_smem_acc_rows_max(int rank) { return fc::smem_acc_rows_max(rank); }

int fc_set_kernel_variant(int pack, int pack_wide) {
  fc::kernel_variant().pack = pack != 0;
  fc::kernel_variant().pack_wide = pack_wide != 0;
  return FC_OK;
}
int fc_tile_elems(void) { return kTile; }

// Row capacity of a direct chunk (several whole super-shards in at most one
// tile, rows stored straight to `out`): the largest multiple of m within the
// 256 counting-sort bins on the fast path; m when merging is not supported.
int64_t fc_chunk_rows_max(int nmodes, int rank, int64_t m) {
  if (m < 1 || m > kMaxBins || nmodes < 2 || nmodes > 4 || rank % 4 != 0 || rank > 64 ||
      m > smem_acc_rows_max(rank))
    return m;
  return kMaxBins / m * m;
}

static int mode_worker_impl(const void *src_crd, const float *src_val, void *dst_crd,
                            float *dst_val, const float *const *factors, const int64_t *dims,
                            float *out, int nmodes, int mode, int rank, int64_t out_rows,
                            int64_t m_mode, const int64_t *chunk_start, const int32_t *chunk_ss,
                            const int32_t *chunk_part, const int32_t *chunk_rows,
                            int64_t tile_rows, int64_t hist_rows, int64_t nchunks,
                            const int64_t *red1, int64_t nred1, const int64_t *red2,
                            int64_t nred2, float *part_ws, float *part_ws2,
                            const uint32_t *dest_slots, int64_t nnz, int do_compute,
                            int do_remap, int acc_in_smem, int32_t *flags,
                            unsigned long long *counters, void *stream, const PeerTable &peers,
                            const int32_t *chunk_owner = nullptr, uint16_t *plan_perm = nullptr,
                            uint16_t *plan_bins = nullptr, int plan = 0) {
  FC_CHECK_ARG(nmodes >= 2 && nmodes <= 8, "nmodes %d outside [2, 8]", nmodes);
  FC_CHECK_ARG(mode >= 0 && mode < nmodes, "mode %d out of range", mode);
  FC_CHECK_ARG(src_crd && flags && counters, "null buffer");
  FC_CHECK_ARG(!do_remap || ((dst_crd || peers.n > 0) && (dest_slots || nnz == 0)),
               "remap needs dst and slots");
  FC_CHECK_ARG(value_embedded(nmodes) || (src_val && (!do_remap || dst_val || peers.n > 0)),
               "N=%d needs separate value arrays", nmodes);
  FC_CHECK_ARG(nnz >= 0 && nnz <= (int64_t)UINT32_MAX, "nnz %lld outside uint32 slots",
               (long long)nnz);
  cudaStream_t st = as_stream(stream);
  const int cw4 = crd_words(nmodes) / 4;
  const bool emb = value_embedded(nmodes);
  if (!do_compute) {
    if (!do_remap || nnz == 0) return FC_OK;
    const int grid = (int)min64((nnz + 255) / 256, 148 * 16);
    ModeArgs r{};
    r.src = static_cast<const int4 *>(src_crd);
    r.src_val = src_val;
    r.dst = static_cast<int4 *>(dst_crd);
    r.dst_val = dst_val;
    r.slots = dest_slots;
    r.nnz = nnz;
    r.flags = flags;
    r.counters = counters;
    r.peers = peers;
    if (cw4 == 1 && emb) remap_only_kernel<1, true><<<grid, 256, 0, st>>>(r, nnz);
    else if (cw4 == 1) remap_only_kernel<1, false><<<grid, 256, 0, st>>>(r, nnz);
    else if (emb) remap_only_kernel<2, true><<<grid, 256, 0, st>>>(r, nnz);
    else remap_only_kernel<2, false><<<grid, 256, 0, st>>>(r, nnz);
    FC_LAUNCH_CHECK();
    return FC_OK;
  }
  FC_CHECK_ARG(factors && out, "null factors/out");
  FC_CHECK_ARG(rank >= 1 && rank <= 256, "rank %d outside [1, 256]", rank);
  FC_CHECK_ARG(m_mode >= 1 && out_rows >= 1, "bad m/out_rows");
  FC_CHECK_ARG(nchunks >= 0 && nchunks < (1ll << 31), "bad chunk count");
  FC_CHECK_ARG(!acc_in_smem || m_mode <= smem_acc_rows_max(rank),
               "m=%lld too large for shared-memory accumulation at rank %d", (long long)m_mode, rank);
  FC_CHECK_ARG(m_mode < (1ll << 30), "interval width too large");
  FC_CHECK_ARG(!chunk_rows || (acc_in_smem && tile_rows >= m_mode && tile_rows <= kMaxBins &&
                               hist_rows <= fc_chunk_rows_max(nmodes, rank, m_mode)),
               "merged chunks need the fast path, tile_rows in [m, 256] and hist_rows <= "
               "fc_chunk_rows_max");
  ModeArgs a{};
  a.src = static_cast<const int4 *>(src_crd);
  a.src_val = src_val;
  a.dst = static_cast<int4 *>(dst_crd);
  a.dst_val = dst_val;
  for (int w = 0; w < nmodes; ++w) {
    FC_CHECK_ARG(w == mode || factors[w], "null factor %d", w);
    a.fac[w] = factors[w];
  }
  a.out = out;
  a.nmodes = nmodes;
  a.mode = mode;
  a.rank = rank;
  a.out_rows = out_rows;
  a.m = m_mode;
  a.chunk_start = chunk_start;
  a.chunk_ss = chunk_ss;
  a.chunk_part = chunk_part;
  a.chunk_rows = chunk_rows;
  a.tile_rows = chunk_rows ? tile_rows : m_mode;
  a.hist_rows = chunk_rows ? (hist_rows > a.tile_rows ? hist_rows : a.tile_rows) : m_mode;
  a.pack_shift = 0;
  if (dims && nmodes == 3) {
    for (int w = 0; w < nmodes; ++w)
      FC_CHECK_ARG(dims[w] >= 1 && dims[w] <= INT32_MAX, "dims[%d] out of range", w);
    const int w1 = mode == 0 ? 1 : 0, w2 = mode == 2 ? 1 : 2;
    const int b1 = bit_length_u64((uint64_t)(dims[w1] - 1));
    const int b2 = bit_length_u64((uint64_t)(dims[w2] - 1));
    if (b2 >= 1 && b1 + b2 <= 32) a.pack_shift = b2;
  }
  a.part_ws = part_ws;
  a.slots = dest_slots;
  a.nnz = nnz;
  a.do_remap = do_remap;
  a.flags = flags;
  a.counters = counters;
  a.peers = peers;
  a.chunk_owner = chunk_owner;
  a.plan_perm = plan_perm;
  a.plan_bins = plan_bins;
  a.plan = plan;
  if (plan) {
    FC_CHECK_ARG(plan_perm && plan_bins, "null tile plan");
    if (!acc_in_smem || !fast_ok(a, true) || (plan == 2 && peers.n > 0)) return FC_ERR_UNSUPPORTED;
  }
  int rc = acc_in_smem ? dispatch<true>(a, nchunks, st) : dispatch<false>(a, nchunks, st);
  if (rc != FC_OK) return rc;
  if (plan == 2) return FC_OK;  // plan emission: no sums to reduce
  if (acc_in_smem && nred1 > 0) {
    FC_CHECK_ARG(red1 && part_ws, "null reduce plan");
    const int64_t cells = m_mode * rank;
    const unsigned gy = (unsigned)((cells + 255) / 256);
    FC_CHECK_ARG(gy < 65536, "super-shard tile too large for the reduce grid");
    reduce_level_kernel<<<dim3((unsigned)nred1, gy), 256, 0, st>>>(red1, 4, part_ws, part_ws2, out,
                                                                   out_rows, m_mode, rank);
    FC_LAUNCH_CHECK();
    if (nred2 > 0) {
      FC_CHECK_ARG(red2 && part_ws2, "null level-2 reduce plan");
      reduce_level_kernel<<<dim3((unsigned)nred2, gy), 256, 0, st>>>(red2, 3, part_ws2, nullptr, out,
                                                                     out_rows, m_mode, rank);
      FC_LAUNCH_CHECK();
    }
  }
  return FC_OK;
}

int fc_mode_worker(const void *src_crd, const float *src_val, void *dst_crd, float *dst_val,
                   const float *const *factors, const int64_t *dims, float *out, int nmodes,
                   int mode, int rank, int64_t out_rows, int64_t m_mode,
                   const int64_t *chunk_start, const int32_t *chunk_ss,
                   const int32_t *chunk_part, const int32_t *chunk_rows, int64_t tile_rows,
                   int64_t hist_rows, int64_t nchunks, const int64_t *red1, int64_t nred1,
                   const int64_t *red2, int64_t nred2, float *part_ws, float *part_ws2,
                   const uint32_t *dest_slots, int64_t nnz, int do_compute, int do_remap,
                   int acc_in_smem, int32_t *flags, unsigned long long *counters, void *stream) {
  PeerTable none{};
  return mode_worker_impl(src_crd, src_val, dst_crd, dst_val, factors, dims, out, nmodes, mode,
                          rank, out_rows, m_mode, chunk_start, chunk_ss, chunk_part, chunk_rows,
                          tile_rows, hist_rows, nchunks, red1, nred1, red2, nred2, part_ws,
                          part_ws2, dest_slots, nnz, do_compute, do_remap, acc_in_smem, flags,
                          counters, stream, none);
}

int fc_mode_worker_planned(const void *src_crd, const float *src_val, void *dst_crd, float *dst_val,
                           const float *const *factors, const int64_t *dims, float *out,
                           int nmodes, int mode, int rank, int64_t out_rows, int64_t m_mode,
                           const int64_t *chunk_start, const int32_t *chunk_ss,
                           const int32_t *chunk_part, const int32_t *chunk_rows,
                           int64_t tile_rows, int64_t hist_rows, int64_t nchunks,
                           const int64_t *red1, int64_t nred1, const int64_t *red2, int64_t nred2,
                           float *part_ws, float *part_ws2, const uint32_t *dest_slots,
                           int64_t nnz, int do_remap, int32_t *flags,
                           unsigned long long *counters, const uint16_t *tile_perm,
                           const uint16_t *tile_bins, void *stream) {
  PeerTable none{};
  return mode_worker_impl(src_crd, src_val, dst_crd, dst_val, factors, dims, out, nmodes, mode,
                          rank, out_rows, m_mode, chunk_start, chunk_ss, chunk_part, chunk_rows,
                          tile_rows, hist_rows, nchunks, red1, nred1, red2, nred2, part_ws,
                          part_ws2, dest_slots, nnz, 1, do_remap, 1, flags, counters, stream, none,
                          nullptr, const_cast<uint16_t *>(tile_perm),
                          const_cast<uint16_t *>(tile_bins), 1);
}

int fc_tile_plan_emit(const void *src_crd, const float *src_val, const float *const *factors,
                      const int64_t *dims, int nmodes, int mode, int rank, int64_t out_rows,
                      int64_t m_mode, const int64_t *chunk_start, const int32_t *chunk_ss,
                      const int32_t *chunk_part, const int32_t *chunk_rows, int64_t tile_rows,
                      int64_t hist_rows, int64_t nchunks, int64_t nnz, int32_t *flags,
                      unsigned long long *counters, uint16_t *tile_perm, uint16_t *tile_bins,
                      void *stream) {
  PeerTable none{};
  // `out` is never written by the emission pass; any non-null pointer passes the checks
  return mode_worker_impl(src_crd, src_val, nullptr, nullptr, factors, dims,
                          reinterpret_cast<float *>(tile_perm), nmodes, mode, rank, out_rows,
                          m_mode, chunk_start, chunk_ss, chunk_part, chunk_rows, tile_rows,
                          hist_rows, nchunks, nullptr, 0, nullptr, 0, nullptr, nullptr, nullptr,
                          nnz, 1, 0, 1, flags, counters, stream, none, nullptr, tile_perm,
                          tile_bins, 2);
}

int64_t fc_tile_plan_keys(int64_t nnz, int64_t nchunks) { return nnz / kTile + nchunks + 2; }

int fc_mode_worker_peers(const void *src_crd, const float *src_val, const float *const *factors,
                         const int64_t *dims, float *out, int nmodes, int mode, int rank,
                         int64_t out_rows, int64_t m_mode, const int64_t *chunk_start,
                         const int32_t *chunk_ss, const int32_t *chunk_part,
                         const int32_t *chunk_rows, int64_t tile_rows, int64_t hist_rows,
                         int64_t nchunks, const int64_t *red1, int64_t nred1,
                         const int64_t *red2, int64_t nred2, float *part_ws, float *part_ws2,
                         const uint32_t *dest_slots, int64_t nnz, int do_compute,
                         int acc_in_smem, int32_t *flags, unsigned long long *counters,
                         int npeers, void *const *peer_crd, float *const *peer_val,
                         const int64_t *peer_base, float *const *peer_part_ws,
                         const int32_t *chunk_owner, void *stream) {
  return fc_mode_worker_peers_planned(src_crd, src_val, factors, dims, out, nmodes, mode, rank,
                                      out_rows, m_mode, chunk_start, chunk_ss, chunk_part,
                                      chunk_rows, tile_rows, hist_rows, nchunks, red1, nred1, red2,
                                      nred2, part_ws, part_ws2, dest_slots, nnz, do_compute,
                                      acc_in_smem, flags, counters, npeers, peer_crd, peer_val,
                                      peer_base, peer_part_ws, chunk_owner, nullptr, nullptr,
                                      stream);
}

int fc_mode_worker_peers_planned(const void *src_crd, const float *src_val,
                                 const float *const *factors, const int64_t *dims, float *out,
                                 int nmodes, int mode, int rank, int64_t out_rows, int64_t m_mode,
                                 const int64_t *chunk_start, const int32_t *chunk_ss,
                                 const int32_t *chunk_part, const int32_t *chunk_rows,
                                 int64_t tile_rows, int64_t hist_rows, int64_t nchunks,
                                 const int64_t *red1, int64_t nred1, const int64_t *red2,
                                 int64_t nred2, float *part_ws, float *part_ws2,
                                 const uint32_t *dest_slots, int64_t nnz, int do_compute,
                                 int acc_in_smem, int32_t *flags, unsigned long long *counters,
                                 int npeers, void *const *peer_crd, float *const *peer_val,
                                 const int64_t *peer_base, float *const *peer_part_ws,
                                 const int32_t *chunk_owner, const uint16_t *tile_perm,
                                 const uint16_t *tile_bins, void *stream) {
  FC_CHECK_ARG(npeers >= 1 && npeers <= kMaxPeers, "npeers %d outside [1, %d]", npeers, kMaxPeers);
  FC_CHECK_ARG(peer_crd && peer_base && (dest_slots || nnz == 0), "null peer table");
  PeerTable t{};
  t.n = npeers;
  FC_CHECK_ARG(peer_base[0] == 0, "peer_base[0] must be 0");
  for (int q = 0; q < npeers; ++q) {
    FC_CHECK_ARG(peer_crd[q], "null peer buffer %d", q);
    FC_CHECK_ARG(value_embedded(nmodes) || (peer_val && peer_val[q]), "null peer values %d", q);
    FC_CHECK_ARG(peer_base[q + 1] >= peer_base[q], "peer_base not monotone");
    t.crd[q] = static_cast<int4 *>(peer_crd[q]);
    t.val[q] = value_embedded(nmodes) ? nullptr : peer_val[q];
    t.base[q] = peer_base[q];
  }
  t.base[npeers] = peer_base[npeers];
  FC_CHECK_ARG(!chunk_owner || peer_part_ws, "chunk owners need the peers' partial workspaces");
  if (peer_part_ws)
    for (int q = 0; q < npeers; ++q) t.part_ws[q] = peer_part_ws[q];
  for (int q = npeers + 1; q <= kMaxPeers; ++q) t.base[q] = t.base[npeers];
  FC_CHECK_ARG(t.base[npeers] <= (int64_t)UINT32_MAX + 1, "global slots exceed uint32");
  return mode_worker_impl(src_crd, src_val, nullptr, nullptr, factors, dims, out, nmodes, mode,
                          rank, out_rows, m_mode, chunk_start, chunk_ss, chunk_part, chunk_rows,
                          tile_rows, hist_rows, nchunks, red1, nred1, red2, nred2, part_ws,
                          part_ws2, dest_slots, nnz, do_compute, 1, acc_in_smem, flags, counters,
                          stream, t, chunk_owner, const_cast<uint16_t *>(tile_perm),
                          const_cast<uint16_t *>(tile_bins), tile_perm && do_compute ? 1 : 0);
}

int fc_reduce_partials(const int64_t *red1, int64_t nred1, const int64_t *red2, int64_t nred2,
                       const float *part_ws, float *part_ws2, float *out, int64_t out_rows,
                       int64_t m_mode, int rank, void *stream) {
  FC_CHECK_ARG(rank >= 1 && rank <= 256, "rank %d outside [1, 256]", rank);
  FC_CHECK_ARG(m_mode >= 1 && out_rows >= 1 && out, "bad output geometry");
  cudaStream_t st = as_stream(stream);
  const int64_t cells = m_mode * rank;
  const unsigned gy = (unsigned)((cells + 255) / 256);
  FC_CHECK_ARG(gy < 65536, "super-shard tile too large for the reduce grid");
  if (nred1 > 0) {
    FC_CHECK_ARG(red1 && part_ws, "null reduce plan");
    reduce_level_kernel<<<dim3((unsigned)nred1, gy), 256, 0, st>>>(red1, 4, part_ws, part_ws2, out,
                                                                   out_rows, m_mode, rank);
    FC_LAUNCH_CHECK();
  }
  if (nred2 > 0) {
    FC_CHECK_ARG(red2 && part_ws2, "null level-2 reduce plan");
    reduce_level_kernel<<<dim3((unsigned)nred2, gy), 256, 0, st>>>(red2, 3, part_ws2, nullptr, out,
                                                                   out_rows, m_mode, rank);
    FC_LAUNCH_CHECK();
  }
  return FC_OK;
}

int fc_remap_cursor(const void *src_crd, const float *src_val, void *dst_crd, float *dst_val,
                    const uint32_t *src_sid, uint32_t *dst_sid, int nmodes, int next_mode,
                    int64_t nnz, const int64_t *dest_base, unsigned long long *cursors,
                    int32_t *flags, void *stream) {
  FC_CHECK_ARG(nmodes >= 2 && nmodes <= 8, "nmodes %d outside [2, 8]", nmodes);
  FC_CHECK_ARG(next_mode >= 0 && next_mode < nmodes, "next_mode %d", next_mode);
  FC_CHECK_ARG(src_crd && dst_crd && src_sid && dst_sid && dest_base && cursors && flags,
               "null buffer");
  const int cw4 = crd_words(nmodes) / 4;
  const bool emb = value_embedded(nmodes);
  FC_CHECK_ARG(emb || (src_val && dst_val), "N=%d needs value arrays", nmodes);
  if (nnz == 0) return FC_OK;
  cudaStream_t st = as_stream(stream);
  const int grid = (int)min64((nnz + 255) / 256, 148 * 16);
  auto s4 = static_cast<const int4 *>(src_crd);
  auto d4 = static_cast<int4 *>(dst_crd);
#define FC_CURSOR(CW, E)                                                                    \
  remap_cursor_kernel<CW, E><<<grid, 256, 0, st>>>(s4, src_val, d4, dst_val, src_sid, dst_sid, \
                                                   nmodes, next_mode, dest_base, cursors, nnz, flags)
  if (cw4 == 1 && emb) FC_CURSOR(1, true);
  else if (cw4 == 1) FC_CURSOR(1, false);
  else if (emb) FC_CURSOR(2, true);
  else FC_CURSOR(2, false);
#undef FC_CURSOR
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_scatter_records(const void *src_crd, const float *src_val, int64_t n, void *dst_crd,
                       float *dst_val, int64_t dst_capacity, const uint32_t *slots, int nmodes,
                       int32_t *flags, unsigned long long *counters, void *stream) {
  FC_CHECK_ARG(nmodes >= 2 && nmodes <= 8, "nmodes %d outside [2, 8]", nmodes);
  FC_CHECK_ARG(n == 0 || (src_crd && dst_crd && slots && flags && counters), "null buffer");
  const int cw4 = crd_words(nmodes) / 4;
  const bool emb = value_embedded(nmodes);
  FC_CHECK_ARG(emb || n == 0 || (src_val && dst_val), "N=%d needs value arrays", nmodes);
  if (n == 0) return FC_OK;
  cudaStream_t st = as_stream(stream);
  const int grid = (int)min64((n + 255) / 256, 148 * 16);
  ModeArgs r{};
  r.src = static_cast<const int4 *>(src_crd);
  r.src_val = src_val;
  r.dst = static_cast<int4 *>(dst_crd);
  r.dst_val = dst_val;
  r.slots = slots;
  r.nnz = dst_capacity;
  r.flags = flags;
  r.counters = counters;
  if (cw4 == 1 && emb) remap_only_kernel<1, true><<<grid, 256, 0, st>>>(r, n);
  else if (cw4 == 1) remap_only_kernel<1, false><<<grid, 256, 0, st>>>(r, n);
  else if (emb) remap_only_kernel<2, true><<<grid, 256, 0, st>>>(r, n);
  else remap_only_kernel<2, false><<<grid, 256, 0, st>>>(r, n);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

}  // extern "C"
