// Fast-path mode pass (K1), specialised on (N, mode, R): see mode_pass.cu for
// the phase structure (A load+remap, B stable row sort, C piece-wise
// gather/Hadamard/segment reduce, D boundary fold).  Requirements: the
// super-shard's accumulator tile is in shared memory, m <= kMaxBins rows,
// N <= 4 (one 16-B coordinate word per record), R % 4 == 0, R <= 64.
//
// Sort: a stable counting sort of each tile by output row.  Warp w ranks
// its items with __match_any_sync (order: warp, item, lane); bases per
// (row, warp) come from one block scan; records are scattered straight into
// a sorted tile padded by one record per piece so that the 4 (or 8) groups of
// a warp read their pieces without bank conflicts.
#pragma once

#include "mode_args.cuh"

#ifndef FAST_MIN_BLOCKS
#define FAST_MIN_BLOCKS 3
#endif

namespace fc {

template <int NM, int LPG>
struct FastPlan {
  static constexpr int G = kBlock / LPG;
  static constexpr int P = kTile / G;
  static constexpr bool EMB = value_embedded(NM);
  static constexpr size_t sorted_bytes = sizeof(int4) * (kTile + G);
  static constexpr size_t sval_bytes = EMB ? 0 : sizeof(float) * (kTile + G);
  static constexpr size_t misc_bytes = 64;
  static constexpr size_t fixed_bytes = sorted_bytes + sval_bytes + misc_bytes;
  // dynamic tail: per-warp row histograms (m ints each), boundary entries,
  // the m x R accumulator tile
  __host__ __device__ static size_t hist_bytes(int64_t m) { return sizeof(int) * kWarps * ((m + 3) / 4 * 4); }
  static size_t total(int rank, int64_t m) {
    return fixed_bytes + hist_bytes(m) + (size_t)2 * G * sizeof(int) +
           (size_t)2 * G * rank * sizeof(float) + (size_t)m * rank * sizeof(float);
  }
};

template <int W>
__device__ __forceinline__ int comp(const int4 &q) {
  static_assert(W >= 0 && W < 4, "one coordinate word per record on the fast path");
  return W == 0 ? q.x : W == 1 ? q.y : W == 2 ? q.z : q.w;
}

template <int W>
__device__ __forceinline__ void set_comp(int4 &q, int v) {
  if (W == 0) q.x = v;
  else if (W == 1) q.y = v;
  else if (W == 2) q.z = v;
  else q.w = v;
}

// Gather the N-1 factor row slices of one element: pr = prod_{w != mode} F_w[c_w, col:col+4].
template <int NM, int MODE, int RT>
__device__ __forceinline__ void element_prod(const ModeArgs &a, int R, int col, const int4 &q,
                                             float (&pr)[4]) {
  bool first = true;
#pragma unroll
  for (int w = 0; w < NM; ++w) {
    if (w == MODE) continue;
    const int c = w == 0 ? q.x : w == 1 ? q.y : w == 2 ? q.z : q.w;
    const float *F = a.fac[w] + (uint64_t)(uint32_t)c * (uint32_t)(RT > 0 ? RT : R) + col;
    const float4 f = __ldg(reinterpret_cast<const float4 *>(F));
    if (first) {
      pr[0] = f.x; pr[1] = f.y; pr[2] = f.z; pr[3] = f.w;
      first = false;
    } else {
      pr[0] *= f.x; pr[1] *= f.y; pr[2] *= f.z; pr[3] *= f.w;
    }
  }
}

// Reference-compatible name used by the pipeline kernel: t = v * prod.
template <int NM, int MODE, int RT>
__device__ __forceinline__ void element_term(const ModeArgs &a, int R, int col, const int4 &q,
                                             float v, float (&t)[4]) {
  float pr[4];
  element_prod<NM, MODE, RT>(a, R, col, q, pr);
#pragma unroll
  for (int k = 0; k < 4; ++k) t[k] = v * pr[k];
}

template <int NM, int MODE, int LPG, int RT>
__global__ void __launch_bounds__(kBlock, FAST_MIN_BLOCKS) mode_pass_fast_kernel(const ModeArgs a) {
  using FP = FastPlan<NM, LPG>;
  constexpr int G = FP::G;
  constexpr int P = FP::P;
  constexpr bool EMB = FP::EMB;
  constexpr int U = 4;
  const int R = RT > 0 ? RT : a.rank;

  extern __shared__ __align__(16) unsigned char smem[];
  const int hstride = (int)((a.m + 3) / 4 * 4);
  int4 *s_sorted = reinterpret_cast<int4 *>(smem);
  float *s_sval = reinterpret_cast<float *>(smem + FP::sorted_bytes);
  int *s_misc = reinterpret_cast<int *>(smem + FP::sorted_bytes + FP::sval_bytes);
  unsigned char *tail = smem + FP::fixed_bytes;
  int *s_hist = reinterpret_cast<int *>(tail);
  tail += FP::hist_bytes(a.m);
  int *s_bnd_row = reinterpret_cast<int *>(tail);
  tail += 2 * G * sizeof(int);
  float *s_bnd = reinterpret_cast<float *>(tail);
  tail += (size_t)2 * G * R * sizeof(float);
  float *s_acc = reinterpret_cast<float *>(tail);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t chunk = blockIdx.x;
  const int64_t start = a.chunk_start[chunk];
  const int64_t end = a.chunk_start[chunk + 1];
  const int64_t ss = a.chunk_ss[chunk];
  const int part = a.chunk_part[chunk];
  const int64_t row0 = ss * a.m;
  const int rows = (int)min64(a.m, a.out_rows - row0);
  const int irow0 = (int)row0;

  for (int i = tid; i < rows * R; i += kBlock) s_acc[i] = 0.f;

  const int gi = tid / LPG;
  const int lg = tid % LPG;
  const int col = lg * 4;
  const bool col_ok = RT > 0 ? true : col < R;
  auto phys = [](int pos) { return pos + pos / P; };
  auto key_of = [&](const int4 &r) {
    const int lr = comp<MODE>(r) - irow0;
    return (lr >= 0 && lr < rows) ? lr : -1;
  };

  for (int64_t t0 = start; t0 < end; t0 += kTile) {
    const int cnt = (int)min64(kTile, end - t0);
    // ---------------------------------------------------------------- A
    int4 rec[kIPT];
    float rv[kIPT];
    uint32_t slot[kIPT];
#pragma unroll
    for (int j = 0; j < kIPT; ++j) {
      const int e = j * kBlock + tid;
      if (e < cnt) {
        const int64_t i = t0 + e;
        rec[j] = ld_stream_v4(a.src + i);
        if (!EMB) rv[j] = ld_stream_f32(a.src_val + i);
        if (a.do_remap) slot[j] = ld_stream_u32(a.slots + i);
      } else {
        rec[j] = make_int4(INT32_MIN, INT32_MIN, INT32_MIN, INT32_MIN);
      }
    }
    for (int b = lane; b < rows; b += 32) s_hist[warp * hstride + b] = 0;
#pragma unroll
    for (int j = 0; j < kIPT; ++j) {
      const int e = j * kBlock + tid;
      if (e < cnt) {
        if (a.do_remap) {
          const uint64_t s = slot[j];
          if (s < (uint64_t)a.nnz) {
            a.dst[s] = rec[j];
            if (!EMB) a.dst_val[s] = rv[j];
          } else {
            atomicOr(a.flags, FC_FLAG_SLOT_RANGE);
          }
        }
        if (key_of(rec[j]) < 0) atomicOr(a.flags, FC_FLAG_ROW_OUTSIDE_SS);
      }
    }
    __syncwarp();
    // ---------------------------------------------------------------- B
    // B1: warp-local ranks.  The rank is parked in the record's mode word
    // as (rank << 8 | local row) until B3 restores the coordinate -- keeps
    // the 8 ranks out of registers.
    int *wh = s_hist + warp * hstride;
#pragma unroll
    for (int j = 0; j < kIPT; ++j) {
      const int k = key_of(rec[j]);
      const unsigned grp = __match_any_sync(0xffffffffu, k >= 0 ? k : -1 - lane);
      int old = 0;
      if (k >= 0) old = wh[k];
      __syncwarp();
      if (k >= 0 && lane == __ffs(grp) - 1) wh[k] = old + __popc(grp);
      __syncwarp();
      set_comp<MODE>(rec[j], k >= 0 ? (((old + __popc(grp & lt_mask)) << 8) | k) : -1);
    }
    __syncthreads();
    {
      int tot = 0;
      int cw[kWarps];
      if (tid < rows) {
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
          cw[w] = s_hist[w * hstride + tid];
          tot += cw[w];
        }
      }
      int incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_misc[warp] = incl;
      __syncthreads();
      int wpre = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) wpre += w < warp ? s_misc[w] : 0;
      if (tid == kBlock - 1) s_misc[kWarps] = wpre + incl;
      if (tid < rows) {
        int base = wpre + incl - tot;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
          s_hist[w * hstride + tid] = base;
          base += cw[w];
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kIPT; ++j) {
      const int x = comp<MODE>(rec[j]);
      if (x >= 0) {
        const int k = x & 255;
        const int pos = wh[k] + (x >> 8);
        set_comp<MODE>(rec[j], irow0 + k);
        s_sorted[phys(pos)] = rec[j];
        if (!EMB) s_sval[phys(pos)] = rv[j];
      }
    }
    __syncthreads();
    const int nvalid = s_misc[kWarps];
    // ---------------------------------------------------------------- C
    if (lg == 0) {
      s_bnd_row[2 * gi] = -1;
      s_bnd_row[2 * gi + 1] = -1;
    }
    const int pb = gi * P;
    const int pe = min(pb + P, nvalid);
    if (pb < nvalid) {
      int cur = comp<MODE>(s_sorted[phys(pb)]);
      bool head = pb > 0 && comp<MODE>(s_sorted[phys(pb - 1)]) == cur;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      auto flush = [&]() {
        if (head) {
          if (lg == 0) s_bnd_row[2 * gi] = cur - irow0;
          if (col_ok) VecT<4>::store(s_bnd + (2 * gi) * R + col, acc);
        } else if (col_ok) {
          float *p = s_acc + (cur - irow0) * R + col;
          float o[4];
          VecT<4>::load(p, o);
#pragma unroll
          for (int v = 0; v < 4; ++v) o[v] += acc[v];
          VecT<4>::store(p, o);
        }
      };
      auto consume = [&](int row, float v, const float (&pr)[4]) {
        if (row != cur) {
          flush();
          head = false;
          cur = row;
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[k] = 0.f;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] = fmaf(v, pr[k], acc[k]);
      };
      // positions of one piece share the pad: phys(p) = p + gi for p in [pb, pb + P)
      const int4 *sp = s_sorted + gi;
      const float *svp = s_sval + gi;
      int p = pb;
      for (; p + U <= pe; p += U) {
        int4 q[U];
        float vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          q[u] = sp[p + u];
          vv[u] = EMB ? __int_as_float(q[u].w) : svp[p + u];
        }
        float pr[U][4];
        if (col_ok) {
#pragma unroll
          for (int u = 0; u < U; ++u) element_prod<NM, MODE, RT>(a, R, col, q[u], pr[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) consume(comp<MODE>(q[u]), vv[u], pr[u]);
      }
      for (; p < pe; ++p) {
        const int4 q = sp[p];
        const float vv = EMB ? __int_as_float(q.w) : svp[p];
        float pr[4];
        if (col_ok) element_prod<NM, MODE, RT>(a, R, col, q, pr);
        consume(comp<MODE>(q), vv, pr);
      }
      const bool tail = pe < nvalid && comp<MODE>(s_sorted[phys(pe)]) == cur;
      if (tail && !head) {
        if (lg == 0) s_bnd_row[2 * gi + 1] = cur - irow0;
        if (col_ok) VecT<4>::store(s_bnd + (2 * gi + 1) * R + col, acc);
      } else {
        flush();
      }
    }
    __syncthreads();
    // ---------------------------------------------------------------- D
    // Boundary entries are in sorted-row order (H0 T0 H1 T1 ...).  Warp w
    // folds every run of equal rows that *starts* in entries
    // [w * E, (w + 1) * E), in entry order -- same sums as one warp walking
    // all entries, spread over the CTA.
    {
      constexpr int E = (2 * G + kWarps - 1) / kWarps;
      constexpr int RC = (LPG * 4 + 31) / 32;
      int ent = warp * E;
      const int ent_end = min(2 * G, ent + E);
      int prev = -1;
      for (int e2 = ent - 1; e2 >= 0; --e2) {  // row of the last valid entry before my range
        const int r2 = s_bnd_row[e2];
        if (r2 >= 0) {
          prev = r2;
          break;
        }
      }
      while (ent < ent_end) {
        const int row = s_bnd_row[ent];
        if (row < 0 || row == prev) {  // invalid, or continues a run started earlier
          if (row >= 0) prev = row;
          ++ent;
          continue;
        }
        float run[RC];
#pragma unroll
        for (int q = 0; q < RC; ++q) run[q] = 0.f;
        int e3 = ent;
        for (; e3 < 2 * G; ++e3) {
          const int r3 = s_bnd_row[e3];
          if (r3 < 0) continue;
          if (r3 != row) break;
#pragma unroll
          for (int q = 0; q < RC; ++q) {
            const int c = q * 32 + lane;
            if (c < R) run[q] += s_bnd[e3 * R + c];
          }
        }
#pragma unroll
        for (int q = 0; q < RC; ++q) {
          const int c = q * 32 + lane;
          if (c < R) s_acc[row * R + c] += run[q];
        }
        prev = row;
        ent = e3;
      }
    }
  }
  __syncthreads();
  float *dstp = part < 0 ? a.out + row0 * R : a.part_ws + (int64_t)part * a.m * R;
  const int n4 = rows * R / 4;
  const float4 *s4 = reinterpret_cast<const float4 *>(s_acc);
  float4 *d4 = reinterpret_cast<float4 *>(dstp);
  for (int i = tid; i < n4; i += kBlock) d4[i] = s4[i];
  if (tid == 0) atomicAdd(a.counters, (unsigned long long)(end - start));
}

template <int NM, int MODE, int LPG, int RT>
int launch_fast(const ModeArgs &a, int64_t nchunks, cudaStream_t st) {
  const size_t smem = FastPlan<NM, LPG>::total(a.rank, a.m);
  auto kern = mode_pass_fast_kernel<NM, MODE, LPG, RT>;
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

}  // namespace fc
