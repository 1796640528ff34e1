// K1 v4: warp-independent mode pass.
//
// A CTA (4 warps) owns one chunk of one super-shard, like the tile kernel,
// but the warps never wait for each other inside the chunk: warp w takes
// the 256-element sub-tiles w, w+4, w+8, ... of the chunk and, per sub-tile,
//   A  streams its records + slots in (lane-consecutive 16-B loads), scatters
//      each record to its remap slot, forms the local output row;
//   B  stable counting sort by row inside the warp: __match_any_sync ranks in
//      (item, lane) order, a warp-level scan of the row histogram, records
//      written to the warp's padded sorted buffer (__syncwarp only);
//   C  its 4 groups of LPG lanes walk 64-element pieces: gather the N-1 factor
//      rows (read-only 16-B loads), FFMA into registers per equal-row segment,
//      interior segments added to the warp's PRIVATE accumulator tile;
//   D  the warp folds its 8 boundary entries in piece order.
// At the chunk's end (the only __syncthreads) the 4 warp tiles are summed in
// warp order and written to `out` (owned rows) or the chunk's partial slot.
// Element -> warp assignment and every summation order are fixed, so results
// are bitwise reproducible; no atomics on data.
#pragma once

#include "fast_kernel.cuh"

namespace fc {

constexpr int kWKWarps = 4;
constexpr int kWKThreads = 32 * kWKWarps;
constexpr int kWKItems = 8;                  // records per lane per sub-tile
constexpr int kWKSub = 32 * kWKItems;        // 256-element sub-tile per warp
constexpr int kWKPiece = 64;                 // elements per group piece (LPG = 8)

template <int NM, int LPG>
struct WarpPlan {
  static constexpr int G = 32 / LPG;         // groups per warp
  static constexpr int P = kWKSub / G;       // piece length
  static constexpr bool EMB = value_embedded(NM);
  static constexpr size_t sorted_bytes = sizeof(int4) * (kWKSub + G);
  static constexpr size_t sval_bytes = EMB ? 0 : sizeof(float) * (kWKSub + G);
  __host__ __device__ static constexpr size_t al16(size_t x) { return (x + 15) / 16 * 16; }
  __host__ __device__ static size_t hist_ints(int64_t m) { return (m + 31) / 32 * 32; }
  // byte offsets inside one warp's region (all 16-B aligned)
  __host__ __device__ static size_t off_hist() { return al16(sorted_bytes + sval_bytes); }
  __host__ __device__ static size_t off_brow(int64_t m) { return al16(off_hist() + 4 * hist_ints(m)); }
  __host__ __device__ static size_t off_bnd(int64_t m) { return al16(off_brow(m) + 8 * G); }
  __host__ __device__ static size_t off_acc(int rank, int64_t m) {
    return al16(off_bnd(m) + (size_t)8 * G * rank);
  }
  __host__ __device__ static size_t per_warp(int rank, int64_t m) {
    return al16(off_acc(rank, m) + (size_t)4 * m * rank);
  }
  static size_t total(int rank, int64_t m) { return kWKWarps * per_warp(rank, m); }
};

template <int NM, int MODE, int LPG, int RT>
__global__ void __launch_bounds__(kWKThreads, 4) mode_pass_warp_kernel(const __grid_constant__ ModeArgs a) {
  using WP = WarpPlan<NM, LPG>;
  constexpr int G = WP::G;
  constexpr int P = WP::P;
  constexpr bool EMB = WP::EMB;
  constexpr int U = 4;
  const int R = RT > 0 ? RT : a.rank;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const unsigned lt_mask = (1u << lane) - 1u;

  extern __shared__ __align__(16) unsigned char smem[];
  const size_t wbytes = WP::per_warp(R, a.tile_rows);
  auto warp_base = [&](int w) { return smem + w * wbytes; };
  unsigned char *base = warp_base(warp);
  int4 *s_sorted = reinterpret_cast<int4 *>(base);
  float *s_sval = reinterpret_cast<float *>(base + WP::sorted_bytes);
  int *s_hist = reinterpret_cast<int *>(base + WP::off_hist());
  int *s_bnd_row = reinterpret_cast<int *>(base + WP::off_brow(a.tile_rows));
  float *s_bnd = reinterpret_cast<float *>(base + WP::off_bnd(a.tile_rows));
  const size_t acc_off = WP::off_acc(R, a.tile_rows);
  float *s_acc = reinterpret_cast<float *>(base + acc_off);

  const int64_t chunk = blockIdx.x;
  const int64_t start = a.chunk_start[chunk];
  const int64_t end = a.chunk_start[chunk + 1];
  const int64_t ss = a.chunk_ss[chunk];
  const int part = a.chunk_part[chunk];
  const int64_t row0 = ss * a.m;
  const int rows = chunk_row_count(a, chunk, row0);
  const int irow0 = (int)row0;

  for (int i = lane; i < rows * R; i += 32) s_acc[i] = 0.f;

  const int gi = lane / LPG;
  const int lg = lane % LPG;
  const int col = lg * 4;
  const bool col_ok = RT > 0 ? true : col < R;
  const int nb = (rows + 31) / 32;  // histogram bins per lane (contiguous)
  auto key_of = [&](const int4 &r) {
    const int lr = comp<MODE>(r) - irow0;
    return (lr >= 0 && lr < rows) ? lr : -1;
  };

  for (int64_t t0 = start + (int64_t)warp * kWKSub; t0 < end; t0 += (int64_t)kWKWarps * kWKSub) {
    const int cnt = (int)min64(kWKSub, end - t0);
    // ---------------------------------------------------------------- A
    int4 rec[kWKItems];
    float rv[kWKItems];
    uint32_t slot[kWKItems];
#pragma unroll
    for (int j = 0; j < kWKItems; ++j) {
      const int e = j * 32 + lane;
      if (e < cnt) {
        const int64_t i = t0 + e;
        rec[j] = ld_stream_v4(a.src + i);
        if (!EMB) rv[j] = ld_stream_f32(a.src_val + i);
        if (a.do_remap) slot[j] = ld_stream_u32(a.slots + i);
      } else {
        rec[j] = make_int4(INT32_MIN, INT32_MIN, INT32_MIN, INT32_MIN);
      }
    }
    for (int b = lane; b < nb * 32; b += 32) s_hist[b] = 0;
#pragma unroll
    for (int j = 0; j < kWKItems; ++j) {
      const int e = j * 32 + lane;
      if (e < cnt) {
        if (a.do_remap) {
          remap_store<1, EMB>(a, slot[j], rec[j], rec[j], EMB ? 0.f : rv[j]);
        }
        if (key_of(rec[j]) < 0) atomicOr(a.flags, FC_FLAG_ROW_OUTSIDE_SS);
      }
    }
    __syncwarp();
    // ---------------------------------------------------------------- B
#pragma unroll
    for (int j = 0; j < kWKItems; ++j) {
      const int k = key_of(rec[j]);
      const unsigned grp = __match_any_sync(0xffffffffu, k >= 0 ? k : -1 - lane);
      int old = 0;
      if (k >= 0) old = s_hist[k];
      __syncwarp();
      if (k >= 0 && lane == __ffs(grp) - 1) s_hist[k] = old + __popc(grp);
      __syncwarp();
      set_comp<MODE>(rec[j], k >= 0 ? ((old + __popc(grp & lt_mask)) << 8) | k : -1);
    }
    // exclusive scan of the histogram: lane l owns bins [l*nb, (l+1)*nb)
    int nvalid;
    {
      int loc = 0;
      for (int q = 0; q < nb; ++q) loc += s_hist[lane * nb + q];
      int incl = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      nvalid = __shfl_sync(0xffffffffu, incl, 31);
      int run = incl - loc;
      __syncwarp();
      for (int q = 0; q < nb; ++q) {
        const int c = s_hist[lane * nb + q];
        s_hist[lane * nb + q] = run;
        run += c;
      }
      __syncwarp();
    }
#pragma unroll
    for (int j = 0; j < kWKItems; ++j) {
      const int x = comp<MODE>(rec[j]);
      if (x >= 0) {
        const int k = x & 255;
        const int pos = s_hist[k] + (x >> 8);
        set_comp<MODE>(rec[j], irow0 + k);
        s_sorted[pos + pos / P] = rec[j];
        if (!EMB) s_sval[pos + pos / P] = rv[j];
      }
    }
    if (lg == 0) {
      s_bnd_row[2 * gi] = -1;
      s_bnd_row[2 * gi + 1] = -1;
    }
    if (col_ok) {
      const float z[4] = {0.f, 0.f, 0.f, 0.f};
      VecT<4>::store(s_bnd + (2 * gi) * R + col, z);
      VecT<4>::store(s_bnd + (2 * gi + 1) * R + col, z);
    }
    __syncwarp();
    // ---------------------------------------------------------------- C
    const int pb = gi * P;
    const int pe = min(pb + P, nvalid);
    if (pb < nvalid) {
      const int4 *sp = s_sorted + gi;  // pad of piece gi
      const float *svp = s_sval + gi;
      int cur = comp<MODE>(sp[pb]);
      bool head = pb > 0 && comp<MODE>(s_sorted[pb - 1 + (pb - 1) / P]) == cur;
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
      const bool tail = pe < nvalid && comp<MODE>(s_sorted[pe + pe / P]) == cur;
      if (tail && !head) {
        if (lg == 0) s_bnd_row[2 * gi + 1] = cur - irow0;
        if (col_ok) VecT<4>::store(s_bnd + (2 * gi + 1) * R + col, acc);
      } else {
        flush();
      }
    }
    __syncwarp();
    // ---------------------------------------------------------------- D
    {
      constexpr int RC = (LPG * 4 + 31) / 32;
      int ent = 0;
      while (ent < 2 * G) {
        const int row = s_bnd_row[ent];
        if (row < 0) {
          ++ent;
          continue;
        }
        int e3 = ent + 1;
        while (e3 < 2 * G) {
          const int r3 = s_bnd_row[e3];
          if (r3 >= 0 && r3 != row) break;
          ++e3;
        }
#pragma unroll
        for (int q = 0; q < RC; ++q) {
          const int c = q * 32 + lane;
          if (c < R) {
            float run = 0.f;
            for (int e = ent; e < e3; ++e) run += s_bnd[e * R + c];
            s_acc[row * R + c] += run;
          }
        }
        ent = e3;
      }
    }
    __syncwarp();
  }
  __syncthreads();
  // sum the warp tiles in warp order, write the super-shard's rows
  float *dstp = part < 0 ? a.out + row0 * R : a.part_ws + (int64_t)part * a.m * R;
  const int n4 = rows * R / 4;
  for (int i = tid; i < n4; i += kWKThreads) {
    float4 s = reinterpret_cast<const float4 *>(warp_base(0) + acc_off)[i];
#pragma unroll
    for (int w = 1; w < kWKWarps; ++w) {
      const float4 t = reinterpret_cast<const float4 *>(warp_base(w) + acc_off)[i];
      s.x += t.x;
      s.y += t.y;
      s.z += t.z;
      s.w += t.w;
    }
    reinterpret_cast<float4 *>(dstp)[i] = s;
  }
  if (tid == 0) atomicAdd(a.counters, (unsigned long long)(end - start));
}

template <int NM, int MODE, int LPG, int RT>
int launch_warp(const ModeArgs &a, int64_t nchunks, cudaStream_t st) {
  const size_t smem = WarpPlan<NM, LPG>::total(a.rank, a.tile_rows);
  auto kern = mode_pass_warp_kernel<NM, MODE, LPG, RT>;
  static size_t configured = 0;
  if (smem > configured) {
    FC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  if (nchunks > 0) {
    kern<<<(unsigned)nchunks, kWKThreads, smem, st>>>(a);
    FC_LAUNCH_CHECK();
  }
  return FC_OK;
}

}  // namespace fc
