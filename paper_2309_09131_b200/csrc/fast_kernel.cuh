// Fast-path mode pass (K1), specialised on (N, mode, R): see mode_pass.cu for
// the phase structure (A load+remap, B stable row sort, C piece-wise
// gather/Hadamard/segment reduce, D boundary fold).  Requirements: the
// super-shard's accumulator tile is in shared memory, m <= kMaxBins rows,
// N <= 4 (one 16-B coordinate word per record), R % 4 == 0, R <= 64.
//
// Sort: a stable counting sort of each tile by output row.  Warp w ranks
// its items with __match_any_sync and one leader atomic per equal-row group
// (order: warp, item, lane); bases per
// (row, warp) come from one block scan; records are scattered straight into
// a sorted tile padded by one record per piece so that the 4 (or 8) groups of
// a warp read their pieces without bank conflicts.
#pragma once

#include "mode_args.cuh"

#ifndef FAST_MIN_BLOCKS
#define FAST_MIN_BLOCKS 3
#endif
#ifndef FAST_U
#define FAST_U 4
#endif
// 4-mode tensors gather three rows per element: 2 elements in flight per
// group keep the 80-register kernel spill-free (c3 19.21 -> 18.8 ms)
#ifndef FAST_U4
#define FAST_U4 2
#endif
#ifndef FAST_IPT
#define FAST_IPT 8
#endif

namespace fc {

#ifndef FAST_BLOCK
#define FAST_BLOCK 256
#endif
// fast-path tile: kFBlock threads x kFIPT records
constexpr int kFBlock = FAST_BLOCK;
constexpr int kFWarps = kFBlock / 32;
constexpr int kFIPT = FAST_IPT;
constexpr int kFTile = kFBlock * kFIPT;


template <int NM, int LPG>
struct FastPlan {
  static constexpr int G = kFBlock / LPG;
  static constexpr int P = kFTile / G;
  static constexpr bool EMB = value_embedded(NM);
  static constexpr size_t sorted_bytes = sizeof(int4) * (kFTile + G);
  static constexpr size_t sval_bytes = EMB ? 0 : sizeof(float) * (kFTile + G);
  static constexpr size_t misc_bytes = 4 * (kFWarps + 4);
  static constexpr size_t fixed_bytes = (sorted_bytes + sval_bytes + misc_bytes + 15) / 16 * 16;
  // dynamic tail: per-warp row histograms (m ints each), boundary entries,
  // the m x R accumulator tile
  __host__ __device__ static size_t hist_bytes(int64_t m) { return sizeof(int) * kFWarps * ((m + 3) / 4 * 4); }
  static size_t total(int rank, int64_t m, int64_t hist_rows = 0) {
    return fixed_bytes + hist_bytes(hist_rows > m ? hist_rows : m) + (size_t)2 * G * sizeof(int) +
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

// Factor bases of the N-1 input modes with the lane's column offset folded
// in, built once per tile so phase C does not re-derive them per element.
template <int NM, int MODE>
struct FacBases {
  const float *p[NM > 1 ? NM - 1 : 1];
  uint32_t stride;
  __device__ __forceinline__ FacBases(const ModeArgs &a, int R, int col) : stride((uint32_t)R) {
    int k = 0;
#pragma unroll
    for (int w = 0; w < NM; ++w) {
      if (w == MODE) continue;
      p[k++] = a.fac[w] + col;
    }
  }
};

template <int NM, int MODE>
__device__ __forceinline__ void element_prod(const FacBases<NM, MODE> &fb, const int4 &q,
                                             float (&pr)[4]) {
  int k = 0;
#pragma unroll
  for (int w = 0; w < NM; ++w) {
    if (w == MODE) continue;
    const int c = w == 0 ? q.x : w == 1 ? q.y : w == 2 ? q.z : q.w;
    const float4 f = __ldg(reinterpret_cast<const float4 *>(fb.p[k] + (uint64_t)(uint32_t)c * fb.stride));
    if (k == 0) {
      pr[0] = f.x; pr[1] = f.y; pr[2] = f.z; pr[3] = f.w;
    } else {
      pr[0] *= f.x; pr[1] *= f.y; pr[2] *= f.z; pr[3] *= f.w;
    }
    ++k;
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

// PLAN: 0 = rank every tile in the kernel; 1 = sorted positions (and, for
// direct chunks, bin starts) from the tile plan; 2 = rank and write the plan
// (nothing else) -- see pack_kernel.cuh.
template <int NM, int MODE, int LPG, int RT, bool PEER = false, int PLAN = 0>
__global__ void __launch_bounds__(kFBlock, FAST_MIN_BLOCKS) mode_pass_fast_kernel(const __grid_constant__ ModeArgs a) {
  using FP = FastPlan<NM, LPG>;
  constexpr int G = FP::G;
  constexpr int P = FP::P;
  constexpr bool EMB = FP::EMB;
  constexpr int U = NM >= 4 ? FAST_U4 : FAST_U;
  const int R = RT > 0 ? RT : a.rank;

  extern __shared__ __align__(16) unsigned char smem[];
  const int hstride = (int)((a.hist_rows + 3) / 4 * 4);
  const int hbits = 32 - __clz((int)(a.hist_rows > 1 ? a.hist_rows - 1 : 1));
  int4 *s_sorted = reinterpret_cast<int4 *>(smem);
  float *s_sval = reinterpret_cast<float *>(smem + FP::sorted_bytes);
  int *s_misc = reinterpret_cast<int *>(smem + FP::sorted_bytes + FP::sval_bytes);
  unsigned char *tail = smem + FP::fixed_bytes;
  int *s_hist = reinterpret_cast<int *>(tail);
  tail += FP::hist_bytes(a.hist_rows);
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
  const int rows = chunk_row_count(a, chunk, row0);
  const int irow0 = (int)row0;

  // direct chunk (part == -2): whole super-shards in <= one tile; every row is
  // complete inside the tile and is stored straight to `out` (no tile acc)
  const bool direct = part == kPartDirect;
  float *out_rows = a.out + row0 * R;
  if (PLAN == 2) {
    if (start == end) return;
  } else if (direct) {
    if (start == end) {  // only empty super-shards: their rows are zero
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int i = tid; i < rows * R / 4; i += kFBlock) reinterpret_cast<float4 *>(out_rows)[i] = z;
      return;
    }
  } else {
    for (int i = tid; i < rows * R; i += kFBlock) s_acc[i] = 0.f;
  }

  const int gi = tid / LPG;
  const int lg = tid % LPG;
  const int col = lg * 4;
  const bool col_ok = RT > 0 ? true : col < R;
  auto phys = [](int pos) { return pos + pos / P; };
  auto key_of = [&](const int4 &r) {
    const int lr = comp<MODE>(r) - irow0;
    return (lr >= 0 && lr < rows) ? lr : -1;
  };

  for (int64_t t0 = start; t0 < end; t0 += kFTile) {
    const int cnt = (int)min64(kFTile, end - t0);
    // ---------------------------------------------------------------- A
    int4 rec[kFIPT];
    float rv[kFIPT];
    uint32_t slot[kFIPT];
    // tile plan: this tile's key, the thread's 8 sorted positions in one word
    const int64_t tkey = t0 / kFTile + chunk;
    static_assert(PLAN == 0 || kFIPT == 8, "the tile plan packs 8 positions per thread");
    uint32_t pw[PLAN != 0 ? 4 : 1] = {};
    if constexpr (PLAN == 1) {
      const int4 w4 = ld_stream_v4(reinterpret_cast<const int4 *>(a.plan_perm + tkey * kFTile) + tid);
      pw[0] = (uint32_t)w4.x, pw[1] = (uint32_t)w4.y, pw[2] = (uint32_t)w4.z, pw[3] = (uint32_t)w4.w;
    }
    if (cnt == kFTile) {  // full tile: no per-item bounds test
#pragma unroll
      for (int j = 0; j < kFIPT; ++j) {
        const int64_t i = t0 + j * kFBlock + tid;
        rec[j] = ld_stream_v4(a.src + i);
        if (!EMB) rv[j] = ld_stream_f32(a.src_val + i);
        if (a.do_remap) slot[j] = ld_stream_u32(a.slots + i);
      }
    } else
    {
#pragma unroll
      for (int j = 0; j < kFIPT; ++j) {
        const int e = j * kFBlock + tid;
        if (e < cnt) {
          const int64_t i = t0 + e;
          rec[j] = ld_stream_v4(a.src + i);
          if (!EMB) rv[j] = ld_stream_f32(a.src_val + i);
          if (a.do_remap) slot[j] = ld_stream_u32(a.slots + i);
        } else {
          rec[j] = make_int4(INT32_MIN, INT32_MIN, INT32_MIN, INT32_MIN);
        }
      }
    }
    if constexpr (PLAN != 1) {
      for (int b = lane; b < rows; b += 32) s_hist[warp * hstride + b] = 0;
    }
#pragma unroll
    for (int j = 0; j < kFIPT; ++j) {
      const int e = j * kFBlock + tid;
      if (e < cnt) {
        if (a.do_remap) {
          remap_store<1, EMB, PEER>(a, slot[j], rec[j], rec[j], EMB ? 0.f : rv[j]);
        }
        if (PLAN != 1 && key_of(rec[j]) < 0) atomicOr(a.flags, FC_FLAG_ROW_OUTSIDE_SS);
      }
    }
    if constexpr (PLAN == 1) {
      // ------------------------------------------------------------ B (planned)
      if (direct && tid < rows) {  // empty rows of a direct chunk are zero
        const uint16_t *tb = a.plan_bins + tkey * a.hist_rows;
        if ((tid + 1 < rows ? (int)tb[tid + 1] : cnt) == (int)tb[tid]) {
          const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int c = 0; c < R; c += 4) *reinterpret_cast<float4 *>(out_rows + tid * R + c) = z;
        }
      }
      if (tid == 0) s_misc[kFWarps] = cnt;
#pragma unroll
      for (int j = 0; j < kFIPT; ++j) {
        if (cnt == kFTile || j * kFBlock + tid < cnt) {
          const int pos = (int)((j & 1) ? pw[j / 2] >> 16 : pw[j / 2] & 0xffffu);
          FC_DCHECK(a, pos >= 0 && pos < cnt);
          s_sorted[phys(pos)] = rec[j];
          if (!EMB) s_sval[phys(pos)] = rv[j];
        }
      }
      __syncthreads();
    } else {
    __syncwarp();
    // ---------------------------------------------------------------- B
    {
    // B1: warp-local ranks.  The rank is parked in the record's mode word
    // as (rank << 8 | local row) until B3 restores the coordinate -- keeps
    // the 8 ranks out of registers.
    int *wh = s_hist + warp * hstride;
    if (a.hist_rows <= 32) {
      // row-owner lanes (pack_kernel.cuh): lane r counts row r; peers and
      // group base come from the owner lane by shuffle
      int cnt = 0;
#pragma unroll
      for (int j = 0; j < kFIPT; ++j) {
        const int k = key_of(rec[j]);
        unsigned own = __ballot_sync(0xffffffffu, k >= 0);
#pragma unroll
        for (int b = 0; b < 5; ++b) {
          const unsigned m = __ballot_sync(0xffffffffu, ((unsigned)k >> b) & 1u);
          own &= m ^ ((((unsigned)lane >> b) & 1u) - 1u);
        }
        const int before = cnt;
        cnt += __popc(own);
        const int src = k & 31;
        const unsigned peers = __shfl_sync(0xffffffffu, own, src);
        const int base = __shfl_sync(0xffffffffu, before, src);
        set_comp<MODE>(rec[j], k >= 0 ? (((base + __popc(peers & lt_mask)) << 8) | k) : -1);
      }
      if (lane < rows) wh[lane] = cnt;
    } else
#pragma unroll
    for (int j = 0; j < kFIPT; ++j) {
      const int k = key_of(rec[j]);
      // equal-row peers from one ballot per key bit (pack_kernel.cuh)
      unsigned peers = __ballot_sync(0xffffffffu, k >= 0);
      auto round = [&](int b) {
        const unsigned bit = ((unsigned)k >> b) & 1u;
        const unsigned m = __ballot_sync(0xffffffffu, bit);
        peers &= m ^ (bit - 1u);
      };
      if (hbits <= 6) {
#pragma unroll
        for (int b = 0; b < 6; ++b) round(b);
      } else {
#pragma unroll
        for (int b = 0; b < 8; ++b) round(b);
      }
      const unsigned grp = k >= 0 ? peers : (1u << lane);
      // the group leader reserves the run and broadcasts its base
      const int leader = __ffs(grp) - 1;
      int old = 0;
      if (k >= 0 && lane == leader) old = atomicAdd(wh + k, __popc(grp));
      old = __shfl_sync(0xffffffffu, old, leader);
      // the next item's leader may be another lane: __syncwarp orders this
      // item's shared atomics before the next item's (memory-model order,
      // not only the warp's in-order issue), keeping the ranks stable
      __syncwarp();
      set_comp<MODE>(rec[j], k >= 0 ? (((old + __popc(grp & lt_mask)) << 8) | k) : -1);
    }
    __syncthreads();
    {
      int tot = 0;
      if (tid < rows) {
#pragma unroll 4
        for (int w = 0; w < kFWarps; ++w) tot += s_hist[w * hstride + tid];
        if (PLAN != 2 && direct && tot == 0) {
          const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int c = 0; c < R; c += 4) *reinterpret_cast<float4 *>(out_rows + tid * R + c) = z;
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
#pragma unroll 4
      for (int w = 0; w < kFWarps; ++w) wpre += w < warp ? s_misc[w] : 0;
      if (tid == kFBlock - 1) s_misc[kFWarps] = wpre + incl;
      if (tid < rows) {
        int base = wpre + incl - tot;
        if constexpr (PLAN == 2) a.plan_bins[tkey * a.hist_rows + tid] = (uint16_t)base;
#pragma unroll 4
        for (int w = 0; w < kFWarps; ++w) {
          const int c = s_hist[w * hstride + tid];
          s_hist[w * hstride + tid] = base;
          base += c;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kFIPT; ++j) {
      const int x = comp<MODE>(rec[j]);
      if (x >= 0) {
        const int k = x & 255;
        const int pos = wh[k] + (x >> 8);
        FC_DCHECK(a, k < rows && pos >= 0 && pos < cnt);
        if constexpr (PLAN == 2) {
          pw[j / 2] |= (uint32_t)pos << (16 * (j & 1));
          continue;
        }
        set_comp<MODE>(rec[j], irow0 + k);
        s_sorted[phys(pos)] = rec[j];
        if (!EMB) s_sval[phys(pos)] = rv[j];
      }
    }
    if constexpr (PLAN == 2) {
      reinterpret_cast<int4 *>(a.plan_perm + tkey * kFTile)[tid] =
          make_int4((int)pw[0], (int)pw[1], (int)pw[2], (int)pw[3]);
    }
    __syncthreads();
    }
    }
    if constexpr (PLAN == 2) continue;
    const int nvalid = s_misc[kFWarps];
    // ---------------------------------------------------------------- C
    if (tid == 0 && t0 + kFTile < end) {  // next tile's records + slots -> L2
      const int64_t n1 = min64(kFTile, end - (t0 + kFTile));
      prefetch_l2(a.src + (t0 + kFTile), n1 * sizeof(int4));
      if (a.do_remap) prefetch_l2(a.slots + (t0 + kFTile), n1 * sizeof(uint32_t));
      if (!EMB) prefetch_l2(a.src_val + (t0 + kFTile), n1 * sizeof(float));
      if constexpr (PLAN == 1) prefetch_l2(a.plan_perm + (tkey + 1) * kFTile, kFTile * sizeof(uint16_t));
    }
    // both boundary entries of every group are (re)written this tile: rows
    // -1 and zero vectors unless a segment lands there
    if (lg == 0) {
      s_bnd_row[2 * gi] = -1;
      s_bnd_row[2 * gi + 1] = -1;
    }
    const int pb = gi * P;
    const int pe = min(pb + P, nvalid);
    if (pb < pe) {
      int cur = comp<MODE>(s_sorted[phys(pb)]);
      bool head = pb > 0 && comp<MODE>(s_sorted[phys(pb - 1)]) == cur;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      auto flush = [&]() {
        if (head) {
          if (lg == 0) s_bnd_row[2 * gi] = cur - irow0;
          if (col_ok) VecT<4>::store(s_bnd + (2 * gi) * R + col, acc);
        } else if (col_ok) {
          FC_DCHECK(a, cur - irow0 >= 0 && cur - irow0 < rows && cur < a.out_rows);
          if (direct) {  // the whole row is this segment
            VecT<4>::store(out_rows + (cur - irow0) * R + col, acc);
            return;
          }
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
      const FacBases<NM, MODE> fb(a, RT > 0 ? RT : R, col);
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
          for (int u = 0; u < U; ++u) element_prod(fb, q[u], pr[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) consume(comp<MODE>(q[u]), vv[u], pr[u]);
      }
      for (; p < pe; ++p) {
        const int4 q = sp[p];
        const float vv = EMB ? __int_as_float(q.w) : svp[p];
        float pr[4];
        if (col_ok) element_prod(fb, q, pr);
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
    // a row crossing pieces a..b: tail(a) + head(a+1) + ... + head(b), in
    // piece order (see pack_kernel.cuh)
    {
      constexpr int RC = (LPG * 4 + 31) / 32;
      for (int t = warp; t < G; t += kFWarps) {
        const int row = s_bnd_row[2 * t + 1];
        if (row < 0) continue;
        FC_DCHECK(a, row < rows);
#pragma unroll
        for (int q = 0; q < RC; ++q) {
          const int c = q * 32 + lane;
          if (c < R) {
            float run = s_bnd[(2 * t + 1) * R + c];
            for (int j = t + 1; j < G && s_bnd_row[2 * j] == row; ++j) run += s_bnd[(2 * j) * R + c];
            if (direct) out_rows[row * R + c] = run;
            else s_acc[row * R + c] += run;
          }
        }
      }
    }
  }
  if constexpr (PLAN == 2) return;
  if (!direct) {
    __syncthreads();
    float *dstp = part < 0 ? out_rows : partial_ws(a, chunk) + (int64_t)part * a.m * R;
    const int n4 = rows * R / 4;
    const float4 *s4 = reinterpret_cast<const float4 *>(s_acc);
    float4 *d4 = reinterpret_cast<float4 *>(dstp);
    for (int i = tid; i < n4; i += kFBlock) d4[i] = s4[i];
  }
  if (tid == 0) atomicAdd(a.counters, (unsigned long long)(end - start));
}

template <int NM, int MODE, int LPG, int RT, bool PEER = false, int PLAN = 0>
int launch_fast(const ModeArgs &a, int64_t nchunks, cudaStream_t st) {
  const size_t smem = FastPlan<NM, LPG>::total(a.rank, a.tile_rows, a.hist_rows);
  auto kern = mode_pass_fast_kernel<NM, MODE, LPG, RT, PEER, PLAN>;
  static size_t configured = 0;
  if (smem > configured) {
    FC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  if (nchunks > 0) {
    kern<<<(unsigned)nchunks, kFBlock, smem, st>>>(a);
    FC_LAUNCH_CHECK();
  }
  return FC_OK;
}

}  // namespace fc
