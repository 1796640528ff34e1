// Warp-specialised persistent mode pass (K1 v3).
//
// One CTA per SM, 24 warps: warps 0..7 are PRODUCERS, warps 8..23
// CONSUMERS, connected by a double-buffered sorted tile in shared memory.
//   producer, per 2048-element tile: stream records + slots in (16-B
//     no-allocate loads), scatter each record to its remap slot, rank the
//     tile by output row (warp __match_any_sync ranks + one scan over the
//     producer warps), write the records into the sorted buffer;
//   consumer, per tile: groups of LPG lanes gather the N-1 factor rows of
//     their piece (read-only 16-B loads), form v * prod in registers, reduce
//     equal-row segments in registers into the super-shard's shared-memory
//     accumulator tile, fold piece-boundary segments in order; at a chunk's
//     last tile write the tile to `out` (owned rows) or to its partial slot.
// The two sides synchronise with named barriers only (FULL[b]: producers
// arrive, consumers sync; EMPTY[b]: consumers arrive, producers sync), so a
// tile's loads, remap stores and sort overlap the previous tile's gathers.
// Chunks are taken round-robin by CTA (results do not depend on which CTA
// runs a chunk: every sum has a fixed order).
#pragma once

#include "fast_kernel.cuh"

namespace fc {

constexpr int kPipeProdWarps = 8;
#ifndef PIPE_CONS_WARPS
#define PIPE_CONS_WARPS 16
#endif
#ifndef PIPE_U
#define PIPE_U 4
#endif
constexpr int kPipeConsWarps = PIPE_CONS_WARPS;
constexpr int kPipeThreads = 32 * (kPipeProdWarps + kPipeConsWarps);
constexpr int kProdThreads = 32 * kPipeProdWarps;
constexpr int kConsThreads = 32 * kPipeConsWarps;
static_assert(kProdThreads * kIPT == kTile, "producers cover one tile");

// named barrier ids (0 is __syncthreads, never used here)
constexpr int kBarProd = 1, kBarCons = 2, kBarFull = 3, kBarEmpty = 5;

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

struct TileMeta {
  int64_t chunk;  // -1: no more work
  int nvalid;
  int first, last;
};

template <int NM, int LPG>
struct PipePlan {
  static constexpr int G = kConsThreads / LPG;
  static constexpr int P = kTile / G;
  static constexpr bool EMB = value_embedded(NM);
  static constexpr size_t sorted_bytes = sizeof(int4) * (kTile + G);
  static constexpr size_t sval_bytes = EMB ? 0 : sizeof(float) * (kTile + G);
  static constexpr size_t buf_bytes = sorted_bytes + sval_bytes;
  static constexpr size_t meta_bytes = 2 * sizeof(TileMeta) + 64;
  static constexpr size_t fixed_bytes = 2 * buf_bytes + meta_bytes;
  __host__ __device__ static size_t hist_bytes(int64_t m) {
    return sizeof(int) * kPipeProdWarps * ((m + 3) / 4 * 4);
  }
  static size_t total(int rank, int64_t m) {
    return fixed_bytes + hist_bytes(m) + (size_t)2 * G * sizeof(int) +
           (size_t)2 * G * rank * sizeof(float) + (size_t)m * rank * sizeof(float);
  }
};

template <int NM, int MODE, int LPG, int RT>
__global__ void __launch_bounds__(kPipeThreads, 1) mode_pass_pipe_kernel(const __grid_constant__ ModeArgs a,
                                                                         int64_t nchunks) {
  using PP = PipePlan<NM, LPG>;
  constexpr int G = PP::G;
  constexpr int P = PP::P;
  constexpr bool EMB = PP::EMB;
  constexpr int U = PIPE_U;
  const int R = RT > 0 ? RT : a.rank;

  extern __shared__ __align__(16) unsigned char smem[];
  const int hstride = (int)((a.hist_rows + 3) / 4 * 4);
  TileMeta *s_meta = reinterpret_cast<TileMeta *>(smem + 2 * PP::buf_bytes);
  int *s_pmisc = reinterpret_cast<int *>(smem + 2 * PP::buf_bytes + 2 * sizeof(TileMeta));
  unsigned char *tail = smem + PP::fixed_bytes;
  int *s_hist = reinterpret_cast<int *>(tail);
  tail += PP::hist_bytes(a.hist_rows);
  int *s_bnd_row = reinterpret_cast<int *>(tail);
  tail += 2 * G * sizeof(int);
  float *s_bnd = reinterpret_cast<float *>(tail);
  tail += (size_t)2 * G * R * sizeof(float);
  float *s_acc = reinterpret_cast<float *>(tail);
  auto sorted_of = [&](int b) { return reinterpret_cast<int4 *>(smem + b * PP::buf_bytes); };
  auto sval_of = [&](int b) {
    return reinterpret_cast<float *>(smem + b * PP::buf_bytes + PP::sorted_bytes);
  };
  auto phys = [](int pos) { return pos + pos / P; };

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  if (warp < kPipeProdWarps) {
    // ============================================================ producer
    const unsigned lt_mask = (1u << lane) - 1u;
    int *wh = s_hist + warp * hstride;
    int tseq = 0;
    for (int64_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
      const int64_t start = a.chunk_start[chunk];
      const int64_t end = a.chunk_start[chunk + 1];
      const int64_t row0 = a.chunk_ss[chunk] * a.m;
      const int rows = chunk_row_count(a, chunk, row0);
      const int irow0 = (int)row0;
      auto key_of = [&](const int4 &r) {
        const int lr = comp<MODE>(r) - irow0;
        return (lr >= 0 && lr < rows) ? lr : -1;
      };
      for (int64_t t0 = start; t0 < end; t0 += kTile, ++tseq) {
        const int b = tseq & 1;
        const int cnt = (int)min64(kTile, end - t0);
        int4 rec[kIPT];
        float rv[kIPT];
        uint32_t slot[kIPT];
#pragma unroll
        for (int j = 0; j < kIPT; ++j) {
          const int e = j * kProdThreads + tid;
          if (e < cnt) {
            const int64_t i = t0 + e;
            rec[j] = ld_stream_v4(a.src + i);
            if (!EMB) rv[j] = ld_stream_f32(a.src_val + i);
            if (a.do_remap) slot[j] = ld_stream_u32(a.slots + i);
          } else {
            rec[j] = make_int4(INT32_MIN, INT32_MIN, INT32_MIN, INT32_MIN);
          }
        }
#pragma unroll
        for (int j = 0; j < kIPT; ++j) {
          const int e = j * kProdThreads + tid;
          if (e < cnt) {
            if (a.do_remap) {
              remap_store<1, EMB>(a, slot[j], rec[j], rec[j], EMB ? 0.f : rv[j]);
            }
            if (key_of(rec[j]) < 0) atomicOr(a.flags, FC_FLAG_ROW_OUTSIDE_SS);
          }
        }
        // the histogram is private to the producers; the previous tile's
        // scatter finished at its last producer barrier
        for (int r = lane; r < rows; r += 32) wh[r] = 0;
        __syncwarp();
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
        named_sync(kBarProd, kProdThreads);
        {
          int tot = 0;
          int cw[kPipeProdWarps];
          if (tid < rows) {
#pragma unroll
            for (int w = 0; w < kPipeProdWarps; ++w) {
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
          if (lane == 31) s_pmisc[warp] = incl;
          named_sync(kBarProd, kProdThreads);
          int wpre = 0;
#pragma unroll
          for (int w = 0; w < kPipeProdWarps; ++w) wpre += w < warp ? s_pmisc[w] : 0;
          if (tid == kProdThreads - 1) s_pmisc[kPipeProdWarps] = wpre + incl;
          if (tid < rows) {
            int base = wpre + incl - tot;
#pragma unroll
            for (int w = 0; w < kPipeProdWarps; ++w) {
              s_hist[w * hstride + tid] = base;
              base += cw[w];
            }
          }
        }
        if (tseq >= 2) named_sync(kBarEmpty + b, kPipeThreads);  // consumers left buffer b
        named_sync(kBarProd, kProdThreads);
        int4 *srt = sorted_of(b);
        float *sv = sval_of(b);
#pragma unroll
        for (int j = 0; j < kIPT; ++j) {
          const int x = comp<MODE>(rec[j]);
          if (x >= 0) {
            const int k = x & 255;
            const int pos = wh[k] + (x >> 8);
            set_comp<MODE>(rec[j], irow0 + k);
            srt[phys(pos)] = rec[j];
            if (!EMB) sv[phys(pos)] = rv[j];
          }
        }
        if (tid == 0) {
          s_meta[b].chunk = chunk;
          s_meta[b].nvalid = s_pmisc[kPipeProdWarps];
          s_meta[b].first = t0 == start;
          s_meta[b].last = t0 + kTile >= end;
          if (t0 + kTile >= end) atomicAdd(a.counters, (unsigned long long)(end - start));
        }
        named_sync(kBarProd, kProdThreads);  // histogram / misc free for the next tile
        named_arrive(kBarFull + b, kPipeThreads);
      }
    }
    // end of stream marker
    const int b = tseq & 1;
    if (tseq >= 2) named_sync(kBarEmpty + b, kPipeThreads);
    if (tid == 0) s_meta[b].chunk = -1;
    named_arrive(kBarFull + b, kPipeThreads);
  } else {
    // ============================================================ consumer
    const int ctid = tid - kProdThreads;
    const int cwarp = ctid >> 5;
    const int gi = ctid / LPG;
    const int lg = ctid % LPG;
    const int col = lg * 4;
    const bool col_ok = RT > 0 ? true : col < R;
    for (int tseq = 0;; ++tseq) {
      const int b = tseq & 1;
      named_sync(kBarFull + b, kPipeThreads);
      const TileMeta meta = s_meta[b];
      if (meta.chunk < 0) break;
      const int64_t chunk = meta.chunk;
      const int64_t row0 = a.chunk_ss[chunk] * a.m;
      const int rows = chunk_row_count(a, chunk, row0);
      const int irow0 = (int)row0;
      if (meta.first) {
        for (int i = ctid; i < rows * R; i += kConsThreads) s_acc[i] = 0.f;
        named_sync(kBarCons, kConsThreads);
      }
      const int4 *srt = sorted_of(b);
      const float *sv = sval_of(b);
      const int nvalid = meta.nvalid;
      if (lg == 0) {
        s_bnd_row[2 * gi] = -1;
        s_bnd_row[2 * gi + 1] = -1;
      }
      const int pb = gi * P;
      const int pe = min(pb + P, nvalid);
      if (pb < nvalid) {
        int cur = comp<MODE>(srt[phys(pb)]);
        bool head = pb > 0 && comp<MODE>(srt[phys(pb - 1)]) == cur;
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
        auto consume = [&](int row, const float (&t)[4]) {
          if (row != cur) {
            flush();
            head = false;
            cur = row;
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[v] = 0.f;
          }
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[v] += t[v];
        };
        int p = pb;
        for (; p + U <= pe; p += U) {
          int4 q[U];
          float vv[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            q[u] = srt[phys(p + u)];
            vv[u] = EMB ? __int_as_float(q[u].w) : sv[phys(p + u)];
          }
          float t[U][4];
          if (col_ok) {
#pragma unroll
            for (int u = 0; u < U; ++u) element_term<NM, MODE, RT>(a, R, col, q[u], vv[u], t[u]);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) consume(comp<MODE>(q[u]), t[u]);
        }
        for (; p < pe; ++p) {
          const int4 q = srt[phys(p)];
          const float vv = EMB ? __int_as_float(q.w) : sv[phys(p)];
          float t[4];
          if (col_ok) element_term<NM, MODE, RT>(a, R, col, q, vv, t);
          consume(comp<MODE>(q), t);
        }
        const bool tail = pe < nvalid && comp<MODE>(srt[phys(pe)]) == cur;
        if (tail && !head) {
          if (lg == 0) s_bnd_row[2 * gi + 1] = cur - irow0;
          if (col_ok) VecT<4>::store(s_bnd + (2 * gi + 1) * R + col, acc);
        } else {
          flush();
        }
      }
      named_sync(kBarCons, kConsThreads);
      named_arrive(kBarEmpty + b, kPipeThreads);  // sorted buffer b no longer read
      // boundary fold, spread over the consumer warps (see fast_kernel.cuh)
      {
        constexpr int E = (2 * G + kPipeConsWarps - 1) / kPipeConsWarps;
        constexpr int RC = (LPG * 4 + 31) / 32;
        int ent = cwarp * E;
        const int ent_end = min(2 * G, ent + E);
        int prev = -1;
        for (int e2 = ent - 1; e2 >= 0; --e2) {
          const int r2 = s_bnd_row[e2];
          if (r2 >= 0) {
            prev = r2;
            break;
          }
        }
        while (ent < ent_end) {
          const int row = s_bnd_row[ent];
          if (row < 0 || row == prev) {
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
      named_sync(kBarCons, kConsThreads);
      if (meta.last) {
        const int part = a.chunk_part[chunk];
        float *dstp = part < 0 ? a.out + row0 * R : a.part_ws + (int64_t)part * a.m * R;
        const int n4 = rows * R / 4;
        const float4 *s4 = reinterpret_cast<const float4 *>(s_acc);
        float4 *d4 = reinterpret_cast<float4 *>(dstp);
        for (int i = ctid; i < n4; i += kConsThreads) d4[i] = s4[i];
        named_sync(kBarCons, kConsThreads);
      }
    }
  }
}

template <int NM, int MODE, int LPG, int RT>
int launch_pipe(const ModeArgs &a, int64_t nchunks, cudaStream_t st) {
  const size_t smem = PipePlan<NM, LPG>::total(a.rank, a.tile_rows);
  auto kern = mode_pass_pipe_kernel<NM, MODE, LPG, RT>;
  static size_t configured = 0;
  if (smem > configured) {
    FC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  static int nsm = 0;
  if (nsm == 0) {
    int dev = 0;
    FC_CUDA_TRY(cudaGetDevice(&dev));
    FC_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  }
  if (nchunks > 0) {
    const int64_t grid = min64(nchunks, (int64_t)nsm);
    kern<<<(unsigned)grid, kPipeThreads, smem, st>>>(a, nchunks);
    FC_LAUNCH_CHECK();
  }
  return FC_OK;
}

}  // namespace fc
