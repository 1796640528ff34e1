// K1, packed-record variant of the tile kernel for 3-mode tensors whose two
// non-output coordinates fit 32 bits together (config 2: 14 + 15 bits).
//
// Same phases and the same sums as mode_pass_fast_kernel (fast_kernel.cuh),
// but the sorted tile holds 8-byte records {c_w1 << shift | c_w2, value}
// instead of 16-byte ones, and phase C takes row boundaries from the sort's
// bin offsets instead of reading a row per element:
//   * shared traffic of the sorted tile halves (one 64-bit load serves the
//     group; the scatter of 8-B records conflicts less);
//   * the tile shrinks by 16 KB, which the SM gives back to L1 -- where the
//     factor-row gathers hit.
#pragma once

#include "fast_kernel.cuh"

// 4 CTAs/SM (its shared footprint is ~36 KB), 3 elements in flight per
// group: no spills at the 64-register cap (profiles/r1_kernel_experiments.md)
#ifndef PACK_MIN_BLOCKS
#define PACK_MIN_BLOCKS 4
#endif
#ifndef PACK_U
#define PACK_U 3
#endif

namespace fc {

// WIDE: 3-mode tensors whose input coordinates do NOT fit 32 bits together
// (c4: 21 + 21 bits): the sorted tile holds {c_w1, c_w2} words plus a
// separate value array (12 B per element instead of the tile kernel's 16,
// rows from the bins as here)
template <int LPG, bool WIDE = false>
struct PackPlan {
  static constexpr int G = kFBlock / LPG;
  static constexpr int P = kFTile / G;
  static constexpr size_t sval_offset = sizeof(uint2) * (kFTile + G);
  static constexpr size_t sorted_bytes = sval_offset + (WIDE ? sizeof(float) * (kFTile + G) : 0);
  static constexpr size_t misc_bytes = 4 * (kFWarps + 4 + G);
  static constexpr size_t fixed_bytes = (sorted_bytes + misc_bytes + 15) / 16 * 16;
  __host__ __device__ static size_t hist_bytes(int64_t m) {
    return sizeof(int) * kFWarps * ((m + 3) / 4 * 4);
  }
  static size_t total(int rank, int64_t m, int64_t hist_rows) {
    return fixed_bytes + hist_bytes(hist_rows > m ? hist_rows : m) + (size_t)2 * G * sizeof(int) +
           (size_t)2 * G * rank * sizeof(float) + (size_t)m * rank * sizeof(float);
  }
};

// PLAN: 0 = rank every tile in the kernel; 1 = the tile plan gives every
// element's sorted position and every tile's bin starts (no ballots, no
// histogram, no scan: two barriers per tile instead of four); 2 = rank as
// PLAN 0 and write the plan (nothing else).  The plan is static because the
// layout is: the same tiles are sorted the same way in every sweep.
template <int MODE, int LPG, int RT, bool PEER = false, bool WIDE = false, int PLAN = 0>
__global__ void __launch_bounds__(kFBlock, PACK_MIN_BLOCKS) mode_pass_pack_kernel(const __grid_constant__ ModeArgs a) {
  using PP = PackPlan<LPG, WIDE>;
  constexpr int G = PP::G;
  constexpr int P = PP::P;
  constexpr int U = PACK_U;
  constexpr int W1 = MODE == 0 ? 1 : 0;  // the two input modes, ascending
  constexpr int W2 = MODE == 2 ? 1 : 2;
  const int R = RT > 0 ? RT : a.rank;
  const int shift = a.pack_shift;
  const uint32_t lowmask = (1u << shift) - 1u;

  extern __shared__ __align__(16) unsigned char smem[];
  const int hstride = (int)((a.hist_rows + 3) / 4 * 4);
  const int hbits = 32 - __clz((int)(a.hist_rows > 1 ? a.hist_rows - 1 : 1));
  const bool hist_rows32 = a.hist_rows <= 32;
  uint2 *s_sorted = reinterpret_cast<uint2 *>(smem);
  float *s_sval = reinterpret_cast<float *>(smem + PP::sval_offset);  // WIDE only
  int *s_misc = reinterpret_cast<int *>(smem + PP::sorted_bytes);
  int *s_piece_bin = s_misc + kFWarps + 4;  // first bin of every piece
  unsigned char *tail = smem + PP::fixed_bytes;
  int *s_hist = reinterpret_cast<int *>(tail);
  tail += PP::hist_bytes(a.hist_rows);
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
  const int part = a.chunk_part[chunk];
  const int64_t row0 = a.chunk_ss[chunk] * a.m;
  const int rows = chunk_row_count(a, chunk, row0);
  const int irow0 = (int)row0;
  const bool direct = part == kPartDirect;
  float *out_rows = a.out + row0 * R;
  if (PLAN == 2) {
    if (start == end) return;
  } else if (direct) {
    if (start == end) {
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
  // start of bin k in the sorted tile (warp 0's base), end = start of k + 1
  auto bin_start = [&](int k) { return s_hist[k]; };

  for (int64_t t0 = start; t0 < end; t0 += kFTile) {
    const int cnt = (int)min64(kFTile, end - t0);
    // ---------------------------------------------------------------- A
    int4 rec[kFIPT];
    uint32_t slot[kFIPT];
    // tile plan: this tile's key, and the thread's 8 sorted positions as one
    // 16-byte word (uint16 each, stored thread-major per tile key)
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
      if (cnt == kFTile || e < cnt) {
        if (a.do_remap) {
          remap_store<1, true, PEER>(a, slot[j], rec[j], rec[j], 0.f);
        }
      }
    }
    if constexpr (PLAN != 1) {  // a record outside the chunk's super-shard rows (invalid items: -1 by design)
      bool bad = false;
#pragma unroll
      for (int j = 0; j < kFIPT; ++j) bad |= (j * kFBlock + tid < cnt) && key_of(rec[j]) < 0;
      if (bad) atomicOr(a.flags, FC_FLAG_ROW_OUTSIDE_SS);
    }
    if constexpr (PLAN == 1) {
      // ------------------------------------------------------------ B (planned)
      // bin starts and the pieces' first bins from the tile plan, records
      // straight to their sorted positions
      if (tid < rows) {
        const uint16_t *tb = a.plan_bins + tkey * a.hist_rows;
        const int bstart = tb[tid];
        const int tot = (tid + 1 < rows ? (int)tb[tid + 1] : cnt) - bstart;
        if (direct && tot == 0) {
          const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int c = 0; c < R; c += 4) *reinterpret_cast<float4 *>(out_rows + tid * R + c) = z;
        }
        s_hist[tid] = bstart;
        for (int j = (bstart + P - 1) / P; j * P < bstart + tot; ++j) s_piece_bin[j] = tid;
      }
      if (tid == 0) s_misc[kFWarps] = cnt;
#pragma unroll
      for (int j = 0; j < kFIPT; ++j) {
        if (cnt == kFTile || j * kFBlock + tid < cnt) {
          const int pos = (int)((j & 1) ? pw[j / 2] >> 16 : pw[j / 2] & 0xffffu);
          FC_DCHECK(a, pos >= 0 && pos < cnt);
          if constexpr (WIDE) {
            s_sorted[phys(pos)] = make_uint2((uint32_t)comp<W1>(rec[j]), (uint32_t)comp<W2>(rec[j]));
            s_sval[phys(pos)] = __int_as_float(rec[j].w);
          } else {
            const uint32_t pk = ((uint32_t)comp<W1>(rec[j]) << shift) | (uint32_t)comp<W2>(rec[j]);
            s_sorted[phys(pos)] = make_uint2(pk, (uint32_t)rec[j].w);
          }
        }
      }
      __syncthreads();
    } else {
    __syncwarp();
    // ---------------------------------------------------------------- B
    int *wh = s_hist + warp * hstride;
    if (hist_rows32) {
      // <= 32 rows: lane r owns row r's count in this warp.  From the key-bit
      // ballots lane r forms `own` = the lanes holding row r; an element's
      // equal-row peers and its group's base are then one shuffle each from
      // the lane owning its row -- no shared atomics, no leader election.
      // Ranks are (count in earlier items) + (lower lanes in this item):
      // the same stable order as the atomic path.
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
    } else {
    // stable per-warp counting: the leader of each equal-row group reserves
    // the group's run with one shared atomic (returns the old count) and
    // broadcasts it; a __syncwarp per item orders the items' atomics, so runs
    // are ordered by (item j, lane)
#pragma unroll
    for (int j = 0; j < kFIPT; ++j) {
      const int k = key_of(rec[j]);
      // equal-row peers from one ballot per key bit (rows < 2^hbits)
      unsigned peers = __ballot_sync(0xffffffffu, k >= 0);
      // bits >= hbits are 0 for every valid lane, so extra rounds only drop
      // invalid lanes again: 5 fixed rounds for <= 32 rows, 6 for <= 64, else 8
      auto round = [&](int b) {
        const unsigned bit = ((unsigned)k >> b) & 1u;
        const unsigned m = __ballot_sync(0xffffffffu, bit);
        peers &= m ^ (bit - 1u);  // m if the bit is set, ~m if not
      };
      if (hbits <= 5) {
#pragma unroll
        for (int b = 0; b < 5; ++b) round(b);
      } else if (hbits <= 6) {
#pragma unroll
        for (int b = 0; b < 6; ++b) round(b);
      } else {
#pragma unroll
        for (int b = 0; b < 8; ++b) round(b);
      }
      const unsigned grp = k >= 0 ? peers : (1u << lane);
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
      // rows <= 32: warp 0 holds every row, so no cross-warp prefix (and no
      // middle barrier) is needed
      const bool one_warp = rows <= 32;
      if (lane == 31) s_misc[warp] = incl;
      if (!one_warp) __syncthreads();
      int wpre = 0;
      if (!one_warp) {
#pragma unroll 4
        for (int w = 0; w < kFWarps; ++w) wpre += w < warp ? s_misc[w] : 0;
      }
      if (tid == (one_warp ? 31 : kFBlock - 1)) s_misc[kFWarps] = wpre + incl;
      if (tid < rows) {
        const int bstart = wpre + incl - tot;
        if constexpr (PLAN == 2) a.plan_bins[tkey * a.hist_rows + tid] = (uint16_t)bstart;
        int base = bstart;
#pragma unroll 4
        for (int w = 0; w < kFWarps; ++w) {
          const int c = s_hist[w * hstride + tid];
          s_hist[w * hstride + tid] = base;
          base += c;
        }
        // pieces whose first element falls in this (non-empty) bin
        for (int j = (bstart + P - 1) / P; j * P < bstart + tot; ++j) s_piece_bin[j] = tid;
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
        if constexpr (WIDE) {
          s_sorted[phys(pos)] = make_uint2((uint32_t)comp<W1>(rec[j]), (uint32_t)comp<W2>(rec[j]));
          s_sval[phys(pos)] = __int_as_float(rec[j].w);
        } else {
          const uint32_t pk = ((uint32_t)comp<W1>(rec[j]) << shift) | (uint32_t)comp<W2>(rec[j]);
          s_sorted[phys(pos)] = make_uint2(pk, (uint32_t)rec[j].w);
        }
      }
    }
    if constexpr (PLAN == 2) {
      reinterpret_cast<int4 *>(a.plan_perm + tkey * kFTile)[tid] =
          make_int4((int)pw[0], (int)pw[1], (int)pw[2], (int)pw[3]);
    }
    __syncthreads();
    }
    if constexpr (PLAN == 2) continue;
    const int nvalid = s_misc[kFWarps];
    // ---------------------------------------------------------------- C
    if (tid == 0 && t0 + kFTile < end) {
      const int64_t n1 = min64(kFTile, end - (t0 + kFTile));
      prefetch_l2(a.src + (t0 + kFTile), n1 * sizeof(int4));
      if (a.do_remap) prefetch_l2(a.slots + (t0 + kFTile), n1 * sizeof(uint32_t));
      if constexpr (PLAN == 1) prefetch_l2(a.plan_perm + (tkey + 1) * kFTile, kFTile * sizeof(uint16_t));
    }
    if (lg == 0) {
      s_bnd_row[2 * gi] = -1;
      s_bnd_row[2 * gi + 1] = -1;
    }
    const int pb = gi * P;
    const int pe = min(pb + P, nvalid);
    if (pb < pe) {
      int cur = s_piece_bin[gi];
      int nxt = cur + 1 < rows ? bin_start(cur + 1) : nvalid;
      bool head = pb > bin_start(cur);
      // 4 columns as two packed fp32 pairs (FMUL2 / FFMA2)
      f32x4p acc = {0ull, 0ull};
      auto put = [](float *p, const f32x4p &x) { *reinterpret_cast<float4 *>(p) = f4u(x); };
      auto flush = [&]() {
        if (head) {
          if (lg == 0) s_bnd_row[2 * gi] = cur;
          if (col_ok) put(s_bnd + (2 * gi) * R + col, acc);
        } else if (col_ok) {
          FC_DCHECK(a, cur >= 0 && cur < rows && row0 + cur < a.out_rows);
          if (direct) {
            put(out_rows + cur * R + col, acc);
            return;
          }
          float *p = s_acc + cur * R + col;
          const f32x4p o = f4p(*reinterpret_cast<const float4 *>(p));
          put(p, {f2_add(o.lo, acc.lo), f2_add(o.hi, acc.hi)});
        }
      };
      auto consume = [&](int p, float v, const f32x4p &pr) {
        if (p == nxt) {  // a new row starts here
          flush();
          head = false;
          do {
            ++cur;
            nxt = cur + 1 < rows ? bin_start(cur + 1) : nvalid;
          } while (nxt == p);
          acc = {0ull, 0ull};
        }
        const f32x2 vv = f2_pack(v, v);
        acc.lo = f2_fma(vv, pr.lo, acc.lo);
        acc.hi = f2_fma(vv, pr.hi, acc.hi);
      };
      // column-offset factor bases, hoisted (the loop rematerialised them
      // from the parameter bank every iteration: 4.84 -> 4.69 ms on c2)
      const float *f1b = a.fac[W1] + col;
      const float *f2b = a.fac[W2] + col;
      const uint32_t rstride = (uint32_t)(RT > 0 ? RT : R);
      // q = {packed coordinates, value bits} or, WIDE, {c_w1, c_w2} (+ s_sval)
      auto prod = [&](const uint2 &q, f32x4p &pr) {
        const uint32_t c1 = WIDE ? q.x : q.x >> shift, c2 = WIDE ? q.y : q.x & lowmask;
        const f32x4p f1 = f4p(__ldg(reinterpret_cast<const float4 *>(f1b + (uint64_t)c1 * rstride)));
        const f32x4p f2 = f4p(__ldg(reinterpret_cast<const float4 *>(f2b + (uint64_t)c2 * rstride)));
        pr.lo = f2_mul(f1.lo, f2.lo);
        pr.hi = f2_mul(f1.hi, f2.hi);
      };
      const uint2 *sp = s_sorted + gi;  // pad of piece gi
      const float *svp = s_sval + gi;
      auto val = [&](const uint2 &q, int at) { return WIDE ? svp[at] : __uint_as_float(q.y); };
      int p = pb;
      for (; p + U <= pe; p += U) {
        uint2 q[U];
        float vq[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          q[u] = sp[p + u];
          vq[u] = val(q[u], p + u);
        }
        f32x4p pr[U];
        if (col_ok) {
#pragma unroll
          for (int u = 0; u < U; ++u) prod(q[u], pr[u]);
        }
        if (p + U <= nxt) {  // no row starts inside [p, p + U)
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const float v = vq[u];
            const f32x2 vv = f2_pack(v, v);
            acc.lo = f2_fma(vv, pr[u].lo, acc.lo);
            acc.hi = f2_fma(vv, pr[u].hi, acc.hi);
          }
          continue;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) consume(p + u, vq[u], pr[u]);
      }
      for (; p < pe; ++p) {
        const uint2 q = sp[p];
        f32x4p pr;
        if (col_ok) prod(q, pr);
        consume(p, val(q, p), pr);
      }
      const bool tail = pe < nvalid && nxt > pe;
      if (tail && !head) {
        if (lg == 0) s_bnd_row[2 * gi + 1] = cur;
        if (col_ok) put(s_bnd + (2 * gi + 1) * R + col, acc);
      } else {
        flush();
      }
    }
    __syncthreads();
    // ---------------------------------------------------------------- D
    // A row that crosses pieces a..b left a tail entry in piece a and a head
    // entry in each of a+1..b; its sum is tail(a) + head(a+1) + ... + head(b)
    // in piece order (the order of the scan-based fold it replaces).
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

template <int MODE, int LPG, int RT, bool PEER = false, bool WIDE = false, int PLAN = 0>
int launch_pack(const ModeArgs &a, int64_t nchunks, cudaStream_t st) {
  const size_t smem = PackPlan<LPG, WIDE>::total(a.rank, a.tile_rows, a.hist_rows);
  auto kern = mode_pass_pack_kernel<MODE, LPG, RT, PEER, WIDE, PLAN>;
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
