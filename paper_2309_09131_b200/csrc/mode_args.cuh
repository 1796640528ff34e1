// Kernel-side definitions shared by the mode-pass translation units.
#pragma once

#include "common.cuh"

namespace fc {

constexpr int kBlock = 256;
constexpr int kIPT = 8;
constexpr int kTile = kBlock * kIPT;  // 2048 elements per tile
constexpr int64_t kSmemAccBytes = 64 * 1024;

// Multi-GPU fused exchange: the remap stores every record straight into
// the back buffer of the GPU that owns its next-mode slot, through NVLink
// peer memory (CUDA IPC mappings).  Slots are global mode-(n+1) positions;
// GPU q owns [base[q], base[q + 1]).  n == 0: single-GPU (dst / nnz).
constexpr int kMaxPeers = 8;
struct PeerTable {
  int n;
  int4 *crd[kMaxPeers];
  float *val[kMaxPeers];
  int64_t base[kMaxPeers + 1];
  float *part_ws[kMaxPeers];  // partial-tile workspaces (super-shards split across GPUs)
};

// Owned output-row ranges of the GPUs (factor-row all-gather).
struct PeerRows {
  int n;
  const float *src[kMaxPeers];
  int64_t row_lo[kMaxPeers + 1];
};

struct ModeArgs {
  const int4 *src;
  const float *src_val;
  int4 *dst;
  float *dst_val;
  const float *fac[8];
  float *out;
  int nmodes, mode, rank;
  int64_t out_rows, m;
  const int64_t *chunk_start;
  const int32_t *chunk_ss;
  const int32_t *chunk_part;
  const int32_t *chunk_rows;  // rows of a chunk merging several small super-shards (or null)
  int64_t tile_rows;          // accumulator tile height (>= m): max rows of non-direct chunks
  int64_t hist_rows;          // max rows of any chunk (counting-sort bins, <= 256)
  int pack_shift;             // N = 3: width of the second input coordinate when both
                              // input coordinates fit 32 bits (8-B sorted records), else 0
  float *part_ws;
  const uint32_t *slots;
  int64_t nnz;
  int do_remap;
  int32_t *flags;
  unsigned long long *counters;
  PeerTable peers;
  // multi-GPU: owner GPU of every chunk's super-shard (null: this GPU).  A
  // super-shard whose chunks span GPUs gets its partial tiles written into
  // the owner's workspace, which reduces them after a barrier.
  const int32_t *chunk_owner;
  // Tile plan (static layout => static per-tile sort): plan = 1 reads every
  // element's position in its row-sorted tile (plan_perm: 2048 uint16 per tile
  // key t0 / tile + chunk, thread-major -- element j * 256 + tid at tid * 8 + j)
  // and every tile's bin starts (plan_bins, hist_rows uint16 per tile key)
  // instead of ranking the tile; plan = 2 ranks as usual and
  // writes them (no compute, no remap).
  uint16_t *plan_perm;
  uint16_t *plan_bins;
  int plan;
};

// Checked build (make CHECKED=1 -> libflycoo_checked.so, FC_DEVICE_CHECKS):
// every shared-tile and output-row index is tested and a miss raises
// FC_FLAG_INDEX_CHECK in the flag word (no trap), which the host turns into
// an exception -- the bounds evidence in place of compute-sanitizer, which
// is closed on this pool.  Compiled out of the product library.
#ifdef FC_DEVICE_CHECKS
#define FC_DCHECK(a, cond)                                                 \
  do {                                                                     \
    if (!(cond)) atomicOr((a).flags, FC_FLAG_INDEX_CHECK);                 \
  } while (0)
#else
#define FC_DCHECK(a, cond) do { } while (0)
#endif

// Partial-tile workspace of chunk c (indexed by the global partial id).
__device__ __forceinline__ float *partial_ws(const ModeArgs &a, int64_t c) {
  return a.chunk_owner ? a.peers.part_ws[a.chunk_owner[c]] : a.part_ws;
}

// Packed fp32 pairs: sm_100's FMUL2 / FFMA2 / FADD2 do two fp32 lanes per
// instruction, each rounded exactly like the scalar op (bitwise-identical
// sums, half the instructions).  A scalar operand packed as (v, v) becomes a
// broadcast operand (no move).
typedef unsigned long long f32x2;
struct f32x4p {
  f32x2 lo, hi;
};
__device__ __forceinline__ f32x2 f2_pack(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(f32x2 r, float &a, float &b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ f32x2 f2_mul(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 f2_fma(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f32x2 f2_add(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x4p f4p(const float4 &x) {
  return {f2_pack(x.x, x.y), f2_pack(x.z, x.w)};
}
__device__ __forceinline__ float4 f4u(const f32x4p &x) {
  float4 r;
  f2_unpack(x.lo, r.x, r.y);
  f2_unpack(x.hi, r.z, r.w);
  return r;
}

// Remap store of one record (CW4 16-byte words + optional separate value)
// to slot s: this GPU's back buffer, or the owning peer's.  Out-of-range
// slots raise FC_FLAG_SLOT_RANGE.
// Remap store of one record (CW4 16-byte words + optional separate value)
// to slot s: this GPU's back buffer, or -- PEER, multi-GPU fused exchange --
// the back buffer of the GPU owning s (peer table; compile-time so the
// single-GPU kernels keep their registers).  Out-of-range slots raise
// FC_FLAG_SLOT_RANGE.
template <int CW4, bool EMB, bool PEER = false>
__device__ __forceinline__ void remap_store(const ModeArgs &a, uint64_t s, const int4 &r0,
                                            const int4 &r1, float v) {
  int4 *d = a.dst;
  float *dv = a.dst_val;
  uint64_t cap = (uint64_t)a.nnz;
  if (PEER) {
    int q = 0;
#pragma unroll
    for (int k = 1; k < kMaxPeers; ++k) q += (k < a.peers.n && s >= (uint64_t)a.peers.base[k]);
    const uint64_t b = (uint64_t)a.peers.base[q];
    cap = (uint64_t)a.peers.base[q + 1] - b;
    s -= b;  // base[0] = 0: no wrap
    d = a.peers.crd[q];
    dv = a.peers.val[q];
  }
  if (s < cap) {
    d[s * CW4] = r0;
    if (CW4 == 2) d[s * CW4 + 1] = r1;
    if (!EMB) dv[s] = v;
  } else {
    atomicOr(a.flags, FC_FLAG_SLOT_RANGE);
  }
}

// chunk_part value of a direct chunk: whole super-shards within one tile,
// rows stored straight to `out` (fast tile kernel only)
constexpr int kPartDirect = -2;

// Output rows [row0, row0 + rows) owned by chunk c: its first super-shard's
// row offset, and either one super-shard's rows or the merged row count.
__device__ __forceinline__ int chunk_row_count(const ModeArgs &a, int64_t c, int64_t row0) {
  const int64_t r = a.chunk_rows ? (int64_t)a.chunk_rows[c] : a.m;
  return (int)min64(r, a.out_rows - row0);
}

__device__ __forceinline__ int4 ld_stream_v4(const int4 *p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t *p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_stream_u16(const uint16_t *p) {
  uint16_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ float ld_stream_f32(const float *p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}

// Prefetch the line holding p into L1 (no register destination).
__device__ __forceinline__ void prefetch_l1(const void *p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Bulk prefetch of [p, p + bytes) into L2 (TMA unit).  The instruction
// needs a 16-B aligned address and a multiple of 16 bytes: widen the range.
__device__ __forceinline__ void prefetch_l2(const void *p, int64_t bytes) {
  const uint64_t a0 = reinterpret_cast<uint64_t>(p) & ~uint64_t(15);
  const uint64_t a1 = (reinterpret_cast<uint64_t>(p) + (uint64_t)bytes + 15) & ~uint64_t(15);
  const uint32_t n = (uint32_t)(a1 - a0);
  if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"(n) : "memory");
}

__device__ __forceinline__ int word_of(const int4 &a, const int4 &b, int w) {
  switch (w) {
    case 0: return a.x;
    case 1: return a.y;
    case 2: return a.z;
    case 3: return a.w;
    case 4: return b.x;
    case 5: return b.y;
    case 6: return b.z;
    default: return b.w;
  }
}

template <int VEC>
struct VecT;
template <>
struct VecT<4> {
  static __device__ __forceinline__ void load_ro(const float *p, float (&v)[4]) {
    const float4 f = __ldg(reinterpret_cast<const float4 *>(p));
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  }
  static __device__ __forceinline__ void load(const float *p, float (&v)[4]) {
    const float4 f = *reinterpret_cast<const float4 *>(p);
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  }
  static __device__ __forceinline__ void store(float *p, const float (&v)[4]) {
    *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <>
struct VecT<1> {
  static __device__ __forceinline__ void load_ro(const float *p, float (&v)[1]) { v[0] = __ldg(p); }
  static __device__ __forceinline__ void load(const float *p, float (&v)[1]) { v[0] = *p; }
  static __device__ __forceinline__ void store(float *p, const float (&v)[1]) { *p = v[0]; }
};

constexpr int kMaxBins = 256;
constexpr int kWarps = kBlock / 32;

// Fast-path launchers, one translation unit per mode count (fast_n*.cu).
int fast_dispatch_n2(const ModeArgs &a, int64_t nchunks, cudaStream_t st);
int fast_dispatch_n3(const ModeArgs &a, int64_t nchunks, cudaStream_t st);
int fast_dispatch_n4(const ModeArgs &a, int64_t nchunks, cudaStream_t st);
// peer-store (multi-GPU fused exchange) instances, fast_n*_peer.cu
int fast_dispatch_peer_n2(const ModeArgs &a, int64_t nchunks, cudaStream_t st);
int fast_dispatch_peer_n3(const ModeArgs &a, int64_t nchunks, cudaStream_t st);
int fast_dispatch_peer_n4(const ModeArgs &a, int64_t nchunks, cudaStream_t st);

// Kernel-variant switches, fixed when the library loads (FLYCOO_PACK=0 /
// FLYCOO_PACK_WIDE=0 in the environment, for A/B runs) or set through
// fc_set_kernel_variant(); never read from the environment on the launch path.
struct KernelVariant {
  bool pack = true;
  bool pack_wide = true;
};
KernelVariant &kernel_variant();

}  // namespace fc
