// Fast-path dispatch: (N, mode, R) -> kernel instance.  The one-CTA-per-chunk
// tile kernel (fast_kernel.cuh) is the default; FLYCOO_KERNEL=pipe|warp select
// the persistent warp-specialised pipeline (pipe_kernel.cuh) or the
// warp-independent kernel (warp_kernel.cuh) for A/B runs -- both slower in
// round 1 (profiles/r1_kernel_experiments.md).
#pragma once

#include <stdlib.h>
#include <string.h>

#include "pipe_kernel.cuh"
#include "warp_kernel.cuh"
#include "pack_kernel.cuh"

namespace fc {

// 1 = tile (default), 0 = warp-independent, 2 = pipeline (FLYCOO_KERNEL=warp|pipe)
inline int kernel_kind() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("FLYCOO_KERNEL");
    v = 1;
    if (e && strcmp(e, "warp") == 0) v = 0;
    if (e && strcmp(e, "pipe") == 0) v = 2;
  }
  return v;
}

inline bool pack_enabled() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("FLYCOO_PACK");
    v = (e && strcmp(e, "0") == 0) ? 0 : 1;
  }
  return v == 1;
}

inline bool pack_wide_enabled() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("FLYCOO_PACK_WIDE");
    v = (e && strcmp(e, "0") == 0) ? 0 : 1;
  }
  return v == 1;
}

template <int NM, int MODE, int LPG, int RT, bool PEER>
int launch_choice(const ModeArgs &a, int64_t nchunks, cudaStream_t st) {
  if constexpr (NM == 3) {
    // 8-byte sorted records when the two input coordinates fit 32 bits
    if (a.pack_shift > 0 && (PEER || kernel_kind() == 1) && pack_enabled())
      return launch_pack<MODE, LPG, RT, PEER>(a, nchunks, st);
    // wider coordinates: {c_w1, c_w2} + value array, rows from the bins
    if (a.pack_shift == 0 && (PEER || kernel_kind() == 1) && pack_wide_enabled())
      return launch_pack<MODE, LPG, RT, PEER, true>(a, nchunks, st);
  }
  // multi-GPU fused exchange: tile kernel only; direct chunks (hist_rows >
  // tile_rows) exist only in the tile kernel
  if (PEER || a.hist_rows > a.tile_rows) return launch_fast<NM, MODE, LPG, RT, PEER>(a, nchunks, st);
  if constexpr (!PEER) {
    switch (kernel_kind()) {
      case 2: return launch_pipe<NM, MODE, LPG, RT>(a, nchunks, st);
      case 0: return launch_warp<NM, MODE, LPG, RT>(a, nchunks, st);
      default: break;
    }
  }
  return launch_fast<NM, MODE, LPG, RT, PEER>(a, nchunks, st);
}

template <int NM, int MODE, bool PEER>
int dispatch_fast_mode(const ModeArgs &a, int64_t nchunks, cudaStream_t st) {
  if (a.rank == 32) return launch_choice<NM, MODE, 8, 32, PEER>(a, nchunks, st);
  if (a.rank == 16) return launch_choice<NM, MODE, 4, 16, PEER>(a, nchunks, st);
  return launch_choice<NM, MODE, 16, 0, PEER>(a, nchunks, st);  // any R % 4 == 0 up to 64
}

template <int NM, bool PEER = false>
int dispatch_fast(const ModeArgs &a, int64_t nchunks, cudaStream_t st) {
  switch (a.mode) {
    case 0: return dispatch_fast_mode<NM, 0, PEER>(a, nchunks, st);
    case 1: return dispatch_fast_mode<NM, 1, PEER>(a, nchunks, st);
    case 2: if constexpr (NM > 2) return dispatch_fast_mode<NM, (NM > 2 ? 2 : 0), PEER>(a, nchunks, st);
            break;
    case 3: if constexpr (NM > 3) return dispatch_fast_mode<NM, (NM > 3 ? 3 : 0), PEER>(a, nchunks, st);
            break;
    default: break;
  }
  set_error("fast path: mode %d out of range for N=%d", a.mode, NM);
  return FC_ERR_ARG;
}

}  // namespace fc
