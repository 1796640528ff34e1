// Fast-path dispatch: (N, mode, R) -> kernel instance.  3-mode tensors run
// the packed kernel (pack_kernel.cuh: 8-B sorted records, or {c_w1, c_w2} +
// value when the input coordinates need more than 32 bits); everything else
// the one-CTA-per-chunk tile kernel (fast_kernel.cuh).
#pragma once

#include "pack_kernel.cuh"

namespace fc {

template <int NM, int MODE, int LPG, int RT, bool PEER>
int launch_choice(const ModeArgs &a, int64_t nchunks, cudaStream_t st) {
  if constexpr (NM == 3) {
    // 8-byte sorted records when the two input coordinates fit 32 bits
    const KernelVariant &kv = kernel_variant();
    if (a.plan) {
      // tile plan: the R = 32 / R = 16 packed kernels of one GPU (tile keys: t0 / kTile + chunk)
      static_assert(kFTile == kTile, "the tile plan is indexed by 2048-element tiles");
      // (the emission pass, plan == 2, never remaps: single-GPU instances only)
      if constexpr (RT == 32 || RT == 16) {
        if (a.pack_shift > 0 && kv.pack) {
          if (a.plan == 1) return launch_pack<MODE, LPG, RT, PEER, false, 1>(a, nchunks, st);
          if constexpr (!PEER) return launch_pack<MODE, LPG, RT, false, false, 2>(a, nchunks, st);
        }
        if (a.pack_shift == 0 && kv.pack_wide) {
          if (a.plan == 1) return launch_pack<MODE, LPG, RT, PEER, true, 1>(a, nchunks, st);
          if constexpr (!PEER) return launch_pack<MODE, LPG, RT, false, true, 2>(a, nchunks, st);
        }
      }
      return FC_ERR_UNSUPPORTED;
    }
    if (a.pack_shift > 0 && kv.pack) return launch_pack<MODE, LPG, RT, PEER>(a, nchunks, st);
    // wider coordinates: {c_w1, c_w2} + value array, rows from the bins
    if (a.pack_shift == 0 && kv.pack_wide) return launch_pack<MODE, LPG, RT, PEER, true>(a, nchunks, st);
  }
  if (a.plan) {  // the 4-mode tile kernels at R = 32 take a plan too
    if constexpr (NM == 4 && RT == 32) {
      static_assert(kFTile == kTile, "the tile plan is indexed by 2048-element tiles");
      if (a.plan == 1) return launch_fast<NM, MODE, LPG, RT, PEER, 1>(a, nchunks, st);
      if constexpr (!PEER) return launch_fast<NM, MODE, LPG, RT, false, 2>(a, nchunks, st);
    }
    return FC_ERR_UNSUPPORTED;
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
