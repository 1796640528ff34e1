// Peer-store (multi-GPU fused exchange) mode-pass instantiations for N = 2.
#include "dispatch.cuh"

namespace fc {
int fast_dispatch_peer_n2(const ModeArgs &a, int64_t nchunks, cudaStream_t st) {
  return dispatch_fast<2, true>(a, nchunks, st);
}
}  // namespace fc
