// Peer-store (multi-GPU fused exchange) mode-pass instantiations for N = 3.
#include "dispatch.cuh"

namespace fc {
int fast_dispatch_peer_n3(const ModeArgs &a, int64_t nchunks, cudaStream_t st) {
  return dispatch_fast<3, true>(a, nchunks, st);
}
}  // namespace fc
