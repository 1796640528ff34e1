// Fast-path mode-pass instantiations for N = 2 (see fast_kernel.cuh).
#include "dispatch.cuh"

namespace fc {
int fast_dispatch_n2(const ModeArgs &a, int64_t nchunks, cudaStream_t st) {
  return dispatch_fast<2>(a, nchunks, st);
}
}  // namespace fc
