// Fast-path mode-pass instantiations for N = 3 (see fast_kernel.cuh).
#include "dispatch.cuh"

namespace fc {
int fast_dispatch_n3(const ModeArgs &a, int64_t nchunks, cudaStream_t st) {
  return dispatch_fast<3>(a, nchunks, st);
}
}  // namespace fc
