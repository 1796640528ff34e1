// Fast-path mode-pass instantiations for N = 3 (see fast_kernel.cuh).
#include "dispatch.cuh"

namespace fc {
int fast_dispatch_n3(const ModeArgs &a, int64_t nchunks, cudaStream_t st) {
  return dispatch_fast<3>(a, nchunks, st);
}
}  // namespace fc

#ifdef FAST_PHASE_TIMING
extern "C" int fc_debug_phase_cycles(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, fc::g_phase_cycles, sizeof(unsigned long long) * 5);
  if (reset) {
    unsigned long long z[5] = {0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(fc::g_phase_cycles, z, sizeof(z));
  }
  return 0;
}
#endif
