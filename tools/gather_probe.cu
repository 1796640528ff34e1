// Probe: throughput of the factor-row gathers alone.  One warp-group of 8
// lanes per element (float4 per lane, R = 32), U elements in flight, rows
// (c1, c2) read from a device array in the order given; sums into a
// per-thread register so nothing can be optimised away.
#include <cstdint>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(256) probe(const uint2 *idx, int64_t n, const float *F1,
                                             const float *F2, float *sink) {
  const int lg = threadIdx.x & 7;
  const int64_t groups = (int64_t)gridDim.x * 32;
  int64_t g = (int64_t)blockIdx.x * 32 + (threadIdx.x >> 3);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t base = g * U; base < n; base += groups * U) {
    float4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint2 c = idx[min(base + u, n - 1)];
      a[u] = __ldg(reinterpret_cast<const float4 *>(F1 + (uint64_t)c.x * 32 + lg * 4));
      b[u] = __ldg(reinterpret_cast<const float4 *>(F2 + (uint64_t)c.y * 32 + lg * 4));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc.x += a[u].x * b[u].x;
      acc.y += a[u].y * b[u].y;
      acc.z += a[u].z * b[u].z;
      acc.w += a[u].w * b[u].w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) sink[0] = acc.x;
}

extern "C" float gather_probe(const uint2 *idx, int64_t n, const float *F1, const float *F2,
                              float *sink, int u, int blocks) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 2; ++it) {
    cudaEventRecord(e0);
    if (u == 1) probe<1><<<blocks, 256>>>(idx, n, F1, F2, sink);
    else if (u == 4) probe<4><<<blocks, 256>>>(idx, n, F1, F2, sink);
    else probe<8><<<blocks, 256>>>(idx, n, F1, F2, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}
