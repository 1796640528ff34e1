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

// TMA variant: one lane per group issues cp.async.bulk copies of the U x 2
// factor rows (128 B each) into a per-group shared staging buffer tracked by
// an mbarrier (double-buffered); the group then reads them with LDS.128.
// No registers are held by in-flight rows.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int U>
__global__ void __launch_bounds__(256) probe_tma(const uint2 *idx, int64_t n, const float *F1,
                                                 const float *F2, float *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int gi = threadIdx.x >> 3, lg = threadIdx.x & 7;
  float4 *stage = reinterpret_cast<float4 *>(sm) + (size_t)gi * 2 * U * 16;  // [2][U][2 rows][8 f4]
  uint64_t *mbar = reinterpret_cast<uint64_t *>(sm + 32 * 2 * U * 256) + gi * 2;
  if (lg == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar + b)));
  }
  __syncwarp();
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncthreads();
  const int64_t groups = (int64_t)gridDim.x * 32;
  const int64_t g = (int64_t)blockIdx.x * 32 + gi;
  float4 acc = make_float4(0, 0, 0, 0);
  auto issue = [&](int64_t base, int b) {
    if (lg == 0) {
      const uint32_t mb = smem_u32(mbar + b);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(U * 256));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint2 c = idx[min(base + u, n - 1)];
        float4 *dst = stage + ((size_t)b * U + u) * 16;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];"
            ::"r"(smem_u32(dst)), "l"(F1 + (uint64_t)c.x * 32), "r"(mb) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];"
            ::"r"(smem_u32(dst + 8)), "l"(F2 + (uint64_t)c.y * 32), "r"(mb) : "memory");
      }
    }
  };
  auto wait = [&](int b, uint32_t parity) {
    const uint32_t mb = smem_u32(mbar + b);
    uint32_t done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(mb), "r"(parity) : "memory");
    }
  };
  int64_t base = g * U;
  uint32_t ph[2] = {0, 0};
  int b = 0;
  if (base < n) issue(base, 0);
  for (; base < n; base += groups * U) {
    const int64_t nxt = base + groups * U;
    if (nxt < n) issue(nxt, b ^ 1);
    wait(b, ph[b]);
    ph[b] ^= 1;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float4 x = stage[((size_t)b * U + u) * 16 + lg];
      const float4 y = stage[((size_t)b * U + u) * 16 + 8 + lg];
      acc.x += x.x * y.x;
      acc.y += x.y * y.y;
      acc.z += x.z * y.z;
      acc.w += x.w * y.w;
    }
    __syncwarp();
    b ^= 1;
  }
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) sink[0] = acc.x;
}

extern "C" float gather_probe_tma(const uint2 *idx, int64_t n, const float *F1, const float *F2,
                                  float *sink, int u, int blocks) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t smem = (size_t)32 * 2 * u * 256 + 32 * 2 * 8;
  if (u == 4) cudaFuncSetAttribute(probe_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  else cudaFuncSetAttribute(probe_tma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int it = 0; it < 2; ++it) {
    cudaEventRecord(e0);
    if (u == 4) probe_tma<4><<<blocks, 256, smem>>>(idx, n, F1, F2, sink);
    else probe_tma<8><<<blocks, 256, smem>>>(idx, n, F1, F2, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ms : -1.f;
}

// TEX variant: factor rows fetched through the texture path
// (tex1Dfetch<float4> on a linear-memory texture object) -- does the TEX
// data path add L1 -> RF bandwidth beside the LSU path?  both = 0: F1 by
// LDG, F2 by TEX; both = 1: both by TEX.
template <int U, int BOTH>
__global__ void __launch_bounds__(256) probe_tex(const uint2 *idx, int64_t n, const float *F1,
                                                 cudaTextureObject_t T1, cudaTextureObject_t T2,
                                                 float *sink) {
  const int lg = threadIdx.x & 7;
  const int64_t groups = (int64_t)gridDim.x * 32;
  int64_t g = (int64_t)blockIdx.x * 32 + (threadIdx.x >> 3);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t base = g * U; base < n; base += groups * U) {
    float4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint2 c = idx[min(base + u, n - 1)];
      if (BOTH) a[u] = tex1Dfetch<float4>(T1, (int)(c.x * 8 + lg));
      else a[u] = __ldg(reinterpret_cast<const float4 *>(F1 + (uint64_t)c.x * 32 + lg * 4));
      b[u] = tex1Dfetch<float4>(T2, (int)(c.y * 8 + lg));
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

static cudaTextureObject_t tex_of(const float *p, int64_t floats) {
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = const_cast<float *>(p);
  rd.res.linear.desc = cudaCreateChannelDesc<float4>();
  rd.res.linear.sizeInBytes = (size_t)floats * 4;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t t = 0;
  cudaCreateTextureObject(&t, &rd, &td, nullptr);
  return t;
}

extern "C" float gather_probe_tex(const uint2 *idx, int64_t n, const float *F1, int64_t f1_floats,
                                  const float *F2, int64_t f2_floats, float *sink, int u,
                                  int blocks, int both) {
  cudaTextureObject_t T1 = tex_of(F1, f1_floats), T2 = tex_of(F2, f2_floats);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 2; ++it) {
    cudaEventRecord(e0);
    if (both) {
      if (u == 4) probe_tex<4, 1><<<blocks, 256>>>(idx, n, F1, T1, T2, sink);
      else probe_tex<8, 1><<<blocks, 256>>>(idx, n, F1, T1, T2, sink);
    } else {
      if (u == 4) probe_tex<4, 0><<<blocks, 256>>>(idx, n, F1, T1, T2, sink);
      else probe_tex<8, 0><<<blocks, 256>>>(idx, n, F1, T1, T2, sink);
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaDestroyTextureObject(T1);
  cudaDestroyTextureObject(T2);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ms : -1.f;
}
