// Shared helpers for the FLYCOO sm_100a kernels: error plumbing for the C ABI,
// record layout, Philox4x32-10, read-only gathers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/flycoo.h"

namespace fc {

// Last error message, reported through fc_last_error().
void set_error(const char *fmt, ...);

#define FC_CHECK_ARG(cond, ...)          \
  do {                                   \
    if (!(cond)) {                       \
      ::fc::set_error(__VA_ARGS__);      \
      return FC_ERR_ARG;                 \
    }                                    \
  } while (0)

#define FC_CUDA_TRY(expr)                                                     \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      ::fc::set_error("%s: %s (%s:%d)", #expr, cudaGetErrorString(_e),        \
                      __FILE__, __LINE__);                                    \
      return FC_ERR_CUDA;                                                     \
    }                                                                         \
  } while (0)

#define FC_LAUNCH_CHECK() FC_CUDA_TRY(cudaGetLastError())

__host__ __device__ inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Record layout (flycoo.h): CW int32 words per element, value embedded in
// word CW-1 when N < CW, else a separate float array.
__host__ __device__ constexpr int crd_words(int n) { return n <= 4 ? 4 : 8; }
__host__ __device__ constexpr bool value_embedded(int n) { return n < crd_words(n); }

__host__ __device__ inline int bit_length_u64(uint64_t x) {
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

// ----------------------------------------------------------------- Philox
// Philox4x32-10 (Salmon et al., SC'11): counter (c0..c3), key (k0, k1).
struct Philox4 {
  uint32_t x, y, z, w;
};

__host__ __device__ inline Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                                 uint32_t c3, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)M0 * c0;
    const uint64_t p1 = (uint64_t)M1 * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += W0;
    k1 += W1;
  }
  return Philox4{c0, c1, c2, c3};
}

// 53-bit uniform double in [0, 1) from two 32-bit words.
__host__ __device__ inline double u01_53(uint32_t a, uint32_t b) {
  const uint64_t hi = a >> 5, lo = b >> 6;  // 27 + 26 bits
  return (double)(hi * 67108864ull + lo) * (1.0 / 9007199254740992.0);
}

// 24-bit uniform float in (0, 1] (open_low) or [0, 1).
__host__ __device__ inline float u01_24(uint32_t a, bool open_low) {
  const uint32_t m = a >> 8;
  return ((float)m + (open_low ? 1.0f : 0.0f)) * (1.0f / 16777216.0f);
}

}  // namespace fc
