// K5: FLYCOO layout build on the device (replaces layout.build_sharded,
// /root/reference/pkg/src/modecycle/layout.py:462-531, and
// morton.interleave, morton.py:20-44), plus K6, the measurement-input
// generator (bench/tests only; coo.synth_tensor's role, coo.py:323-399).
//
// The canonical mode-n order is lexsort(seq, lo, hi, iv_n): elements sorted
// by super-shard, then Morton key of all modes' interval coordinates, ties
// by input position.  On the device that is a chain of stable LSD radix
// sorts (CUB onesweep) of element ids that start in input order, so "ties
// by input position" comes for free.  Everything here is integer work and
// bit-exact with the reference.
#include <cub/device/device_radix_sort.cuh>

#include <stdarg.h>
#include <string.h>

#include "common.cuh"

namespace fc {

static thread_local char g_err[512];

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

namespace {

constexpr int kMaxModes = 8;

struct MortonPlan {
  int nmodes;
  int maxw;
  int width[kMaxModes];
  int64_t m[kMaxModes];
};

// morton.py:20-44: level b, then mode w ascending; bit position grows by one
// for every (b, w) with b < width[w]; positions >= 64 land in hi.
__global__ void morton_kernel(const int32_t *coords, int64_t nnz, MortonPlan mp, uint64_t *hi,
                              uint64_t *lo) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t iv[kMaxModes];
#pragma unroll
    for (int w = 0; w < kMaxModes; ++w)
      iv[w] = w < mp.nmodes ? (uint64_t)(coords[i * mp.nmodes + w] / mp.m[w]) : 0;
    uint64_t h = 0, l = 0;
    int pos = 0;
    for (int b = 0; b < mp.maxw; ++b) {
#pragma unroll
      for (int w = 0; w < kMaxModes; ++w) {
        if (w >= mp.nmodes || b >= mp.width[w]) continue;
        const uint64_t bit = (iv[w] >> b) & 1ull;
        if (pos < 64) l |= bit << pos;
        else h |= bit << (pos - 64);
        ++pos;
      }
    }
    if (hi) hi[i] = h;
    lo[i] = l;
  }
}

__global__ void gather_key_kernel(const uint32_t *ids, int64_t n, int what, const uint64_t *hi,
                                  const uint64_t *lo, const int32_t *coords, int nmodes, int mode,
                                  int64_t m, int shift, uint64_t *keys) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t id = ids[p];
    uint64_t k;
    switch (what) {
      case 0: k = lo[id]; break;
      case 1: k = hi[id]; break;
      case 2: k = (uint64_t)(coords[(int64_t)id * nmodes + mode] / m); break;
      default:
        k = ((uint64_t)(coords[(int64_t)id * nmodes + mode] / m) << shift) | lo[id];
        break;
    }
    keys[p] = k;
  }
}

__global__ void ss_hist_kernel(const int32_t *coords, int64_t nnz, int nmodes, int mode, int64_t m,
                               int64_t k, unsigned long long *hist) {
  extern __shared__ unsigned int sh[];
  const bool use_smem = k <= 8192;
  if (use_smem) {
    for (int64_t b = threadIdx.x; b < k; b += blockDim.x) sh[b] = 0;
    __syncthreads();
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = coords[i * nmodes + mode] / m;
    if (use_smem) atomicAdd(&sh[b], 1u);
    else atomicAdd(&hist[b], 1ull);
  }
  if (use_smem) {
    __syncthreads();
    for (int64_t b = threadIdx.x; b < k; b += blockDim.x)
      if (sh[b]) atomicAdd(&hist[b], (unsigned long long)sh[b]);
  }
}

// layout.py:491-492: sid = first[iv] + (pos - offs[iv]) // g, pos = p.
__global__ void shard_id_kernel(const uint32_t *order, int64_t nnz, const int32_t *coords,
                                int nmodes, int mode, int64_t m, const int64_t *offs,
                                const int64_t *first, int64_t g, uint32_t *sid) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t id = order[p];
    const int64_t iv = coords[(int64_t)id * nmodes + mode] / m;
    sid[id] = (uint32_t)(first[iv] + (p - offs[iv]) / g);
  }
}

__global__ void device_key_kernel(const uint32_t *ids, int64_t n, const uint32_t *sid_mode,
                                  const uint32_t *sid_prev, uint64_t *keys) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t id = ids[p];
    keys[p] = ((uint64_t)sid_mode[id] << 32) | sid_prev[id];
  }
}

__global__ void invert_kernel(const uint32_t *order, int64_t n, uint32_t *pos) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    pos[order[p]] = (uint32_t)p;
}

__global__ void slots_kernel(const uint32_t *order, const uint32_t *pos_next, int64_t n,
                             uint32_t *slot) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    slot[p] = pos_next[order[p]];
}

// slot[pos_n[id]] = pos_next[id]: the slot map from positions only (no orders)
__global__ void slots_scatter_kernel(const uint32_t *pos_n, const uint32_t *pos_next, int64_t n,
                                     uint32_t *slot) {
  for (int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; id < n;
       id += (int64_t)gridDim.x * blockDim.x)
    slot[pos_n[id]] = pos_next[id];
}

// crd[pos[id]] = record of input element id
__global__ void records_scatter_kernel(const uint32_t *pos, int64_t n, int nmodes,
                                       const int32_t *coords, const float *vals, int32_t *crd,
                                       float *val_out) {
  const int cw = crd_words(nmodes);
  const bool emb = value_embedded(nmodes);
  for (int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; id < n;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = pos[id];
    int32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int q = 0; q < nmodes; ++q) w[q] = coords[id * nmodes + q];
    const float v = vals[id];
    if (emb) w[cw - 1] = __float_as_int(v);
    else val_out[p] = v;
    int4 *dst = reinterpret_cast<int4 *>(crd + p * cw);
    dst[0] = make_int4(w[0], w[1], w[2], w[3]);
    if (cw == 8) dst[1] = make_int4(w[4], w[5], w[6], w[7]);
  }
}

__global__ void records_kernel(const uint32_t *order, int64_t n, int nmodes, const int32_t *coords,
                               const float *vals, int32_t *crd, float *val_out) {
  const int cw = crd_words(nmodes);
  const bool emb = value_embedded(nmodes);
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t id = order[p];
    int32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int q = 0; q < nmodes; ++q) w[q] = coords[(int64_t)id * nmodes + q];
    const float v = vals[id];
    if (emb) w[cw - 1] = __float_as_int(v);
    else val_out[p] = v;
    int4 *dst = reinterpret_cast<int4 *>(crd + p * cw);
    dst[0] = make_int4(w[0], w[1], w[2], w[3]);
    if (cw == 8) dst[1] = make_int4(w[4], w[5], w[6], w[7]);
  }
}

// ------------------------------------------------------------------ K6
struct SynthPlan {
  int nmodes;
  int64_t dims[kMaxModes];
  const double *cdf[kMaxModes];
  int64_t cdf_len[kMaxModes];
};

__global__ void synth_draw_kernel(uint64_t seed, int64_t ndraws, SynthPlan sp, int32_t *coords) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < ndraws;
       j += (int64_t)gridDim.x * blockDim.x) {
    for (int w = 0; w < sp.nmodes; ++w) {
      const Philox4 r = philox4x32_10((uint32_t)j, (uint32_t)((uint64_t)j >> 32), (uint32_t)w,
                                      0x5EEDu, k0, k1);
      const double u = u01_53(r.x, r.y);
      int64_t idx;
      if (sp.cdf[w] == nullptr) {
        idx = (int64_t)(u * (double)sp.dims[w]);
        if (idx >= sp.dims[w]) idx = sp.dims[w] - 1;
      } else {
        // smallest i with u < cdf[i]
        int64_t lo = 0, hi = sp.cdf_len[w] - 1;
        const double *c = sp.cdf[w];
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (u < c[mid]) hi = mid;
          else lo = mid + 1;
        }
        idx = lo;
      }
      coords[j * sp.nmodes + w] = (int32_t)idx;
    }
  }
}

// Mixed-radix linear key (mode 0 most significant) as a 128-bit (hi, lo).
__global__ void synth_keys_kernel(const int32_t *coords, int64_t n, int nmodes, SynthPlan sp,
                                  uint64_t *hi, uint64_t *lo) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    unsigned __int128 key = 0;
    for (int w = 0; w < nmodes; ++w)
      key = key * (unsigned __int128)sp.dims[w] + (unsigned __int128)coords[i * nmodes + w];
    hi[i] = (uint64_t)(key >> 64);
    lo[i] = (uint64_t)key;
  }
}

__global__ void mark_first_kernel(const uint64_t *hs, const uint64_t *ls, const uint32_t *ids,
                                  int64_t n, uint8_t *keep) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const bool first = p == 0 || hs[p] != hs[p - 1] || ls[p] != ls[p - 1];
    keep[ids[p]] = first ? 1 : 0;
  }
}

__global__ void uniform_kernel(uint64_t seed, uint32_t sid, int64_t n, float *out, int open_low) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Philox4 r = philox4x32_10((uint32_t)i, (uint32_t)((uint64_t)i >> 32), sid, 0xF00Du, k0, k1);
    out[i] = u01_24(r.x, open_low != 0);
  }
}

// ---------------------------------------------- lean build (c5-size tensors)
// Same orders as above with 32-bit sort keys and records read in place
// (coordinates at a stride of crd_words), so the whole build runs inside the
// memory of the final layout (layout.build_device_sharded_lean).
__global__ void iota_kernel(uint32_t *out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)i;
}

__global__ void morton32_kernel(const int32_t *crd, int64_t n, int cs, MortonPlan mp, uint32_t *key) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t iv[kMaxModes];
#pragma unroll
    for (int w = 0; w < kMaxModes; ++w)
      iv[w] = w < mp.nmodes ? (uint32_t)(crd[i * cs + w] / mp.m[w]) : 0u;
    uint32_t l = 0;
    int pos = 0;
    for (int b = 0; b < mp.maxw; ++b) {
#pragma unroll
      for (int w = 0; w < kMaxModes; ++w) {
        if (w >= mp.nmodes || b >= mp.width[w]) continue;
        l |= ((iv[w] >> b) & 1u) << pos;
        ++pos;
      }
    }
    key[i] = l;
  }
}

__global__ void iv_key32_kernel(const uint32_t *ids, int64_t n, const int32_t *crd, int cs, int mode,
                                int64_t m, uint32_t *keys) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    keys[p] = (uint32_t)(crd[(int64_t)ids[p] * cs + mode] / m);
}

__global__ void gather_u32_kernel(const uint32_t *ids, int64_t n, const uint32_t *src, uint32_t *dst) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    dst[p] = src[ids[p]];
}

// dst[pos[i]] = src[i] for 16-byte records (src = a batch of the input order)
__global__ void scatter_rec16_kernel(const uint32_t *pos, int64_t n, const int4 *src, int4 *dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[pos[i]] = src[i];
}

// coordinates of modes [w0, w1) of the draws js[i] (same law as synth_draw_kernel)
__global__ void synth_draw_at_kernel(uint64_t seed, const int64_t *js, int64_t n, SynthPlan sp,
                                     int w0, int w1, int32_t *out, int cs) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t j = (uint64_t)js[i];
    for (int w = w0; w < w1; ++w) {
      const Philox4 r = philox4x32_10((uint32_t)j, (uint32_t)(j >> 32), (uint32_t)w, 0x5EEDu, k0, k1);
      const double u = u01_53(r.x, r.y);
      int64_t idx;
      if (sp.cdf[w] == nullptr) {
        idx = (int64_t)(u * (double)sp.dims[w]);
        if (idx >= sp.dims[w]) idx = sp.dims[w] - 1;
      } else {
        int64_t lo = 0, hi = sp.cdf_len[w] - 1;
        const double *c = sp.cdf[w];
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (u < c[mid]) hi = mid;
          else lo = mid + 1;
        }
        idx = lo;
      }
      out[i * cs + (w - w0)] = (int32_t)idx;
    }
  }
}

inline int grid_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return (int)(b < 148 * 32 ? (b > 0 ? b : 1) : 148 * 32);
}

}  // namespace
}  // namespace fc

using namespace fc;

extern "C" {

int fc_version(void) { return 1; }
const char *fc_last_error(void) { return g_err; }
int fc_crd_words(int nmodes) { return (nmodes >= 2 && nmodes <= 8) ? crd_words(nmodes) : -1; }
int fc_value_embedded(int nmodes) { return (nmodes >= 2 && nmodes <= 8) ? (value_embedded(nmodes) ? 1 : 0) : -1; }

int fc_build_morton(const int32_t *coords, int64_t nnz, int nmodes, const int64_t *m,
                    const int64_t *k, uint64_t *hi, uint64_t *lo, void *stream) {
  FC_CHECK_ARG(nmodes >= 2 && nmodes <= kMaxModes, "nmodes %d", nmodes);
  FC_CHECK_ARG(coords && lo && m && k, "null argument");
  MortonPlan mp{};
  mp.nmodes = nmodes;
  int total = 0;
  for (int w = 0; w < nmodes; ++w) {
    FC_CHECK_ARG(m[w] >= 1 && k[w] >= 1, "bad m/k");
    mp.m[w] = m[w];
    mp.width[w] = bit_length_u64((uint64_t)(k[w] - 1));
    total += mp.width[w];
    if (mp.width[w] > mp.maxw) mp.maxw = mp.width[w];
  }
  if (total > 128) {
    set_error("morton key would need %d bits (> 128)", total);
    return FC_ERR_UNSUPPORTED;
  }
  FC_CHECK_ARG(hi || total <= 64, "hi word needed for a %d-bit key", total);
  if (nnz == 0) return FC_OK;
  morton_kernel<<<grid_for(nnz), 256, 0, as_stream(stream)>>>(coords, nnz, mp, hi, lo);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int64_t fc_build_sort_temp_bytes(int64_t nnz) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                  (const uint32_t *)nullptr, (uint32_t *)nullptr, nnz, 0, 64);
  return (int64_t)bytes;
}

int fc_build_sort_pairs(const uint64_t *keys_in, uint64_t *keys_out, const uint32_t *ids_in,
                        uint32_t *ids_out, int64_t nnz, int end_bit, void *temp,
                        int64_t temp_bytes, void *stream) {
  FC_CHECK_ARG(end_bit >= 1 && end_bit <= 64, "end_bit %d", end_bit);
  if (nnz == 0) return FC_OK;
  size_t bytes = (size_t)temp_bytes;
  FC_CUDA_TRY(cub::DeviceRadixSort::SortPairs(temp, bytes, keys_in, keys_out, ids_in, ids_out, nnz,
                                              0, end_bit, as_stream(stream)));
  return FC_OK;
}

int fc_build_gather_key(const uint32_t *ids, int64_t nnz, int what, const uint64_t *hi,
                        const uint64_t *lo, const int32_t *coords, int nmodes, int mode, int64_t m,
                        int shift, uint64_t *keys, void *stream) {
  FC_CHECK_ARG(what >= 0 && what <= 3, "what %d", what);
  if (nnz == 0) return FC_OK;
  gather_key_kernel<<<grid_for(nnz), 256, 0, as_stream(stream)>>>(ids, nnz, what, hi, lo, coords,
                                                                  nmodes, mode, m, shift, keys);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_build_ss_hist(const int32_t *coords, int64_t nnz, int nmodes, int mode, int64_t m, int64_t k,
                     unsigned long long *hist, void *stream) {
  FC_CHECK_ARG(coords && hist && m >= 1 && k >= 1, "bad argument");
  FC_CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * k, as_stream(stream)));
  if (nnz == 0) return FC_OK;
  const size_t sh = k <= 8192 ? sizeof(unsigned) * k : 0;
  ss_hist_kernel<<<grid_for(nnz), 256, sh, as_stream(stream)>>>(coords, nnz, nmodes, mode, m, k, hist);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_build_shard_ids(const uint32_t *order, int64_t nnz, const int32_t *coords, int nmodes,
                       int mode, int64_t m, const int64_t *ss_offs, const int64_t *ss_first,
                       int64_t g, uint32_t *sid, void *stream) {
  FC_CHECK_ARG(g >= 1, "g %lld", (long long)g);
  if (nnz == 0) return FC_OK;
  shard_id_kernel<<<grid_for(nnz), 256, 0, as_stream(stream)>>>(order, nnz, coords, nmodes, mode, m,
                                                                ss_offs, ss_first, g, sid);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_build_device_key(const uint32_t *ids, int64_t nnz, const uint32_t *sid_mode,
                        const uint32_t *sid_prev, uint64_t *keys, void *stream) {
  if (nnz == 0) return FC_OK;
  device_key_kernel<<<grid_for(nnz), 256, 0, as_stream(stream)>>>(ids, nnz, sid_mode, sid_prev, keys);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_build_invert(const uint32_t *order, int64_t nnz, uint32_t *pos, void *stream) {
  if (nnz == 0) return FC_OK;
  invert_kernel<<<grid_for(nnz), 256, 0, as_stream(stream)>>>(order, nnz, pos);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_build_slots(const uint32_t *order, const uint32_t *pos_next, int64_t nnz, uint32_t *slot,
                   void *stream) {
  if (nnz == 0) return FC_OK;
  slots_kernel<<<grid_for(nnz), 256, 0, as_stream(stream)>>>(order, pos_next, nnz, slot);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_build_slots_scatter(const uint32_t *pos_n, const uint32_t *pos_next, int64_t nnz,
                           uint32_t *slot, void *stream) {
  if (nnz == 0) return FC_OK;
  slots_scatter_kernel<<<grid_for(nnz), 256, 0, as_stream(stream)>>>(pos_n, pos_next, nnz, slot);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_build_records_scatter(const uint32_t *pos, int64_t nnz, int nmodes, const int32_t *coords,
                             const float *vals, void *crd, float *val_out, void *stream) {
  FC_CHECK_ARG(nmodes >= 2 && nmodes <= kMaxModes, "nmodes %d", nmodes);
  FC_CHECK_ARG(value_embedded(nmodes) || val_out, "separate value array required");
  if (nnz == 0) return FC_OK;
  records_scatter_kernel<<<grid_for(nnz), 256, 0, as_stream(stream)>>>(
      pos, nnz, nmodes, coords, vals, static_cast<int32_t *>(crd), val_out);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_build_records(const uint32_t *order, int64_t nnz, int nmodes, const int32_t *coords,
                     const float *vals, void *crd, float *val_out, void *stream) {
  FC_CHECK_ARG(nmodes >= 2 && nmodes <= kMaxModes, "nmodes %d", nmodes);
  FC_CHECK_ARG(value_embedded(nmodes) || val_out, "separate value array required");
  if (nnz == 0) return FC_OK;
  records_kernel<<<grid_for(nnz), 256, 0, as_stream(stream)>>>(order, nnz, nmodes, coords, vals,
                                                               static_cast<int32_t *>(crd), val_out);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_synth_draw(uint64_t seed, int64_t ndraws, int nmodes, const int64_t *dims,
                  const double *const *cdfs, const int64_t *cdf_len, int32_t *coords,
                  void *stream) {
  FC_CHECK_ARG(nmodes >= 2 && nmodes <= kMaxModes, "nmodes %d", nmodes);
  SynthPlan sp{};
  sp.nmodes = nmodes;
  for (int w = 0; w < nmodes; ++w) {
    FC_CHECK_ARG(dims[w] >= 1 && dims[w] <= INT32_MAX, "dims[%d]", w);
    sp.dims[w] = dims[w];
    sp.cdf[w] = cdfs ? cdfs[w] : nullptr;
    sp.cdf_len[w] = (cdfs && cdfs[w]) ? cdf_len[w] : 0;
  }
  if (ndraws == 0) return FC_OK;
  synth_draw_kernel<<<grid_for(ndraws), 256, 0, as_stream(stream)>>>(seed, ndraws, sp, coords);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_synth_keys(const int32_t *coords, int64_t n, int nmodes, const int64_t *dims, uint64_t *hi,
                  uint64_t *lo, void *stream) {
  FC_CHECK_ARG(nmodes >= 2 && nmodes <= kMaxModes, "nmodes %d", nmodes);
  SynthPlan sp{};
  sp.nmodes = nmodes;
  double bits = 0;
  for (int w = 0; w < nmodes; ++w) {
    sp.dims[w] = dims[w];
    bits += log2((double)dims[w]);
  }
  FC_CHECK_ARG(bits <= 127.0, "coordinate space too large for 128-bit keys");
  if (n == 0) return FC_OK;
  synth_keys_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(coords, n, nmodes, sp, hi, lo);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_synth_mark_first(const uint64_t *hi_sorted, const uint64_t *lo_sorted,
                        const uint32_t *ids_sorted, int64_t n, uint8_t *keep, void *stream) {
  if (n == 0) return FC_OK;
  mark_first_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(hi_sorted, lo_sorted, ids_sorted, n, keep);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_synth_uniform(uint64_t seed, uint32_t stream_id, int64_t n, float *out, int open_low,
                     void *stream) {
  if (n == 0) return FC_OK;
  uniform_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(seed, stream_id, n, out, open_low);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

// ---------------------------------------------- lean build (c5-size tensors)
int fc_build_iota(uint32_t *out, int64_t n, void *stream) {
  if (n == 0) return FC_OK;
  iota_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(out, n);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_build_morton32(const int32_t *crd, int64_t nnz, int nmodes, int cstride, const int64_t *m,
                      const int64_t *k, uint32_t *key, void *stream) {
  FC_CHECK_ARG(nmodes >= 2 && nmodes <= kMaxModes && cstride >= nmodes, "nmodes %d", nmodes);
  FC_CHECK_ARG(crd && key && m && k, "null argument");
  MortonPlan mp{};
  mp.nmodes = nmodes;
  int total = 0;
  for (int w = 0; w < nmodes; ++w) {
    FC_CHECK_ARG(m[w] >= 1 && k[w] >= 1, "bad m/k");
    mp.m[w] = m[w];
    mp.width[w] = bit_length_u64((uint64_t)(k[w] - 1));
    total += mp.width[w];
    if (mp.width[w] > mp.maxw) mp.maxw = mp.width[w];
  }
  if (total > 32) {
    set_error("morton key needs %d bits (> 32): use fc_build_morton", total);
    return FC_ERR_UNSUPPORTED;
  }
  if (nnz == 0) return FC_OK;
  morton32_kernel<<<grid_for(nnz), 256, 0, as_stream(stream)>>>(crd, nnz, cstride, mp, key);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int64_t fc_build_sort32_temp_bytes(int64_t nnz) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                  (const uint32_t *)nullptr, (uint32_t *)nullptr, nnz, 0, 32);
  return (int64_t)bytes;
}

int fc_build_sort_pairs32(const uint32_t *keys_in, uint32_t *keys_out, const uint32_t *ids_in,
                          uint32_t *ids_out, int64_t nnz, int end_bit, void *temp, int64_t temp_bytes,
                          void *stream) {
  FC_CHECK_ARG(end_bit >= 1 && end_bit <= 32, "end_bit %d", end_bit);
  if (nnz == 0) return FC_OK;
  size_t bytes = (size_t)temp_bytes;
  FC_CUDA_TRY(cub::DeviceRadixSort::SortPairs(temp, bytes, keys_in, keys_out, ids_in, ids_out, nnz,
                                              0, end_bit, as_stream(stream)));
  return FC_OK;
}

int fc_build_iv_key32(const uint32_t *ids, int64_t n, const int32_t *crd, int cstride, int mode,
                      int64_t m, uint32_t *keys, void *stream) {
  FC_CHECK_ARG(m >= 1 && cstride > mode, "bad argument");
  if (n == 0) return FC_OK;
  iv_key32_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(ids, n, crd, cstride, mode, m, keys);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_build_gather_u32(const uint32_t *ids, int64_t n, const uint32_t *src, uint32_t *dst,
                        void *stream) {
  if (n == 0) return FC_OK;
  gather_u32_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(ids, n, src, dst);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_build_scatter_rec16(const uint32_t *pos, int64_t n, const void *src, void *dst, void *stream) {
  if (n == 0) return FC_OK;
  scatter_rec16_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(
      pos, n, static_cast<const int4 *>(src), static_cast<int4 *>(dst));
  FC_LAUNCH_CHECK();
  return FC_OK;
}

int fc_synth_draw_at(uint64_t seed, const int64_t *js, int64_t n, int nmodes, const int64_t *dims,
                     const double *const *cdfs, const int64_t *cdf_len, int mode_lo, int mode_hi,
                     int32_t *out, int cstride, void *stream) {
  FC_CHECK_ARG(nmodes >= 2 && nmodes <= kMaxModes, "nmodes %d", nmodes);
  FC_CHECK_ARG(0 <= mode_lo && mode_lo < mode_hi && mode_hi <= nmodes && cstride >= mode_hi - mode_lo,
               "modes [%d, %d)", mode_lo, mode_hi);
  SynthPlan sp{};
  sp.nmodes = nmodes;
  for (int w = 0; w < nmodes; ++w) {
    FC_CHECK_ARG(dims[w] >= 1 && dims[w] <= INT32_MAX, "dims[%d]", w);
    sp.dims[w] = dims[w];
    sp.cdf[w] = cdfs ? cdfs[w] : nullptr;
    sp.cdf_len[w] = (cdfs && cdfs[w]) ? cdf_len[w] : 0;
  }
  if (n == 0) return FC_OK;
  synth_draw_at_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(seed, js, n, sp, mode_lo, mode_hi,
                                                                   out, cstride);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

}  // extern "C"
