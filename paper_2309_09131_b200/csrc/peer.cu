// Peer-memory plumbing for the multi-GPU fused exchange (dist.py, exchange
// "p2p"): IPC-shareable device allocations, their handles, peer mappings and
// stream-ordered copies between them.  One process per GPU; the handles are
// exchanged through torch.distributed on the host.  Allocations come from
// cudaMalloc (not torch's allocator) because legacy IPC handles cover whole
// cudaMalloc allocations and torch's expandable segments are not IPC-able.
#include <cuda.h>
#include <string.h>

#include "common.cuh"
#include "mode_args.cuh"

using namespace fc;

namespace {
// One launch for the factor-row all-gather of the fused exchange: GPU q's
// owned rows [row_lo[q], row_lo[q+1]) are read from q's output buffer over
// NVLink (16-B loads) into this GPU's copy.  Blocks stride over the rows of
// all peers; the local range (self) is skipped.
__global__ void __launch_bounds__(256) gather_peer_rows_kernel(float4 *dst, PeerRows pr, int self,
                                                               int64_t row_vec) {
  for (int q = 0; q < pr.n; ++q) {
    if (q == self) continue;
    const float4 *src = reinterpret_cast<const float4 *>(pr.src[q]);
    const int64_t v0 = pr.row_lo[q] * row_vec, v1 = pr.row_lo[q + 1] * row_vec;
    for (int64_t v = v0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < v1;
         v += (int64_t)gridDim.x * blockDim.x)
      dst[v] = src[v];
  }
}

// Stream memory operations, resolved through the runtime so the library has
// no link-time dependency on libcuda (it loads on hosts without a driver).
typedef CUresult (*StreamValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

StreamValueFn driver_fn(const char *name) {
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion(name, &fn, 12000, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<StreamValueFn>(fn);
}

// Whether the current device can flush remote (NVLink) writes ahead of a
// stream wait (CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES), queried once per
// device -- a query, not a stream operation, so it is also safe while the
// stream is being captured into a graph.  -1 on a query failure.
int can_flush_remote_writes() {
  typedef CUresult (*AttrFn)(int *, CUdevice_attribute, CUdevice);
  static AttrFn attr = [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuDeviceGetAttribute", &fn, 12000, cudaEnableDefault, &q) !=
            cudaSuccess || q != cudaDriverEntryPointSuccess)
      return (AttrFn) nullptr;
    return reinterpret_cast<AttrFn>(fn);
  }();
  static int cached[64];
  static bool init = [] {
    for (int &c : cached) c = -2;
    return true;
  }();
  (void)init;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || !attr) return -1;
  if (cached[dev] == -2) {
    int v = 0;
    cached[dev] = attr(&v, CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES, (CUdevice)dev) == CUDA_SUCCESS
                      ? (v != 0)
                      : -1;
  }
  return cached[dev];
}
}  // namespace

extern "C" {

int fc_ipc_handle_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }

int fc_ipc_alloc(int64_t bytes, void **ptr) {
  FC_CHECK_ARG(ptr && bytes > 0, "bad allocation request");
  *ptr = nullptr;
  FC_CUDA_TRY(cudaMalloc(ptr, (size_t)bytes));
  return FC_OK;
}

int fc_ipc_free(void *ptr) {
  if (ptr) FC_CUDA_TRY(cudaFree(ptr));
  return FC_OK;
}

int fc_ipc_handle(const void *ptr, void *handle) {
  FC_CHECK_ARG(ptr && handle, "null pointer");
  cudaIpcMemHandle_t h;
  FC_CUDA_TRY(cudaIpcGetMemHandle(&h, const_cast<void *>(ptr)));
  memcpy(handle, &h, sizeof(h));
  return FC_OK;
}

int fc_ipc_open(const void *handle, void **ptr) {
  FC_CHECK_ARG(ptr && handle, "null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  *ptr = nullptr;
  FC_CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return FC_OK;
}

int fc_ipc_close(void *ptr) {
  if (ptr) FC_CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return FC_OK;
}

int fc_copy_async(void *dst, const void *src, int64_t bytes, void *stream) {
  FC_CHECK_ARG(bytes >= 0 && (bytes == 0 || (dst && src)), "bad copy");
  if (bytes == 0) return FC_OK;
  FC_CUDA_TRY(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, as_stream(stream)));
  return FC_OK;
}

int fc_gather_peer_rows(float *dst, const float *const *peer_src, const int64_t *row_lo,
                        int npeers, int self, int64_t row_floats, void *stream) {
  FC_CHECK_ARG(npeers >= 1 && npeers <= kMaxPeers, "npeers %d outside [1, %d]", npeers, kMaxPeers);
  FC_CHECK_ARG(dst && peer_src && row_lo, "null argument");
  FC_CHECK_ARG(row_floats > 0 && row_floats % 4 == 0, "row width must be a multiple of 4 floats");
  PeerRows pr{};
  pr.n = npeers;
  int64_t vecs = 0;
  for (int q = 0; q < npeers; ++q) {
    FC_CHECK_ARG(q == self || peer_src[q], "null peer rows %d", q);
    FC_CHECK_ARG(row_lo[q + 1] >= row_lo[q], "row ranges not monotone");
    pr.src[q] = peer_src[q];
    pr.row_lo[q] = row_lo[q];
    if (q != self) vecs += (row_lo[q + 1] - row_lo[q]) * (row_floats / 4);
  }
  pr.row_lo[npeers] = row_lo[npeers];
  if (vecs == 0) return FC_OK;
  const int grid = (int)min64((vecs + 255) / 256, 148 * 8);
  gather_peer_rows_kernel<<<grid, 256, 0, as_stream(stream)>>>(reinterpret_cast<float4 *>(dst), pr,
                                                             self, row_floats / 4);
  FC_LAUNCH_CHECK();
  return FC_OK;
}

// Cross-GPU ordering without the host (fused exchange barrier): the GPU's
// front end writes / waits on 32-bit flags in (peer-mapped) device memory.
// The write fences the stream's prior memory operations, so a peer that
// observes the flag also observes this GPU's records and output rows.  No
// SM spins: safe even when several processes share one GPU.
int fc_stream_signal(void *flag, uint32_t value, void *stream) {
  static StreamValueFn fn = driver_fn("cuStreamWriteValue32");
  FC_CHECK_ARG(flag, "null flag");
  if (!fn) {
    set_error("cuStreamWriteValue32 unavailable");
    return FC_ERR_CUDA;
  }
  CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value, 0);
  if (r != CUDA_SUCCESS) {
    set_error("cuStreamWriteValue32 failed (%d)", (int)r);
    return FC_ERR_CUDA;
  }
  return FC_OK;
}

int fc_stream_wait_flush_supported(void) { return can_flush_remote_writes(); }

int fc_stream_wait(const void *flag, uint32_t value, void *stream) {
  static StreamValueFn fn = driver_fn("cuStreamWaitValue32");
  FC_CHECK_ARG(flag, "null flag");
  if (!fn) {
    set_error("cuStreamWaitValue32 unavailable");
    return FC_ERR_CUDA;
  }
  // FLUSH (devices that support it, per the device attribute): the peers'
  // NVLink stores that precede their flag write are visible to this stream's
  // later kernels.  Any failure of the wait itself is an error.
  const int flush = can_flush_remote_writes();
  if (flush < 0) {
    set_error("cuDeviceGetAttribute(CAN_FLUSH_REMOTE_WRITES) failed");
    return FC_ERR_CUDA;
  }
  const unsigned flags = CU_STREAM_WAIT_VALUE_GEQ | (flush ? CU_STREAM_WAIT_VALUE_FLUSH : 0u);
  const CUresult r = fn(reinterpret_cast<CUstream>(stream),
                        reinterpret_cast<CUdeviceptr>(const_cast<void *>(flag)), value, flags);
  if (r != CUDA_SUCCESS) {
    set_error("cuStreamWaitValue32 failed (%d)", (int)r);
    return FC_ERR_CUDA;
  }
  return FC_OK;
}

}  // extern "C"
