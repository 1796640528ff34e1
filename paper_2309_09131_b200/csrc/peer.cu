// Peer-memory plumbing for the multi-GPU fused exchange (dist.py, exchange
// "p2p"): IPC-shareable device allocations, their handles, peer mappings and
// stream-ordered copies between them.  One process per GPU; the handles are
// exchanged through torch.distributed on the host.  Allocations come from
// cudaMalloc (not torch's allocator) because legacy IPC handles cover whole
// cudaMalloc allocations and torch's expandable segments are not IPC-able.
#include <cuda.h>
#include <string.h>

#include "common.cuh"

using namespace fc;

namespace {
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

int fc_stream_wait(const void *flag, uint32_t value, void *stream) {
  static StreamValueFn fn = driver_fn("cuStreamWaitValue32");
  FC_CHECK_ARG(flag, "null flag");
  if (!fn) {
    set_error("cuStreamWaitValue32 unavailable");
    return FC_ERR_CUDA;
  }
  CUresult r = fn(reinterpret_cast<CUstream>(stream),
                  reinterpret_cast<CUdeviceptr>(const_cast<void *>(flag)), value,
                  CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) {
    set_error("cuStreamWaitValue32 failed (%d)", (int)r);
    return FC_ERR_CUDA;
  }
  return FC_OK;
}

}  // extern "C"
