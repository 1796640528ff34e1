// Peer-memory plumbing for the multi-GPU fused exchange (dist.py, exchange
// "p2p"): IPC-shareable device allocations, their handles, peer mappings and
// stream-ordered copies between them.  One process per GPU; the handles are
// exchanged through torch.distributed on the host.  Allocations come from
// cudaMalloc (not torch's allocator) because legacy IPC handles cover whole
// cudaMalloc allocations and torch's expandable segments are not IPC-able.
#include "common.cuh"

using namespace fc;

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

}  // extern "C"
