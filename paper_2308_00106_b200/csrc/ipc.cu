// ipc.cu — device buffers shared between the ranks of one node (CUDA IPC), so a
// kernel on one GPU can store straight into another rank's buffer over NVLink
// (sme_spmv_seg_epi_peers).  The buffers are whole cudaMalloc allocations, so an
// opened handle maps to the buffer's first byte (no caching-allocator offsets).
#include <string.h>

#include "common.cuh"

static_assert(sizeof(cudaIpcMemHandle_t) == SME_IPC_HANDLE_BYTES, "IPC handle size");

SME_API int sme_ipc_malloc(size_t bytes, void** d_ptr) {
  SME_REQUIRE(d_ptr && bytes > 0, "bad arguments");
  SME_CUDA(cudaMalloc(d_ptr, bytes));
  return SME_OK;
}

SME_API int sme_ipc_free(void* d_ptr) {
  SME_CUDA(cudaFree(d_ptr));
  return SME_OK;
}

SME_API int sme_ipc_get_handle(void* d_ptr, uint8_t* handle) {
  SME_REQUIRE(d_ptr && handle, "bad arguments");
  cudaIpcMemHandle_t h;
  SME_CUDA(cudaIpcGetMemHandle(&h, d_ptr));
  memcpy(handle, &h, sizeof(h));
  return SME_OK;
}

SME_API int sme_ipc_open(const uint8_t* handle, void** d_ptr) {
  SME_REQUIRE(d_ptr && handle, "bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  SME_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return SME_OK;
}

SME_API int sme_ipc_close(void* d_ptr) {
  SME_CUDA(cudaIpcCloseMemHandle(d_ptr));
  return SME_OK;
}
