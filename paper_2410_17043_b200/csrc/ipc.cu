// Peer-memory plumbing for the multi-GPU layer: CUDA IPC handles for the
// buffers other GPUs store into (receive / return rows, arrival counters).
// The engine then writes those peers' HBM directly over NVSwitch.
#include <cuda.h>
#include <string.h>

#include "common.cuh"

namespace {
typedef CUresult (*GetRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

GetRangeFn get_range_fn() {
  static GetRangeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<GetRangeFn>(p);
  }
  return fn;
}
}  // namespace

extern "C" int aurora_ipc_get(const void* ptr, void* handle, int64_t* offset) {
  if (!ptr || !handle || !offset) return AURORA_EINVAL;
  GetRangeFn fn = get_range_fn();
  if (!fn) return AURORA_ECUDA;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return AURORA_ECUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, (void*)base) != cudaSuccess) return AURORA_ECUDA;
  memcpy(handle, &h, sizeof(h));
  *offset = (int64_t)((CUdeviceptr)ptr - base);
  return AURORA_OK;
}

extern "C" int aurora_ipc_open(const void* handle, int64_t offset, void** out) {
  if (!handle || !out) return AURORA_EINVAL;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return AURORA_ECUDA;
  *out = (char*)base + offset;
  return AURORA_OK;
}

extern "C" int aurora_ipc_close(void* base) {
  return cudaIpcCloseMemHandle(base) == cudaSuccess ? AURORA_OK : AURORA_ECUDA;
}

extern "C" int aurora_ipc_handle_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }
