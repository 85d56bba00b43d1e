// wavefuse-b200: CUDA IPC helpers for the peer-memory halo path of the strip
// driver (strips.py, PeerHalos).
//
// With one process per GPU, every rank exports the allocation that holds its
// PAN/MS strip (cudaIpcGetMemHandle on the allocation BASE plus the byte
// offset of the tensor inside it -- PyTorch's caching allocator sub-allocates,
// so the base comes from the driver's cuMemGetAddressRange), the handles are
// all-gathered once, and each rank maps its two ring neighbours' strips
// (cudaIpcOpenMemHandle with lazy peer access). The D4 strip kernel's
// producer then bulk-copies the neighbours' halo rows straight out of peer
// HBM over NVLink: no separate exchange step and no collective inside a
// fusion step.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <string.h>

namespace wf {

typedef int (*MemGetAddressRange)(unsigned long long*, size_t*, unsigned long long);

static MemGetAddressRange address_range_fn() {
  static MemGetAddressRange fn = [] {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libcuda.so.1", RTLD_NOW);
    if (!h) return (MemGetAddressRange) nullptr;
    return (MemGetAddressRange)dlsym(h, "cuMemGetAddressRange_v2");
  }();
  return fn;
}

cudaError_t ipc_export(const void* ptr, void* handle64, uint64_t* offset) {
  MemGetAddressRange range = address_range_fn();
  if (!range) return cudaErrorNotSupported;
  unsigned long long base = 0;
  size_t size = 0;
  if (range(&base, &size, (unsigned long long)(uintptr_t)ptr) != 0) return cudaErrorInvalidValue;
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base);
  if (e != cudaSuccess) return e;
  memcpy(handle64, &h, sizeof h);
  *offset = (uint64_t)((uintptr_t)ptr - (uintptr_t)base);
  return cudaSuccess;
}

cudaError_t ipc_open(const void* handle64, void** base) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof h);
  return cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess);
}

cudaError_t ipc_close(void* base) { return cudaIpcCloseMemHandle(base); }

}  // namespace wf
