// mpix_heap.cpp — symmetric heap for multi-process mode (one process per GPU).
//
// Every process reserves the same virtual range [base, base + n * slice) and
// maps each rank's physical allocation at base + q * slice, so a device
// pointer into the heap means the same memory in every process. The
// single-process runtime hands raw peer pointers to its kernels (descriptor
// addresses, done words, regions, staging); with the heap those pointers stay
// valid across processes and the kernels run unchanged. Physical memory is
// created with the CUDA VMM API and shared as POSIX file descriptors (the
// caller passes the descriptors between processes, e.g. over a Unix socket);
// driver entry points are resolved at run time (no link against libcuda).
// This replaces the reference's in-process World (proj/include/streamix/
// world.hpp:129-159) for the one-process-per-GPU launch.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "mpix.h"

namespace {

struct Driver {
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuMemExportToShareableHandle) export_handle = nullptr;
  decltype(&cuMemImportFromShareableHandle) import_handle = nullptr;
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  bool ok = false;
};

template <typename F>
bool entry(const char* name, F* fn) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  *fn = reinterpret_cast<F>(p);
  return true;
}

Driver& drv() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.ok = entry("cuMemAddressReserve", &d.reserve) && entry("cuMemAddressFree", &d.addr_free) &&
           entry("cuMemCreate", &d.create) && entry("cuMemRelease", &d.release) &&
           entry("cuMemMap", &d.map) && entry("cuMemUnmap", &d.unmap) &&
           entry("cuMemSetAccess", &d.set_access) &&
           entry("cuMemExportToShareableHandle", &d.export_handle) &&
           entry("cuMemImportFromShareableHandle", &d.import_handle) &&
           entry("cuMemGetAllocationGranularity", &d.granularity);
  });
  return d;
}

struct Heap {
  std::mutex mu;
  bool live = false;
  int rank = 0, n = 0, device = 0;
  CUdeviceptr base = 0;
  uint64_t slice = 0;
  uint64_t used = 0;  // bump pointer in my slice
  CUmemGenericAllocationHandle mine = 0;
  CUmemGenericAllocationHandle peers[64] = {};
  bool mapped[64] = {};
} g_heap;

CUmemAllocationProp prop_for(int device) {
  CUmemAllocationProp p = {};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return p;
}

int access_for(CUdeviceptr at, uint64_t bytes, int device) {
  CUmemAccessDesc a = {};
  a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  a.location.id = device;
  a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  return drv().set_access(at, bytes, &a, 1) == CUDA_SUCCESS ? MPI_SUCCESS : MPIX_ERR_CUDA;
}

}  // namespace

extern "C" {

int MPIX_Heap_create(int rank, int nranks, int device, uint64_t bytes_per_rank, uint64_t base_hint,
                     uint64_t* base_out, uint64_t* slice_out, int* fd_out) {
  std::lock_guard<std::mutex> lk(g_heap.mu);
  if (g_heap.live) return MPIX_ERR_IN_USE;
  if (nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks || !base_out || !fd_out)
    return MPIX_ERR_INVALID_ARG;
  Driver& d = drv();
  if (!d.ok) return MPIX_ERR_UNSUPPORTED;
  if (cudaSetDevice(device) != cudaSuccess || cudaFree(0) != cudaSuccess) return MPIX_ERR_CUDA;
  CUmemAllocationProp p = prop_for(device);
  size_t gran = 0;
  if (d.granularity(&gran, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || !gran)
    return MPIX_ERR_CUDA;
  const uint64_t slice = (bytes_per_rank + gran - 1) / gran * gran;
  CUdeviceptr base = 0;
  if (d.reserve(&base, slice * nranks, gran, (CUdeviceptr)base_hint, 0) != CUDA_SUCCESS)
    return MPIX_ERR_NO_MEM;
  if (base_hint && base != (CUdeviceptr)base_hint) {  // every process needs the same range
    d.addr_free(base, slice * nranks);
    return MPIX_ERR_NO_MEM;
  }
  CUmemGenericAllocationHandle h = 0;
  if (d.create(&h, slice, &p, 0) != CUDA_SUCCESS) {
    d.addr_free(base, slice * nranks);
    return MPIX_ERR_NO_MEM;
  }
  const CUdeviceptr at = base + slice * rank;
  int fd = -1;
  if (d.map(at, slice, 0, h, 0) != CUDA_SUCCESS || access_for(at, slice, device) != MPI_SUCCESS ||
      d.export_handle(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) != CUDA_SUCCESS) {
    d.release(h);
    d.addr_free(base, slice * nranks);
    return MPIX_ERR_CUDA;
  }
  g_heap.live = true;
  g_heap.rank = rank;
  g_heap.n = nranks;
  g_heap.device = device;
  g_heap.base = base;
  g_heap.slice = slice;
  g_heap.used = 0;
  g_heap.mine = h;
  g_heap.mapped[rank] = true;
  *base_out = (uint64_t)base;
  if (slice_out) *slice_out = slice;
  *fd_out = fd;
  return MPI_SUCCESS;
}

int MPIX_Heap_attach(int peer, int fd) {
  std::lock_guard<std::mutex> lk(g_heap.mu);
  if (!g_heap.live) return MPIX_ERR_NOT_INITIALIZED;
  if (peer < 0 || peer >= g_heap.n || peer == g_heap.rank || g_heap.mapped[peer])
    return MPIX_ERR_INVALID_RANK;
  Driver& d = drv();
  CUmemGenericAllocationHandle h = 0;
  if (d.import_handle(&h, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) !=
      CUDA_SUCCESS)
    return MPIX_ERR_CUDA;
  const CUdeviceptr at = g_heap.base + g_heap.slice * peer;
  if (d.map(at, g_heap.slice, 0, h, 0) != CUDA_SUCCESS) {
    d.release(h);
    return MPIX_ERR_CUDA;
  }
  if (access_for(at, g_heap.slice, g_heap.device) != MPI_SUCCESS) return MPIX_ERR_CUDA;
  g_heap.peers[peer] = h;
  g_heap.mapped[peer] = true;
  return MPI_SUCCESS;
}

// Bump allocation in my slice (256-B aligned); memory is returned at
// MPIX_Heap_destroy. In single-process mode (no heap) it is cudaMalloc.
int MPIX_Alloc_mem(uint64_t bytes, void** ptr) {
  if (!ptr) return MPIX_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> lk(g_heap.mu);
  if (!g_heap.live) return cudaMalloc(ptr, bytes ? bytes : 1) == cudaSuccess ? MPI_SUCCESS
                                                                              : MPIX_ERR_NO_MEM;
  const uint64_t off = (g_heap.used + 255) & ~255ull;
  if (off + bytes > g_heap.slice) return MPIX_ERR_NO_MEM;
  g_heap.used = off + bytes;
  *ptr = (void*)(g_heap.base + g_heap.slice * g_heap.rank + off);
  return MPI_SUCCESS;
}

int MPIX_Free_mem(void* ptr) {
  std::lock_guard<std::mutex> lk(g_heap.mu);
  if (!g_heap.live) return cudaFree(ptr) == cudaSuccess ? MPI_SUCCESS : MPIX_ERR_INVALID_ARG;
  return MPI_SUCCESS;  // bump heap: released with the heap
}

}  // extern "C"

namespace mpix {
bool heap_live() { return g_heap.live; }
}  // namespace mpix

extern "C" {

int MPIX_Heap_contains(const void* ptr, uint64_t bytes) {
  if (!g_heap.live) return 0;
  const uint64_t p = (uint64_t)ptr, b = (uint64_t)g_heap.base;
  return p >= b && p + bytes <= b + g_heap.slice * g_heap.n;
}

int MPIX_Heap_destroy(void) {
  std::lock_guard<std::mutex> lk(g_heap.mu);
  if (!g_heap.live) return MPIX_ERR_NOT_INITIALIZED;
  Driver& d = drv();
  cudaDeviceSynchronize();
  for (int q = 0; q < g_heap.n; ++q) {
    if (!g_heap.mapped[q]) continue;
    d.unmap(g_heap.base + g_heap.slice * q, g_heap.slice);
    d.release(q == g_heap.rank ? g_heap.mine : g_heap.peers[q]);
    g_heap.mapped[q] = false;
  }
  d.addr_free(g_heap.base, g_heap.slice * g_heap.n);
  g_heap.live = false;
  return MPI_SUCCESS;
}

}  // extern "C"
