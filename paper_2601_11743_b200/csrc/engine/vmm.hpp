// CUDA virtual-memory-management (VMM) helpers for the exportable device
// arena (internal header).
//
// The interposer path (csrc/shim, csrc/daemon) needs the GPU tier's frames to
// be mappable into every application's own address space at stable virtual
// addresses ("reserve GPU virtual addresses, and map these
// addresses to different physical allocations before and after chunk
// migrations"; modeled in the reference by Chunk::logical_base,
// proj/include/nixie/mem_model.hpp:72). The daemon therefore backs each 2 MiB
// frame of the arena with its own cuMemCreate allocation, exportable as a
// POSIX file descriptor; each shim imports every frame once at start-up and
// maps frames under its applications' reserved ranges as blocks move.
//
// Driver entry points are resolved at run time through the runtime's
// cudaGetDriverEntryPoint, so the product library still loads without a
// driver (the CPU tests dlopen it).
#pragma once

#include <cuda.h>

#include <cstdint>
#include <vector>

#include "nixie/units.hpp"

namespace nixie::b200 {

struct VmmApi {
  CUresult (*mem_create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*mem_release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*addr_reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addr_free)(CUdeviceptr, size_t) = nullptr;
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*export_handle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long) = nullptr;
  CUresult (*get_error_string)(CUresult, const char**) = nullptr;
};

// Resolved once; throws CudaFailure when an entry point is missing.
const VmmApi& vmm_api();

// The GPU tier as a row of exportable physical slabs (cuMemMap maps a handle
// only from offset 0, so whatever an application maps on its own must be its
// own allocation), mapped contiguously at a fresh virtual range of this
// process. On the pool's B200s the driver charges ~0.1-0.4 ms of
// cuMemSetAccess and ~0.08 ms of cuMemUnmap per mapping whatever its size,
// and 5-7 ms to export/import a handle (tools/vmm_probe.cu,
// profiles/r01_vmm_probe.txt), so slabs are large (128 MiB = 64 frames).
class ExportableArena {
 public:
  // `reserve_bytes` (>= bytes) of virtual space is reserved up front so
  // grow() can append slabs at contiguous addresses later.
  void init(int device, Bytes bytes, Bytes slab_bytes, Bytes reserve_bytes = 0);
  ~ExportableArena();
  // Creates, maps and opens one more slab (a dropped slot first, else after
  // the last); returns its index. Throws when the reserved range is full.
  std::uint32_t grow();
  // Unmaps and releases slab `f` (its slot stays reserved; grow() refills it).
  // Shims holding an imported handle keep the memory alive until they
  // release it too.
  void drop(std::uint32_t f);
  std::uint8_t* base() const { return reinterpret_cast<std::uint8_t*>(va_); }
  Bytes bytes() const { return bytes_; }
  std::uint32_t slabs() const { return static_cast<std::uint32_t>(handles_.size()); }
  Bytes slab_bytes() const { return slab_; }
  // A new descriptor for slab `s`'s physical allocation (the caller owns
  // it; it is sent to a shim with SCM_RIGHTS and closed).
  int export_fd(std::uint32_t s) const;

 private:
  std::vector<CUmemGenericAllocationHandle> handles_;
  CUdeviceptr va_ = 0;
  Bytes bytes_ = 0;
  Bytes reserved_ = 0;
  Bytes slab_ = 0;
  int device_ = 0;
  std::uint32_t mapped_ = 0;  // slots in use (dropped ones included)
  void add_slab();
  void create_at(std::uint32_t f);
};

}  // namespace nixie::b200
