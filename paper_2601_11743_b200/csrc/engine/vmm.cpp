// Exportable VMM arena (vmm.hpp).
#include "vmm.hpp"

#include <cuda_runtime.h>

#include <string>

#include "phys.hpp"

namespace nixie::b200 {

namespace {

template <typename F>
void resolve(F& fn, const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  NX_CUDA(cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q));
  if (!p || q != cudaDriverEntryPointSuccess) throw CudaFailure(std::string("driver entry point ") + name + " unavailable");
  fn = reinterpret_cast<F>(p);
}

void check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  const char* s = "unknown";
  if (vmm_api().get_error_string) vmm_api().get_error_string(r, &s);
  throw CudaFailure(std::string(what) + ": CUresult " + std::to_string(static_cast<int>(r)) + " (" + s + ")");
}

}  // namespace

const VmmApi& vmm_api() {
  static const VmmApi api = [] {
    VmmApi a;
    resolve(a.mem_create, "cuMemCreate");
    resolve(a.mem_release, "cuMemRelease");
    resolve(a.addr_reserve, "cuMemAddressReserve");
    resolve(a.addr_free, "cuMemAddressFree");
    resolve(a.map, "cuMemMap");
    resolve(a.unmap, "cuMemUnmap");
    resolve(a.set_access, "cuMemSetAccess");
    resolve(a.granularity, "cuMemGetAllocationGranularity");
    resolve(a.export_handle, "cuMemExportToShareableHandle");
    resolve(a.get_error_string, "cuGetErrorString");
    return a;
  }();
  return api;
}

namespace {
CUmemAllocationProp slab_prop(int device) {
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return prop;
}
}  // namespace

void ExportableArena::init(int device, Bytes bytes, Bytes slab_bytes, Bytes reserve_bytes) {
  const VmmApi& v = vmm_api();
  NX_CUDA(cudaFree(nullptr));  // the primary context is current on this thread
  device_ = device;
  const CUmemAllocationProp prop = slab_prop(device);
  size_t gran = 0;
  check(v.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM), "cuMemGetAllocationGranularity");
  if (gran == 0 || kBlockBytes % gran != 0)
    throw CudaFailure("VMM granularity " + std::to_string(gran) + " does not divide the 2 MiB frame");
  if (slab_bytes == 0 || slab_bytes % kBlockBytes || bytes % slab_bytes)
    throw SimError(Err::ValidationError, "exportable arena: bytes must be a multiple of the slab, the slab of 2 MiB");
  slab_ = slab_bytes;
  reserved_ = std::max(bytes, reserve_bytes) / slab_ * slab_;
  check(v.addr_reserve(&va_, reserved_, slab_, 0, 0), "cuMemAddressReserve(arena)");
  const auto n = static_cast<std::uint32_t>(bytes / slab_);
  for (std::uint32_t f = 0; f < n; ++f) add_slab();
}

// Creates slab `f`'s physical allocation and maps it at its slot.
void ExportableArena::create_at(std::uint32_t f) {
  const VmmApi& v = vmm_api();
  const CUmemAllocationProp prop = slab_prop(device_);
  CUmemGenericAllocationHandle h = 0;
  check(v.mem_create(&h, slab_, &prop, 0), "cuMemCreate(exportable slab)");
  if (handles_.size() <= f) handles_.resize(f + 1, 0);
  handles_[f] = h;
  const CUdeviceptr at = va_ + static_cast<CUdeviceptr>(f) * slab_;
  check(v.map(at, slab_, 0, h, 0), "cuMemMap(slab)");
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device_;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  check(v.set_access(at, slab_, &acc, 1), "cuMemSetAccess(slab)");
}

void ExportableArena::add_slab() {
  create_at(mapped_);
  ++mapped_;
  bytes_ = static_cast<Bytes>(mapped_) * slab_;
}

std::uint32_t ExportableArena::grow() {
  for (std::uint32_t f = 0; f < mapped_; ++f)
    if (handles_[f] == 0) {  // a dropped slot comes back first
      create_at(f);
      bytes_ += slab_;
      return f;
    }
  if (static_cast<Bytes>(mapped_ + 1) * slab_ > reserved_)
    throw InvariantViolation("exportable arena: the reserved range is full (" + std::to_string(mapped_) + " slabs)");
  add_slab();
  return mapped_ - 1;
}

void ExportableArena::drop(std::uint32_t f) {
  if (f >= mapped_ || handles_[f] == 0) throw InvariantViolation("exportable arena: drop of a missing slab");
  const VmmApi& v = vmm_api();
  NX_CUDA(cudaDeviceSynchronize());  // nothing of ours may still touch it
  check(v.unmap(va_ + static_cast<CUdeviceptr>(f) * slab_, slab_), "cuMemUnmap(slab)");
  check(v.mem_release(handles_[f]), "cuMemRelease(slab)");
  handles_[f] = 0;
  bytes_ -= slab_;
}

ExportableArena::~ExportableArena() {
  if (!va_) return;
  const VmmApi& v = vmm_api();
  for (std::uint32_t f = 0; f < mapped_; ++f)
    if (handles_[f]) v.unmap(va_ + static_cast<CUdeviceptr>(f) * slab_, slab_);
  for (CUmemGenericAllocationHandle h : handles_)
    if (h) v.mem_release(h);
  v.addr_free(va_, reserved_);
}

int ExportableArena::export_fd(std::uint32_t f) const {
  if (f >= handles_.size() || handles_[f] == 0) throw SimError(Err::InvalidState, "export of slab " + std::to_string(f) + ": none");
  int fd = -1;
  check(vmm_api().export_handle(&fd, handles_[f], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "cuMemExportToShareableHandle");
  return fd;
}

}  // namespace nixie::b200
