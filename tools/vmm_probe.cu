// VMM cost probe (tools/): what does each driver VMM operation the
// interposer path uses cost on this B200? Times per call, N frames of 2 MiB:
//   create (exportable), export fd, import fd (same process), map,
//   set_access (per block and per range), unmap, and the same for
//   non-exportable handles; and map/unmap of larger physical sizes.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/vmm_probe.cu -o /tmp/vmm_probe -lcuda
#include <cuda.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <vector>

#define CK(x)                                                      \
  do {                                                             \
    CUresult r_ = (x);                                             \
    if (r_ != CUDA_SUCCESS) {                                      \
      const char* s = nullptr;                                     \
      cuGetErrorString(r_, &s);                                    \
      std::printf("%s failed: %d %s\n", #x, (int)r_, s ? s : "?"); \
      return 1;                                                    \
    }                                                              \
  } while (0)

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 1024;
  const size_t blk = 2ull << 20;
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  CK(cuDevicePrimaryCtxRetain(&ctx, dev));
  CK(cuCtxSetCurrent(ctx));
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  CUmemAccessDesc acc{};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;

  for (int exportable = 0; exportable < 2; ++exportable) {
    prop.requestedHandleTypes = exportable ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_NONE;
    std::vector<CUmemGenericAllocationHandle> h(n), imp(n);
    double t0 = now_us();
    for (int i = 0; i < n; ++i) CK(cuMemCreate(&h[i], blk, &prop, 0));
    double t1 = now_us();
    std::printf("[%s] create            %.2f us/frame\n", exportable ? "exportable" : "plain", (t1 - t0) / n);
    std::vector<CUmemGenericAllocationHandle>* use = &h;
    if (exportable) {
      std::vector<int> fds(n);
      t0 = now_us();
      for (int i = 0; i < n; ++i) CK(cuMemExportToShareableHandle(&fds[i], h[i], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
      t1 = now_us();
      for (int i = 0; i < n; ++i)
        CK(cuMemImportFromShareableHandle(&imp[i], (void*)(uintptr_t)fds[i], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
      double t2 = now_us();
      for (int i = 0; i < n; ++i) close(fds[i]);
      std::printf("[exportable] export fd         %.2f us/frame\n", (t1 - t0) / n);
      std::printf("[exportable] import fd         %.2f us/frame\n", (t2 - t1) / n);
      use = &imp;
    }
    CUdeviceptr va;
    CK(cuMemAddressReserve(&va, n * blk, blk, 0, 0));
    for (int round = 0; round < 3; ++round) {
      t0 = now_us();
      for (int i = 0; i < n; ++i) CK(cuMemMap(va + i * blk, blk, 0, (*use)[i], 0));
      t1 = now_us();
      if (round == 0) {
        for (int i = 0; i < n; ++i) CK(cuMemSetAccess(va + i * blk, blk, &acc, 1));
      } else {
        CK(cuMemSetAccess(va, n * blk, &acc, 1));
      }
      double t2 = now_us();
      CK(cuCtxSynchronize());
      double t3 = now_us();
      // reverse frames on the next map (scattered placement)
      for (int i = 0; i < n; ++i) CK(cuMemUnmap(va + i * blk, blk));
      double t4 = now_us();
      std::printf("[%s] round %d: map %.2f us/blk, set_access %s %.2f us/blk, unmap %.2f us/blk\n",
                  exportable ? "exportable" : "plain", round, (t1 - t0) / n, round == 0 ? "per-block" : "one-range",
                  (t2 - t1) / n, (t4 - t3) / n);
    }
    // unmap as one range after mapping a range of separate handles?
    for (int i = 0; i < n; ++i) CK(cuMemMap(va + i * blk, blk, 0, (*use)[i], 0));
    CK(cuMemSetAccess(va, n * blk, &acc, 1));
    t0 = now_us();
    CUresult r = cuMemUnmap(va, n * blk);
    t1 = now_us();
    std::printf("[%s] unmap whole range of %d mappings: %s %.2f us total\n", exportable ? "exportable" : "plain", n,
                r == CUDA_SUCCESS ? "ok" : "FAILED", t1 - t0);
    if (r != CUDA_SUCCESS)
      for (int i = 0; i < n; ++i) cuMemUnmap(va + i * blk, blk);
    CK(cuMemAddressFree(va, n * blk));
    if (exportable)
      for (auto x : imp) CK(cuMemRelease(x));
    for (auto x : h) CK(cuMemRelease(x));
  }
  // Larger physical granularity: one handle of 64 MiB / 128 MiB map+unmap.
  for (size_t mb : {8, 32, 128}) {
    prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    const int k = 32;
    std::vector<CUmemGenericAllocationHandle> h(k);
    for (int i = 0; i < k; ++i) CK(cuMemCreate(&h[i], mb << 20, &prop, 0));
    CUdeviceptr va;
    CK(cuMemAddressReserve(&va, k * (mb << 20), blk, 0, 0));
    double t0 = now_us();
    for (int i = 0; i < k; ++i) CK(cuMemMap(va + i * (mb << 20), mb << 20, 0, h[i], 0));
    double t1 = now_us();
    CK(cuMemSetAccess(va, k * (mb << 20), &acc, 1));
    double t2 = now_us();
    for (int i = 0; i < k; ++i) CK(cuMemUnmap(va + i * (mb << 20), mb << 20));
    double t3 = now_us();
    std::printf("[%zu MiB handles] map %.2f us, set_access(range) %.2f us total, unmap %.2f us per handle\n", mb,
                (t1 - t0) / k, t2 - t1, (t3 - t2) / k);
    CK(cuMemAddressFree(va, k * (mb << 20)));
    for (auto x : h) CK(cuMemRelease(x));
  }
  return 0;
}
