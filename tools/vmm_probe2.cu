// VMM mapping cost for 128 MiB slabs (the interposer's unit): sequential vs
// several threads, with the link idle and under bidirectional copy load.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/vmm_probe2.cu -o tools/vmm_probe2 -lcuda -lpthread
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>

#define CK(x)                                                 \
  do {                                                        \
    CUresult r_ = (x);                                        \
    if (r_ != CUDA_SUCCESS) {                                 \
      std::printf("%s failed: %d\n", #x, (int)r_);            \
      std::exit(1);                                           \
    }                                                         \
  } while (0)

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  const size_t slab = 128ull << 20;
  const int n = 64;
  cudaFree(0);
  CUcontext ctx;
  CK(cuCtxGetCurrent(&ctx));
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemAccessDesc acc{};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  std::vector<CUmemGenericAllocationHandle> h(n);
  for (auto& x : h) CK(cuMemCreate(&x, slab, &prop, 0));
  CUdeviceptr va;
  CK(cuMemAddressReserve(&va, n * slab, slab, 0, 0));
  // load: 1 GiB H2D + D2H copies looping on two streams
  void *hbuf, *dbuf;
  cudaHostAlloc(&hbuf, 2ull << 30, cudaHostAllocPortable);
  cudaMalloc(&dbuf, 2ull << 30);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  for (int load = 0; load < 2; ++load) {
    for (int threads : {1, 2, 4, 8}) {
      if (load)
        for (int r = 0; r < 8; ++r) {
          cudaMemcpyAsync(dbuf, hbuf, 1ull << 30, cudaMemcpyHostToDevice, s1);
          cudaMemcpyAsync((char*)hbuf + (1ull << 30), (char*)dbuf + (1ull << 30), 1ull << 30, cudaMemcpyDeviceToHost, s2);
        }
      double t0 = now_ms();
      std::vector<std::thread> th;
      for (int t = 0; t < threads; ++t)
        th.emplace_back([&, t] {
          cuCtxSetCurrent(ctx);
          for (int i = t; i < n; i += threads) {
            CK(cuMemMap(va + i * slab, slab, 0, h[i], 0));
            CK(cuMemSetAccess(va + i * slab, slab, &acc, 1));
          }
        });
      for (auto& x : th) x.join();
      double t1 = now_ms();
      th.clear();
      for (int t = 0; t < threads; ++t)
        th.emplace_back([&, t] {
          cuCtxSetCurrent(ctx);
          for (int i = t; i < n; i += threads) CK(cuMemUnmap(va + i * slab, slab));
        });
      for (auto& x : th) x.join();
      double t2 = now_ms();
      std::printf("%s threads %d: map+access %.3f ms/slab  unmap %.3f ms/slab\n", load ? "loaded" : "idle  ", threads,
                  (t1 - t0) / n, (t2 - t1) / n);
      cudaStreamSynchronize(s1);
      cudaStreamSynchronize(s2);
    }
  }
  return 0;
}
