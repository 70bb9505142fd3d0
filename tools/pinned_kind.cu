// Does the kind of pinned host memory change the bidirectional link rate at
// the pinned ring's working-set size? (tools/probe_sizes.py: the free-running
// H2D rate drops from ~48.7 GB/s over 1-2 GiB buffers to 45-46 over 8 GiB,
// which points at IOMMU/IOTLB reach or host-page effects.) Per kind:
//   hostalloc   cudaHostAlloc(portable | mapped)          (the ring today)
//   thp         mmap + madvise(MADV_HUGEPAGE) + touch + cudaHostRegister
//   hugetlb     mmap(MAP_HUGETLB) + cudaHostRegister     (if the host has huge pages)
// both directions at once in 64 MiB calls, `gib` GiB per direction, best of 3;
// the D2H source and H2D destination are device buffers of the same size.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/pinned_kind.cu -o tools/pinned_kind
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>

#define CK(x)                                                        \
  do {                                                               \
    cudaError_t e_ = (x);                                            \
    if (e_ != cudaSuccess) {                                         \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));  \
      std::exit(1);                                                  \
    }                                                                \
  } while (0)

static long anon_huge_kb() {
  std::ifstream f("/proc/self/smaps_rollup");
  std::string k;
  long v;
  std::string unit;
  while (f >> k) {
    if (k == "AnonHugePages:") {
      f >> v;
      return v;
    }
  }
  return -1;
}

static void* alloc_kind(int kind, size_t bytes) {
  void* p = nullptr;
  if (kind == 0) {
    if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) return nullptr;
  } else {
    const int flags = MAP_PRIVATE | MAP_ANONYMOUS | (kind == 2 ? MAP_HUGETLB : 0);
    p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, flags, -1, 0);
    if (p == MAP_FAILED) return nullptr;
    if (kind == 1) madvise(p, bytes, MADV_HUGEPAGE);
    std::memset(p, 1, bytes);
    if (cudaHostRegister(p, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped) != cudaSuccess) {
      munmap(p, bytes);
      return nullptr;
    }
  }
  std::memset(p, 3, bytes);
  return p;
}

static void free_kind(int kind, void* p, size_t bytes) {
  if (kind == 0) {
    cudaFreeHost(p);
  } else {
    cudaHostUnregister(p);
    munmap(p, bytes);
  }
}

int main(int argc, char** argv) {
  const char* names[] = {"hostalloc", "thp", "hugetlb"};
  cudaStream_t up, dn;
  CK(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&dn, cudaStreamNonBlocking));
  cudaEvent_t a, zu, zd;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&zu));
  CK(cudaEventCreate(&zd));
  const size_t ch = 64ull << 20;
  for (int round = 0; round < 2; ++round) {
    for (int gib : {2, 8}) {
      const size_t bytes = static_cast<size_t>(gib) << 30;
      void *d_src, *d_dst;
      CK(cudaMalloc(&d_src, bytes));
      CK(cudaMalloc(&d_dst, bytes));
      for (int kind = 0; kind < 3; ++kind) {
        const long huge0 = anon_huge_kb();
        void* h_src = alloc_kind(kind, bytes);
        void* h_dst = h_src ? alloc_kind(kind, bytes) : nullptr;
        if (!h_src || !h_dst) {
          std::printf("{\"round\": %d, \"gib\": %d, \"kind\": \"%s\", \"unavailable\": true}\n", round, gib, names[kind]);
          if (h_src) free_kind(kind, h_src, bytes);
          continue;
        }
        const long huge1 = anon_huge_kb();
        double best = 0, bh = 0, bd = 0;
        for (int rep = 0; rep < 4; ++rep) {
          CK(cudaDeviceSynchronize());
          CK(cudaEventRecord(a, 0));
          CK(cudaStreamWaitEvent(up, a, 0));
          CK(cudaStreamWaitEvent(dn, a, 0));
          for (size_t o = 0; o < bytes; o += ch) {
            CK(cudaMemcpyAsync((char*)d_dst + o, (char*)h_src + o, ch, cudaMemcpyHostToDevice, up));
            CK(cudaMemcpyAsync((char*)h_dst + o, (char*)d_src + o, ch, cudaMemcpyDeviceToHost, dn));
          }
          CK(cudaEventRecord(zu, up));
          CK(cudaEventRecord(zd, dn));
          CK(cudaDeviceSynchronize());
          if (rep == 0) continue;
          float mu = 0, md = 0;
          CK(cudaEventElapsedTime(&mu, a, zu));
          CK(cudaEventElapsedTime(&md, a, zd));
          const double tot = 2.0 * bytes / (std::max(mu, md) * 1e-3) / 1e9;
          if (tot > best) {
            best = tot;
            bh = bytes / (mu * 1e-3) / 1e9;
            bd = bytes / (md * 1e-3) / 1e9;
          }
        }
        std::printf(
            "{\"round\": %d, \"gib\": %d, \"kind\": \"%s\", \"bidir_gbs\": %.2f, \"h2d_gbs\": %.2f, \"d2h_gbs\": %.2f, "
            "\"anon_huge_mib_added\": %ld}\n",
            round, gib, names[kind], best, bh, bd, (huge1 - huge0) / 1024);
        std::fflush(stdout);
        free_kind(kind, h_src, bytes);
        free_kind(kind, h_dst, bytes);
      }
      CK(cudaFree(d_src));
      CK(cudaFree(d_dst));
    }
  }
  return 0;
}
