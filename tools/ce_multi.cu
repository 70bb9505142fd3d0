// Does more than one copy stream per direction raise simultaneous H2D+D2H
// throughput? k streams per direction, 64 MiB chunks, 4 GiB each way.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/ce_multi.cu -o tools/ce_multi
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

int main() {
  const size_t total = 4ull << 30, chunk = 64ull << 20;
  void *h1, *h2, *d1, *d2;
  cudaHostAlloc(&h1, total, cudaHostAllocPortable);
  cudaHostAlloc(&h2, total, cudaHostAllocPortable);
  cudaMalloc(&d1, total);
  cudaMalloc(&d2, total);
  for (int chunk_mib : {64, 256}) {
    const size_t ch = static_cast<size_t>(chunk_mib) << 20;
    for (int k : {1, 2, 4}) {
      std::vector<cudaStream_t> up(k), dn(k);
      for (auto& s : up) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      for (auto& s : dn) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      cudaEvent_t a, z;
      cudaEventCreate(&a);
      cudaEventCreate(&z);
      for (int rep = 0; rep < 3; ++rep) {
        cudaDeviceSynchronize();
        cudaEventRecord(a, 0);
        for (auto& s : up) cudaStreamWaitEvent(s, a, 0);
        for (auto& s : dn) cudaStreamWaitEvent(s, a, 0);
        for (size_t off = 0, i = 0; off < total; off += ch, ++i) {
          cudaMemcpyAsync((char*)d1 + off, (char*)h1 + off, ch, cudaMemcpyHostToDevice, up[i % k]);
          cudaMemcpyAsync((char*)h2 + off, (char*)d2 + off, ch, cudaMemcpyDeviceToHost, dn[i % k]);
        }
        for (auto& s : up) {
          cudaEvent_t e;
          cudaEventCreate(&e);
          cudaEventRecord(e, s);
          cudaStreamWaitEvent(0, e, 0);
        }
        for (auto& s : dn) {
          cudaEvent_t e;
          cudaEventCreate(&e);
          cudaEventRecord(e, s);
          cudaStreamWaitEvent(0, e, 0);
        }
        cudaEventRecord(z, 0);
        cudaEventSynchronize(z);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, z);
        if (rep == 2) std::printf("chunk %d MiB, %d stream(s) per direction: %.1f GB/s bidirectional\n", chunk_mib, k, 2.0 * total / (ms * 1e-3) / 1e9);
      }
    }
  }
  return 0;
}
