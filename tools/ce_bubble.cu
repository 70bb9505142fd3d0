// Where do the ~0.05 ms (D2H) / ~0.1 ms (H2D) gaps between consecutive copy
// batches on one stream come from (tools/timeline.py on config 2), and do
// they go away with two streams per direction? Both directions copy 4 GiB at
// once, as batches of `batch` MiB, in these shapes:
//   plain      1 stream/dir, one cudaMemcpyAsync per batch, no events
//   events     1 stream/dir, event record before and after every batch (the engine's shape)
//   split      1 stream/dir, events, every batch as 2 MiB cudaMemcpyAsync calls
//   2streams   2 streams/dir alternating, events
//   2split     2 streams/dir alternating, events, 2 MiB calls
// Prints GB/s of both directions together (best of 3).
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/ce_bubble.cu -o tools/ce_bubble
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

int main() {
  const size_t total = 4ull << 30;
  void *h1, *h2, *d1, *d2;
  cudaHostAlloc(&h1, total, cudaHostAllocPortable);
  cudaHostAlloc(&h2, total, cudaHostAllocPortable);
  cudaMalloc(&d1, total);
  cudaMalloc(&d2, total);
  std::memset(h1, 1, total);
  cudaMemset(d2, 2, total);
  std::vector<cudaEvent_t> evs(1 << 16);
  for (auto& e : evs) cudaEventCreate(&e);
  const char* names[] = {"plain", "events", "split", "2streams", "2split", "3streams"};
  cudaStream_t up[3], dn[3];
  for (int i = 0; i < 3; ++i) {
    cudaStreamCreateWithFlags(&up[i], cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&dn[i], cudaStreamNonBlocking);
  }
  cudaEvent_t a, z;
  cudaEventCreate(&a);
  cudaEventCreate(&z);
  for (int batch_mib : {32, 128, 256}) {
    const size_t ch = static_cast<size_t>(batch_mib) << 20;
    for (int mode = 0; mode < 6; ++mode) {
      const int k = mode == 5 ? 3 : (mode >= 3 ? 2 : 1);
      const bool events = mode != 0, split = mode == 2 || mode == 4;
      double best = 0;
      for (int rep = 0; rep < 3; ++rep) {
        size_t ev = 0;
        cudaDeviceSynchronize();
        cudaEventRecord(a, 0);
        for (int i = 0; i < k; ++i) {
          cudaStreamWaitEvent(up[i], a, 0);
          cudaStreamWaitEvent(dn[i], a, 0);
        }
        for (size_t off = 0, i = 0; off < total; off += ch, ++i) {
          for (int dir = 0; dir < 2; ++dir) {
            cudaStream_t s = dir == 0 ? up[i % k] : dn[i % k];
            if (events) cudaEventRecord(evs[ev++ % evs.size()], s);
            const size_t step = split ? (2ull << 20) : ch;
            for (size_t o = 0; o < ch; o += step) {
              if (dir == 0) cudaMemcpyAsync((char*)d1 + off + o, (char*)h1 + off + o, step, cudaMemcpyHostToDevice, s);
              else cudaMemcpyAsync((char*)h2 + off + o, (char*)d2 + off + o, step, cudaMemcpyDeviceToHost, s);
            }
            if (events) {
              cudaEventRecord(evs[ev++ % evs.size()], s);
              cudaEventRecord(evs[ev++ % evs.size()], s);
            }
          }
        }
        for (int i = 0; i < k; ++i) {
          cudaEventRecord(evs[ev % evs.size()], up[i]);
          cudaStreamWaitEvent(0, evs[ev++ % evs.size()], 0);
          cudaEventRecord(evs[ev % evs.size()], dn[i]);
          cudaStreamWaitEvent(0, evs[ev++ % evs.size()], 0);
        }
        cudaEventRecord(z, 0);
        cudaEventSynchronize(z);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, z);
        best = std::max(best, 2.0 * total / (ms * 1e-3) / 1e9);
      }
      std::printf("{\"batch_mib\": %d, \"mode\": \"%s\", \"bidir_gbs\": %.2f}\n", batch_mib, names[mode], best);
    }
  }
  return 0;
}
