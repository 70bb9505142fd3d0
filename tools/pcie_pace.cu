// Does pacing the D2H direction behind H2D shorten an equal-bytes exchange?
//
// On a bidirectional PCIe exchange the upstream link (GPU -> host) carries the
// D2H data AND the read requests of the H2D copies; with both directions
// saturated the H2D copy engine runs slower than D2H (config-2 timelines:
// H2D ~47 vs D2H ~50 GB/s), D2H finishes first and H2D finishes alone. Both
// directions copy the same bytes here, in `chunk` MiB calls, in these shapes:
//   free        one stream per direction, no coupling (the same-run probe's shape)
//   pace<k>     D2H chunk i waits for H2D chunk i-k to land (D2H never runs more
//               than k chunks ahead; H2D is never held)
//   sleep<us>   D2H chunks separated by a device-side sleep of <us> microseconds
// Prints, per shape: time to move both directions, the end time of each
// direction, and bytes/time of the whole exchange (best of `reps`).
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/pcie_pace.cu -o tools/pcie_pace
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

__global__ void sleep_kernel(unsigned ns) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 >= ns) break;
  }
}

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));            \
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

int main(int argc, char** argv) {
  const size_t total = (argc > 1 ? std::atoll(argv[1]) : 4ll) << 30;
  const int reps = argc > 2 ? std::atoi(argv[2]) : 3;
  void *h_src, *h_dst, *d_src, *d_dst;
  CK(cudaHostAlloc(&h_src, total, cudaHostAllocPortable));
  CK(cudaHostAlloc(&h_dst, total, cudaHostAllocPortable));
  CK(cudaMalloc(&d_src, total));
  CK(cudaMalloc(&d_dst, total));
  std::memset(h_src, 1, total);
  std::memset(h_dst, 0, total);
  CK(cudaMemset(d_src, 2, total));
  cudaStream_t up, dn, sl;
  CK(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&dn, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sl, cudaStreamNonBlocking));
  const size_t max_chunks = total / (2ull << 20) + 1;
  std::vector<cudaEvent_t> h_done(max_chunks), d_done(max_chunks);
  for (auto& e : h_done) CK(cudaEventCreate(&e));
  for (auto& e : d_done) CK(cudaEventCreate(&e));
  cudaEvent_t a, zu, zd;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&zu));
  CK(cudaEventCreate(&zd));
  struct Shape {
    std::string name;
    int pace;      // >0: D2H chunk i waits for H2D chunk i-pace
    int sleep_us;  // >0: sleep between D2H chunks
  };
  std::vector<Shape> shapes = {{"free", 0, 0},     {"pace1", 1, 0},     {"pace2", 2, 0},    {"pace4", 4, 0},
                               {"pace8", 8, 0},    {"sleep20", 0, 20},  {"sleep50", 0, 50}, {"sleep100", 0, 100},
                               {"free", 0, 0}};
  for (int chunk_mib : {64, 256}) {
    const size_t ch = static_cast<size_t>(chunk_mib) << 20;
    const size_t n = total / ch;
    for (const Shape& sh : shapes) {
      double best_t = 1e30, best_u = 0, best_d = 0;
      for (int rep = 0; rep < reps; ++rep) {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a, 0));
        CK(cudaStreamWaitEvent(up, a, 0));
        CK(cudaStreamWaitEvent(dn, a, 0));
        for (size_t i = 0; i < n; ++i) {
          CK(cudaMemcpyAsync((char*)d_dst + i * ch, (char*)h_src + i * ch, ch, cudaMemcpyHostToDevice, up));
          CK(cudaEventRecord(h_done[i], up));
          if (sh.pace > 0 && i >= static_cast<size_t>(sh.pace)) CK(cudaStreamWaitEvent(dn, h_done[i - sh.pace], 0));
          if (sh.sleep_us > 0 && i > 0) sleep_kernel<<<1, 1, 0, dn>>>(sh.sleep_us * 1000u);
          CK(cudaMemcpyAsync((char*)h_dst + i * ch, (char*)d_src + i * ch, ch, cudaMemcpyDeviceToHost, dn));
        }
        CK(cudaEventRecord(zu, up));
        CK(cudaEventRecord(zd, dn));
        CK(cudaDeviceSynchronize());
        float mu = 0, md = 0;
        CK(cudaEventElapsedTime(&mu, a, zu));
        CK(cudaEventElapsedTime(&md, a, zd));
        const double t = std::max(mu, md);
        if (t < best_t) {
          best_t = t;
          best_u = mu;
          best_d = md;
        }
      }
      std::printf(
          "{\"chunk_mib\": %d, \"shape\": \"%s\", \"ms\": %.2f, \"h2d_end_ms\": %.2f, \"d2h_end_ms\": %.2f, "
          "\"h2d_gbs\": %.2f, \"d2h_gbs\": %.2f, \"bidir_gbs\": %.2f}\n",
          chunk_mib, sh.name.c_str(), best_t, best_u, best_d, total / (best_u * 1e-3) / 1e9,
          total / (best_d * 1e-3) / 1e9, 2.0 * total / (best_t * 1e-3) / 1e9);
      std::fflush(stdout);
    }
  }
  return 0;
}
