// nx_uvm_rr — the UVM comparator on real hardware (the
// reference models it in proj/src/uvm.cpp, PAPER.md:93 explains why it is
// slow: fault-driven, half-duplex evict-then-fetch). Two "apps" share one GPU
// through cudaMallocManaged, round-robin, like nvshare: a device balloon
// (cudaMalloc) leaves only --cap-gib of device memory for managed pages, and
// each app's kernel touches its whole --ws-gib working set, so every switch
// evicts the other app and faults this one back in.
//
//   nx_uvm_rr --cap-gib C --ws-gib W --rounds R [--prefetch 0|1]
//
// --prefetch 1 issues cudaMemPrefetchAsync of the app's buffer before its
// kernel (bulk migration instead of demand faults: UVM's best case).
// Per switch: kernel time with the data elsewhere minus the same kernel's
// time when resident = the switch cost. Prints one JSON line.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) {                                                                    \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(2);                                                                             \
    }                                                                                           \
  } while (0)

__global__ void touch(std::uint64_t* p, std::uint64_t n, std::uint64_t add, unsigned long long* sum) {
  unsigned long long acc = 0;
  for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
    const std::uint64_t v = p[i] + add;
    p[i] = v;
    acc += v;
  }
  atomicAdd(sum, acc);
}

__global__ void fill(std::uint64_t* p, std::uint64_t n, std::uint64_t salt) {
  for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x)
    p[i] = (i * 0x9E3779B97F4A7C15ull) ^ salt;
}

// Counts words that differ from fill(salt) + `adds` touches: the data
// survived every fault-driven migration.
__global__ void check(const std::uint64_t* p, std::uint64_t n, std::uint64_t salt, std::uint64_t adds,
                      unsigned long long* bad) {
  unsigned long long b = 0;
  for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x)
    b += p[i] != ((i * 0x9E3779B97F4A7C15ull) ^ salt) + adds;
  atomicAdd(bad, b);
}

// Peak resident host memory of this process (kB, /proc/self/status VmHWM):
// with UVM, evicted managed pages live in host memory, so this is the host
// mirror the reference models as UVM's pinned peak (proj/include/nixie/uvm.hpp:58-63).
static long vm_hwm_kb() {
  FILE* f = std::fopen("/proc/self/status", "r");
  if (!f) return -1;
  char line[256];
  long kb = -1;
  while (std::fgets(line, sizeof(line), f))
    if (std::sscanf(line, "VmHWM: %ld kB", &kb) == 1) break;
  std::fclose(f);
  return kb;
}

// Host memory in use system-wide (MemTotal - MemAvailable, bytes): sampled
// around the round robin, its rise is what UVM's managed backing took on
// the host (the driver's own pinned pages included).
static long long host_used_bytes() {
  FILE* f = std::fopen("/proc/meminfo", "r");
  if (!f) return -1;
  char line[256];
  long long total = -1, avail = -1, v = 0;
  while (std::fgets(line, sizeof(line), f)) {
    if (std::sscanf(line, "MemTotal: %lld kB", &v) == 1) total = v;
    if (std::sscanf(line, "MemAvailable: %lld kB", &v) == 1) avail = v;
  }
  std::fclose(f);
  return total < 0 || avail < 0 ? -1 : (total - avail) * 1024;
}

static double ms_since(std::chrono::steady_clock::time_point t) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}

int main(int argc, char** argv) {
  double cap_gib = 17, ws_gib = 16;
  int rounds = 3, prefetch = 0;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string a = argv[i];
    if (a == "--cap-gib") cap_gib = std::atof(argv[i + 1]);
    else if (a == "--ws-gib") ws_gib = std::atof(argv[i + 1]);
    else if (a == "--rounds") rounds = std::atoi(argv[i + 1]);
    else if (a == "--prefetch") prefetch = std::atoi(argv[i + 1]);
  }
  int dev = 0;
  CK(cudaSetDevice(dev));
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  const std::size_t cap = static_cast<std::size_t>(cap_gib * (1ull << 30));
  void* balloon = nullptr;
  if (free_b > cap) CK(cudaMalloc(&balloon, free_b - cap));
  const long long host0 = host_used_bytes();
  long long host_peak = host0;
  const std::size_t ws = static_cast<std::size_t>(ws_gib * (1ull << 30));
  const std::uint64_t n = ws / 8;
  std::uint64_t* app[2];
  for (auto& p : app) {
    CK(cudaMallocManaged(&p, ws));
    CK(cudaMemAdvise(p, ws, cudaMemAdviseSetPreferredLocation, dev));
  }
  unsigned long long* sum = nullptr;
  CK(cudaMalloc(&sum, sizeof(unsigned long long)));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  auto run = [&](int a, std::uint64_t add) {
    const auto t = std::chrono::steady_clock::now();
    if (prefetch) {
      cudaMemLocation loc{};
      loc.type = cudaMemLocationTypeDevice;
      loc.id = dev;
      CK(cudaMemPrefetchAsync(app[a], ws, loc, 0, s));
    }
    touch<<<148 * 8, 512, 0, s>>>(app[a], n, add, sum);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    const double ms = ms_since(t);
    host_peak = std::max(host_peak, host_used_bytes());
    return ms;
  };
  // populate both (first touch on the GPU), then round-robin
  for (int a = 0; a < 2; ++a) {
    fill<<<148 * 8, 512, 0, s>>>(app[a], n, 0x5157ull + a);
    CK(cudaStreamSynchronize(s));
  }
  run(0, 1);
  run(1, 1);
  std::vector<double> sw, res;
  for (int r = 0; r < rounds; ++r)
    for (int a = 0; a < 2; ++a) {
      sw.push_back(run(a, 1));   // the other app's pages occupy the GPU
      res.push_back(run(a, 1));  // resident now: compute only
    }
  unsigned long long* bad = nullptr;
  CK(cudaMallocManaged(&bad, sizeof(unsigned long long)));
  *bad = 0;
  for (int a = 0; a < 2; ++a) check<<<148 * 8, 512, 0, s>>>(app[a], n, 0x5157ull + a, 1 + 2ull * rounds, bad);
  CK(cudaStreamSynchronize(s));
  const unsigned long long mismatches = *bad;
  std::vector<double> cost;
  for (std::size_t i = 0; i < sw.size(); ++i) cost.push_back(sw[i] - res[i]);
  std::sort(cost.begin(), cost.end());
  const double med = cost[cost.size() / 2];
  std::printf("{\"mode\": \"%s\", \"cap_gib\": %.2f, \"ws_gib\": %.2f, \"switch_cost_ms\": [", prefetch ? "uvm+prefetch" : "uvm",
              cap_gib, ws_gib);
  for (std::size_t i = 0; i < cost.size(); ++i) std::printf("%s%.2f", i ? ", " : "", cost[i]);
  std::printf("], \"median_ms\": %.2f, \"resident_kernel_ms\": %.2f, \"bidir_equiv_gbps\": %.2f, \"mismatches\": %llu"
              ", \"host_peak_rss_bytes\": %lld, \"host_mem_used_peak_bytes\": %lld}\n", med, res.back(),
              2.0 * ws / (med * 1e-3) / 1e9, mismatches, static_cast<long long>(vm_hwm_kb()) * 1024,
              host0 < 0 ? -1LL : host_peak - host0);
  return 0;
}
