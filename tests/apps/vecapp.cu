// nx_vecapp — an ordinary CUDA application used to test the interposer
// (libnixie_shim.so + nixied). It knows nothing about Nixie: it allocates
// with cudaMalloc, launches kernels with <<<>>>, synchronises, thinks, and at
// the end copies everything back and checks it on the host. Built with
// `-cudart shared` so LD_PRELOAD can interpose the runtime.
//
//   nx_vecapp --mib N --buffers K --iters I --think-ms T --seed S [--name X] [--host-check 0|1] [--driver 0|1]
//             [--passes P]   (P step kernels over the working set per iteration)
//             [--graph 0|1|2|3] (iterations as launches of one captured CUDA graph;
//                              1: thread-local capture, 2: global, 3: relaxed)
//             [--capture-alloc-ms T] (--graph: while capturing, sleep T ms, cudaMalloc
//                              a 4 MiB buffer (a managed allocation: a daemon round
//                              trip), sleep T ms again: a pause arriving meanwhile
//                              must wait for the capture without deadlocking)
//             [--driver 2|3]  (2: cuLaunchKernelEx from cudaGetDriverEntryPoint;
//                              3: cuLaunchKernelEx called through the PLT, -lcuda)
//             [--alloc rt|pitch|3d|drvpitch|async]  (how the working set is allocated:
//                              cudaMalloc, cudaMallocPitch, cudaMalloc3D,
//                              cuMemAllocPitch, cuMemAllocAsync)
//             [--streams N]   (creates N streams first: implicit allocations)
//             [--stack-kib K] (cudaDeviceSetLimit(cudaLimitStackSize, K KiB) first: an implicit
//                              device reservation that grows with the per-thread stack)
//             [--sync-ops 1]  (every iteration also reads back part of the working set with
//                              cudaMemcpy2D and cudaMemcpy3D, and memsets + checks a scratch
//                              buffer with cudaMemset2D and cuMemsetD32: synchronous calls that
//                              must wait for the GPU like launches)
//
// Every word of every buffer holds hash(seed, buffer, index) + iteration; each
// iteration's kernel checks the expected value and increments it, so a byte
// lost or misplaced across a context switch is counted (device errors) and
// the final host check compares every word. Prints one JSON line.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <numeric>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

__host__ __device__ inline std::uint32_t mix(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return static_cast<std::uint32_t>(x ^ (x >> 31));
}

__host__ __device__ inline std::uint32_t expect(std::uint64_t seed, int buf, std::uint64_t i) {
  return mix(seed ^ (static_cast<std::uint64_t>(buf) << 48) ^ i);
}

__global__ void fill(std::uint32_t* p, std::uint64_t n, std::uint64_t seed, int buf) {
  for (std::uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = expect(seed, buf, i);
}

__global__ void step(std::uint32_t* p, std::uint64_t n, std::uint64_t seed, int buf, std::uint32_t iter,
                     unsigned long long* errors) {
  unsigned long long bad = 0;
  for (std::uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const std::uint32_t want = expect(seed, buf, i) + iter;
    const std::uint32_t v = p[i];
    bad += v != want;
    p[i] = v + 1;
  }
  if (bad) atomicAdd(errors, bad);
}

__global__ void step_dev(std::uint32_t* p, std::uint64_t n, std::uint64_t seed, int buf, const std::uint32_t* iter,
                         unsigned long long* errors) {
  const std::uint32_t it = *iter;
  unsigned long long bad = 0;
  for (std::uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const std::uint32_t want = expect(seed, buf, i) + it;
    const std::uint32_t v = p[i];
    bad += v != want;
    p[i] = v + 1;
  }
  if (bad) atomicAdd(errors, bad);
}

__global__ void bump(std::uint32_t* k) { *k += 1; }

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) {                                                                    \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(2);                                                                             \
    }                                                                                           \
  } while (0)

int main(int argc, char** argv) {
  double mib = 512;
  int buffers = 4, iters = 10;
  double think_ms = 50;
  std::uint64_t seed = 1;
  std::string name = "vecapp";
  int host_check = 1;
  int driver = 0;  // 1: launch `step` through the driver API (cuLaunchKernel from cudaGetDriverEntryPoint)
  int passes = 1;  // step kernels over the whole working set per iteration (compute per request)
  int graph = 0;   // 1: each iteration is one cudaGraphLaunch of a graph captured once (per pass offset)
  std::string alloc = "rt";
  int streams = 0, sync_ops = 0, stack_kib = 0;
  double capture_alloc_ms = 0;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string a = argv[i];
    if (a == "--mib") mib = std::atof(argv[i + 1]);
    else if (a == "--buffers") buffers = std::atoi(argv[i + 1]);
    else if (a == "--iters") iters = std::atoi(argv[i + 1]);
    else if (a == "--think-ms") think_ms = std::atof(argv[i + 1]);
    else if (a == "--seed") seed = std::strtoull(argv[i + 1], nullptr, 0);
    else if (a == "--name") name = argv[i + 1];
    else if (a == "--host-check") host_check = std::atoi(argv[i + 1]);
    else if (a == "--driver") driver = std::atoi(argv[i + 1]);
    else if (a == "--passes") passes = std::atoi(argv[i + 1]);
    else if (a == "--graph") graph = std::atoi(argv[i + 1]);
    else if (a == "--alloc") alloc = argv[i + 1];
    else if (a == "--streams") streams = std::atoi(argv[i + 1]);
    else if (a == "--sync-ops") sync_ops = std::atoi(argv[i + 1]);
    else if (a == "--stack-kib") stack_kib = std::atoi(argv[i + 1]);
    else if (a == "--capture-alloc-ms") capture_alloc_ms = std::atof(argv[i + 1]);
  }
  const auto t_start = std::chrono::steady_clock::now();
  // Pitched allocations: rows of kRow bytes (a multiple of 512, so the pitch
  // equals the row and the buffer is contiguous).
  constexpr std::uint64_t kRow = 1 << 16;
  std::uint64_t bytes_each = static_cast<std::uint64_t>(mib * 1048576.0 / buffers) / 4 * 4;
  if (alloc != "rt" && alloc != "async") bytes_each = std::max<std::uint64_t>(1, bytes_each / kRow) * kRow;
  const std::uint64_t n = bytes_each / 4;
  if (stack_kib > 0) CK(cudaDeviceSetLimit(cudaLimitStackSize, static_cast<size_t>(stack_kib) * 1024));
  std::vector<cudaStream_t> extra_streams(streams);
  for (auto& st : extra_streams) CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  std::vector<std::uint32_t*> buf(buffers);
  for (auto& p : buf) {
    if (alloc == "rt") {
      CK(cudaMalloc(&p, bytes_each));
    } else if (alloc == "pitch") {
      size_t pitch = 0;
      CK(cudaMallocPitch(reinterpret_cast<void**>(&p), &pitch, kRow, bytes_each / kRow));
      if (pitch != kRow) { std::fprintf(stderr, "pitch %zu != %llu\n", pitch, (unsigned long long)kRow); return 2; }
    } else if (alloc == "3d") {
      cudaPitchedPtr pp{};
      CK(cudaMalloc3D(&pp, make_cudaExtent(kRow, bytes_each / kRow / 4, 4)));
      if (pp.pitch != kRow || (bytes_each / kRow) % 4) { std::fprintf(stderr, "3d pitch %zu\n", pp.pitch); return 2; }
      p = static_cast<std::uint32_t*>(pp.ptr);
    } else if (alloc == "drvpitch") {
      CUdeviceptr d = 0;
      size_t pitch = 0;
      if (cuMemAllocPitch(&d, &pitch, kRow, bytes_each / kRow, 16) != CUDA_SUCCESS || pitch != kRow) {
        std::fprintf(stderr, "cuMemAllocPitch failed (pitch %zu)\n", pitch);
        return 2;
      }
      p = reinterpret_cast<std::uint32_t*>(d);
    } else if (alloc == "async") {
      CUdeviceptr d = 0;
      if (cuMemAllocAsync(&d, bytes_each, nullptr) != CUDA_SUCCESS) { std::fprintf(stderr, "cuMemAllocAsync failed\n"); return 2; }
      CK(cudaStreamSynchronize(nullptr));
      p = reinterpret_cast<std::uint32_t*>(d);
    } else {
      std::fprintf(stderr, "unknown --alloc %s\n", alloc.c_str());
      return 2;
    }
  }
  // Scratch buffer for --sync-ops (memset, then read back and checked).
  constexpr std::uint64_t kScratch = 4 << 20;
  std::uint8_t* scratch = nullptr;
  if (sync_ops) CK(cudaMalloc(&scratch, kScratch));
  std::uint64_t sync_mismatch = 0, sync_calls = 0;
  unsigned long long* d_err = nullptr;  // a small allocation (passes through)
  CK(cudaMalloc(&d_err, sizeof(unsigned long long)));
  CK(cudaMemset(d_err, 0, sizeof(unsigned long long)));
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  for (int b = 0; b < buffers; ++b) fill<<<1184, 256>>>(buf[b], n, seed, b);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  using LaunchFn = CUresult (*)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                                void**, void**);
  LaunchFn cu_launch = nullptr;
  using LaunchExFn = CUresult (*)(const CUlaunchConfig*, CUfunction, void**, void**);
  LaunchExFn cu_launch_ex = driver == 3 ? &cuLaunchKernelEx : nullptr;
  using MemsetD32Fn = CUresult (*)(CUdeviceptr, unsigned, size_t);
  MemsetD32Fn cu_memset32 = nullptr;
  CUfunction step_fn = nullptr;
  if (sync_ops) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CK(cudaGetDriverEntryPoint("cuMemsetD32", &p, cudaEnableDefault, &q));
    cu_memset32 = reinterpret_cast<MemsetD32Fn>(p);
  }
  if (driver) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CK(cudaGetDriverEntryPoint(driver == 2 ? "cuLaunchKernelEx" : "cuLaunchKernel", &p, cudaEnableDefault, &q));
    if (driver == 2) cu_launch_ex = reinterpret_cast<LaunchExFn>(p);
    else cu_launch = reinterpret_cast<LaunchFn>(p);
    cudaFunction_t f = nullptr;
    CK(cudaGetFuncBySymbol(&f, reinterpret_cast<const void*>(&step)));
    step_fn = reinterpret_cast<CUfunction>(f);
  }
  std::vector<double> lat;
  std::uint32_t k = 0;  // passes done so far: every word holds expect() + k
  // --graph: the step kernels read the pass counter from device memory, so one
  // captured graph (steps + counter increment) serves every iteration.
  std::uint32_t* d_k = nullptr;
  cudaStream_t gs = nullptr;
  cudaGraphExec_t gexec = nullptr;
  if (graph) {
    CK(cudaMalloc(&d_k, sizeof(std::uint32_t)));
    CK(cudaMemset(d_k, 0, sizeof(std::uint32_t)));
    CK(cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(gs, graph == 2   ? cudaStreamCaptureModeGlobal
                                  : graph == 3 ? cudaStreamCaptureModeRelaxed
                                               : cudaStreamCaptureModeThreadLocal));
    void* in_capture = nullptr;
    if (capture_alloc_ms > 0) {
      std::this_thread::sleep_for(std::chrono::duration<double, std::milli>(capture_alloc_ms));
      CK(cudaMalloc(&in_capture, 4 << 20));
      std::this_thread::sleep_for(std::chrono::duration<double, std::milli>(capture_alloc_ms));
    }
    for (int pass = 0; pass < passes; ++pass) {
      for (int b = 0; b < buffers; ++b) step_dev<<<1184, 256, 0, gs>>>(buf[b], n, seed, b, d_k, d_err);
      bump<<<1, 1, 0, gs>>>(d_k);
    }
    CK(cudaStreamEndCapture(gs, &g));
    if (in_capture) CK(cudaFree(in_capture));
    CK(cudaGraphInstantiate(&gexec, g, 0));
    CK(cudaGraphDestroy(g));
  }
  for (int it = 0; it < iters && graph; ++it) {
    const auto t0 = std::chrono::steady_clock::now();
    CK(cudaGraphLaunch(gexec, gs));
    CK(cudaStreamSynchronize(gs));
    k += passes;
    lat.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    if (think_ms > 0) std::this_thread::sleep_for(std::chrono::duration<double, std::milli>(think_ms));
  }
  std::vector<std::uint32_t> rows(sync_ops ? 2 * kRow / 4 : 0);
  std::vector<std::uint8_t> sc(sync_ops ? kScratch : 0);
  for (int it = 0; it < iters && !graph; ++it) {
    const auto t0 = std::chrono::steady_clock::now();
    if (sync_ops) {
      // The first call after a think gap may find the app switched out: each
      // of these must wait at the gate for its working set to come back.
      const int b = it % buffers;
      CK(cudaMemcpy2D(rows.data(), kRow, buf[b], kRow, kRow, 2, cudaMemcpyDeviceToHost));
      cudaMemcpy3DParms p3{};
      p3.srcPtr = make_cudaPitchedPtr(buf[b], kRow, kRow, 2);
      p3.dstPtr = make_cudaPitchedPtr(rows.data(), kRow, kRow, 2);
      p3.extent = make_cudaExtent(kRow, 2, 1);
      p3.kind = cudaMemcpyDeviceToHost;
      std::vector<std::uint32_t> rows2(rows.size());
      CK(cudaMemcpy2D(rows2.data(), kRow, buf[b], kRow, kRow, 2, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy3D(&p3));
      for (std::uint64_t i = 0; i < rows.size() && i < n; ++i)
        sync_mismatch += (rows[i] != expect(seed, b, i) + k) + (rows2[i] != rows[i]);
      const int v = (it * 37 + 11) & 0xff;
      CK(cudaMemset2D(scratch, kRow, v, kRow, kScratch / kRow));
      CK(cudaMemcpy(sc.data(), scratch, kScratch, cudaMemcpyDeviceToHost));
      for (std::uint8_t x : sc) sync_mismatch += x != v;
      const unsigned w = 0x01010101u * static_cast<unsigned>((v + 1) & 0xff);
      if (cu_memset32(reinterpret_cast<CUdeviceptr>(scratch), w, kScratch / 4) != CUDA_SUCCESS) return 2;
      CK(cudaMemcpy(sc.data(), scratch, kScratch, cudaMemcpyDeviceToHost));
      for (std::uint8_t x : sc) sync_mismatch += x != ((v + 1) & 0xff);
      sync_calls += 7;
    }
    for (int pass = 0; pass < passes; ++pass, ++k)
    for (int b = 0; b < buffers; ++b) {
      if (driver) {
        std::uint32_t* pb = buf[b];
        std::uint64_t nn = n, sd = seed;
        int bb = b;
        std::uint32_t itv = k;
        void* args[] = {&pb, &nn, &sd, &bb, &itv, &d_err};
        CUresult r;
        if (cu_launch_ex) {
          CUlaunchConfig cfg{};
          cfg.gridDimX = 1184; cfg.gridDimY = cfg.gridDimZ = 1;
          cfg.blockDimX = 256; cfg.blockDimY = cfg.blockDimZ = 1;
          r = cu_launch_ex(&cfg, step_fn, args, nullptr);
        } else {
          r = cu_launch(step_fn, 1184, 1, 1, 256, 1, 1, 0, nullptr, args, nullptr);
        }
        if (r != CUDA_SUCCESS) {
          std::fprintf(stderr, "driver launch failed (%d)\n", static_cast<int>(r));
          return 2;
        }
      } else {
        step<<<1184, 256>>>(buf[b], n, seed, b, k, d_err);
      }
    }
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    lat.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    if (think_ms > 0) std::this_thread::sleep_for(std::chrono::duration<double, std::milli>(think_ms));
  }
  unsigned long long dev_errors = 0;
  CK(cudaMemcpy(&dev_errors, d_err, sizeof(dev_errors), cudaMemcpyDeviceToHost));
  std::uint64_t host_mismatch = 0;
  std::vector<std::uint32_t> h(host_check ? n : 0);
  for (int b = 0; b < buffers && host_check; ++b) {
    CK(cudaMemcpy(h.data(), buf[b], bytes_each, cudaMemcpyDeviceToHost));
    for (std::uint64_t i = 0; i < n; ++i) host_mismatch += h[i] != expect(seed, b, i) + k;
  }
  size_t free_end = 0, total_end = 0;
  CK(cudaMemGetInfo(&free_end, &total_end));
  if (alloc == "async" || alloc == "drvpitch") {
    for (auto p : buf) {
      CUresult r = alloc == "async" ? cuMemFreeAsync(reinterpret_cast<CUdeviceptr>(p), nullptr) : cuMemFree(reinterpret_cast<CUdeviceptr>(p));
      if (r != CUDA_SUCCESS) return 2;
    }
    CK(cudaStreamSynchronize(nullptr));
  } else {
    for (auto p : buf) CK(cudaFree(p));
  }
  for (auto st : extra_streams) CK(cudaStreamDestroy(st));
  if (scratch) CK(cudaFree(scratch));
  CK(cudaFree(d_err));
  std::vector<double> s = lat;
  std::sort(s.begin(), s.end());
  auto q = [&](double f) { return s.empty() ? 0.0 : s[std::min(s.size() - 1, static_cast<std::size_t>(f * s.size()))]; };
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  std::printf("{\"name\": \"%s\", \"bytes\": %llu, \"iters\": %d, \"device_errors\": %llu, \"host_mismatch\": %llu, "
              "\"host_checked\": %d, \"memgetinfo\": [%zu, %zu], \"memgetinfo_end\": [%zu, %zu], \"alloc\": \"%s\", "
              "\"streams\": %d, \"sync_calls\": %llu, \"sync_mismatch\": %llu, \"iter_ms\": {\"p50\": %.3f, \"p99\": %.3f, \"max\": %.3f, \"mean\": %.3f}, \"wall_s\": %.3f}\n",
              name.c_str(), static_cast<unsigned long long>(bytes_each * buffers), iters, dev_errors,
              static_cast<unsigned long long>(host_mismatch), host_check, free_b, total_b, free_end, total_end, alloc.c_str(), streams,
              static_cast<unsigned long long>(sync_calls), static_cast<unsigned long long>(sync_mismatch), q(0.5), q(0.99), s.empty() ? 0.0 : s.back(),
              s.empty() ? 0.0 : std::accumulate(s.begin(), s.end(), 0.0) / s.size(), wall);
  return dev_errors == 0 && host_mismatch == 0 && sync_mismatch == 0 ? 0 : 1;
}
