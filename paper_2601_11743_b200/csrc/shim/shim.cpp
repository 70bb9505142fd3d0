// libnixie_shim.so — the Nixie shim: LD_PRELOAD it into an
// unmodified CUDA application (one that links the CUDA runtime dynamically)
// and set NIXIE_SOCKET to a running nixied's socket.
//
// Interposed ("memory allocation and free ... kernel/graph
// launches ... APIs that implicitly allocate memory ... memory usage"):
//   cudaMalloc / cudaFree, cudaMallocAsync[_ptsz] / cudaFreeAsync, cudaMallocPitch,
//   cudaMalloc3D, cuMemAlloc_v2 / cuMemFree_v2, cuMemAllocPitch_v2,
//   cuMemAllocAsync / cuMemFreeAsync
//       allocations >= min_bytes (2 MiB) become daemon chunks: the shim
//       are placed in a virtual range the shim reserved once (stable
//       addresses); every 128 MiB virtual slab of it that holds GPU-resident
//       blocks is mapped to one physical slab of the daemon's arena (imported
//       once at start-up), so a restore costs one mapping per 64 blocks; smaller
//       ones pass through. Reference registry anchor:
//       MemState::allocate / free_chunk (proj/src/mem_model.cpp:48-116),
//       Chunk::logical_base (proj/include/nixie/mem_model.hpp:72).
//   cudaLaunchKernel[_ptsz], cudaLaunchKernelExC[_ptsz],
//   cudaLaunchCooperativeKernel[_ptsz], cudaGraphLaunch[_ptsz], cuLaunchKernel,
//   cuLaunchKernelEx, cuLaunchCooperativeKernel, cuGraphLaunch, and every
//   copy/memset that can touch device memory: cudaMemcpy{,2D,3D,Peer,3DPeer}
//   [Async] and cudaMemset{,2D,3D}[Async] (with their _ptds/_ptsz
//   per-thread-stream twins); the driver's
//   cuMemcpy*/cuMemset* (synchronous and async) through the PLT and through
//   the cuGetProcAddress table
//       the launch gate (PAPER.md:116 steps 1-2 and 6): pass while the
//       execution flag is set; otherwise ask the daemon (Acquire) and hold
//       the calling thread until a Grant has mapped the app's slabs.
//   cublasLtMatmul, cublasGemmEx, cublasGemmStridedBatchedEx, cublasSgemm_v2,
//   cublasSgemmStridedBatched, cudnnBackendExecute
//       gated too: cuBLAS and cuDNN launch through their static runtimes'
//       private driver tables, which no public hook sees.
//   cudaDeviceSynchronize, cudaStreamSynchronize, cudaEventSynchronize,
//   cudaMemcpy (sync)
//       blocking-call brackets for the MLFQ's idleness test (§6.1).
//   cudaStreamBeginCapture / cudaStreamEndCapture
//       capture guard: launches into a capturing stream are
//       not gated and a pause waits for captures to end before it calls any
//       CUDA API.
//   cudaMemGetInfo
//       reports the daemon's budget as total and budget - own usage as free
//       (PAPER.md:147); own usage = managed + passthrough + implicit bytes.
//   cudaStreamCreate*, cuStreamCreate*, cudaDeviceSetLimit,
//   cudaGraphInstantiate*, cublasCreate_v2, cublasLtCreate, cudnnCreate (and
//   their destroys)
//       implicitly allocating APIs: the device memory a call
//       takes (the drop of the device's free memory across it, measured under
//       a process lock) is charged to the app: the daemon admits managed
//       allocations only while managed + passthrough + implicit bytes fit the
//       budget, and cudaMemGetInfo reports it.
//
// The shim never copies application data: the daemon's swap engine moves
// every byte (both PCIe directions at once) through its own mapping of the
// same physical slabs; the shim only maps, unmaps and gates.
#include <cublasLt.h>
#include <cublas_api.h>
#include <cuda.h>
#include <cuda_runtime_api.h>
#include <dlfcn.h>
#include <sys/mman.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "nixie_ipc.hpp"
#include "range_alloc.hpp"

// Per-thread-default-stream variants (declared by cuda_runtime_api.h only
// when that mode is compiled in; libcudart exports them regardless).
extern "C" {
cudaError_t cudaLaunchKernel_ptsz(const void*, dim3, dim3, void**, size_t, cudaStream_t);
cudaError_t cudaLaunchKernelExC_ptsz(const cudaLaunchConfig_t*, const void*, void**);
cudaError_t cudaLaunchCooperativeKernel_ptsz(const void*, dim3, dim3, void**, size_t, cudaStream_t);
cudaError_t cudaGraphLaunch_ptsz(cudaGraphExec_t, cudaStream_t);
cudaError_t cudaMemcpyAsync_ptsz(void*, const void*, size_t, cudaMemcpyKind, cudaStream_t);
cudaError_t cudaMemsetAsync_ptsz(void*, int, size_t, cudaStream_t);
cudaError_t cudaMallocAsync_ptsz(void**, size_t, cudaStream_t);
cudaError_t cudaMemcpy_ptds(void*, const void*, size_t, cudaMemcpyKind);
cudaError_t cudaMemcpy2D_ptds(void*, size_t, const void*, size_t, size_t, size_t, cudaMemcpyKind);
cudaError_t cudaMemcpy2DAsync_ptsz(void*, size_t, const void*, size_t, size_t, size_t, cudaMemcpyKind, cudaStream_t);
cudaError_t cudaMemcpy3D_ptds(const cudaMemcpy3DParms*);
cudaError_t cudaMemcpy3DAsync_ptsz(const cudaMemcpy3DParms*, cudaStream_t);
cudaError_t cudaMemcpy3DPeer_ptds(const cudaMemcpy3DPeerParms*);
cudaError_t cudaMemcpy3DPeerAsync_ptsz(const cudaMemcpy3DPeerParms*, cudaStream_t);
cudaError_t cudaMemset_ptds(void*, int, size_t);
cudaError_t cudaMemset2D_ptds(void*, size_t, int, size_t, size_t);
cudaError_t cudaMemset2DAsync_ptsz(void*, size_t, int, size_t, size_t, cudaStream_t);
cudaError_t cudaMemset3D_ptds(cudaPitchedPtr, int, cudaExtent);
cudaError_t cudaMemset3DAsync_ptsz(cudaPitchedPtr, int, cudaExtent, cudaStream_t);
}

namespace ipc = nixie::ipc;

namespace {

constexpr std::uint64_t kBlock = 2ull << 20;

// ---- real entry points --------------------------------------------------------
void* cudart_handle() {
  static void* h = [] {
    void* p = dlopen("libcudart.so.12", RTLD_NOW | RTLD_NOLOAD);
    if (!p) p = dlopen("libcudart.so", RTLD_NOW | RTLD_NOLOAD);
    return p;
  }();
  return h;
}

void* real_sym(const char* name) {
  void* p = dlsym(RTLD_NEXT, name);
  if (!p && cudart_handle()) p = dlsym(cudart_handle(), name);
  for (const char* lib : {"libcublasLt.so.12", "libcublas.so.12", "libcudnn.so.9"}) {  // loaded RTLD_LOCAL by the app
    if (p) break;
    if (void* h = dlopen(lib, RTLD_NOW | RTLD_NOLOAD)) p = dlsym(h, name);
  }
  if (!p) {
    static void* cuda = dlopen("libcuda.so.1", RTLD_NOW);
    if (cuda) p = dlsym(cuda, name);
  }
  if (!p) {
    std::fprintf(stderr, "[nixie-shim] cannot resolve %s\n", name);
    std::abort();
  }
  return p;
}

#define REAL(name) \
  static auto real_##name = reinterpret_cast<decltype(&::name)>(real_sym(#name))

// Driver entry points the shim itself uses (never the interposed names).
struct Drv {
  CUresult (*import_handle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
  CUresult (*addr_reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*addr_free)(CUdeviceptr, size_t);
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*unmap)(CUdeviceptr, size_t);
  CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*ctx_get_current)(CUcontext*);
  CUresult (*ctx_set_current)(CUcontext);
  CUresult (*release)(CUmemGenericAllocationHandle);
};

Drv& drv() {
  static Drv d = [] {
    Drv x{};
    void* h = dlopen("libcuda.so.1", RTLD_NOW);
    if (!h) {
      std::fprintf(stderr, "[nixie-shim] libcuda.so.1 not found\n");
      std::abort();
    }
    auto get = [h](const char* n) {
      void* p = dlsym(h, n);
      if (!p) {
        std::fprintf(stderr, "[nixie-shim] libcuda lacks %s\n", n);
        std::abort();
      }
      return p;
    };
    x.import_handle = reinterpret_cast<decltype(x.import_handle)>(get("cuMemImportFromShareableHandle"));
    x.addr_reserve = reinterpret_cast<decltype(x.addr_reserve)>(get("cuMemAddressReserve"));
    x.addr_free = reinterpret_cast<decltype(x.addr_free)>(get("cuMemAddressFree"));
    x.map = reinterpret_cast<decltype(x.map)>(get("cuMemMap"));
    x.unmap = reinterpret_cast<decltype(x.unmap)>(get("cuMemUnmap"));
    x.set_access = reinterpret_cast<decltype(x.set_access)>(get("cuMemSetAccess"));
    x.ctx_get_current = reinterpret_cast<decltype(x.ctx_get_current)>(get("cuCtxGetCurrent"));
    x.ctx_set_current = reinterpret_cast<decltype(x.ctx_set_current)>(get("cuCtxSetCurrent"));
    x.release = reinterpret_cast<decltype(x.release)>(get("cuMemRelease"));
    return x;
  }();
  return d;
}

struct Shim;
extern Shim& g;
bool exiting();

thread_local bool t_listener = false;

void die(const char* what, CUresult r = CUDA_SUCCESS) {
  // At exit the driver tears down under the listener thread: not an error;
  // the thread parks and the process finishes exiting with its own status.
  if (t_listener && (r == CUDA_ERROR_DEINITIALIZED || exiting()))
    for (;;) pause();
  std::fprintf(stderr, "[nixie-shim] fatal: %s (CUresult %d)\n", what, static_cast<int>(r));
  std::abort();
}

// ---- state ----------------------------------------------------------------------
// A virtual slab (slab_blocks x 2 MiB window of the shim's range) and
// the physical arena slab mapped under it.
struct VSlab {
  std::uint32_t want = ipc::kNoFrame;  // physical slab the daemon placed it on (kNoFrame: none)
  std::uint32_t have = ipc::kNoFrame;  // physical slab mapped now
  std::uint64_t epoch = 0;             // newest daemon message applied to `want`
};

struct Region {
  std::uint64_t first = 0, blocks = 0;  // placement in the range, 2 MiB blocks
  std::vector<std::uint32_t> chunks;
};

struct Shim {
  bool active = false;
  int device = 0;
  std::uint32_t app = 0;
  std::uint64_t budget = 0, min_bytes = kBlock, slab_bytes = 0, slab_blocks = 0;
  int rpc = -1, ev = -1;
  ipc::CtlPage* ctl = nullptr;
  std::vector<CUmemGenericAllocationHandle> slabs;  // imported arena slabs (0: none)
  std::vector<std::uint32_t> slab_gen;             // generation of each imported slab
  std::vector<std::uint32_t> slab_gone_gen;        // highest dropped generation per slot
  std::vector<std::uint64_t> slab_drop_epoch;      // epoch of the last Drop per slot
  CUcontext ctx = nullptr;
  CUdeviceptr range = 0;          // reserved once; managed allocations live here
  std::uint64_t range_blocks = 0;

  std::mutex rpc_mu;            // one request in flight on the rpc socket
  std::mutex mu;                // everything below (slow paths only)
  std::condition_variable cv;
  nixie::shim::RangeAlloc ranges;  // managed allocations in the range, 2 MiB blocks
  std::map<CUdeviceptr, Region> regions;
  std::unordered_map<std::uint32_t, VSlab> vslabs;
  std::map<void*, std::size_t> small;  // passthrough allocations (for cudaMemGetInfo)
  std::uint64_t managed_bytes = 0, small_bytes = 0;

  std::atomic<bool> granted{false};
  std::atomic<bool> exiting{false};  // the process is exiting: the driver may be torn down
  std::atomic<int> inflight{0};
  std::atomic<int> capturing{0};         // stream captures in progress (any mode)
  std::atomic<int> capturing_global{0};  // ... in global mode: no other thread may call unsafe APIs
};

constexpr std::uint64_t kRangeBytes = 1ull << 40;  // 1 TiB of virtual space per process

// Never destroyed: the listener thread may still run while the process exits.
Shim& g = *new Shim;
bool exiting() { return g.exiting.load(); }
std::once_flag g_once;
thread_local int t_capturing = 0;  // this thread began a stream capture
thread_local std::vector<bool> t_capture_global;  // mode of each open capture of this thread
thread_local int t_gate_depth = 0; // this thread holds a gate slot (nested gated calls pass)
thread_local int t_in_shim = 0;    // re-entrancy guard

void now_api() {
  if (g.ctl) g.ctl->last_api_ns.store(ipc::mono_ns(), std::memory_order_release);
}

void ensure_ctx() {
  CUcontext cur = nullptr;
  drv().ctx_get_current(&cur);
  if (cur != g.ctx && g.ctx) drv().ctx_set_current(g.ctx);
}

void listener();

int connect_to(const char* path) {
  const int fd = ::socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
  sockaddr_un addr{};
  addr.sun_family = AF_UNIX;
  std::strncpy(addr.sun_path, path, sizeof(addr.sun_path) - 1);
  if (::connect(fd, reinterpret_cast<sockaddr*>(&addr), sizeof(addr)) != 0) {
    ::close(fd);
    return -1;
  }
  return fd;
}

void init_once() {
  const char* path = std::getenv("NIXIE_SOCKET");
  if (!path || !*path) return;  // inactive: pure passthrough
  t_in_shim++;
  REAL(cudaFree);
  REAL(cudaGetDevice);
  real_cudaFree(nullptr);  // primary context current on this thread
  real_cudaGetDevice(&g.device);
  drv().ctx_get_current(&g.ctx);
  g.rpc = connect_to(path);
  if (g.rpc < 0) {
    std::fprintf(stderr, "[nixie-shim] cannot connect to %s\n", path);
    std::abort();
  }
  ipc::HelloReq req{};
  req.pid = getpid();
  req.device = g.device;
  FILE* f = std::fopen("/proc/self/comm", "r");
  if (f) {
    if (!std::fgets(req.name, sizeof(req.name), f)) req.name[0] = 0;
    std::fclose(f);
    req.name[strcspn(req.name, "\n")] = 0;
  }
  ipc::Msg type;
  std::vector<std::uint8_t> body;
  int ctl_fd = -1;
  if (!ipc::send_msg(g.rpc, ipc::Msg::Hello, &req, sizeof(req)) || !ipc::recv_msg(g.rpc, type, body) ||
      type != ipc::Msg::Hello || body.size() < sizeof(ipc::HelloRep) || !ipc::recv_fds(g.rpc, &ctl_fd, 1))
    die("hello with the daemon failed");
  ipc::HelloRep rep;
  std::memcpy(&rep, body.data(), sizeof(rep));
  if (rep.status != 0) die("the daemon serves another device");
  g.app = rep.app;
  g.budget = rep.gpu_budget;
  g.min_bytes = rep.min_bytes;
  g.slab_bytes = rep.slab_bytes;
  if (g.slab_bytes == 0 || g.slab_bytes % kBlock != 0) die("bad slab size from the daemon");
  g.slab_blocks = g.slab_bytes / kBlock;
  g.slabs.resize(rep.slabs, 0);
  g.slab_gen.assign(rep.slabs, 1);
  std::vector<int> fds(ipc::kFdBatch);
  for (std::uint64_t f = 0; f < rep.slabs; f += ipc::kFdBatch) {
    const int n = static_cast<int>(std::min<std::uint64_t>(ipc::kFdBatch, rep.slabs - f));
    if (!ipc::recv_fds(g.rpc, fds.data(), n)) die("receiving the arena's slab descriptors");
    for (int k = 0; k < n; ++k) {
      const CUresult r = drv().import_handle(&g.slabs[f + k], reinterpret_cast<void*>(static_cast<std::uintptr_t>(fds[k])),
                                             CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
      if (r != CUDA_SUCCESS) die("cuMemImportFromShareableHandle(slab)", r);
      ::close(fds[k]);
    }
  }
  {
    const CUresult r = drv().addr_reserve(&g.range, kRangeBytes, g.slab_bytes, 0, 0);
    if (r != CUDA_SUCCESS) die("cuMemAddressReserve(range)", r);
    g.range_blocks = kRangeBytes / kBlock;
    const char* ff = std::getenv("NIXIE_SHIM_FIRST_FIT");  // reuse freed ranges (scatters eviction order)
    g.ranges.reset(g.range_blocks, ff && *ff == '1');
  }
  void* p = ::mmap(nullptr, 4096, PROT_READ | PROT_WRITE, MAP_SHARED, ctl_fd, 0);
  if (p == MAP_FAILED) die("mmap control page");
  ::close(ctl_fd);
  g.ctl = static_cast<ipc::CtlPage*>(p);
  g.ev = connect_to(path);
  ipc::EventHelloReq eh{g.app, 0};
  if (g.ev < 0 || !ipc::send_msg(g.ev, ipc::Msg::EventHello, &eh, sizeof(eh))) die("event connection");
  g.active = true;
  std::atexit([] { g.exiting.store(true); });
  std::thread(listener).detach();
  t_in_shim--;
}

bool active() {
  std::call_once(g_once, init_once);
  return g.active;
}

// ---- mapping ---------------------------------------------------------------------
CUmemAccessDesc access_desc() {
  CUmemAccessDesc a{};
  a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  a.location.id = g.device;
  a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  return a;
}

// Makes vslab v's mapping equal `want` (caller holds g.mu): one cuMemUnmap
// and/or one cuMemMap + cuMemSetAccess of a whole slab.
void sync_vslab(std::uint32_t v, VSlab& s, std::uint64_t& maps, std::uint64_t& unmaps) {
  if (s.have == s.want) return;
  ensure_ctx();
  const CUdeviceptr va = g.range + static_cast<CUdeviceptr>(v) * g.slab_bytes;
  const std::uint64_t t0 = ipc::mono_ns();
  if (s.have != ipc::kNoFrame) {
    const CUresult e = drv().unmap(va, g.slab_bytes);
    if (e != CUDA_SUCCESS) die("cuMemUnmap", e);
    s.have = ipc::kNoFrame;
    ++unmaps;
  }
  const std::uint64_t t1 = ipc::mono_ns();
  if (s.want != ipc::kNoFrame) {
    if (s.want >= g.slabs.size() || g.slabs[s.want] == 0) die("the daemon named a slab this shim has no handle for");
    CUresult e = drv().map(va, g.slab_bytes, 0, g.slabs[s.want], 0);
    if (e != CUDA_SUCCESS) die("cuMemMap", e);
    const CUmemAccessDesc acc = access_desc();
    e = drv().set_access(va, g.slab_bytes, &acc, 1);
    if (e != CUDA_SUCCESS) die("cuMemSetAccess", e);
    s.have = s.want;
    ++maps;
  }
  const std::uint64_t t2 = ipc::mono_ns();
  if (g.ctl) {
    g.ctl->unmap_ns.fetch_add(t1 - t0, std::memory_order_relaxed);
    g.ctl->map_ns.fetch_add(t2 - t1, std::memory_order_relaxed);
  }
}

// Applies a daemon placement if it is newer than what the vslab has seen.
void place(std::uint32_t v, std::uint32_t phys, std::uint64_t epoch, std::uint64_t& maps, std::uint64_t& unmaps) {
  VSlab& s = g.vslabs[v];
  if (epoch <= s.epoch) return;
  // A placement older than a Drop of its slab is stale: the slab was freed
  // (the vslab evicted) after it was sent; a later message places the vslab.
  if (phys != ipc::kNoFrame && phys < g.slab_drop_epoch.size() && epoch < g.slab_drop_epoch[phys]) phys = ipc::kNoFrame;
  s.want = phys;
  s.epoch = epoch;
  sync_vslab(v, s, maps, unmaps);
}

// A global-mode capture forbids other threads' unsafe CUDA calls (they would
// invalidate it): the listener's VMM calls wait until it ends.
void wait_for_global_captures() {
  while (g.capturing_global.load() != 0) std::this_thread::sleep_for(std::chrono::microseconds(50));
}

// ---- event socket: Pause / Unmap / Grant ----------------------------------------------
void on_pause(const std::vector<std::uint8_t>& body) {
  ipc::EpochMsg m{};
  std::memcpy(&m, body.data(), std::min(body.size(), sizeof(m)));
  const std::uint64_t t0 = ipc::mono_ns();
  g.granted.store(false, std::memory_order_seq_cst);
  if (g.ctl) g.ctl->granted.store(0);
  while (g.inflight.load(std::memory_order_seq_cst) != 0 || g.capturing.load() != 0) std::this_thread::yield();
  REAL(cudaDeviceSynchronize);
  t_in_shim++;
  ensure_ctx();
  real_cudaDeviceSynchronize();  // outstanding kernels finish before any eviction
  t_in_shim--;
  if (g.ctl) g.ctl->drain_ns.fetch_add(ipc::mono_ns() - t0, std::memory_order_relaxed);
  ipc::send_msg(g.ev, ipc::Msg::Drained, &m, sizeof(m));
}

void on_unmap(const std::vector<std::uint8_t>& body) {
  wait_for_global_captures();
  ipc::Reader r{body};
  const auto m = r.get<ipc::SlabsMsg>();
  std::uint64_t maps = 0, unmaps = 0;
  std::lock_guard<std::mutex> lk(g.mu);
  for (std::uint32_t i = 0; i < m.n && r.ok; ++i) place(r.get<std::uint32_t>(), ipc::kNoFrame, m.epoch, maps, unmaps);
}

std::uint64_t g_premap_ns = 0, g_premap_calls = 0, g_premap_unmap_ns = 0;  // listener thread only

void on_map(const std::vector<std::uint8_t>& body) {
  wait_for_global_captures();
  const std::uint64_t t0 = ipc::mono_ns();
  const std::uint64_t u0 = g.ctl ? g.ctl->unmap_ns.load() : 0;
  ipc::Reader r{body};
  const auto m = r.get<ipc::SlabsMsg>();
  std::uint64_t maps = 0, unmaps = 0;
  {
    std::lock_guard<std::mutex> lk(g.mu);
    for (std::uint32_t i = 0; i < m.n && r.ok; ++i) {
      const auto sm = r.get<ipc::SlabMap>();
      place(sm.vslab, sm.phys, m.epoch, maps, unmaps);
    }
  }
  g_premap_ns += ipc::mono_ns() - t0;
  g_premap_calls += maps;
  if (g.ctl) g_premap_unmap_ns += g.ctl->unmap_ns.load() - u0;
}

void on_grant(const std::vector<std::uint8_t>& body) {
  const std::uint64_t recv = ipc::mono_ns();
  wait_for_global_captures();
  ipc::Reader r{body};
  const auto m = r.get<ipc::SlabsMsg>();
  const std::uint64_t t0 = ipc::mono_ns();
  std::uint64_t maps = 0, unmaps = 0;
  {
    std::lock_guard<std::mutex> lk(g.mu);
    std::unordered_set<std::uint32_t> listed;
    for (std::uint32_t k = 0; k < m.n && r.ok; ++k) {
      const auto sm = r.get<ipc::SlabMap>();
      listed.insert(sm.vslab);
      place(sm.vslab, sm.phys, m.epoch, maps, unmaps);
    }
    // The grant lists every backed vslab of the app: anything else is stale.
    for (auto& [v, st] : g.vslabs)
      if (!listed.count(v) && st.have != ipc::kNoFrame && m.epoch > st.epoch) place(v, ipc::kNoFrame, m.epoch, maps, unmaps);
    g.granted.store(true, std::memory_order_seq_cst);
    if (g.ctl) g.ctl->granted.store(1);
  }
  g.cv.notify_all();
  ipc::GrantedMsg ack{m.epoch, ipc::mono_ns() - t0, maps, unmaps, recv, g_premap_ns, g_premap_calls, g_premap_unmap_ns};
  g_premap_ns = g_premap_calls = g_premap_unmap_ns = 0;
  ipc::send_msg(g.ev, ipc::Msg::Granted, &ack, sizeof(ack));
}

// The daemon's arena grew: import the new slab (its fd follows the message).
// Unmaps every vslab currently mapped to physical slab `p` (caller holds g.mu).
void unmap_slab_users(std::uint32_t p, std::uint64_t epoch) {
  std::uint64_t maps = 0, unmaps = 0;
  for (auto& [v, st] : g.vslabs)
    if (st.have == p) {
      st.want = ipc::kNoFrame;
      st.epoch = std::max(st.epoch, epoch);
      sync_vslab(v, st, maps, unmaps);
    }
}

void grow_slot_tables(std::uint32_t p) {
  if (g.slabs.size() <= p) g.slabs.resize(p + 1, 0);
  if (g.slab_gen.size() <= p) g.slab_gen.resize(p + 1, 0);
  if (g.slab_gone_gen.size() <= p) g.slab_gone_gen.resize(p + 1, 0);
  if (g.slab_drop_epoch.size() <= p) g.slab_drop_epoch.resize(p + 1, 0);
}

// A (re)created slab, on whichever socket the daemon is about to name it on.
void on_slab(int sock, const std::vector<std::uint8_t>& body) {
  ipc::SlabFdMsg m{};
  std::memcpy(&m, body.data(), std::min(body.size(), sizeof(m)));
  int fd = -1;
  if (!ipc::recv_fds(sock, &fd, 1)) die("receiving a new slab's descriptor");
  {
    std::lock_guard<std::mutex> lk(g.mu);
    grow_slot_tables(m.slab);
    if (g.slab_gen[m.slab] >= m.gen || g.slab_gone_gen[m.slab] >= m.gen) {  // seen through the other socket, or dropped
      ::close(fd);
      return;
    }
  }
  CUmemGenericAllocationHandle h = 0;
  ensure_ctx();
  const CUresult r = drv().import_handle(&h, reinterpret_cast<void*>(static_cast<std::uintptr_t>(fd)), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  ::close(fd);
  if (r != CUDA_SUCCESS) die("cuMemImportFromShareableHandle(new slab)", r);
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.slab_gen[m.slab] >= m.gen) {  // raced with the other socket
    drv().release(h);
    return;
  }
  if (g.slabs[m.slab] != 0) {  // an older generation of the slot: nothing may map it any more
    unmap_slab_users(m.slab, 0);
    drv().release(g.slabs[m.slab]);
  }
  g.slabs[m.slab] = h;
  g.slab_gen[m.slab] = m.gen;
}

// The daemon released a grown slab: drop every mapping of it and the handle.
void on_drop(const std::vector<std::uint8_t>& body) {
  ipc::DropMsg m{};
  std::memcpy(&m, body.data(), std::min(body.size(), sizeof(m)));
  wait_for_global_captures();
  std::lock_guard<std::mutex> lk(g.mu);
  grow_slot_tables(m.slab);
  g.slab_gone_gen[m.slab] = std::max(g.slab_gone_gen[m.slab], m.gen);
  g.slab_drop_epoch[m.slab] = std::max(g.slab_drop_epoch[m.slab], m.epoch);
  if (g.slab_gen[m.slab] != m.gen || g.slabs[m.slab] == 0) return;  // superseded already
  ensure_ctx();
  unmap_slab_users(m.slab, m.epoch);
  drv().release(g.slabs[m.slab]);
  g.slabs[m.slab] = 0;
  g.slab_gen[m.slab] = 0;
}

void listener() {
  t_listener = true;
  t_in_shim++;
  REAL(cudaSetDevice);
  REAL(cudaFree);
  real_cudaSetDevice(g.device);
  real_cudaFree(nullptr);
  ensure_ctx();
  ipc::Msg type;
  std::vector<std::uint8_t> body;
  while (ipc::recv_msg(g.ev, type, body)) {
    switch (type) {
      case ipc::Msg::Pause: on_pause(body); break;
      case ipc::Msg::Unmap: on_unmap(body); break;
      case ipc::Msg::Grant: on_grant(body); break;
      case ipc::Msg::Map: on_map(body); break;
      case ipc::Msg::Slab: on_slab(g.ev, body); break;
      case ipc::Msg::Drop: on_drop(body); break;
      default:
        std::fprintf(stderr, "[nixie-shim] unexpected event %u\n", static_cast<unsigned>(type));
    }
  }
  // The daemon went away: keep the application alive only if it holds its
  // memory; otherwise any further gated call would hang forever.
  std::fprintf(stderr, "[nixie-shim] daemon connection closed\n");
  std::_Exit(3);
}

// ---- rpc ----------------------------------------------------------------------------
bool rpc(ipc::Msg type, const void* p, std::size_t n, ipc::Msg& rtype, std::vector<std::uint8_t>& body) {
  std::lock_guard<std::mutex> lk(g.rpc_mu);
  if (!ipc::send_msg(g.rpc, type, p, n)) return false;
  for (;;) {  // new slabs the reply may name come first
    if (!ipc::recv_msg(g.rpc, rtype, body)) return false;
    if (rtype != ipc::Msg::Slab) return true;
    t_in_shim++;
    on_slab(g.rpc, body);
    t_in_shim--;
  }
}

// ---- the gate -------------------------------------------------------------------------
// Held at the gate: the thread waits for the GPU like a blocking call (the
// MLFQ must not see a waiting app as idle the moment it is granted).
void acquire_slow() {
  const std::uint64_t t0 = ipc::mono_ns();
  g.ctl->blocking.fetch_add(1, std::memory_order_acq_rel);
  g.ctl->last_block_ns.store(t0, std::memory_order_release);
  std::unique_lock<std::mutex> lk(g.mu);
  auto last_ask = std::chrono::steady_clock::now() - std::chrono::hours(1);
  while (!g.granted.load(std::memory_order_seq_cst)) {
    if (std::chrono::steady_clock::now() - last_ask > std::chrono::seconds(1)) {
      lk.unlock();
      ipc::Msg rt;
      std::vector<std::uint8_t> body;
      if (!rpc(ipc::Msg::Acquire, nullptr, 0, rt, body)) die("acquire: daemon connection lost");
      last_ask = std::chrono::steady_clock::now();
      lk.lock();
      continue;
    }
    g.cv.wait_for(lk, std::chrono::milliseconds(200));
  }
  const std::uint64_t t1 = ipc::mono_ns();
  g.ctl->last_block_ns.store(t1, std::memory_order_release);
  g.ctl->last_api_ns.store(t1, std::memory_order_release);
  g.ctl->blocking.fetch_sub(1, std::memory_order_acq_rel);
  if (g.ctl) {
    g.ctl->gate_waits.fetch_add(1, std::memory_order_relaxed);
    g.ctl->gate_wait_ns.fetch_add(ipc::mono_ns() - t0, std::memory_order_relaxed);
  }
}

// Entry of every gated call: returns true holding an in-flight slot (a pause
// waits for it), false when the call need not be gated.
bool gate_enter() {
  if (t_in_shim || t_gate_depth || !active()) return false;
  if (t_capturing) {
    // Recorded into a capture, not executed: no gate (the graph launch is
    // gated), but it is activity, so a capturing holder is not seen as idle
    // by the MLFQ and preempted mid-capture.
    g.ctl->captured_launches.fetch_add(1, std::memory_order_relaxed);
    g.ctl->launches.fetch_add(1, std::memory_order_relaxed);
    now_api();
    return false;
  }
  for (;;) {
    g.inflight.fetch_add(1, std::memory_order_seq_cst);
    if (g.granted.load(std::memory_order_seq_cst)) break;
    g.inflight.fetch_sub(1, std::memory_order_seq_cst);
    acquire_slow();
  }
  g.ctl->launches.fetch_add(1, std::memory_order_relaxed);
  return true;
}

// A runtime call the shim gates reaches the driver through cudart's entry
// table, which the shim also wraps (cuGetProcAddress below): the nested
// driver call passes on the outer call's slot (t_gate_depth).
struct Gate {
  bool held;
  Gate() : held(gate_enter()) {
    if (held) ++t_gate_depth;
  }
  ~Gate() {
    if (held) {
      --t_gate_depth;
      g.inflight.fetch_sub(1, std::memory_order_seq_cst);
      now_api();
    }
  }
};

struct Blocking {
  bool on;
  Blocking() : on(!t_in_shim && active()) {
    if (on) {
      g.ctl->blocking.fetch_add(1, std::memory_order_acq_rel);
      g.ctl->last_block_ns.store(ipc::mono_ns(), std::memory_order_release);
    }
  }
  ~Blocking() {
    if (on) {
      const std::uint64_t t = ipc::mono_ns();
      g.ctl->last_block_ns.store(t, std::memory_order_release);
      g.ctl->last_api_ns.store(t, std::memory_order_release);
      g.ctl->blocking.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
};

// ---- implicitly allocating APIs ---------------------------------------------
// The device memory such a call takes is the drop of the device's free memory
// across it, measured under a process-wide lock so this process's other
// implicit calls cannot interleave. The charge is kept per handle and
// returned when the handle is destroyed. While a global-mode capture is open
// nothing is measured (cudaMemGetInfo must not run then).
std::mutex g_implicit_mu;
std::unordered_map<const void*, std::uint64_t> g_implicit;  // handle (or limit tag) -> bytes charged

std::size_t device_free_bytes() {
  REAL(cudaMemGetInfo);
  std::size_t f = 0, t = 0;
  t_in_shim++;
  real_cudaMemGetInfo(&f, &t);
  t_in_shim--;
  return f;
}

struct ImplicitScope {
  bool on;
  std::size_t before = 0;
  std::unique_lock<std::mutex> lk;
  ImplicitScope() : on(!t_in_shim && active() && g.capturing_global.load() == 0) {
    if (!on) return;
    lk = std::unique_lock<std::mutex>(g_implicit_mu);
    before = device_free_bytes();
  }
  // Free-memory change across the call: > 0 taken, < 0 returned.
  std::int64_t delta() const {
    const std::size_t after = device_free_bytes();
    return static_cast<std::int64_t>(before) - static_cast<std::int64_t>(after);
  }
};

// Caller holds g_implicit_mu (through an ImplicitScope).
void implicit_adjust(const void* key, std::int64_t bytes) {
  std::uint64_t& have = g_implicit[key];
  if (bytes < 0) bytes = -static_cast<std::int64_t>(std::min<std::uint64_t>(have, static_cast<std::uint64_t>(-bytes)));
  have += static_cast<std::uint64_t>(bytes);
  g.ctl->implicit_bytes.fetch_add(static_cast<std::uint64_t>(bytes), std::memory_order_relaxed);
  if (have == 0) g_implicit.erase(key);
}

void implicit_release(const void* key) {
  if (t_in_shim || !active()) return;
  std::lock_guard<std::mutex> lk(g_implicit_mu);
  auto it = g_implicit.find(key);
  if (it == g_implicit.end()) return;
  g.ctl->implicit_bytes.fetch_sub(it->second, std::memory_order_relaxed);
  g_implicit.erase(it);
}

// Runs a creating call and charges what it took to the handle it returns.
template <typename R, typename H, typename Fn>
R implicit_create(R ok, H* out, Fn&& call) {
  ImplicitScope sc;
  const R e = call();
  if (sc.on && e == ok && out) {
    const std::int64_t d = sc.delta();
    if (d > 0) implicit_adjust(reinterpret_cast<const void*>(*out), d);
  }
  return e;
}

void small_add(void* p, std::size_t bytes) {
  if (!p || !g.active || t_in_shim) return;
  std::lock_guard<std::mutex> lk(g.mu);
  g.small[p] = bytes;
  g.small_bytes += bytes;
  g.ctl->small_bytes.store(g.small_bytes, std::memory_order_relaxed);
}

void small_remove(void* p) {
  std::lock_guard<std::mutex> lk(g.mu);
  auto it = g.small.find(p);
  if (it == g.small.end()) return;
  g.small_bytes -= it->second;
  g.small.erase(it);
  g.ctl->small_bytes.store(g.small_bytes, std::memory_order_relaxed);
}

// cudaMallocPitch / cudaMalloc3D / cuMemAllocPitch pitch for managed
// allocations: rows aligned to 512 bytes (>= the texture pitch alignment).
constexpr std::size_t kPitchAlign = 512;
std::size_t pitch_of(std::size_t width) { return (width + kPitchAlign - 1) / kPitchAlign * kPitchAlign; }

// ---- allocation -------------------------------------------------------------------------
int managed_alloc(void** out, std::size_t bytes) {
  const std::uint64_t n = (bytes + kBlock - 1) / kBlock;
  std::uint64_t first = 0;
  {
    std::lock_guard<std::mutex> lk(g.mu);
    if (!g.ranges.take(n, g.slab_blocks, first)) return 2;
  }
  ipc::AllocReq req{bytes, first};
  ipc::Msg rt;
  std::vector<std::uint8_t> body;
  if (!rpc(ipc::Msg::Alloc, &req, sizeof(req), rt, body) || rt != ipc::Msg::Alloc || body.size() < sizeof(ipc::AllocRep))
    die("alloc: daemon connection lost");
  ipc::Reader r{body};
  const auto rep = r.get<ipc::AllocRep>();
  std::lock_guard<std::mutex> lk(g.mu);
  if (rep.status != 0) {
    g.ranges.give(first, n);
    return 2;
  }
  Region reg{first, n, {}};
  for (std::uint32_t k = 0; k < rep.n_chunks; ++k) reg.chunks.push_back(r.get<std::uint32_t>());
  std::uint64_t maps = 0, unmaps = 0;
  for (std::uint32_t k = 0; k < rep.n_slabs && r.ok; ++k) {
    const auto sm = r.get<ipc::SlabMap>();
    place(sm.vslab, sm.phys, rep.epoch, maps, unmaps);
  }
  const CUdeviceptr va = g.range + first * kBlock;
  g.regions[va] = reg;
  g.managed_bytes += n * kBlock;
  *out = reinterpret_cast<void*>(va);
  return 0;
}

// Returns true if `p` was a managed allocation (and frees it).
bool managed_free(void* p) {
  const auto va = reinterpret_cast<CUdeviceptr>(p);
  Region reg;
  {
    std::lock_guard<std::mutex> lk(g.mu);
    auto it = g.regions.find(va);
    if (it == g.regions.end()) return false;
    reg = it->second;
    g.regions.erase(it);
  }
  if (g.granted.load()) {  // cudaFree's implicit synchronisation
    REAL(cudaDeviceSynchronize);
    t_in_shim++;
    real_cudaDeviceSynchronize();
    t_in_shim--;
  }
  ipc::Writer w;
  w.put(static_cast<std::uint32_t>(reg.chunks.size()));
  w.put_u32s(reg.chunks);
  ipc::Msg rt;
  std::vector<std::uint8_t> body;
  if (!rpc(ipc::Msg::Free, w.buf.data(), w.buf.size(), rt, body) || rt != ipc::Msg::Free || body.size() < sizeof(ipc::FreeRep))
    die("free: daemon connection lost");
  ipc::Reader r{body};
  const auto rep = r.get<ipc::FreeRep>();
  std::lock_guard<std::mutex> lk(g.mu);
  std::uint64_t maps = 0, unmaps = 0;
  for (std::uint32_t k = 0; k < rep.n && r.ok; ++k) place(r.get<std::uint32_t>(), ipc::kNoFrame, rep.epoch, maps, unmaps);
  g.ranges.give(reg.first, reg.blocks);
  g.managed_bytes -= reg.blocks * kBlock;
  return true;
}

// ---- driver entry points handed out by cuGetProcAddress -----------------------------
// Libraries that link the CUDA runtime statically (cuBLAS, cuDNN) and cudart
// itself reach the driver through cuGetProcAddress, not the PLT. The shim
// wraps dlsym's answer for cuGetProcAddress and returns gated wrappers for
// the launch and async-copy entry points (legacy and per-thread-stream
// variants); everything else is returned untouched.
// Each (symbol, real pointer) pair gets its own wrapper slot: libraries built
// against different CUDA versions may receive different implementations for
// the same name (and the per-thread-stream flavour is another pointer).
constexpr int kSlots = 8;

#define NX_DRV(id, ret, params, args)                                                       \
  ret(*real_##id[kSlots]) params = {};                                                      \
  template <int K>                                                                          \
  ret wrap_##id params {                                                                    \
    Gate gate_;                                                                             \
    if (gate_.held) g.ctl->table_launches.fetch_add(1, std::memory_order_relaxed);          \
    return real_##id[K] args;                                                               \
  }                                                                                         \
  void* const wraps_##id[kSlots] = {                                                        \
      reinterpret_cast<void*>(&wrap_##id<0>), reinterpret_cast<void*>(&wrap_##id<1>),       \
      reinterpret_cast<void*>(&wrap_##id<2>), reinterpret_cast<void*>(&wrap_##id<3>),       \
      reinterpret_cast<void*>(&wrap_##id<4>), reinterpret_cast<void*>(&wrap_##id<5>),       \
      reinterpret_cast<void*>(&wrap_##id<6>), reinterpret_cast<void*>(&wrap_##id<7>)};

NX_DRV(LaunchKernel, CUresult,
       (CUfunction f, unsigned gx, unsigned gy, unsigned gz, unsigned bx, unsigned by, unsigned bz, unsigned sm,
        CUstream st, void** p, void** e),
       (f, gx, gy, gz, bx, by, bz, sm, st, p, e))
NX_DRV(LaunchKernelEx, CUresult, (const CUlaunchConfig* c, CUfunction f, void** p, void** e), (c, f, p, e))
NX_DRV(LaunchCoop, CUresult,
       (CUfunction f, unsigned gx, unsigned gy, unsigned gz, unsigned bx, unsigned by, unsigned bz, unsigned sm,
        CUstream st, void** p),
       (f, gx, gy, gz, bx, by, bz, sm, st, p))
NX_DRV(GraphLaunch, CUresult, (CUgraphExec e, CUstream st), (e, st))
NX_DRV(MemcpyAsync, CUresult, (CUdeviceptr d, CUdeviceptr s, size_t n, CUstream st), (d, s, n, st))
NX_DRV(MemcpyHtoDAsync, CUresult, (CUdeviceptr d, const void* s, size_t n, CUstream st), (d, s, n, st))
NX_DRV(MemcpyDtoHAsync, CUresult, (void* d, CUdeviceptr s, size_t n, CUstream st), (d, s, n, st))
NX_DRV(MemcpyDtoDAsync, CUresult, (CUdeviceptr d, CUdeviceptr s, size_t n, CUstream st), (d, s, n, st))
NX_DRV(MemsetD8Async, CUresult, (CUdeviceptr d, unsigned char v, size_t n, CUstream st), (d, v, n, st))
NX_DRV(MemsetD32Async, CUresult, (CUdeviceptr d, unsigned v, size_t n, CUstream st), (d, v, n, st))
NX_DRV(MemsetD16Async, CUresult, (CUdeviceptr d, unsigned short v, size_t n, CUstream st), (d, v, n, st))
NX_DRV(MemsetD2D8Async, CUresult, (CUdeviceptr d, size_t p, unsigned char v, size_t w, size_t h, CUstream st), (d, p, v, w, h, st))
NX_DRV(MemsetD2D16Async, CUresult, (CUdeviceptr d, size_t p, unsigned short v, size_t w, size_t h, CUstream st), (d, p, v, w, h, st))
NX_DRV(MemsetD2D32Async, CUresult, (CUdeviceptr d, size_t p, unsigned v, size_t w, size_t h, CUstream st), (d, p, v, w, h, st))
NX_DRV(Memcpy2DAsync, CUresult, (const CUDA_MEMCPY2D* c, CUstream st), (c, st))
NX_DRV(Memcpy3DAsync, CUresult, (const CUDA_MEMCPY3D* c, CUstream st), (c, st))
NX_DRV(MemcpyPeerAsync, CUresult, (CUdeviceptr d, CUcontext dc, CUdeviceptr s, CUcontext sc, size_t n, CUstream st),
       (d, dc, s, sc, n, st))
NX_DRV(Memcpy3DPeerAsync, CUresult, (const CUDA_MEMCPY3D_PEER* c, CUstream st), (c, st))
// Synchronous copies and memsets: a paused app's thread must not touch device
// memory either (its mappings may be gone or, kept stale, another app's).
NX_DRV(Memcpy, CUresult, (CUdeviceptr d, CUdeviceptr s, size_t n), (d, s, n))
NX_DRV(MemcpyHtoD, CUresult, (CUdeviceptr d, const void* s, size_t n), (d, s, n))
NX_DRV(MemcpyDtoH, CUresult, (void* d, CUdeviceptr s, size_t n), (d, s, n))
NX_DRV(MemcpyDtoD, CUresult, (CUdeviceptr d, CUdeviceptr s, size_t n), (d, s, n))
NX_DRV(Memcpy2D, CUresult, (const CUDA_MEMCPY2D* c), (c))
NX_DRV(Memcpy2DUnaligned, CUresult, (const CUDA_MEMCPY2D* c), (c))
NX_DRV(Memcpy3D, CUresult, (const CUDA_MEMCPY3D* c), (c))
NX_DRV(MemcpyPeer, CUresult, (CUdeviceptr d, CUcontext dc, CUdeviceptr s, CUcontext sc, size_t n), (d, dc, s, sc, n))
NX_DRV(Memcpy3DPeer, CUresult, (const CUDA_MEMCPY3D_PEER* c), (c))
NX_DRV(MemsetD8, CUresult, (CUdeviceptr d, unsigned char v, size_t n), (d, v, n))
NX_DRV(MemsetD16, CUresult, (CUdeviceptr d, unsigned short v, size_t n), (d, v, n))
NX_DRV(MemsetD32, CUresult, (CUdeviceptr d, unsigned v, size_t n), (d, v, n))
NX_DRV(MemsetD2D8, CUresult, (CUdeviceptr d, size_t p, unsigned char v, size_t w, size_t h), (d, p, v, w, h))
NX_DRV(MemsetD2D16, CUresult, (CUdeviceptr d, size_t p, unsigned short v, size_t w, size_t h), (d, p, v, w, h))
NX_DRV(MemsetD2D32, CUresult, (CUdeviceptr d, size_t p, unsigned v, size_t w, size_t h), (d, p, v, w, h))

struct DrvWrap {
  const char* name;
  void** real;        // kSlots real pointers
  void* const* wrap;  // kSlots wrappers
};

#define NX_ENTRY(id, sym) \
  DrvWrap { sym, reinterpret_cast<void**>(real_##id), wraps_##id }

const DrvWrap kDrvWraps[] = {
    NX_ENTRY(LaunchKernel, "cuLaunchKernel"),       NX_ENTRY(LaunchKernelEx, "cuLaunchKernelEx"),
    NX_ENTRY(LaunchCoop, "cuLaunchCooperativeKernel"), NX_ENTRY(GraphLaunch, "cuGraphLaunch"),
    NX_ENTRY(MemcpyAsync, "cuMemcpyAsync"),         NX_ENTRY(MemcpyHtoDAsync, "cuMemcpyHtoDAsync"),
    NX_ENTRY(MemcpyDtoHAsync, "cuMemcpyDtoHAsync"), NX_ENTRY(MemcpyDtoDAsync, "cuMemcpyDtoDAsync"),
    NX_ENTRY(MemsetD8Async, "cuMemsetD8Async"),     NX_ENTRY(MemsetD32Async, "cuMemsetD32Async"),
    NX_ENTRY(MemsetD16Async, "cuMemsetD16Async"),   NX_ENTRY(MemsetD2D8Async, "cuMemsetD2D8Async"),
    NX_ENTRY(MemsetD2D16Async, "cuMemsetD2D16Async"), NX_ENTRY(MemsetD2D32Async, "cuMemsetD2D32Async"),
    NX_ENTRY(Memcpy2DAsync, "cuMemcpy2DAsync"),     NX_ENTRY(Memcpy3DAsync, "cuMemcpy3DAsync"),
    NX_ENTRY(MemcpyPeerAsync, "cuMemcpyPeerAsync"), NX_ENTRY(Memcpy3DPeerAsync, "cuMemcpy3DPeerAsync"),
    NX_ENTRY(Memcpy, "cuMemcpy"),                   NX_ENTRY(MemcpyHtoD, "cuMemcpyHtoD"),
    NX_ENTRY(MemcpyDtoH, "cuMemcpyDtoH"),           NX_ENTRY(MemcpyDtoD, "cuMemcpyDtoD"),
    NX_ENTRY(Memcpy2D, "cuMemcpy2D"),               NX_ENTRY(Memcpy2DUnaligned, "cuMemcpy2DUnaligned"),
    NX_ENTRY(Memcpy3D, "cuMemcpy3D"),               NX_ENTRY(MemcpyPeer, "cuMemcpyPeer"),
    NX_ENTRY(Memcpy3DPeer, "cuMemcpy3DPeer"),       NX_ENTRY(MemsetD8, "cuMemsetD8"),
    NX_ENTRY(MemsetD16, "cuMemsetD16"),             NX_ENTRY(MemsetD32, "cuMemsetD32"),
    NX_ENTRY(MemsetD2D8, "cuMemsetD2D8"),           NX_ENTRY(MemsetD2D16, "cuMemsetD2D16"),
    NX_ENTRY(MemsetD2D32, "cuMemsetD2D32"),
};

// dlsym names carry the ABI version and stream flavour (cuMemcpyHtoD_v2,
// cuMemsetD8_v2_ptds, cuLaunchKernel_ptsz); cuGetProcAddress takes the base
// name. The positional arguments are the same across versions.
std::string base_symbol(const char* name) {
  std::string n = name;
  for (const char* suf : {"_ptds", "_ptsz"})
    if (n.size() > 5 && n.compare(n.size() - 5, 5, suf) == 0) n.resize(n.size() - 5);
  for (const char* suf : {"_v2", "_v3"})
    if (n.size() > 3 && n.compare(n.size() - 3, 3, suf) == 0) n.resize(n.size() - 3);
  return n;
}

std::mutex g_drv_mu;

// Replaces *pfn with a gated wrapper when `symbol` is one of ours. The real
// pointer is kept per (symbol, stream flavour); a library asking twice gets
// the same answer.
bool debug_on() {
  static const bool on = [] {
    const char* e = std::getenv("NIXIE_SHIM_DEBUG");
    return e && *e == '1';
  }();
  return on;
}

void wrap_proc(const char* symbol, void** pfn, cuuint64_t flags) {
  if (!symbol || !pfn || !*pfn) return;
  for (const DrvWrap& w : kDrvWraps) {
    if (std::strcmp(symbol, w.name) != 0) continue;
    std::lock_guard<std::mutex> lk(g_drv_mu);
    for (int k = 0; k < kSlots; ++k) {
      if (*pfn == w.wrap[k]) return;  // already ours
      if (w.real[k] == nullptr) w.real[k] = *pfn;
      if (w.real[k] == *pfn) {
        if (debug_on())
          std::fprintf(stderr, "[nixie-shim] wrapped %s (flags %llu) slot %d\n", symbol, static_cast<unsigned long long>(flags), k);
        *pfn = w.wrap[k];
        return;
      }
    }
    std::fprintf(stderr, "[nixie-shim] warning: %s has more than %d implementations; not gated\n", symbol, kSlots);
    return;
  }
}

using GetProcV2 = CUresult (*)(const char*, void**, int, cuuint64_t, CUdriverProcAddressQueryResult*);
using GetProcV1 = CUresult (*)(const char*, void**, int, cuuint64_t);
GetProcV2 real_gpa_v2 = nullptr;
GetProcV1 real_gpa_v1 = nullptr;
CUresult wrap_gpa_v1(const char* symbol, void** pfn, int ver, cuuint64_t flags);

CUresult wrap_gpa_v2(const char* symbol, void** pfn, int ver, cuuint64_t flags, CUdriverProcAddressQueryResult* st) {
  const CUresult r = real_gpa_v2(symbol, pfn, ver, flags, st);
  if (debug_on()) std::fprintf(stderr, "[nixie-shim] gpa %s ver %d flags %llu -> %d\n", symbol, ver, static_cast<unsigned long long>(flags), static_cast<int>(r));
  if (r == CUDA_SUCCESS && symbol) {
    if (std::strcmp(symbol, "cuGetProcAddress") == 0) {
      if (ver >= 12000) {
        real_gpa_v2 = real_gpa_v2 ? real_gpa_v2 : reinterpret_cast<GetProcV2>(*pfn);
        *pfn = reinterpret_cast<void*>(&wrap_gpa_v2);
      } else {
        real_gpa_v1 = reinterpret_cast<GetProcV1>(*pfn);
        *pfn = reinterpret_cast<void*>(&wrap_gpa_v1);
      }
    } else {
      wrap_proc(symbol, pfn, flags);
    }
  }
  return r;
}

CUresult wrap_gpa_v1(const char* symbol, void** pfn, int ver, cuuint64_t flags) {
  const CUresult r = real_gpa_v1(symbol, pfn, ver, flags);
  if (debug_on()) std::fprintf(stderr, "[nixie-shim] gpa1 %s ver %d flags %llu -> %d\n", symbol, ver, static_cast<unsigned long long>(flags), static_cast<int>(r));
  if (r == CUDA_SUCCESS) wrap_proc(symbol, pfn, flags);
  return r;
}

using DlsymFn = void* (*)(void*, const char*);
DlsymFn real_dlsym() {
  static DlsymFn f = [] {
    auto p = reinterpret_cast<DlsymFn>(dlvsym(RTLD_NEXT, "dlsym", "GLIBC_2.34"));
    if (!p) p = reinterpret_cast<DlsymFn>(dlvsym(RTLD_NEXT, "dlsym", "GLIBC_2.2.5"));
    return p;
  }();
  return f;
}

}  // namespace

// The one libc entry point the shim wraps: libraries find the driver with
// dlopen("libcuda.so.1") + dlsym("cuGetProcAddress[_v2]").
extern "C" void* dlsym(void* handle, const char* name) {
  void* p = real_dlsym()(handle, name);
  if (!p || std::strncmp(name, "cu", 2) != 0) return p;
  if (std::strncmp(name, "cuGetProcAddress", 16) != 0) {
    // Direct lookups of the gated entry points (launchers that dlopen libcuda).
    wrap_proc(base_symbol(name).c_str(), &p, 0);
    return p;
  }
  if (debug_on()) std::fprintf(stderr, "[nixie-shim] dlsym(%s)\n", name);
  if (std::strcmp(name, "cuGetProcAddress_v2") == 0) {
    if (!real_gpa_v2) real_gpa_v2 = reinterpret_cast<GetProcV2>(p);
    return reinterpret_cast<void*>(&wrap_gpa_v2);
  }
  if (std::strcmp(name, "cuGetProcAddress") == 0) {
    if (!real_gpa_v1) real_gpa_v1 = reinterpret_cast<GetProcV1>(p);
    return reinterpret_cast<void*>(&wrap_gpa_v1);
  }
  return p;
}

// =================================================================================
// Interposed CUDA runtime API
// =================================================================================
extern "C" {

cudaError_t cudaMalloc(void** devPtr, size_t size) {
  REAL(cudaMalloc);
  if (t_in_shim || !active() || size < g.min_bytes) {
    const cudaError_t e = real_cudaMalloc(devPtr, size);
    if (e == cudaSuccess) small_add(*devPtr, size);
    return e;
  }
  return managed_alloc(devPtr, size) == 0 ? cudaSuccess : cudaErrorMemoryAllocation;
}

cudaError_t cudaFree(void* devPtr) {
  REAL(cudaFree);
  if (t_in_shim || !devPtr || !active()) return real_cudaFree(devPtr);
  if (managed_free(devPtr)) return cudaSuccess;
  small_remove(devPtr);
  return real_cudaFree(devPtr);
}

// Stream-ordered allocation (cudaMallocAsync / cudaFreeAsync, e.g. PyTorch's
// cudaMallocAsync backend): managed sizes take the cudaMalloc path (memory
// usable on return is valid stream-ordered semantics); a managed free waits
// for the stream's queued work first, then frees.
cudaError_t cudaMallocAsync(void** devPtr, size_t size, cudaStream_t stream) {
  REAL(cudaMallocAsync);
  if (t_in_shim || !active() || size < g.min_bytes) return real_cudaMallocAsync(devPtr, size, stream);
  return managed_alloc(devPtr, size) == 0 ? cudaSuccess : cudaErrorMemoryAllocation;
}

cudaError_t cudaFreeAsync(void* devPtr, cudaStream_t stream) {
  REAL(cudaFreeAsync);
  if (t_in_shim || !devPtr || !active()) return real_cudaFreeAsync(devPtr, stream);
  bool managed = false;
  {
    std::lock_guard<std::mutex> lk(g.mu);
    managed = g.regions.count(reinterpret_cast<CUdeviceptr>(devPtr)) != 0;
  }
  if (!managed) return real_cudaFreeAsync(devPtr, stream);
  REAL(cudaStreamSynchronize);
  t_in_shim++;
  const cudaError_t e = real_cudaStreamSynchronize(stream);
  t_in_shim--;
  if (e != cudaSuccess) return e;
  managed_free(devPtr);
  return cudaSuccess;
}

cudaError_t cudaMallocAsync_ptsz(void** devPtr, size_t size, cudaStream_t stream) {
  REAL(cudaMallocAsync_ptsz);
  if (t_in_shim || !active() || size < g.min_bytes) return real_cudaMallocAsync_ptsz(devPtr, size, stream);
  return managed_alloc(devPtr, size) == 0 ? cudaSuccess : cudaErrorMemoryAllocation;
}

// Pitched allocations: managed ones get rows of pitch_of(width) bytes in the
// shim's range (any pitch >= width with that alignment is a valid answer).
cudaError_t cudaMallocPitch(void** devPtr, size_t* pitch, size_t width, size_t height) {
  REAL(cudaMallocPitch);
  const std::size_t pt = pitch_of(width);
  if (t_in_shim || !active() || width == 0 || height == 0 || pt * height < g.min_bytes) {
    const cudaError_t e = real_cudaMallocPitch(devPtr, pitch, width, height);
    if (e == cudaSuccess && pitch) small_add(*devPtr, *pitch * height);
    return e;
  }
  if (managed_alloc(devPtr, pt * height) != 0) return cudaErrorMemoryAllocation;
  *pitch = pt;
  return cudaSuccess;
}

cudaError_t cudaMalloc3D(cudaPitchedPtr* pp, cudaExtent ext) {
  REAL(cudaMalloc3D);
  const std::size_t pt = pitch_of(ext.width);
  const std::size_t bytes = pt * ext.height * ext.depth;
  if (t_in_shim || !active() || bytes == 0 || bytes < g.min_bytes) {
    const cudaError_t e = real_cudaMalloc3D(pp, ext);
    if (e == cudaSuccess) small_add(pp->ptr, pp->pitch * ext.height * ext.depth);
    return e;
  }
  void* p = nullptr;
  if (managed_alloc(&p, bytes) != 0) return cudaErrorMemoryAllocation;
  pp->ptr = p;
  pp->pitch = pt;
  pp->xsize = ext.width;
  pp->ysize = ext.height;
  return cudaSuccess;
}

// ---- implicitly allocating runtime / library calls ---------------------------------------
cudaError_t cudaStreamCreate(cudaStream_t* st) {
  REAL(cudaStreamCreate);
  return implicit_create(cudaSuccess, st, [&] { return real_cudaStreamCreate(st); });
}
cudaError_t cudaStreamCreateWithFlags(cudaStream_t* st, unsigned flags) {
  REAL(cudaStreamCreateWithFlags);
  return implicit_create(cudaSuccess, st, [&] { return real_cudaStreamCreateWithFlags(st, flags); });
}
cudaError_t cudaStreamCreateWithPriority(cudaStream_t* st, unsigned flags, int prio) {
  REAL(cudaStreamCreateWithPriority);
  return implicit_create(cudaSuccess, st, [&] { return real_cudaStreamCreateWithPriority(st, flags, prio); });
}
cudaError_t cudaStreamDestroy(cudaStream_t st) {
  REAL(cudaStreamDestroy);
  const cudaError_t e = real_cudaStreamDestroy(st);
  implicit_release(st);
  return e;
}
cudaError_t cudaGraphInstantiate(cudaGraphExec_t* ge, cudaGraph_t gr, unsigned long long flags) {
  REAL(cudaGraphInstantiate);
  return implicit_create(cudaSuccess, ge, [&] { return real_cudaGraphInstantiate(ge, gr, flags); });
}
cudaError_t cudaGraphInstantiateWithFlags(cudaGraphExec_t* ge, cudaGraph_t gr, unsigned long long flags) {
  REAL(cudaGraphInstantiateWithFlags);
  return implicit_create(cudaSuccess, ge, [&] { return real_cudaGraphInstantiateWithFlags(ge, gr, flags); });
}
cudaError_t cudaGraphExecDestroy(cudaGraphExec_t ge) {
  REAL(cudaGraphExecDestroy);
  const cudaError_t e = real_cudaGraphExecDestroy(ge);
  implicit_release(ge);
  return e;
}
// Stack / heap / printf-FIFO limits resize device reservations: the net
// change is charged per limit.
cudaError_t cudaDeviceSetLimit(cudaLimit limit, size_t value) {
  REAL(cudaDeviceSetLimit);
  ImplicitScope sc;
  const cudaError_t e = real_cudaDeviceSetLimit(limit, value);
  if (sc.on && e == cudaSuccess) implicit_adjust(reinterpret_cast<const void*>(static_cast<std::uintptr_t>(0x10 + limit)), sc.delta());
  return e;
}
cublasStatus_t cublasCreate_v2(cublasHandle_t* h) {
  static auto real = reinterpret_cast<cublasStatus_t (*)(cublasHandle_t*)>(real_sym("cublasCreate_v2"));
  return implicit_create(CUBLAS_STATUS_SUCCESS, h, [&] { return real(h); });
}
cublasStatus_t cublasDestroy_v2(cublasHandle_t h) {
  static auto real = reinterpret_cast<cublasStatus_t (*)(cublasHandle_t)>(real_sym("cublasDestroy_v2"));
  const cublasStatus_t e = real(h);
  implicit_release(h);
  return e;
}
cublasStatus_t cublasLtCreate(cublasLtHandle_t* h) {
  static auto real = reinterpret_cast<cublasStatus_t (*)(cublasLtHandle_t*)>(real_sym("cublasLtCreate"));
  return implicit_create(CUBLAS_STATUS_SUCCESS, h, [&] { return real(h); });
}
cublasStatus_t cublasLtDestroy(cublasLtHandle_t h) {
  static auto real = reinterpret_cast<cublasStatus_t (*)(cublasLtHandle_t)>(real_sym("cublasLtDestroy"));
  const cublasStatus_t e = real(h);
  implicit_release(h);
  return e;
}
int cudnnCreate(void** h) {
  static auto real = reinterpret_cast<int (*)(void**)>(real_sym("cudnnCreate"));
  return implicit_create(0, h, [&] { return real(h); });
}
int cudnnDestroy(void* h) {
  static auto real = reinterpret_cast<int (*)(void*)>(real_sym("cudnnDestroy"));
  const int e = real(h);
  implicit_release(h);
  return e;
}

cudaError_t cudaMemGetInfo(size_t* free_b, size_t* total_b) {
  REAL(cudaMemGetInfo);
  if (t_in_shim || !active()) return real_cudaMemGetInfo(free_b, total_b);
  std::lock_guard<std::mutex> lk(g.mu);
  const std::uint64_t used = g.managed_bytes + g.small_bytes + g.ctl->implicit_bytes.load(std::memory_order_relaxed);
  if (total_b) *total_b = g.budget;
  if (free_b) *free_b = used >= g.budget ? 0 : g.budget - used;
  return cudaSuccess;
}

#define GATED(ret, name, params, args) \
  ret name params {                    \
    REAL(name);                        \
    Gate gate_;                        \
    return real_##name args;           \
  }

GATED(cudaError_t, cudaLaunchKernel, (const void* f, dim3 g_, dim3 b, void** a, size_t s, cudaStream_t st), (f, g_, b, a, s, st))
GATED(cudaError_t, cudaLaunchKernel_ptsz, (const void* f, dim3 g_, dim3 b, void** a, size_t s, cudaStream_t st), (f, g_, b, a, s, st))
GATED(cudaError_t, cudaLaunchKernelExC, (const cudaLaunchConfig_t* c, const void* f, void** a), (c, f, a))
GATED(cudaError_t, cudaLaunchKernelExC_ptsz, (const cudaLaunchConfig_t* c, const void* f, void** a), (c, f, a))
GATED(cudaError_t, cudaLaunchCooperativeKernel, (const void* f, dim3 g_, dim3 b, void** a, size_t s, cudaStream_t st), (f, g_, b, a, s, st))
GATED(cudaError_t, cudaLaunchCooperativeKernel_ptsz, (const void* f, dim3 g_, dim3 b, void** a, size_t s, cudaStream_t st), (f, g_, b, a, s, st))
GATED(cudaError_t, cudaGraphLaunch, (cudaGraphExec_t e, cudaStream_t st), (e, st))
GATED(cudaError_t, cudaGraphLaunch_ptsz, (cudaGraphExec_t e, cudaStream_t st), (e, st))
GATED(cudaError_t, cudaMemcpyAsync, (void* d, const void* s, size_t n, cudaMemcpyKind k, cudaStream_t st), (d, s, n, k, st))
GATED(cudaError_t, cudaMemcpyAsync_ptsz, (void* d, const void* s, size_t n, cudaMemcpyKind k, cudaStream_t st), (d, s, n, k, st))
GATED(cudaError_t, cudaMemcpy2DAsync, (void* d, size_t dp, const void* s, size_t sp, size_t w, size_t h, cudaMemcpyKind k, cudaStream_t st), (d, dp, s, sp, w, h, k, st))
GATED(cudaError_t, cudaMemsetAsync, (void* d, int v, size_t n, cudaStream_t st), (d, v, n, st))
GATED(cudaError_t, cudaMemsetAsync_ptsz, (void* d, int v, size_t n, cudaStream_t st), (d, v, n, st))
GATED(cudaError_t, cudaMemset, (void* d, int v, size_t n), (d, v, n))
GATED(cudaError_t, cudaMemset_ptds, (void* d, int v, size_t n), (d, v, n))
GATED(cudaError_t, cudaMemcpy2DAsync_ptsz, (void* d, size_t dp, const void* s, size_t sp, size_t w, size_t h, cudaMemcpyKind k, cudaStream_t st), (d, dp, s, sp, w, h, k, st))
GATED(cudaError_t, cudaMemcpy3DAsync, (const cudaMemcpy3DParms* p, cudaStream_t st), (p, st))
GATED(cudaError_t, cudaMemcpy3DAsync_ptsz, (const cudaMemcpy3DParms* p, cudaStream_t st), (p, st))
GATED(cudaError_t, cudaMemcpyPeerAsync, (void* d, int dd, const void* s, int sd, size_t n, cudaStream_t st), (d, dd, s, sd, n, st))
GATED(cudaError_t, cudaMemcpy3DPeerAsync, (const cudaMemcpy3DPeerParms* p, cudaStream_t st), (p, st))
GATED(cudaError_t, cudaMemcpy3DPeerAsync_ptsz, (const cudaMemcpy3DPeerParms* p, cudaStream_t st), (p, st))
GATED(cudaError_t, cudaMemset2D, (void* d, size_t p, int v, size_t w, size_t h), (d, p, v, w, h))
GATED(cudaError_t, cudaMemset2D_ptds, (void* d, size_t p, int v, size_t w, size_t h), (d, p, v, w, h))
GATED(cudaError_t, cudaMemset2DAsync, (void* d, size_t p, int v, size_t w, size_t h, cudaStream_t st), (d, p, v, w, h, st))
GATED(cudaError_t, cudaMemset2DAsync_ptsz, (void* d, size_t p, int v, size_t w, size_t h, cudaStream_t st), (d, p, v, w, h, st))
GATED(cudaError_t, cudaMemset3D, (cudaPitchedPtr p, int v, cudaExtent e), (p, v, e))
GATED(cudaError_t, cudaMemset3D_ptds, (cudaPitchedPtr p, int v, cudaExtent e), (p, v, e))
GATED(cudaError_t, cudaMemset3DAsync, (cudaPitchedPtr p, int v, cudaExtent e, cudaStream_t st), (p, v, e, st))
GATED(cudaError_t, cudaMemset3DAsync_ptsz, (cudaPitchedPtr p, int v, cudaExtent e, cudaStream_t st), (p, v, e, st))

// Synchronous copies: gated, and blocking calls for the MLFQ's idleness test.
#define GATED_SYNC(ret, name, params, args) \
  ret name params {                         \
    REAL(name);                             \
    Gate gate_;                             \
    Blocking b_;                            \
    return real_##name args;                \
  }

GATED_SYNC(cudaError_t, cudaMemcpy2D, (void* d, size_t dp, const void* s, size_t sp, size_t w, size_t h, cudaMemcpyKind k), (d, dp, s, sp, w, h, k))
GATED_SYNC(cudaError_t, cudaMemcpy2D_ptds, (void* d, size_t dp, const void* s, size_t sp, size_t w, size_t h, cudaMemcpyKind k), (d, dp, s, sp, w, h, k))
GATED_SYNC(cudaError_t, cudaMemcpy_ptds, (void* d, const void* s, size_t n, cudaMemcpyKind k), (d, s, n, k))
GATED_SYNC(cudaError_t, cudaMemcpy3D, (const cudaMemcpy3DParms* p), (p))
GATED_SYNC(cudaError_t, cudaMemcpy3D_ptds, (const cudaMemcpy3DParms* p), (p))
GATED_SYNC(cudaError_t, cudaMemcpyPeer, (void* d, int dd, const void* s, int sd, size_t n), (d, dd, s, sd, n))
GATED_SYNC(cudaError_t, cudaMemcpy3DPeer, (const cudaMemcpy3DPeerParms* p), (p))
GATED_SYNC(cudaError_t, cudaMemcpy3DPeer_ptds, (const cudaMemcpy3DPeerParms* p), (p))

// Like GATED, for names the C++ headers overload (the real symbol is the C one).
#define GATED_C(ret, name, params, args)                                               \
  ret name params {                                                                    \
    static auto real_##name = reinterpret_cast<ret(*) params>(real_sym(#name));       \
    Gate gate_;                                                                        \
    if (gate_.held) g.ctl->blas_calls.fetch_add(1, std::memory_order_relaxed);        \
    return real_##name args;                                                           \
  }

// cuBLAS / cuBLASLt GEMM entry points. cuBLAS links a static CUDA runtime
// and launches through its private driver table, which no public hook sees;
// gating its API calls holds the app's GEMMs at the gate like its own kernels
// (their internal launches happen inside the call, on the held slot).
GATED_C(cublasStatus_t, cublasLtMatmul,
      (cublasLtHandle_t h, cublasLtMatmulDesc_t cd, const void* al, const void* A, cublasLtMatrixLayout_t Ad, const void* B,
       cublasLtMatrixLayout_t Bd, const void* be, const void* C, cublasLtMatrixLayout_t Cd, void* D, cublasLtMatrixLayout_t Dd,
       const cublasLtMatmulAlgo_t* algo, void* ws, size_t wss, cudaStream_t st),
      (h, cd, al, A, Ad, B, Bd, be, C, Cd, D, Dd, algo, ws, wss, st))
GATED_C(cublasStatus_t, cublasGemmEx,
      (cublasHandle_t h, cublasOperation_t ta, cublasOperation_t tb, int m, int n, int k, const void* al, const void* A,
       cudaDataType At, int lda, const void* B, cudaDataType Bt, int ldb, const void* be, void* C, cudaDataType Ct, int ldc,
       cublasComputeType_t ct, cublasGemmAlgo_t algo),
      (h, ta, tb, m, n, k, al, A, At, lda, B, Bt, ldb, be, C, Ct, ldc, ct, algo))
GATED_C(cublasStatus_t, cublasGemmStridedBatchedEx,
      (cublasHandle_t h, cublasOperation_t ta, cublasOperation_t tb, int m, int n, int k, const void* al, const void* A,
       cudaDataType At, int lda, long long sa, const void* B, cudaDataType Bt, int ldb, long long sb, const void* be, void* C,
       cudaDataType Ct, int ldc, long long sc, int bc, cublasComputeType_t ct, cublasGemmAlgo_t algo),
      (h, ta, tb, m, n, k, al, A, At, lda, sa, B, Bt, ldb, sb, be, C, Ct, ldc, sc, bc, ct, algo))
GATED_C(cublasStatus_t, cublasSgemm_v2,
      (cublasHandle_t h, cublasOperation_t ta, cublasOperation_t tb, int m, int n, int k, const float* al, const float* A,
       int lda, const float* B, int ldb, const float* be, float* C, int ldc),
      (h, ta, tb, m, n, k, al, A, lda, B, ldb, be, C, ldc))
GATED_C(cublasStatus_t, cublasSgemmStridedBatched,
      (cublasHandle_t h, cublasOperation_t ta, cublasOperation_t tb, int m, int n, int k, const float* al, const float* A,
       int lda, long long sa, const float* B, int ldb, long long sb, const float* be, float* C, int ldc, long long sc, int bc),
      (h, ta, tb, m, n, k, al, A, lda, sa, B, ldb, sb, be, C, ldc, sc, bc))

// cuDNN 9 executes every backend (graph API) plan through one entry point;
// PyTorch's convolutions go through it. Handles are opaque pointers and the
// status an enum, so no cuDNN header is needed.
GATED_C(int, cudnnBackendExecute, (void* handle, void* plan, void* variant_pack), (handle, plan, variant_pack))

cudaError_t cudaMemcpy(void* d, const void* s, size_t n, cudaMemcpyKind k) {
  REAL(cudaMemcpy);
  Gate gate_;
  Blocking b_;
  return real_cudaMemcpy(d, s, n, k);
}

cudaError_t cudaDeviceSynchronize(void) {
  REAL(cudaDeviceSynchronize);
  Blocking b_;
  return real_cudaDeviceSynchronize();
}

cudaError_t cudaStreamSynchronize(cudaStream_t st) {
  REAL(cudaStreamSynchronize);
  Blocking b_;
  return real_cudaStreamSynchronize(st);
}

cudaError_t cudaEventSynchronize(cudaEvent_t ev) {
  REAL(cudaEventSynchronize);
  Blocking b_;
  return real_cudaEventSynchronize(ev);
}

cudaError_t cudaStreamBeginCapture(cudaStream_t st, cudaStreamCaptureMode mode) {
  REAL(cudaStreamBeginCapture);
  // Capture records work; the app must hold the GPU when the graph is later
  // launched (gated), not while it is built.
  const cudaError_t e = real_cudaStreamBeginCapture(st, mode);
  if (e == cudaSuccess && !t_in_shim) {
    ++t_capturing;
    g.capturing.fetch_add(1);
    t_capture_global.push_back(mode == cudaStreamCaptureModeGlobal);
    if (mode == cudaStreamCaptureModeGlobal) g.capturing_global.fetch_add(1);
  }
  return e;
}

cudaError_t cudaStreamEndCapture(cudaStream_t st, cudaGraph_t* graph) {
  REAL(cudaStreamEndCapture);
  const cudaError_t e = real_cudaStreamEndCapture(st, graph);
  if (!t_in_shim && t_capturing > 0) {
    --t_capturing;
    g.capturing.fetch_sub(1);
    if (!t_capture_global.empty()) {
      if (t_capture_global.back()) g.capturing_global.fetch_sub(1);
      t_capture_global.pop_back();
    }
  }
  return e;
}

// ---- driver API (applications that call it directly through the PLT) ----------------
CUresult cuMemAlloc_v2(CUdeviceptr* dptr, size_t bytes) {
  REAL(cuMemAlloc_v2);
  if (t_in_shim || !active() || bytes < g.min_bytes) return real_cuMemAlloc_v2(dptr, bytes);
  void* p = nullptr;
  if (managed_alloc(&p, bytes) != 0) return CUDA_ERROR_OUT_OF_MEMORY;
  *dptr = reinterpret_cast<CUdeviceptr>(p);
  return CUDA_SUCCESS;
}

CUresult cuMemFree_v2(CUdeviceptr dptr) {
  REAL(cuMemFree_v2);
  if (t_in_shim || !dptr || !active()) return real_cuMemFree_v2(dptr);
  if (managed_free(reinterpret_cast<void*>(dptr))) return CUDA_SUCCESS;
  return real_cuMemFree_v2(dptr);
}

CUresult cuLaunchKernel(CUfunction f, unsigned gx, unsigned gy, unsigned gz, unsigned bx, unsigned by, unsigned bz,
                        unsigned smem, CUstream st, void** params, void** extra) {
  REAL(cuLaunchKernel);
  Gate gate_;
  return real_cuLaunchKernel(f, gx, gy, gz, bx, by, bz, smem, st, params, extra);
}

CUresult cuMemAllocPitch_v2(CUdeviceptr* dptr, size_t* pitch, size_t width, size_t height, unsigned elem) {
  REAL(cuMemAllocPitch_v2);
  const std::size_t pt = pitch_of(width);
  if (t_in_shim || !active() || width == 0 || height == 0 || pt * height < g.min_bytes)
    return real_cuMemAllocPitch_v2(dptr, pitch, width, height, elem);
  if (elem != 4 && elem != 8 && elem != 16) return CUDA_ERROR_INVALID_VALUE;
  void* p = nullptr;
  if (managed_alloc(&p, pt * height) != 0) return CUDA_ERROR_OUT_OF_MEMORY;
  *dptr = reinterpret_cast<CUdeviceptr>(p);
  *pitch = pt;
  return CUDA_SUCCESS;
}

// Stream-ordered driver allocations: as cudaMallocAsync / cudaFreeAsync.
CUresult cuMemAllocAsync(CUdeviceptr* dptr, size_t bytes, CUstream st) {
  REAL(cuMemAllocAsync);
  if (t_in_shim || !active() || bytes < g.min_bytes) return real_cuMemAllocAsync(dptr, bytes, st);
  void* p = nullptr;
  if (managed_alloc(&p, bytes) != 0) return CUDA_ERROR_OUT_OF_MEMORY;
  *dptr = reinterpret_cast<CUdeviceptr>(p);
  return CUDA_SUCCESS;
}

CUresult cuMemFreeAsync(CUdeviceptr dptr, CUstream st) {
  REAL(cuMemFreeAsync);
  if (t_in_shim || !dptr || !active()) return real_cuMemFreeAsync(dptr, st);
  bool managed = false;
  {
    std::lock_guard<std::mutex> lk(g.mu);
    managed = g.regions.count(dptr) != 0;
  }
  if (!managed) return real_cuMemFreeAsync(dptr, st);
  static auto sync = reinterpret_cast<CUresult (*)(CUstream)>(real_sym("cuStreamSynchronize"));
  t_in_shim++;
  const CUresult e = sync(st);
  t_in_shim--;
  if (e != CUDA_SUCCESS) return e;
  managed_free(reinterpret_cast<void*>(dptr));
  return CUDA_SUCCESS;
}

CUresult cuStreamCreate(CUstream* st, unsigned flags) {
  REAL(cuStreamCreate);
  return implicit_create(CUDA_SUCCESS, st, [&] { return real_cuStreamCreate(st, flags); });
}
CUresult cuStreamCreateWithPriority(CUstream* st, unsigned flags, int prio) {
  REAL(cuStreamCreateWithPriority);
  return implicit_create(CUDA_SUCCESS, st, [&] { return real_cuStreamCreateWithPriority(st, flags, prio); });
}
CUresult cuStreamDestroy_v2(CUstream st) {
  REAL(cuStreamDestroy_v2);
  const CUresult e = real_cuStreamDestroy_v2(st);
  implicit_release(st);
  return e;
}

// Driver launches, graph launches, copies and memsets called through the PLT
// (applications linked against libcuda): the same gate as the table entries.
#define GATED_DRV(name, params, args) \
  CUresult name params {              \
    REAL(name);                       \
    Gate gate_;                       \
    return real_##name args;          \
  }

GATED_DRV(cuLaunchKernelEx, (const CUlaunchConfig* c, CUfunction f, void** p, void** e), (c, f, p, e))
GATED_DRV(cuLaunchCooperativeKernel,
          (CUfunction f, unsigned gx, unsigned gy, unsigned gz, unsigned bx, unsigned by, unsigned bz, unsigned sm, CUstream st, void** p),
          (f, gx, gy, gz, bx, by, bz, sm, st, p))
GATED_DRV(cuGraphLaunch, (CUgraphExec e, CUstream st), (e, st))
GATED_DRV(cuMemcpy, (CUdeviceptr d, CUdeviceptr s, size_t n), (d, s, n))
GATED_DRV(cuMemcpyAsync, (CUdeviceptr d, CUdeviceptr s, size_t n, CUstream st), (d, s, n, st))
GATED_DRV(cuMemcpyHtoD_v2, (CUdeviceptr d, const void* s, size_t n), (d, s, n))
GATED_DRV(cuMemcpyDtoH_v2, (void* d, CUdeviceptr s, size_t n), (d, s, n))
GATED_DRV(cuMemcpyDtoD_v2, (CUdeviceptr d, CUdeviceptr s, size_t n), (d, s, n))
GATED_DRV(cuMemcpyHtoDAsync_v2, (CUdeviceptr d, const void* s, size_t n, CUstream st), (d, s, n, st))
GATED_DRV(cuMemcpyDtoHAsync_v2, (void* d, CUdeviceptr s, size_t n, CUstream st), (d, s, n, st))
GATED_DRV(cuMemcpyDtoDAsync_v2, (CUdeviceptr d, CUdeviceptr s, size_t n, CUstream st), (d, s, n, st))
GATED_DRV(cuMemcpy2D_v2, (const CUDA_MEMCPY2D* c), (c))
GATED_DRV(cuMemcpy2DUnaligned_v2, (const CUDA_MEMCPY2D* c), (c))
GATED_DRV(cuMemcpy2DAsync_v2, (const CUDA_MEMCPY2D* c, CUstream st), (c, st))
GATED_DRV(cuMemcpy3D_v2, (const CUDA_MEMCPY3D* c), (c))
GATED_DRV(cuMemcpy3DAsync_v2, (const CUDA_MEMCPY3D* c, CUstream st), (c, st))
GATED_DRV(cuMemcpyPeer, (CUdeviceptr d, CUcontext dc, CUdeviceptr s, CUcontext sc, size_t n), (d, dc, s, sc, n))
GATED_DRV(cuMemcpyPeerAsync, (CUdeviceptr d, CUcontext dc, CUdeviceptr s, CUcontext sc, size_t n, CUstream st), (d, dc, s, sc, n, st))
GATED_DRV(cuMemsetD8_v2, (CUdeviceptr d, unsigned char v, size_t n), (d, v, n))
GATED_DRV(cuMemsetD16_v2, (CUdeviceptr d, unsigned short v, size_t n), (d, v, n))
GATED_DRV(cuMemsetD32_v2, (CUdeviceptr d, unsigned v, size_t n), (d, v, n))
GATED_DRV(cuMemsetD8Async, (CUdeviceptr d, unsigned char v, size_t n, CUstream st), (d, v, n, st))
GATED_DRV(cuMemsetD16Async, (CUdeviceptr d, unsigned short v, size_t n, CUstream st), (d, v, n, st))
GATED_DRV(cuMemsetD32Async, (CUdeviceptr d, unsigned v, size_t n, CUstream st), (d, v, n, st))
GATED_DRV(cuMemsetD2D8_v2, (CUdeviceptr d, size_t p, unsigned char v, size_t w, size_t h), (d, p, v, w, h))
GATED_DRV(cuMemsetD2D16_v2, (CUdeviceptr d, size_t p, unsigned short v, size_t w, size_t h), (d, p, v, w, h))
GATED_DRV(cuMemsetD2D32_v2, (CUdeviceptr d, size_t p, unsigned v, size_t w, size_t h), (d, p, v, w, h))

// Introspection for tests: 1 when the shim is connected to a daemon.
int nixie_shim_active(void) { return active() ? 1 : 0; }
unsigned nixie_shim_app(void) { return active() ? g.app : 0xFFFFFFFFu; }

}  // extern "C"
