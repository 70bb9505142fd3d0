// Tier backing stores, NUMA placement and the host copy pool (phys.hpp).
#include "phys.hpp"
#include "vmm.hpp"

#include <pthread.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <immintrin.h>

#include <cctype>
#include <cstring>
#include <fstream>
#include <sstream>

namespace nixie::b200 {

std::string cuda_msg(cudaError_t e, const char* what) {
  return std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
}

namespace {

std::string read_line(const std::string& path) {
  std::ifstream f(path);
  std::string s;
  if (f) std::getline(f, s);
  return s;
}

std::vector<int> parse_cpulist(const std::string& s) {
  std::vector<int> cpus;
  std::stringstream ss(s);
  std::string part;
  while (std::getline(ss, part, ',')) {
    if (part.empty()) continue;
    const auto dash = part.find('-');
    try {
      if (dash == std::string::npos) {
        cpus.push_back(std::stoi(part));
      } else {
        const int lo = std::stoi(part.substr(0, dash)), hi = std::stoi(part.substr(dash + 1));
        for (int c = lo; c <= hi; ++c) cpus.push_back(c);
      }
    } catch (const std::exception&) {
    }
  }
  return cpus;
}

// The node holding most of `cpus` (sysfs node*/cpulist), or -1. Used when the
// device's numa_node reads -1 (firmware did not describe the affinity) but
// its local_cpulist is narrower than the machine.
int node_of_cpus(const std::vector<int>& cpus) {
  if (cpus.empty()) return -1;
  int best = -1;
  std::size_t best_n = 0, nodes = 0;
  for (int n = 0; n < 1024; ++n) {
    const std::string list = read_line("/sys/devices/system/node/node" + std::to_string(n) + "/cpulist");
    if (list.empty()) {
      if (n > 64) break;
      continue;
    }
    ++nodes;
    const std::vector<int> nc = parse_cpulist(list);
    std::size_t hit = 0;
    for (int c : cpus)
      for (int d : nc) hit += (c == d);
    if (hit > best_n) {
      best_n = hit;
      best = n;
    }
  }
  // One node, or the local list spans several nodes evenly: nothing to bind to.
  if (nodes <= 1 || best_n * 2 <= cpus.size()) return -1;
  return best;
}

}  // namespace

NumaInfo numa_for_device(int device) {
  NumaInfo info;
  char bus[64] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), device) != cudaSuccess) return info;
  std::string id(bus);
  for (char& c : id) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  // sysfs uses a 4-digit domain; CUDA may print 8.
  if (id.size() > 12 && id.find(':') == 8) id = id.substr(4);
  info.pci_bus_id = id;
  const std::string dir = "/sys/bus/pci/devices/" + id;
  const std::string node = read_line(dir + "/numa_node");
  try {
    info.node = node.empty() ? -1 : std::stoi(node);
  } catch (const std::exception&) {
    info.node = -1;
  }
  info.cpus = parse_cpulist(read_line(dir + "/local_cpulist"));
  if (info.node < 0) {
    info.node = node_of_cpus(info.cpus);
    info.node_from_cpus = info.node >= 0;
  }
  // Keep only CPUs this process may run on.
  cpu_set_t allowed;
  CPU_ZERO(&allowed);
  if (sched_getaffinity(0, sizeof(allowed), &allowed) == 0) {
    std::vector<int> ok;
    for (int c : info.cpus)
      if (c >= 0 && c < CPU_SETSIZE && CPU_ISSET(c, &allowed)) ok.push_back(c);
    info.cpus = ok;
  }
  return info;
}

void prefer_numa_node(int node) {
  constexpr int kMpolDefault = 0, kMpolPreferred = 1;
  if (node < 0) {
    syscall(SYS_set_mempolicy, kMpolDefault, nullptr, 0);
    return;
  }
  unsigned long mask[16] = {0};
  if (node >= static_cast<int>(sizeof(mask) * 8)) return;
  mask[node / (8 * sizeof(unsigned long))] |= 1ul << (node % (8 * sizeof(unsigned long)));
  syscall(SYS_set_mempolicy, kMpolPreferred, mask, sizeof(mask) * 8);
}

void pin_thread_to(const std::vector<int>& cpus) {
  if (cpus.empty()) return;
  cpu_set_t set;
  CPU_ZERO(&set);
  for (int c : cpus)
    if (c >= 0 && c < CPU_SETSIZE) CPU_SET(c, &set);
  pthread_setaffinity_np(pthread_self(), sizeof(set), &set);
}

void DeviceArena::init(Bytes capacity, bool exportable, int device, Bytes slab_bytes, Bytes reserve) {
  const auto units = static_cast<std::uint32_t>(capacity / kBlockBytes);
  if (units > 0) {
    if (exportable) {
      vmm_ = new ExportableArena();
      vmm_->init(device, static_cast<Bytes>(units) * kBlockBytes, slab_bytes ? slab_bytes : kBlockBytes, reserve);
      base_ = vmm_->base();
    } else {
      NX_CUDA(cudaMalloc(&base_, static_cast<std::size_t>(units) * kBlockBytes));
    }
  }
  ring.reset(units);
}

DeviceArena::~DeviceArena() {
  if (vmm_) {
    delete vmm_;
  } else if (base_) {
    cudaFree(base_);
  }
}

int DeviceArena::export_fd(std::uint32_t slab) const { return vmm_ ? vmm_->export_fd(slab) : -1; }

std::uint32_t DeviceArena::grow_slab() {
  if (!vmm_) throw SimError(Err::InvalidState, "only an exportable arena grows");
  const std::uint32_t s = vmm_->grow();
  const auto per = static_cast<std::uint32_t>(vmm_->slab_bytes() / kBlockBytes);
  const auto frames = static_cast<std::uint32_t>((s + 1) * per);
  if (frames > ring.units()) ring.reset(frames);  // the frame count (the placer owns the frames)
  return s;
}

void DeviceArena::drop_slab(std::uint32_t slab) {
  if (!vmm_) throw SimError(Err::InvalidState, "only an exportable arena shrinks");
  vmm_->drop(slab);
}

void PinnedRing::init(Bytes capacity, int numa_node) {
  const auto units = static_cast<std::uint32_t>(capacity / kBlockBytes);
  bytes_ = static_cast<Bytes>(units) * kBlockBytes;
  if (units > 0) {
    prefer_numa_node(numa_node);
    void* p = nullptr;
    const cudaError_t e = cudaHostAlloc(&p, bytes_, cudaHostAllocMapped | cudaHostAllocPortable);
    prefer_numa_node(-1);
    NX_CUDA(e);
    host_ = static_cast<std::uint8_t*>(p);
    void* d = nullptr;
    NX_CUDA(cudaHostGetDevicePointer(&d, p, 0));
    dev_ = static_cast<std::uint8_t*>(d);
  }
  ring.reset(units);
}

PinnedRing::~PinnedRing() {
  if (host_) cudaFreeHost(host_);
}

void PagedStore::init(Bytes capacity) {
  const Bytes capped = capacity == kUnbounded ? 4096 * kGiB : capacity;
  const auto units = static_cast<std::uint32_t>(capped / kBlockBytes);
  regions_.assign((units + kUnitsPerRegion - 1) / kUnitsPerRegion, nullptr);
  ring.reset(units);
}

std::uint8_t* PagedStore::unit(std::uint32_t u) {
  const std::uint32_t r = u / kUnitsPerRegion;
  if (regions_[r] == nullptr) {
    const std::size_t len = static_cast<std::size_t>(kUnitsPerRegion) * kBlockBytes;
    void* p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) throw SimError(Err::IoError, "mmap of a paged-tier region failed");
    madvise(p, len, MADV_HUGEPAGE);
    regions_[r] = static_cast<std::uint8_t*>(p);
  }
  return regions_[r] + static_cast<std::size_t>(u % kUnitsPerRegion) * kBlockBytes;
}

PagedStore::~PagedStore() {
  for (std::uint8_t* p : regions_)
    if (p) munmap(p, static_cast<std::size_t>(kUnitsPerRegion) * kBlockBytes);
}

void HostCopyPool::start(int threads, const std::vector<int>& cpus, int active) {
  if (threads < 1) threads = 1;
  active_.store(active > 0 ? std::min(active, threads) : threads);
  for (int i = 0; i < threads; ++i) threads_.emplace_back(&HostCopyPool::worker, this, i, cpus);
}

void HostCopyPool::set_active(int n) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    active_.store(std::max(1, std::min(n, static_cast<int>(threads_.size()))));
  }
  idle_cv_.notify_all();
  cv_.notify_all();
}

HostCopyPool::~HostCopyPool() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  idle_cv_.notify_all();
  for (auto& t : threads_) t.join();
}

namespace {
// 256 bytes per iteration: eight 32-byte loads, eight streaming stores. The
// sfence makes the stores visible before the completion is published.
__attribute__((target("avx2"))) void stream_copy(void* dst, const void* src, std::size_t bytes) {
  auto* d = static_cast<__m256i*>(dst);
  const auto* s = static_cast<const __m256i*>(src);
  const std::size_t n = bytes / 32;
  std::size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    const __m256i a0 = _mm256_load_si256(s + i), a1 = _mm256_load_si256(s + i + 1), a2 = _mm256_load_si256(s + i + 2),
                  a3 = _mm256_load_si256(s + i + 3), a4 = _mm256_load_si256(s + i + 4), a5 = _mm256_load_si256(s + i + 5),
                  a6 = _mm256_load_si256(s + i + 6), a7 = _mm256_load_si256(s + i + 7);
    _mm256_stream_si256(d + i, a0);
    _mm256_stream_si256(d + i + 1, a1);
    _mm256_stream_si256(d + i + 2, a2);
    _mm256_stream_si256(d + i + 3, a3);
    _mm256_stream_si256(d + i + 4, a4);
    _mm256_stream_si256(d + i + 5, a5);
    _mm256_stream_si256(d + i + 6, a6);
    _mm256_stream_si256(d + i + 7, a7);
  }
  for (; i < n; ++i) _mm256_stream_si256(d + i, _mm256_load_si256(s + i));
  _mm_sfence();
  std::memcpy(static_cast<char*>(dst) + n * 32, static_cast<const char*>(src) + n * 32, bytes - n * 32);
}
bool have_avx2() {
  static const bool ok = __builtin_cpu_supports("avx2");
  return ok;
}
}  // namespace

void HostCopyPool::worker(int index, std::vector<int> cpus) {
  pin_thread_to(cpus);
  while (true) {
    Job j;
    {
      std::unique_lock<std::mutex> lk(mu_);
      for (;;) {
        if (stop_ && jobs_.empty()) return;
        if (!stop_ && index >= active_.load()) {  // parked: waits on its own condition
          cv_.notify_one();                        // pass on a wake-up it may have taken
          idle_cv_.wait(lk);
          continue;
        }
        if (!jobs_.empty()) break;
        cv_.wait(lk);
      }
      j = jobs_.front();
      jobs_.pop_front();
    }
    if (streaming_.load(std::memory_order_relaxed) && have_avx2() &&
        ((reinterpret_cast<std::uintptr_t>(j.dst) | reinterpret_cast<std::uintptr_t>(j.src)) & 31) == 0)
      stream_copy(j.dst, j.src, j.bytes);
    else
      std::memcpy(j.dst, j.src, j.bytes);
    {
      std::lock_guard<std::mutex> lk(done_mu_);
      done_.push_back(j.token);
    }
    done_count_.fetch_add(1, std::memory_order_release);
  }
}

void HostCopyPool::submit(void* dst, const void* src, std::size_t bytes, std::uint64_t token) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    jobs_.push_back(Job{dst, src, bytes, token});
  }
  cv_.notify_one();
}

bool HostCopyPool::drain(std::vector<std::uint64_t>& out) {
  if (done_count_.load(std::memory_order_acquire) == drained_) return false;
  std::lock_guard<std::mutex> lk(done_mu_);
  drained_ += done_.size();
  out.insert(out.end(), done_.begin(), done_.end());
  done_.clear();
  return true;
}

void HostCopyPool::copy_all(const std::vector<std::pair<void*, const void*>>& pairs, std::size_t bytes) {
  constexpr std::uint64_t kBulkTag = 1ull << 63;
  for (std::size_t i = 0; i < pairs.size(); ++i) submit(pairs[i].first, pairs[i].second, bytes, kBulkTag | i);
  std::size_t got = 0;
  std::vector<std::uint64_t> toks;
  while (got < pairs.size()) {
    toks.clear();
    if (drain(toks)) got += toks.size();
    else std::this_thread::yield();
  }
}

}  // namespace nixie::b200
