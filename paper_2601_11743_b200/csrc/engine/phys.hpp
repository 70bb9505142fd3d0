// Physical backing of the three tiers the CUDA engine serves, and the host
// copy pool for the pinned<->paged lanes (internal header).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "nixie/errors.hpp"
#include "nixie/units.hpp"

namespace nixie::b200 {

std::string cuda_msg(cudaError_t e, const char* what);

// A failed CUDA call (reported as NX_E_CUDA through the C ABI).
class CudaFailure : public SimError {
 public:
  explicit CudaFailure(const std::string& what) : SimError(Err::IoError, what) {}
};

#define NX_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t nx_e_ = (call);                                                            \
    if (nx_e_ != cudaSuccess) throw ::nixie::b200::CudaFailure(::nixie::b200::cuda_msg(nx_e_, #call)); \
  } while (0)

// A fixed set of 2 MiB units handed out FIFO (a ring: freed units go to the
// back). acquire() failing means the registry let a tier overcommit.
// acquire_after(prev) hands out the unit right after `prev` when it is free:
// consecutive acquisitions of one stream of legs (a lane's departures into
// the pinned ring) then stay contiguous, so their copies merge into long
// copy-engine calls even after the ring's free order has fragmented. A unit
// taken that way stays in the FIFO as a stale entry, skipped when reached.
class UnitRing {
 public:
  static constexpr std::uint32_t kNone = ~0u;
  void reset(std::uint32_t units) {
    free_.clear();
    is_free_.assign(units, 1);
    for (std::uint32_t u = 0; u < units; ++u) free_.push_back(u);
    units_ = units;
    n_free_ = units;
  }
  std::uint32_t acquire(const char* tier) {
    while (!free_.empty() && !is_free_[free_.front()]) free_.pop_front();  // stale entries
    if (free_.empty()) throw InvariantViolation(std::string(tier) + " has no free 2 MiB unit (budget overcommitted)");
    const std::uint32_t u = free_.front();
    free_.pop_front();
    take(u);
    return u;
  }
  std::uint32_t acquire_after(std::uint32_t prev, const char* tier) {
    if (prev != kNone && prev + 1 < units_ && is_free_[prev + 1]) {
      take(prev + 1);
      return prev + 1;
    }
    return acquire(tier);
  }
  void release(std::uint32_t u) {
    is_free_[u] = 1;
    ++n_free_;
    free_.push_back(u);
    if (free_.size() > 2 * static_cast<std::size_t>(units_) + 64) compact();
  }
  std::uint32_t units() const { return units_; }
  std::size_t free_units() const { return n_free_; }

 private:
  void take(std::uint32_t u) {
    is_free_[u] = 0;
    --n_free_;
  }
  // Drops stale and duplicate entries, keeping the FIFO order of the rest.
  void compact() {
    std::vector<std::uint8_t> seen(units_, 0);
    std::deque<std::uint32_t> keep;
    for (std::uint32_t u : free_)
      if (is_free_[u] && !seen[u]) {
        seen[u] = 1;
        keep.push_back(u);
      }
    free_.swap(keep);
  }
  std::deque<std::uint32_t> free_;
  std::vector<std::uint8_t> is_free_;
  std::uint32_t units_ = 0;
  std::size_t n_free_ = 0;
};

// NUMA placement of the GPU's host-side resources.
struct NumaInfo {
  int node = -1;
  bool node_from_cpus = false;  // sysfs numa_node was -1; derived from local_cpulist
  std::vector<int> cpus;        // local CPU list (allowed by this process's affinity)
  std::string pci_bus_id;
};
NumaInfo numa_for_device(int device);
// Prefer `node` for this thread's future page allocations (-1: default policy).
void prefer_numa_node(int node);
void pin_thread_to(const std::vector<int>& cpus);

class ExportableArena;

// tier 0: one allocation of the capped budget: cudaMalloc, or (exportable,
// for the interposer daemon) one VMM allocation whose handle the shims import
// to map frames at their applications' stable virtual addresses (vmm.hpp).
class DeviceArena {
 public:
  void init(Bytes capacity, bool exportable = false, int device = 0, Bytes slab_bytes = 0, Bytes reserve = 0);
  // Exportable arenas only: one more slab at the end (frames grow with it).
  std::uint32_t grow_slab();
  void drop_slab(std::uint32_t slab);
  ~DeviceArena();
  std::uint8_t* frame(std::uint32_t u) const { return base_ + static_cast<std::size_t>(u) * kBlockBytes; }
  std::uint8_t* base() const { return base_; }
  int export_fd(std::uint32_t slab) const;  // -1 unless exportable
  UnitRing ring;

 private:
  std::uint8_t* base_ = nullptr;
  ExportableArena* vmm_ = nullptr;
};

// tier 1: the pinned staging ring, exactly `capacity` bytes of
// cudaHostAlloc(mapped | portable) memory (not write-combined: host threads
// read it on the pinned->paged lane).
class PinnedRing {
 public:
  void init(Bytes capacity, int numa_node);
  ~PinnedRing();
  std::uint8_t* host(std::uint32_t u) const { return host_ + static_cast<std::size_t>(u) * kBlockBytes; }
  std::uint8_t* dev(std::uint32_t u) const { return dev_ + static_cast<std::size_t>(u) * kBlockBytes; }
  Bytes bytes() const { return bytes_; }
  UnitRing ring;

 private:
  std::uint8_t* host_ = nullptr;
  std::uint8_t* dev_ = nullptr;
  Bytes bytes_ = 0;
};

// tier 2: pageable memory in 64 MiB regions mapped on first use.
class PagedStore {
 public:
  void init(Bytes capacity);
  ~PagedStore();
  std::uint8_t* unit(std::uint32_t u);
  UnitRing ring;

 private:
  static constexpr std::uint32_t kUnitsPerRegion = 32;
  std::vector<std::uint8_t*> regions_;
};

// Fixed worker pool for 2 MiB host memcpy legs; completions are drained by
// the engine thread.
class HostCopyPool {
 public:
  // Starts `threads` workers; the first `active` of them take jobs (the rest
  // wait until set_active raises the count: the engine sizes the pool from a
  // measurement, SwapEngine::calibrate_host).
  void start(int threads, const std::vector<int>& cpus, int active = 0);
  void set_active(int n);
  // Copy with non-temporal (streaming) stores when the CPU has AVX2 and the
  // buffers are 32-byte aligned: no read-for-ownership of the destination, so
  // a copied byte costs two DRAM transfers instead of three.
  void set_streaming(bool on) { streaming_.store(on); }
  int active() const { return active_.load(); }
  int size() const { return static_cast<int>(threads_.size()); }
  ~HostCopyPool();
  void submit(void* dst, const void* src, std::size_t bytes, std::uint64_t token);
  // Moves finished tokens into `out`; cheap when nothing finished.
  bool drain(std::vector<std::uint64_t>& out);
  // Parallel memcpy of many buffers, blocking (setup paths only).
  void copy_all(const std::vector<std::pair<void*, const void*>>& pairs, std::size_t bytes);

 private:
  struct Job {
    void* dst;
    const void* src;
    std::size_t bytes;
    std::uint64_t token;
  };
  void worker(int index, std::vector<int> cpus);
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_;       // active workers wait here for jobs
  std::condition_variable idle_cv_;  // workers beyond the active count
  std::deque<Job> jobs_;
  std::mutex done_mu_;
  std::vector<std::uint64_t> done_;
  std::atomic<std::uint64_t> done_count_{0};
  std::uint64_t drained_ = 0;
  bool stop_ = false;
  std::atomic<int> active_{0};
  std::atomic<bool> streaming_{false};
};

}  // namespace nixie::b200
