// CUDA swap engine: the shared lane state machine (csrc/host/lanes.hpp)
// driven by real copies. See include/nixie/swap_engine.hpp for the tier
// backing; this file is the per-switch control loop.
//
// Control loop of execute():
//   LaneSet::begin() starts the FIFO heads of every lane (up to the in-flight
//   limit), each start = MemState::begin_move + a physical unit for the
//   destination. Started PCIe legs are batched into K1 launches (or CE
//   batches) on the lane's stream; started host legs go straight to the copy
//   pool. The loop then polls batch-end events and pool completions, commits
//   finished legs in per-lane FIFO order (LaneSet::finish_hop: commit_move,
//   next hop, window, pump), and launches whatever the commits unblocked.
//   A fetch into a full GPU therefore starts the moment the eviction that
//   frees its frame has landed, with several launches queued per stream so
//   the link never waits on the host.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <limits>
#include <array>
#include <chrono>
#include <cstring>
#include <functional>
#include <deque>
#include <map>
#include <thread>

#include "lanes.hpp"
#include "nixie/swap_engine.hpp"
#include "nx_kernels.h"
#include "phys.hpp"

namespace nixie::b200 {

namespace {

using Clock = std::chrono::steady_clock;
double secs_since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

constexpr int kH2D = 0;  // stream / PCIe lane index (lane 0 = pinned -> GPU)
constexpr int kD2H = 1;  // (lane 1 = GPU -> pinned)
constexpr std::uint32_t kBounceUnits = 64;  // 128 MiB pinned bounce for paged fills / compares

int log2_bucket(int n) {
  int k = 0;
  while ((1 << (k + 1)) <= n) ++k;
  return k;
}

}  // namespace

struct ExecOptions {
  cudaStream_t drain = nullptr;
  cudaEvent_t gate_event = nullptr;              // recorded on the H2D stream after the last fetch
  void (*gate_callback)(void*) = nullptr;        // then called (launch-gate release)
  void* gate_ctx = nullptr;
};

struct SwapEngine::Impl final : detail::LaneSink {
  EngineConfig cfg;
  MemState mem;
  HardwareConfig hw;
  NumaInfo numa;
  DeviceArena arena;
  FramePlacer* placer = nullptr;
  std::function<void()> progress;  // called on the engine thread after commits
  PinnedRing pinned;
  PagedStore paged;
  HostCopyPool pool;
  cudaStream_t st[2] = {nullptr, nullptr};
  cudaStream_t aux = nullptr;
  int sm_count = 0;
  int max_ctas = 0;
  int k3_ctas = 0;  // checksum-only launches: HBM-bound, want more resident warps

  // Per-block state, indexed by BlockId.
  std::vector<std::uint32_t> unit;  // frame / slot / paged unit of the block's current (source) tier
  NxCkTables ck{};
  std::size_t ck_cap = 0;
  std::uint64_t* d_frames = nullptr;  // device frame table
  std::uint64_t* h_frames = nullptr;  // pinned mirror
  std::uint64_t* h_frames_stage = nullptr;
  NxScratch scratch[4]{};  // [0..1] lane streams, [2..3] checksum side streams
  cudaStream_t cks[2] = {nullptr, nullptr};
  std::uint8_t* bounce = nullptr;  // pinned, kBounceUnits slots (outside the budget)
  NxDevStatus status_seen{};
  std::vector<bool> auto_sm;
  std::uint64_t launches_total = 0;

  // Per-execute state.
  struct Leg {
    std::size_t mi;
    BlockId block;
    TierId from, to;
    std::uint32_t src_u, dst_u;
    int lane;
    bool done;
    double t_start;
    std::size_t rec;
  };
  struct Batch {
    std::vector<std::uint32_t> legs;
    cudaEvent_t ev_start, ev_end;
    cudaEvent_t ev_copied = nullptr;  // CE batch: its copies landed
    double host_submit = 0, host_done = 0;
    int stream;
    bool ce;
    bool end_on_side = false;                        // CE batch: ends on the checksum side stream
    cudaEvent_t dep_done = nullptr;                  // grouped K3: the record launch covering its departures
    // CE departure batch (grouped K3): commit groups inside the batch, each
    // ending at legs[end] (exclusive) behind its own copy event; the last
    // group is the batch itself (ev_end / dep_done).
    struct SubCommit {
      std::uint32_t end;
      cudaEvent_t copied;
      cudaEvent_t dep_done;  // the record launch covering the group's departures
    };
    std::vector<SubCommit> subs;
    bool early = false;  // departures committed at submission (early_frame_release)
    std::size_t sub_next = 0, committed = 0;  // next group to poll; legs completed so far
    std::vector<std::array<cudaEvent_t, 2>> k3ev;    // CE batch: K3 launch start/end
    std::vector<std::uint32_t> k3slot;               // device-clock slot per K3 launch
    Bytes k3_bytes = 0;
  };
  std::array<int, 2> batches_sent{};  // per PCIe lane this execute (batch-size ramp)
  std::size_t d2h_legs_sent = 0;      // departures submitted this execute (commit-group ramp)
  std::size_t batches_submitted = 0;  // PCIe batches submitted since construction

  // early_frame_release: a departure commits when its copy is queued. Its
  // GPU frame is free "as of" the event ending its group (seq, 1-based, in
  // D2H stream order) and of the record launch covering it; a fetch into the
  // frame waits for both on the H2D stream. Its pinned slot holds data in
  // flight until the batch lands (a second hop out of it waits).
  bool early_mode = false;
  std::vector<std::uint32_t> frame_seq;   // arena frame -> group seq freeing it (0: free)
  std::vector<cudaEvent_t> frame_dep;     // arena frame -> record launch covering its departure
  std::vector<cudaEvent_t> seq_events;    // seq - 1 -> event
  std::vector<std::uint8_t> slot_inflight;  // pinned slot -> early-committed copy still landing
  std::uint32_t h2d_seq_waited = 0;
  bool h2d_waited_head = false, h2d_waited_all = false;
  std::vector<std::uint32_t> early_done;  // departures to commit once the current flush pass ends
  std::vector<std::uint32_t> host_wait;   // host legs waiting for their pinned source to land

  // Pacing (EngineConfig::pace_lag_legs, early frame release only): the D2H
  // group starting at departure x waits on the device for the fetches to have
  // landed up to x - lag. Fetch copies leave marks (fetch legs copied so far,
  // event after them) on the H2D stream; a departure group is submitted only
  // once the mark it needs exists (device waits are enqueued after the work
  // that satisfies them), unless nothing on the H2D side can move without it.
  bool pacing = false;
  std::vector<std::pair<std::size_t, cudaEvent_t>> h2d_marks;
  std::size_t h2d_marked = 0;     // fetch legs covered by marks this execute
  std::size_t d2h_mark_next = 0;  // marks before this one are already waited on by the D2H stream

  // Fetch legs that must have landed before the departure group starting at x.
  std::size_t pace_need(std::size_t x) const {
    const auto lag = static_cast<std::size_t>(cfg.pace_lag_legs);
    if (!pacing || x <= lag || x - lag > fetches_total) return 0;  // nothing (left) to pace against
    return x - lag;
  }
  std::size_t d2h_group_legs(std::size_t sent) const {
    const std::size_t small = static_cast<std::size_t>(std::max(1, cfg.first_batch_legs));
    return sent < 32 * small ? small : static_cast<std::size_t>(std::max(1, cfg.d2h_commit_legs));
  }
  void pace_wait(std::size_t x) {
    const std::size_t need = pace_need(x);
    if (need == 0) return;
    if (d2h_mark_next > 0 && h2d_marks[d2h_mark_next - 1].first >= need) return;  // already waited on
    std::size_t m = d2h_mark_next;
    while (m < h2d_marks.size() && h2d_marks[m].first < need) ++m;
    if (m == h2d_marks.size()) return;  // not queued yet (flush_pass let it go unpaced)
    NX_CUDA(cudaStreamWaitEvent(st[kD2H], h2d_marks[m].second, 0));
    ++stats.pace_waits;
    d2h_mark_next = m + 1;
  }

  template <typename T>
  static T& at_grow(std::vector<T>& v, std::size_t i) {
    if (i >= v.size()) v.resize(i + 1, T{});
    return v[i];
  }

  // Grouped K3 (CE path, one K3 stream): one table launch records every
  // departing block of the switch at its start; arrival checks run per group
  // of landed batches. Descriptors live in a device table (uploaded from a
  // pinned stage) so a launch covers any number of legs.
  struct GroupK3 {
    cudaEvent_t a, z;
    int legs;
    int lane;
    std::uint32_t slot;
  };
  bool grouped = false;
  NxLeg* d_ktab = nullptr;
  NxLeg* h_ktab = nullptr;
  std::size_t ktab_cap = 0, ktab_used = 0;
  NxScratch tscratch{};
  std::size_t tscratch_cap = 0;
  std::vector<GroupK3> gk3;
  std::vector<NxLeg> vgroup;          // landed-or-landing arrivals not yet checked
  std::vector<std::uint32_t> dep_pos;  // block -> position in the switch's departure order (grouped K3)
  std::size_t dep_head = 0;            // departures covered by the first record launch
  cudaEvent_t rec_head = nullptr, rec_all = nullptr;
  cudaEvent_t vgroup_copied = nullptr;
  std::vector<K3Launch> k3_trace;     // last execute's K3 launches (device times)
  std::vector<BatchTrace> batch_tr;   // last execute's PCIe batches (timeline)
  std::uint32_t k3_slots_used = 0;    // device-clock slots handed out this execute

  // Capacity for `n` table legs this execute (grown before any work is queued).
  void reserve_table(std::size_t n) {
    if (n > ktab_cap) {
      NX_CUDA(cudaDeviceSynchronize());
      if (d_ktab) cudaFree(d_ktab);
      if (h_ktab) cudaFreeHost(h_ktab);
      const std::size_t cap = std::max<std::size_t>(n, 2 * ktab_cap);
      NX_CUDA(cudaMalloc(&d_ktab, sizeof(NxLeg) * cap));
      void* h = nullptr;
      NX_CUDA(cudaHostAlloc(&h, sizeof(NxLeg) * cap, cudaHostAllocPortable | cudaHostAllocMapped));  // read by launch_table_upload
      h_ktab = static_cast<NxLeg*>(h);
      ktab_cap = cap;
    }
    if (n > tscratch_cap) {
      NX_CUDA(cudaDeviceSynchronize());
      cudaFree(tscratch.part_sums);
      cudaFree(tscratch.part_count);
      cudaFree(tscratch.leg_acc);
      const std::size_t cap = std::max<std::size_t>(n, 2 * tscratch_cap);
      NX_CUDA(cudaMalloc(&tscratch.part_sums, sizeof(unsigned long long)));
      NX_CUDA(cudaMalloc(&tscratch.part_count, sizeof(unsigned int) * cap));
      NX_CUDA(cudaMemset(tscratch.part_count, 0, sizeof(unsigned int) * cap));
      NX_CUDA(cudaMalloc(&tscratch.leg_acc, sizeof(unsigned long long) * cap));
      NX_CUDA(cudaMemset(tscratch.leg_acc, 0, sizeof(unsigned long long) * cap));
      tscratch_cap = cap;
    }
  }

  // One K3 table launch on the (single) K3 stream over `l`.
  void k3_table_launch(const std::vector<NxLeg>& l, bool arriving, int lane) {
    const std::size_t n = l.size();
    if (ktab_used + n > ktab_cap) throw InvariantViolation("K3 descriptor table overflow");
    std::memcpy(h_ktab + ktab_used, l.data(), sizeof(NxLeg) * n);
    cudaStream_t cs = cks[0];
    NX_CUDA(launch_table_upload(d_ktab + ktab_used, h_ktab + ktab_used, static_cast<int>(n), cs));
    ++launches_total;
    GroupK3 g{take_event(), take_event(), static_cast<int>(n), lane,
              k3_slots_used < kClockSlots ? k3_slots_used++ : kNoClockSlot};
    NX_CUDA(cudaEventRecord(g.a, cs));
    NX_CUDA(launch_checksum_tma_table(d_ktab + ktab_used, static_cast<int>(n), arriving, cfg.verify ? kNxVerify : 0u, ck,
                                      tscratch, sm_count, cs, g.slot));
    NX_CUDA(cudaEventRecord(g.z, cs));
    ktab_used += n;
    gk3.push_back(g);
    ++stats.launches[lane == 0 ? kH2D : kD2H];
    ++launches_total;
  }

  // Checks the arrivals collected so far (after their copies landed). Nothing
  // in the switch waits on it: an arrived block belongs to the incoming app,
  // which cannot run before the gate release (which waits for this stream),
  // and the status is read once every launch has finished.
  void flush_verify() {
    if (vgroup.empty()) return;
    NX_CUDA(cudaStreamWaitEvent(cks[0], vgroup_copied, 0));  // copies land in order on the H2D stream
    k3_table_launch(vgroup, true, 0);
    vgroup.clear();
  }

  // K3 checksum-only launch of a CE batch (record on departure, verify on arrival).
  void k3_launch(Batch& B, const std::vector<NxLeg>& l, bool arriving, cudaStream_t cs, std::uint32_t flags) {
    const int n = static_cast<int>(l.size());
    cudaEvent_t a = take_event(), z = take_event();
    NX_CUDA(cudaEventRecord(a, cs));
    if (cfg.k3_tma)
      NX_CUDA(launch_checksum_tma(l.data(), n, arriving, flags, ck, scratch[2 + B.stream], sm_count, cs,
                                  k3_slots_used < kClockSlots ? k3_slots_used : kNoClockSlot));
    else
      NX_CUDA(launch_swap(l.data(), arriving ? 0 : n, arriving ? n : 0, flags, ck, scratch[2 + B.stream], k3_ctas, cs));
    NX_CUDA(cudaEventRecord(z, cs));
    B.k3ev.push_back({a, z});
    B.k3slot.push_back(cfg.k3_tma && k3_slots_used < kClockSlots ? k3_slots_used++ : kNoClockSlot);
    B.k3_bytes += static_cast<Bytes>(n) * kBlockBytes;
    ++stats.launches[B.stream];
    ++launches_total;
  }
  detail::LaneSet* lanes = nullptr;
  bool finished = false;
  std::vector<Leg> legs;
  std::array<std::vector<std::uint32_t>, detail::kLaneCount> pending;
  std::array<std::deque<std::uint32_t>, detail::kLaneCount> host_fifo;
  std::array<std::deque<Batch>, 2> inflight;
  std::vector<Batch> landed;
  std::vector<cudaEvent_t> events;
  std::size_t events_used = 0;
  cudaEvent_t ev0 = nullptr;
  Clock::time_point t0;
  SwitchStats stats;
  std::array<std::vector<LegTrace>, detail::kLaneCount> trace;
  std::vector<TransferRecord>* records = nullptr;
  const ExecOptions* opts = nullptr;
  std::size_t fetches_total = 0, fetches_submitted = 0;
  AppId incoming = kNoApp;
  bool gate_done = false;

  explicit Impl(const EngineConfig& c) : cfg(c) {
    pinned_prev.fill(UnitRing::kNone);
    if (cfg.gpu_capacity % kBlockBytes || cfg.pinned_capacity % kBlockBytes ||
        (cfg.paged_capacity != kUnbounded && cfg.paged_capacity % kBlockBytes))
      throw SimError(Err::ValidationError, "tier budgets must be multiples of 2 MiB");
    if (cfg.legs_per_launch < 1 || cfg.legs_per_launch > kMaxLegsPerLaunch)
      throw SimError(Err::ValidationError, "legs_per_launch must be in [1, 256]");
    if (cfg.k3_verify_group < 1) throw SimError(Err::ValidationError, "k3_verify_group must be >= 1");
    NX_CUDA(cudaSetDevice(cfg.device));
    sm_count = device_sm_count(cfg.device);
    max_ctas = cfg.max_ctas > 0 ? cfg.max_ctas : 2 * std::max(sm_count, 1);
    k3_ctas = 4 * std::max(sm_count, 1);
    if (cfg.numa_bind) numa = numa_for_device(cfg.device);

    hw.tier_capacity[0] = cfg.gpu_capacity;
    hw.tier_capacity[1] = cfg.pinned_capacity;
    hw.tier_capacity[2] = cfg.paged_capacity;
    hw.tier_capacity[3] = 0;
    hw.apply_to(mem);

    arena.init(cfg.gpu_physical ? cfg.gpu_physical : cfg.gpu_capacity, cfg.exportable_arena, cfg.device, cfg.arena_slab_bytes,
               cfg.gpu_physical_max);
    pinned.init(cfg.pinned_capacity, numa.node);
    paged.init(cfg.paged_capacity);
    {
      const int ncpu = numa.cpus.empty() ? static_cast<int>(std::thread::hardware_concurrency()) : static_cast<int>(numa.cpus.size());
      const int maxt = std::max(1, std::min(ncpu, 32));
      pool.start(std::max(cfg.host_threads, maxt), numa.cpus, cfg.host_threads > 0 ? cfg.host_threads : maxt);
      pool.set_streaming(cfg.host_streaming_copy);
    }
    for (auto& s : st) NX_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    NX_CUDA(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
    // K3 checksum launches of both lanes share one stream by default, so they
    // never compete for the SMs (each is a full-GPU TMA pipeline). This
    // cannot deadlock: a fetch is submitted only after the eviction batch that
    // frees its frames has ended (record included), so a verify never waits
    // on a copy that waits on a record queued behind it.
    NX_CUDA(cudaStreamCreateWithFlags(&cks[0], cudaStreamNonBlocking));
    if (cfg.k3_one_stream) cks[1] = cks[0];
    else NX_CUDA(cudaStreamCreateWithFlags(&cks[1], cudaStreamNonBlocking));
    NX_CUDA(cudaMalloc(&ck.status, sizeof(NxDevStatus)));
    NX_CUDA(cudaMalloc(&ck.kstart, sizeof(unsigned long long) * kClockSlots));
    NX_CUDA(cudaMalloc(&ck.kend, sizeof(unsigned long long) * kClockSlots));
    NX_CUDA(cudaMemset(ck.status, 0, sizeof(NxDevStatus)));
    for (auto& s : scratch) {
      NX_CUDA(cudaMalloc(&s.part_sums, sizeof(unsigned long long) * (kMaxLegsPerLaunch << kMaxPartsLog2)));
      NX_CUDA(cudaMalloc(&s.part_count, sizeof(unsigned int) * kMaxLegsPerLaunch));
      NX_CUDA(cudaMemset(s.part_count, 0, sizeof(unsigned int) * kMaxLegsPerLaunch));
      NX_CUDA(cudaMalloc(&s.leg_acc, sizeof(unsigned long long) * kMaxLegsPerLaunch));
      NX_CUDA(cudaMemset(s.leg_acc, 0, sizeof(unsigned long long) * kMaxLegsPerLaunch));
    }
    void* b = nullptr;
    NX_CUDA(cudaHostAlloc(&b, static_cast<std::size_t>(kBounceUnits) * kBlockBytes, cudaHostAllocMapped | cudaHostAllocPortable));
    bounce = static_cast<std::uint8_t*>(b);
    NX_CUDA(cudaEventCreate(&ev0));
    grow_tables(65536);
    if (cfg.host_threads <= 0) calibrate_host(256 * kMiB);
  }

  HostCalibration host_cal;

  HostCalibration calibrate_host(Bytes bytes) {
    if (!pf_queue.empty() || !pf_inflight.empty()) prefetch_quiesce();  // the pool's completions must all be ours
    constexpr std::size_t kSpan = 64 * kMiB;  // per direction per round
    const std::size_t rounds = std::max<std::size_t>(1, bytes / kSpan);
    void* pin = nullptr;
    NX_CUDA(cudaHostAlloc(&pin, 2 * kSpan, cudaHostAllocPortable));
    auto* pg = static_cast<std::uint8_t*>(std::aligned_alloc(4096, 2 * kSpan));
    if (!pg) {
      cudaFreeHost(pin);
      throw SimError(Err::IoError, "calibrate_host: out of host memory");
    }
    std::memset(pg, 0x5A, 2 * kSpan);
    std::memset(pin, 0xA5, 2 * kSpan);
    auto* pn = static_cast<std::uint8_t*>(pin);
    std::vector<std::pair<void*, const void*>> pairs;
    for (std::size_t r = 0; r < rounds; ++r)
      for (std::size_t o = 0; o < kSpan; o += kBlockBytes) {
        pairs.emplace_back(pg + o, pn + o);                  // demote: pinned -> paged
        pairs.emplace_back(pn + kSpan + o, pg + kSpan + o);  // promote: paged -> pinned
      }
    HostCalibration c;
    const int before = pool.active();
    for (int t : {1, 2, 4, 6, 8, 12, 16, 24, 32}) {
      if (t > pool.size()) break;
      pool.set_active(t);
      pool.copy_all(std::vector<std::pair<void*, const void*>>(pairs.begin(), pairs.begin() + std::min<std::size_t>(pairs.size(), 64)),
                    kBlockBytes);  // warm the workers
      const auto t0 = Clock::now();
      pool.copy_all(pairs, kBlockBytes);
      const double s = secs_since(t0);
      c.threads.push_back(t);
      c.gbps.push_back(static_cast<double>(pairs.size()) * kBlockBytes / s / 1e9);
    }
    std::free(pg);
    cudaFreeHost(pin);
    if (c.gbps.empty()) {
      pool.set_active(before);
      return c;
    }
    c.peak_gbps = *std::max_element(c.gbps.begin(), c.gbps.end());
    for (std::size_t i = 0; i < c.gbps.size(); ++i)
      if (c.gbps[i] >= 0.98 * c.peak_gbps) {
        c.chosen = c.threads[i];
        break;
      }
    pool.set_active(c.chosen);
    host_cal = c;
    return c;
  }

  // Synchronises only the engine's own streams: a device-wide sync could wait
  // on an application stream parked behind a launch gate.
  void sync_own() {
    for (auto s : st) NX_CUDA(cudaStreamSynchronize(s));
    for (auto s : cks) NX_CUDA(cudaStreamSynchronize(s));
    NX_CUDA(cudaStreamSynchronize(aux));
  }

  ~Impl() override {
    for (auto s : st) cudaStreamSynchronize(s);
    for (auto s : cks) cudaStreamSynchronize(s);
    cudaStreamSynchronize(aux);
    for (cudaEvent_t e : events) cudaEventDestroy(e);
    if (ev0) cudaEventDestroy(ev0);
    cudaFree(ck.ck_ref);
    cudaFree(ck.ck_seen);
    cudaFree(ck.ck_valid);
    cudaFree(ck.status);
    cudaFree(ck.kstart);
    cudaFree(ck.kend);
    cudaFree(d_frames);
    if (h_frames) cudaFreeHost(h_frames);
    if (h_frames_stage) cudaFreeHost(h_frames_stage);
    for (auto& s : scratch) {
      cudaFree(s.part_sums);
      cudaFree(s.part_count);
      cudaFree(s.leg_acc);
    }
    if (bounce) cudaFreeHost(bounce);
    if (d_ktab) cudaFree(d_ktab);
    if (h_ktab) cudaFreeHost(h_ktab);
    cudaFree(tscratch.part_sums);
    cudaFree(tscratch.part_count);
    cudaFree(tscratch.leg_acc);
    for (auto& s : st) cudaStreamDestroy(s);
    cudaStreamDestroy(aux);
    cudaStreamDestroy(cks[0]);
    if (cks[1] != cks[0]) cudaStreamDestroy(cks[1]);
  }

  // ---- per-block tables -------------------------------------------------
  template <typename T>
  void grow_dev(T*& p, std::size_t old_n, std::size_t new_n) {
    T* q = nullptr;
    NX_CUDA(cudaMalloc(&q, sizeof(T) * new_n));
    NX_CUDA(cudaMemset(q, 0, sizeof(T) * new_n));
    if (p) {
      NX_CUDA(cudaMemcpy(q, p, sizeof(T) * old_n, cudaMemcpyDeviceToDevice));
      cudaFree(p);
    }
    p = q;
  }

  void grow_tables(std::size_t need) {
    if (need <= ck_cap) return;
    const std::size_t cap = std::max(need, 2 * ck_cap);
    NX_CUDA(cudaDeviceSynchronize());
    grow_dev(ck.ck_ref, ck_cap, cap);
    grow_dev(ck.ck_seen, ck_cap, cap);
    grow_dev(ck.ck_valid, ck_cap, cap);
    grow_dev(d_frames, ck_cap, cap);
    for (std::uint64_t** h : {&h_frames, &h_frames_stage}) {
      void* q = nullptr;
      NX_CUDA(cudaHostAlloc(&q, sizeof(std::uint64_t) * cap, cudaHostAllocPortable));
      std::memset(q, 0, sizeof(std::uint64_t) * cap);
      if (*h) {
        std::memcpy(q, *h, sizeof(std::uint64_t) * ck_cap);
        cudaFreeHost(*h);
      }
      *h = static_cast<std::uint64_t*>(q);
    }
    ck_cap = cap;
  }

  UnitRing& ring_of(TierId t) {
    switch (t) {
      case TierId::Gpu: return arena.ring;
      case TierId::PinnedHost: return pinned.ring;
      case TierId::PagedHost: return paged.ring;
      default: throw SimError(Err::InvalidState, "the disk tier is not backed by the CUDA swap engine");
    }
  }

  // Pinned slots of one lane's legs are taken contiguously when they can be
  // (UnitRing::acquire_after), so departures and the later fetches of the
  // same blocks copy in long runs even after the ring's free order fragments.
  std::array<std::uint32_t, detail::kLaneCount> pinned_prev;
  std::uint32_t take_unit(TierId t, BlockId b, int lane = -1) {
    if (t == TierId::Gpu && placer) return placer->acquire(b);
    if (t == TierId::PinnedHost && lane >= 0) {
      const std::uint32_t u = pinned.ring.acquire_after(pinned_prev[lane], tier_name(t));
      pinned_prev[lane] = u;
      return u;
    }
    return ring_of(t).acquire(tier_name(t));
  }
  void give_unit(TierId t, BlockId b, std::uint32_t u) {
    if (t == TierId::Gpu && placer) return placer->release(b, u);
    ring_of(t).release(u);
  }

  // Device-visible address of a unit (GPU frame or mapped pinned slot).
  void* dev_addr(TierId t, std::uint32_t u) {
    if (t == TierId::Gpu) return arena.frame(u);
    if (t == TierId::PinnedHost) return pinned.dev(u);
    throw InvariantViolation("PCIe leg touches a non-PCIe tier");
  }
  std::uint8_t* host_addr(TierId t, std::uint32_t u) {
    if (t == TierId::PinnedHost) return pinned.host(u);
    if (t == TierId::PagedHost) return paged.unit(u);
    throw InvariantViolation("host leg touches a non-host tier");
  }

  // ---- registry entry points ---------------------------------------------
  std::vector<ChunkId> allocate(AppId app, Bytes size, TierId tier) {
    if (tier == TierId::Disk) throw SimError(Err::InvalidState, "the disk tier is not backed by the CUDA swap engine");
    const std::size_t first = mem.block_count();
    std::vector<ChunkId> out = mem.allocate(app, size, tier);
    const std::size_t last = mem.block_count();
    grow_tables(last);
    unit.resize(last);
    for (std::size_t b = first; b < last; ++b) {
      unit[b] = take_unit(tier, b);
      h_frames[b] = tier == TierId::Gpu ? reinterpret_cast<std::uint64_t>(arena.frame(unit[b])) : 0;
    }
    if (tier == TierId::PagedHost)  // touch now, not inside a timed switch
      for (std::size_t b = first; b < last; ++b) std::memset(paged.unit(unit[b]), 0, 4096);
    push_frame_table(aux);
    NX_CUDA(cudaStreamSynchronize(aux));
    return out;
  }

  Bytes free_chunk(AppId app, ChunkId c) {
    std::vector<std::pair<BlockId, TierId>> where;
    if (mem.has_chunk(c))
      for (BlockId b : mem.chunk(c).blocks) where.emplace_back(b, mem.block(b).loc.tier);
    const Bytes released = mem.free_chunk(app, c);  // throws before any physical change
    for (auto [b, t] : where) {
      give_unit(t, b, unit[b]);
      h_frames[b] = 0;
    }
    return released;
  }

  void push_frame_table(cudaStream_t s) {
    const std::size_t n = mem.block_count();
    if (n == 0) return;
    NX_CUDA(cudaMemcpyAsync(d_frames, h_frames, sizeof(std::uint64_t) * n, cudaMemcpyHostToDevice, s));
  }

  // ---- K4 pattern fill / compare ----------------------------------------
  std::vector<BlockId> blocks_of(AppId app) {
    std::vector<BlockId> out;
    for (ChunkId c : mem.chunks_of(app))
      for (BlockId b : mem.chunk(c).blocks) {
        if (!mem.block(b).loc.is_resident()) throw SimError(Err::InvalidState, "block in flight");
        out.push_back(b);
      }
    return out;
  }

  void fill_pattern(AppId app, std::uint64_t seed) {
    std::vector<NxLeg> direct;
    std::vector<BlockId> paged_blocks;
    for (BlockId b : blocks_of(app)) {
      const TierId t = mem.block(b).loc.tier;
      if (t == TierId::PagedHost)
        paged_blocks.push_back(b);
      else
        direct.push_back(NxLeg{nullptr, dev_addr(t, unit[b]), static_cast<std::uint32_t>(b), app});
    }
    NX_CUDA(launch_fill(direct.data(), static_cast<int>(direct.size()), seed, ck, aux));
    launches_total += (direct.size() + kMaxLegsPerLaunch - 1) / kMaxLegsPerLaunch;
    for (std::size_t i = 0; i < paged_blocks.size(); i += kBounceUnits) {
      const std::size_t n = std::min<std::size_t>(kBounceUnits, paged_blocks.size() - i);
      std::vector<NxLeg> legs;
      std::vector<std::pair<void*, const void*>> copies;
      for (std::size_t k = 0; k < n; ++k) {
        const BlockId b = paged_blocks[i + k];
        std::uint8_t* slot = bounce + k * kBlockBytes;
        legs.push_back(NxLeg{nullptr, slot, static_cast<std::uint32_t>(b), app});
        copies.emplace_back(paged.unit(unit[b]), slot);
      }
      NX_CUDA(launch_fill(legs.data(), static_cast<int>(n), seed, ck, aux));
      ++launches_total;
      NX_CUDA(cudaStreamSynchronize(aux));
      pool.copy_all(copies, kBlockBytes);
    }
    NX_CUDA(cudaStreamSynchronize(aux));
  }

  // Sums per-leg mismatch counts of one compare launch.
  std::uint64_t compare_into(const std::vector<NxLeg>& legs_, std::uint64_t seed, unsigned long long* d_mis) {
    if (legs_.empty()) return 0;
    NX_CUDA(cudaMemsetAsync(d_mis, 0, sizeof(unsigned long long) * legs_.size(), aux));
    NX_CUDA(launch_compare(legs_.data(), static_cast<int>(legs_.size()), seed, d_mis, aux));
    launches_total += (legs_.size() + kMaxLegsPerLaunch - 1) / kMaxLegsPerLaunch;
    std::vector<unsigned long long> h(legs_.size());
    NX_CUDA(cudaMemcpyAsync(h.data(), d_mis, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, aux));
    NX_CUDA(cudaStreamSynchronize(aux));
    std::uint64_t bad = 0;
    for (auto v : h) bad += v;
    return bad;
  }

  std::uint64_t verify_pattern(AppId app, std::uint64_t seed) {
    std::vector<NxLeg> direct;
    std::vector<BlockId> paged_blocks;
    for (BlockId b : blocks_of(app)) {
      const TierId t = mem.block(b).loc.tier;
      if (t == TierId::PagedHost)
        paged_blocks.push_back(b);
      else
        direct.push_back(NxLeg{dev_addr(t, unit[b]), nullptr, static_cast<std::uint32_t>(b), app});
    }
    unsigned long long* d_mis = nullptr;
    NX_CUDA(cudaMalloc(&d_mis, sizeof(unsigned long long) * std::max<std::size_t>(direct.size(), kBounceUnits)));
    std::uint64_t bad = 0;
    try {
      bad += compare_into(direct, seed, d_mis);
      for (std::size_t i = 0; i < paged_blocks.size(); i += kBounceUnits) {
        const std::size_t n = std::min<std::size_t>(kBounceUnits, paged_blocks.size() - i);
        std::vector<std::pair<void*, const void*>> copies;
        std::vector<NxLeg> batch;
        for (std::size_t k = 0; k < n; ++k) {
          const BlockId b = paged_blocks[i + k];
          copies.emplace_back(bounce + k * kBlockBytes, paged.unit(unit[b]));
          batch.push_back(NxLeg{bounce + k * kBlockBytes, nullptr, static_cast<std::uint32_t>(b), app});
        }
        pool.copy_all(copies, kBlockBytes);
        bad += compare_into(batch, seed, d_mis);
      }
    } catch (...) {
      cudaFree(d_mis);
      throw;
    }
    cudaFree(d_mis);
    return bad;
  }

  // ---- lane sink ----------------------------------------------------------
  void leg_started(int lane, std::size_t mi, TierId from, TierId to, bool) override {
    const BlockId b = lanes->move(mi).block;
    Leg L{mi, b, from, to, unit[b], take_unit(to, b, lane), lane, false, secs_since(t0), 0};
    const auto idx = static_cast<std::uint32_t>(legs.size());
    legs.push_back(L);
    trace[lane].push_back(LegTrace{b, from, to});
    if (lane == kH2D || lane == kD2H) {
      pending[lane].push_back(idx);
    } else {
      host_fifo[lane].push_back(idx);
      stats.host_bytes += kBlockBytes;
      ++stats.host_legs;
      if (from == TierId::PinnedHost && at_grow(slot_inflight, L.src_u)) host_wait.push_back(idx);  // still landing
      else pool.submit(host_addr(to, L.dst_u), host_addr(from, L.src_u), kBlockBytes, idx);
    }
  }

  void plan_finished() override { finished = true; }

  cudaEvent_t take_event() {
    if (events_used == events.size()) {
      cudaEvent_t e;
      NX_CUDA(cudaEventCreate(&e));
      events.push_back(e);
    }
    return events[events_used++];
  }

  bool use_sm_kernel(int n_legs) const {
    switch (cfg.path) {
      case CopyPath::SmKernel: return true;
      case CopyPath::CopyEngine: return false;
      case CopyPath::Auto: {
        const auto k = static_cast<std::size_t>(log2_bucket(n_legs));
        // Uncalibrated: the copy engines, the faster mechanism measured on
        // B200 PCIe Gen5 x16 at every batch size; calibrate()
        // re-measures on the box.
        return auto_sm.empty() ? false : auto_sm[std::min(k, auto_sm.size() - 1)];
      }
    }
    return true;
  }

  // The SM copy path: K1T (TMA bulk copies) when cfg.sm_tma_ctas > 0, else K1.
  cudaError_t sm_copy_launch(const NxLeg* l, int n_d2h, int n_h2d, std::uint32_t flags, const NxScratch& sc, cudaStream_t s) {
    const int tma = cfg.sm_tma_ctas < 0 ? std::max(1, sm_count / 2) : cfg.sm_tma_ctas;
    return tma > 0 ? launch_swap_tma(l, n_d2h, n_h2d, flags, ck, sc, tma, s) : launch_swap(l, n_d2h, n_h2d, flags, ck, sc, max_ctas, s);
  }

  NxLeg kernel_leg(const Leg& L) {
    return NxLeg{dev_addr(L.from, L.src_u), dev_addr(L.to, L.dst_u), static_cast<std::uint32_t>(L.block), 0};
  }

  // Submits `d2h` and `h2d` legs as one batch on stream `s`.
  void submit(int s, const std::vector<std::uint32_t>& d2h, const std::vector<std::uint32_t>& h2d) {
    ++batches_submitted;
    Batch B;
    B.stream = s;
    B.legs = d2h;
    B.legs.insert(B.legs.end(), h2d.begin(), h2d.end());
    B.ev_start = take_event();
    B.ev_end = take_event();
    B.ce = !use_sm_kernel(static_cast<int>(B.legs.size()));
    B.host_submit = secs_since(t0);
    const std::uint32_t flags = cfg.verify ? kNxVerify : 0u;
    NX_CUDA(cudaEventRecord(B.ev_start, st[s]));
    if (!B.ce) {
      std::vector<NxLeg> kl;
      kl.reserve(B.legs.size());
      for (auto i : B.legs) kl.push_back(kernel_leg(legs[i]));
      NX_CUDA(sm_copy_launch(kl.data(), static_cast<int>(d2h.size()), static_cast<int>(h2d.size()), flags, scratch[s], st[s]));
      ++stats.launches[s];
      ++launches_total;
    } else {
      // K2: the copy engines move the bytes on st[s]; the K3 checksum
      // launches run on the side stream cks[s] so the copy stream never
      // waits for them: the departure checksum reads the frames while the
      // DMA reads them, the arrival check runs after the batch landed. The
      // batch ends (and may commit) only when both are done.
      cudaStream_t cs = cks[s];
      std::vector<NxLeg> ckl;
      auto dep_event = [&](std::size_t a, std::size_t z) {
        std::uint32_t last = 0;
        for (std::size_t k = a; k < z; ++k) last = std::max(last, dep_pos[legs[d2h[k]].block]);
        return last < dep_head ? rec_head : rec_all;
      };
      if (grouped && !d2h.empty()) B.dep_done = dep_event(0, d2h.size());
      if (!grouped) {
        NX_CUDA(cudaStreamWaitEvent(cs, B.ev_start, 0));
        for (auto i : d2h) ckl.push_back(NxLeg{dev_addr(legs[i].from, legs[i].src_u), nullptr, static_cast<std::uint32_t>(legs[i].block), 0});
        if (!ckl.empty()) k3_launch(B, ckl, false, cs, flags);
      }  // grouped: the switch-wide record launch already covers these departures
      const bool record_covered = grouped && h2d.empty();  // departures only: ends on the copy stream
      if (record_covered && early_mode) {
        // Early frame release: event groups; every departure commits after
        // this flush pass, its frame tagged with its group's event.
        const std::size_t small = static_cast<std::size_t>(std::max(1, cfg.first_batch_legs));
        std::size_t i = 0;
        while (i < d2h.size()) {
          std::size_t g = d2h_legs_sent < 32 * small ? small : static_cast<std::size_t>(cfg.d2h_commit_legs);
          if (g == 0) g = d2h.size();
          const std::size_t j = std::min(d2h.size(), i + g);
          pace_wait(d2h_legs_sent);
          copy_runs(d2h.data() + i, j - i, s, cudaMemcpyDeviceToHost);
          d2h_legs_sent += j - i;
          cudaEvent_t e = take_event();
          NX_CUDA(cudaEventRecord(e, st[s]));
          seq_events.push_back(e);
          const auto seq = static_cast<std::uint32_t>(seq_events.size());
          for (std::size_t k = i; k < j; ++k) {
            const Leg& L = legs[d2h[k]];
            at_grow(frame_seq, L.src_u) = seq;
            at_grow(frame_dep, L.src_u) = dep_event(k, k + 1);
            at_grow(slot_inflight, L.dst_u) = 1;
            early_done.push_back(d2h[k]);
          }
          i = j;
        }
        B.early = true;
        B.committed = B.legs.size();
      } else if (record_covered && cfg.d2h_commit_legs > 0 && !cfg.early_frame_release) {
        // Commit groups: small ones while the fetches ramp up, then
        // d2h_commit_legs; each behind an event the poll loop checks.
        const std::size_t small = static_cast<std::size_t>(std::max(1, cfg.first_batch_legs));
        std::size_t i = 0;
        while (i < d2h.size()) {
          const std::size_t g = d2h_legs_sent < 32 * small ? small : static_cast<std::size_t>(cfg.d2h_commit_legs);
          const std::size_t j = std::min(d2h.size(), i + g);
          copy_runs(d2h.data() + i, j - i, s, cudaMemcpyDeviceToHost);
          d2h_legs_sent += j - i;
          if (j < d2h.size()) {
            cudaEvent_t e = take_event();
            NX_CUDA(cudaEventRecord(e, st[s]));
            B.subs.push_back({static_cast<std::uint32_t>(j), e, dep_event(0, j)});
          }
          i = j;
        }
      } else {
        copy_runs(d2h.data(), d2h.size(), s, cudaMemcpyDeviceToHost);
        d2h_legs_sent += d2h.size();
      }
      if (early_mode && !h2d.empty()) copy_runs_after_frames(h2d.data(), h2d.size(), s);
      else copy_runs(h2d.data(), h2d.size(), s, cudaMemcpyHostToDevice);
      cudaEvent_t copied = take_event();
      NX_CUDA(cudaEventRecord(copied, st[s]));
      B.ev_copied = copied;
      const bool group_check = grouped && !h2d.empty() && d2h.empty();
      if (group_check) {
        for (auto i : h2d) vgroup.push_back(NxLeg{dev_addr(legs[i].to, legs[i].dst_u), nullptr, static_cast<std::uint32_t>(legs[i].block), 0});
        vgroup_copied = copied;  // the batch commits when its copy lands; a group launch checks it
      } else if (!record_covered) {
        NX_CUDA(cudaStreamWaitEvent(cs, copied, 0));
        ckl.clear();
        for (auto i : h2d) ckl.push_back(NxLeg{dev_addr(legs[i].to, legs[i].dst_u), nullptr, static_cast<std::uint32_t>(legs[i].block), 0});
        if (!ckl.empty()) k3_launch(B, ckl, true, cs, flags);
      }
      ++stats.ce_batches[s];
      B.end_on_side = !group_check && !record_covered;
    }
    NX_CUDA(cudaEventRecord(B.ev_end, B.end_on_side ? cks[s] : st[s]));
    stats.pcie_d2h_bytes += d2h.size() * kBlockBytes;
    for (auto i : h2d) {
      stats.pcie_h2d_bytes += kBlockBytes;
      const Leg& L = legs[i];
      h_frames[L.block] = reinterpret_cast<std::uint64_t>(arena.frame(L.dst_u));
      if (lanes->move(L.mi).dst == TierId::Gpu) ++fetches_submitted;
    }
    inflight[s].push_back(std::move(B));
    // Group arrival checks; in the tail (fewer fetches left than a group) a
    // check covers at least three times the legs that remain to be
    // submitted, so group sizes shrink geometrically towards the end: the
    // last check after the last copy is one small batch and the tail takes
    // ~3 launches (each pays ~30 us of launch cost under PCIe load, §3),
    // not one per batch.
    const std::size_t remaining = fetches_total - fetches_submitted;
    if (!vgroup.empty() && (static_cast<int>(vgroup.size()) >= cfg.k3_verify_group ||
                            (remaining < static_cast<std::size_t>(cfg.k3_verify_group) && vgroup.size() >= 3 * remaining)))
      flush_verify();
    maybe_release_gate();
  }

  // Fetches under early frame release: each leg's frame may still be being
  // vacated; the H2D stream waits for the newest group event (and departure
  // record) its legs need before the copies that need it. Waits are monotone
  // (D2H groups end in stream order), so a batch adds only the waits it
  // needs beyond the ones already queued.
  void copy_runs_after_frames(const std::uint32_t* idx, std::size_t count, int s) {
    std::size_t i = 0;
    while (i < count) {
      std::size_t j = i;
      // extend the segment while no new wait is needed
      while (j < count) {
        const std::uint32_t f = legs[idx[j]].dst_u;
        const std::uint32_t need = f < frame_seq.size() ? frame_seq[f] : 0;
        const cudaEvent_t dep = f < frame_dep.size() ? frame_dep[f] : nullptr;
        const bool dep_needed = dep != nullptr && !h2d_waited_all && !(dep == rec_head && h2d_waited_head);
        if (need > h2d_seq_waited || dep_needed) {
          if (j > i) break;  // copy what needs nothing new first
          if (need > h2d_seq_waited) {
            NX_CUDA(cudaStreamWaitEvent(st[s], seq_events[need - 1], 0));
            h2d_seq_waited = need;
          }
          if (dep_needed) {
            NX_CUDA(cudaStreamWaitEvent(st[s], dep, 0));
            if (dep == rec_all) h2d_waited_all = true;
            h2d_waited_head = true;
          }
        }
        ++j;
      }
      copy_runs(idx + i, j - i, s, cudaMemcpyHostToDevice);
      if (pacing) {
        h2d_marked += j - i;
        cudaEvent_t e = take_event();
        NX_CUDA(cudaEventRecord(e, st[s]));
        h2d_marks.emplace_back(h2d_marked, e);
      }
      i = j;
    }
  }

  // cudaMemcpyAsync over runs of legs whose source and destination are both contiguous.
  void copy_runs(const std::uint32_t* idx, std::size_t count, int s, cudaMemcpyKind kind) {
    std::size_t i = 0;
    while (i < count) {
      const Leg& a = legs[idx[i]];
      auto* src = static_cast<std::uint8_t*>(dev_addr(a.from, a.src_u));
      auto* dst = static_cast<std::uint8_t*>(dev_addr(a.to, a.dst_u));
      std::size_t n = 1;
      while (i + n < count) {
        const Leg& c = legs[idx[i + n]];
        const bool src_ok = dev_addr(c.from, c.src_u) == src + n * kBlockBytes;
        const bool dst_ok = dev_addr(c.to, c.dst_u) == dst + n * kBlockBytes;
        if (!src_ok || !dst_ok) {
          const int d = kind == cudaMemcpyHostToDevice ? 0 : 1;
          stats.run_breaks_src[d] += !src_ok;
          stats.run_breaks_dst[d] += !dst_ok;
          break;
        }
        ++n;
      }
      NX_CUDA(cudaMemcpyAsync(dst, src, n * kBlockBytes, kind, st[s]));
      ++stats.ce_calls;
      ++stats.ce_calls_dir[kind == cudaMemcpyHostToDevice ? 0 : 1];
      i += n;
    }
  }

  // Once every fetch has been submitted, publish the incoming app's frame
  // table and open its launch gate on the H2D stream (device side).
  void maybe_release_gate() {
    if (gate_done || opts == nullptr || fetches_submitted < fetches_total) return;
    gate_done = true;
    flush_verify();
    for (ChunkId c : mem.chunks_of(incoming))
      for (BlockId b : mem.chunk(c).blocks) {
        const Location& loc = mem.block(b).loc;
        if (loc.is_resident() && loc.tier == TierId::Gpu) h_frames[b] = reinterpret_cast<std::uint64_t>(arena.frame(unit[b]));
      }
    const std::size_t n = mem.block_count();
    std::memcpy(h_frames_stage, h_frames, sizeof(std::uint64_t) * n);
    NX_CUDA(cudaMemcpyAsync(d_frames, h_frames_stage, sizeof(std::uint64_t) * n, cudaMemcpyHostToDevice, st[kH2D]));
    if (cfg.verify) {
      // The arrival checks of the CE path run on the K3 stream: the app may
      // start only after they have read the restored frames (its kernels
      // may overwrite them).
      cudaEvent_t checked = take_event();
      NX_CUDA(cudaEventRecord(checked, cks[kH2D]));
      NX_CUDA(cudaStreamWaitEvent(st[kH2D], checked, 0));
    }
    if (opts->gate_event != nullptr) NX_CUDA(cudaEventRecord(opts->gate_event, st[kH2D]));
    if (opts->gate_callback != nullptr) opts->gate_callback(opts->gate_ctx);
  }

  // Submits pending legs; departures committed early (at submission) are
  // committed between passes, which may admit more fetches.
  // Under early frame release a pass submits one departure batch at most, so
  // the fetches its commits admit go out right behind it instead of after
  // every departure batch of the switch has been queued (~0.5 ms of host time).
  void flush() {
    for (;;) {
      const std::size_t before = batches_submitted;
      flush_pass(early_mode ? 1 : std::numeric_limits<int>::max());
      if (!early_done.empty()) {
        std::vector<std::uint32_t> v;
        v.swap(early_done);
        for (auto i : v) complete(i);
        continue;
      }
      if (batches_submitted == before) break;
    }
  }

  void flush_pass(int max_d2h_batches) {
    const int L = cfg.legs_per_launch;
    if (cfg.fused_launch) {
      while (!pending[kD2H].empty() || !pending[kH2D].empty()) {
        if (inflight[kD2H].size() >= 2 && static_cast<int>(pending[kD2H].size() + pending[kH2D].size()) < L) break;
        const int take_h = std::min<int>(static_cast<int>(pending[kH2D].size()), std::max(L / 2, L - static_cast<int>(pending[kD2H].size())));
        const int take_d = std::min<int>(static_cast<int>(pending[kD2H].size()), L - take_h);
        std::vector<std::uint32_t> d(pending[kD2H].begin(), pending[kD2H].begin() + take_d);
        std::vector<std::uint32_t> h(pending[kH2D].begin(), pending[kH2D].begin() + take_h);
        pending[kD2H].erase(pending[kD2H].begin(), pending[kD2H].begin() + take_d);
        pending[kH2D].erase(pending[kH2D].begin(), pending[kH2D].begin() + take_h);
        submit(kD2H, d, h);
      }
      return;
    }
    int d2h_batches = 0;
    for (int lane : {kD2H, kH2D}) {
      auto& p = pending[lane];
      while (!p.empty()) {
        if (lane == kD2H && d2h_batches >= max_d2h_batches) break;
        // Batches ramp up from first_batch_legs so the first fetches can start
        // (into frames the first evictions free) after a short first batch.
        int cap = std::min<int>(L, std::max(1, cfg.first_batch_legs) << std::min(batches_sent[lane], 12));
        // Ramp down at the end of the evictions: the fetches trail the
        // evictions by one batch (they need the frames a landed batch frees),
        // so smaller last eviction batches shorten the fetch-only tail.
        if (lane == kD2H) {
          const int left = static_cast<int>(p.size() + lanes->queued(kD2H));
          cap = std::min(cap, std::max(std::max(1, cfg.first_batch_legs), left / 4));
        }
        if (lane == kD2H && pacing) {
          // Only groups whose pacing mark exists (or needs none).
          std::size_t allow = 0;
          while (allow < static_cast<std::size_t>(cap) && allow < p.size()) {
            const std::size_t x = d2h_legs_sent + allow;
            const std::size_t need = pace_need(x);
            if (need > h2d_marked) break;
            allow += d2h_group_legs(x);
          }
          if (allow == 0) {
            // The fetches in flight or pending will land and leave marks; with
            // none, nothing moves without more departures: go unpaced.
            if (!pending[kH2D].empty() || !inflight[kH2D].empty()) break;
          } else {
            cap = std::min<int>(cap, static_cast<int>(allow));
          }
        }
        // Enough queued on the stream to hide the host: wait for a full batch
        // (paced: the fetch backlog stays within the lag, so a smaller one).
        int hold = cap;
        if (lane == kH2D && pacing)
          hold = std::min(cap, std::max(std::max(1, cfg.d2h_commit_legs), cfg.pace_lag_legs));
        if (inflight[lane].size() >= 2 && static_cast<int>(p.size()) < hold) break;
        const int take = std::min<int>(static_cast<int>(p.size()), cap);
        ++batches_sent[lane];
        std::vector<std::uint32_t> part(p.begin(), p.begin() + take);
        p.erase(p.begin(), p.begin() + take);
        if (lane == kD2H) {
          submit(kD2H, part, {});
          ++d2h_batches;
        } else {
          submit(kH2D, {}, part);
        }
      }
    }
  }

  void complete(std::uint32_t idx) {
    Leg& L = legs[idx];
    L.done = true;
    give_unit(L.from, L.block, L.src_u);
    unit[L.block] = L.dst_u;
    if (L.from == TierId::Gpu) h_frames[L.block] = 0;
    if (records) {
      L.rec = records->size();
      records->push_back(TransferRecord{L.t_start, secs_since(t0), L.block, L.from, L.to, kBlockBytes});
    }
    lanes->finish_hop(L.lane, L.mi, L.to);
  }

  bool poll() {
    bool progress = false;
    for (int s = 0; s < 2; ++s) {
      while (!inflight[s].empty()) {
        Batch& F = inflight[s].front();
        // Commit groups of a departure batch that have landed (and whose
        // departures are recorded): their frames are free for the fetches.
        while (F.sub_next < F.subs.size()) {
          const Batch::SubCommit& g = F.subs[F.sub_next];
          const cudaError_t r = cudaEventQuery(g.dep_done);
          if (r == cudaErrorNotReady) break;
          NX_CUDA(r);
          const cudaError_t c = cudaEventQuery(g.copied);
          if (c == cudaErrorNotReady) break;
          NX_CUDA(c);
          for (; F.committed < g.end; ++F.committed) complete(F.legs[F.committed]);
          ++F.sub_next;
          progress = true;
        }
        if (F.sub_next < F.subs.size()) break;
        if (F.dep_done != nullptr && !F.early) {  // its departures must be recorded before its frames are reused
          const cudaError_t r = cudaEventQuery(F.dep_done);
          if (r == cudaErrorNotReady) break;
          NX_CUDA(r);
        }
        const cudaError_t e = cudaEventQuery(F.ev_end);
        if (e == cudaErrorNotReady) break;
        NX_CUDA(e);
        Batch B = std::move(inflight[s].front());
        inflight[s].pop_front();
        B.host_done = secs_since(t0);
        for (; B.committed < B.legs.size(); ++B.committed) complete(B.legs[B.committed]);
        if (B.early) {  // landed: second hops out of these pinned slots may start
          for (auto i : B.legs) slot_inflight[legs[i].dst_u] = 0;
          for (std::size_t k = 0; k < host_wait.size();) {
            const Leg& L = legs[host_wait[k]];
            if (!slot_inflight[L.src_u]) {
              pool.submit(host_addr(L.to, L.dst_u), host_addr(L.from, L.src_u), kBlockBytes, host_wait[k]);
              host_wait.erase(host_wait.begin() + static_cast<std::ptrdiff_t>(k));
            } else {
              ++k;
            }
          }
        }
        landed.push_back(std::move(B));
        progress = true;
      }
    }
    static thread_local std::vector<std::uint64_t> toks;
    toks.clear();
    if (pool.drain(toks)) {
      for (auto t : toks) legs[t].done = true;  // committed below, in FIFO order
      progress = true;
    }
    for (int lane = 2; lane < detail::kLaneCount; ++lane) {
      auto& q = host_fifo[lane];
      while (!q.empty() && legs[q.front()].done) {
        const std::uint32_t i = q.front();
        q.pop_front();
        complete(i);
      }
    }
    return progress;
  }

  // ---- prefetch (reference plan_prefetch, planner.cpp:218-242,
  // run by an Orchestrator and preempted with cancel_pending,
  // transfer.cpp:89-113): paged -> pinned host legs on the copy pool while
  // the current app computes. The owning thread pumps it; commits happen in
  // the pump, so the registry stays single-writer.
  static constexpr std::uint64_t kPrefetchTag = 1ull << 62;
  struct PfLeg {
    BlockId block;
    std::uint32_t src_u, dst_u;
    bool done;
  };
  std::deque<BlockId> pf_queue;   // not started
  std::deque<PfLeg> pf_inflight;  // started, FIFO
  Bytes pf_committed = 0;
  std::vector<BlockId> pf_log;    // committed prefetch legs not yet taken (take_prefetch_commits)

  void prefetch_begin(const MigrationPlan& plan) {
    if (!pf_queue.empty() || !pf_inflight.empty()) throw SimError(Err::InvalidState, "a prefetch is already running");
    for (const Move& m : plan.moves)
      if (m.kind != MoveKind::PrefetchToPinned || m.src != TierId::PagedHost || m.dst != TierId::PinnedHost)
        throw SimError(Err::InvalidState, "prefetch plans move paged -> pinned only");
    for (const Move& m : plan.moves) pf_queue.push_back(m.block);
    prefetch_pump();
  }

  bool prefetch_pump() {
    static thread_local std::vector<std::uint64_t> toks;
    toks.clear();
    if (pool.drain(toks))
      for (auto t : toks) {
        if (!(t & kPrefetchTag)) throw InvariantViolation("host copy completion outside a switch");
        for (PfLeg& L : pf_inflight)
          if (L.block == (t & ~kPrefetchTag)) L.done = true;
      }
    while (!pf_inflight.empty() && pf_inflight.front().done) {
      const PfLeg L = pf_inflight.front();
      pf_inflight.pop_front();
      mem.commit_move(L.block, TierId::PinnedHost);
      give_unit(TierId::PagedHost, L.block, L.src_u);
      unit[L.block] = L.dst_u;
      pf_committed += kBlockBytes;
      pf_log.push_back(L.block);
    }
    while (!pf_queue.empty() && static_cast<int>(pf_inflight.size()) < cfg.host_legs_in_flight) {
      const BlockId b = pf_queue.front();
      pf_queue.pop_front();
      const Location& loc = mem.block(b).loc;
      if (!loc.is_resident() || loc.tier != TierId::PagedHost) continue;  // moved since planned
      if (mem.tier(TierId::PinnedHost).free_bytes() < kBlockBytes) {  // room went to a switch: stop here
        pf_queue.clear();
        break;
      }
      mem.begin_move(b, TierId::PinnedHost, false);
      const std::uint32_t dst = take_unit(TierId::PinnedHost, b);
      pf_inflight.push_back(PfLeg{b, unit[b], dst, false});
      pool.submit(pinned.host(dst), paged.unit(unit[b]), kBlockBytes, kPrefetchTag | b);
    }
    return !pf_queue.empty() || !pf_inflight.empty();
  }

  // cancel_pending + wait until quiesced: queued legs are dropped (their
  // blocks stay where they are), legs on the copy pool land and commit.
  void prefetch_quiesce() {
    pf_queue.clear();
    while (prefetch_pump()) std::this_thread::yield();
  }

  void prefetch_wait() {  // every queued leg, to the end
    while (prefetch_pump()) std::this_thread::yield();
  }

  ExecResult execute(const MigrationPlan& plan, const PlannerConfig& pcfg, const ExecOptions& o) {
    if (!pf_queue.empty() || !pf_inflight.empty()) prefetch_quiesce();  // plan_switch needs a quiescent registry
    for (const Move& m : plan.moves)
      if (m.src == TierId::Disk || m.dst == TierId::Disk)
        throw SimError(Err::InvalidState, "plan touches the disk tier, which the CUDA swap engine does not back");
    ExecResult res;
    stats = SwitchStats{};
    stats.bytes_in = plan.bytes_in;
    stats.bytes_out = plan.bytes_out;
    for (auto& t : trace) t.clear();
    legs.clear();
    landed.clear();
    detail_pending = false;
    events_used = 0;
    batches_sent = {0, 0};
    d2h_legs_sent = 0;
    std::fill(frame_seq.begin(), frame_seq.end(), 0u);
    std::fill(frame_dep.begin(), frame_dep.end(), nullptr);
    std::fill(slot_inflight.begin(), slot_inflight.end(), std::uint8_t{0});
    seq_events.clear();
    h2d_seq_waited = 0;
    h2d_waited_head = h2d_waited_all = false;
    early_done.clear();
    host_wait.clear();
    k3_slots_used = 0;
    NX_CUDA(cudaMemsetAsync(ck.kstart, 0xFF, sizeof(unsigned long long) * kClockSlots, aux));
    NX_CUDA(cudaMemsetAsync(ck.kend, 0, sizeof(unsigned long long) * kClockSlots, aux));
    NX_CUDA(cudaStreamSynchronize(aux));
    records = &res.events;
    opts = &o;
    incoming = plan.incoming_app;
    gate_done = false;
    fetches_total = 0;
    fetches_submitted = 0;
    for (const Move& m : plan.moves)
      if (m.dst == TierId::Gpu) ++fetches_total;
    grouped = cfg.k3_grouped && cfg.k3_tma && cks[0] == cks[1] && cfg.path != CopyPath::SmKernel;
    // Early frame release needs every departure batch on the copy engines
    // (an SM-kernel batch records and moves in one launch).
    early_mode = cfg.early_frame_release && grouped && !cfg.fused_launch &&
                 (cfg.path == CopyPath::CopyEngine || (cfg.path == CopyPath::Auto && std::none_of(auto_sm.begin(), auto_sm.end(), [](bool b) { return b; })));
    pacing = early_mode && cfg.pace_lag_legs >= 0 && fetches_total > 0;
    h2d_marks.clear();
    h2d_marked = 0;
    d2h_mark_next = 0;
    gk3.clear();
    vgroup.clear();
    ktab_used = 0;
    rec_head = rec_all = nullptr;
    dep_head = 0;
    std::vector<NxLeg> departing;
    if (grouped) {
      for (const Move& m : plan.moves)
        if (m.src == TierId::Gpu)
          departing.push_back(NxLeg{arena.frame(unit[m.block]), nullptr, static_cast<std::uint32_t>(m.block), 0});
      reserve_table(departing.size() + fetches_total);
    }

    detail::LaneSet ls(mem, hw);
    ls.set_limit(kH2D, cfg.pcie_legs_in_flight);
    ls.set_limit(kD2H, cfg.pcie_legs_in_flight);
    ls.set_limit(2, cfg.host_legs_in_flight);
    ls.set_limit(3, cfg.host_legs_in_flight);
    ls.set_fetch_first(cfg.fetch_first_pump);
    lanes = &ls;
    finished = false;

    t0 = Clock::now();
    NX_CUDA(cudaEventRecord(ev0, st[kD2H]));
    if (o.drain != nullptr) {
      cudaEvent_t d = take_event();
      NX_CUDA(cudaEventRecord(d, o.drain));
      NX_CUDA(cudaStreamWaitEvent(st[kD2H], d, 0));
      if (cfg.fused_launch) NX_CUDA(cudaStreamWaitEvent(st[kH2D], d, 0));
    }
    if (!departing.empty()) {
      // Record every departing block's checksum once, after the incumbent's
      // drain (everything queued on the D2H stream so far), concurrently with
      // the DMA reading the same frames; D2H batches end on this stream after
      // it, so no frame is reused before it is recorded.
      cudaEvent_t drained = take_event();
      NX_CUDA(cudaEventRecord(drained, st[kD2H]));
      NX_CUDA(cudaStreamWaitEvent(cks[0], drained, 0));
      // The D2H lane starts its legs in plan order: a small first launch
      // covers the first (ramp) batches so they can end early, one launch
      // the rest of the switch.
      const std::size_t head = std::min<std::size_t>(departing.size(), 4 * static_cast<std::size_t>(cfg.first_batch_legs) +
                                                                           static_cast<std::size_t>(cfg.legs_per_launch));
      k3_table_launch(std::vector<NxLeg>(departing.begin(), departing.begin() + head), false, 1);
      rec_head = gk3.back().z;
      rec_all = rec_head;
      if (head < departing.size()) {
        k3_table_launch(std::vector<NxLeg>(departing.begin() + head, departing.end()), false, 1);
        rec_all = gk3.back().z;
      }
      dep_head = head;
      if (dep_pos.size() < mem.block_count()) dep_pos.resize(mem.block_count());
      for (std::size_t i = 0; i < departing.size(); ++i) dep_pos[departing[i].block] = static_cast<std::uint32_t>(i);
    }
    AppId owner = kNoApp;
    for (const Move& m : plan.moves)
      if (m.kind == MoveKind::EvictFromGpu) {
        owner = mem.block(m.block).app;
        break;
      }
    try {
      ls.begin(plan, pcfg, /*gate_evictions=*/false, owner, this);
      maybe_release_gate();  // no fetches at all: open immediately
      flush();
      auto last = Clock::now();
      while (!finished) {
        if (poll()) {
          flush();
          if (progress) progress();
          last = Clock::now();
        } else {
          if (std::chrono::duration<double>(Clock::now() - last).count() > 120.0)
            throw InvariantViolation("swap engine made no progress for 120 s");
          std::this_thread::yield();
        }
      }
    } catch (...) {
      lanes = nullptr;
      cudaStreamSynchronize(st[0]);
      cudaStreamSynchronize(st[1]);
      cudaStreamSynchronize(cks[0]);
      cudaStreamSynchronize(cks[1]);
      throw;
    }
    // Early-committed departures nothing waited on may still be landing.
    while (!inflight[kD2H].empty() || !inflight[kH2D].empty())
      if (!poll()) std::this_thread::yield();
    if (!host_wait.empty()) throw InvariantViolation("swap engine finished with host legs still waiting");
    lanes = nullptr;
    if (grouped) NX_CUDA(cudaStreamSynchronize(cks[0]));  // the last arrival check (the switch is verified)
    stats.wall_s = secs_since(t0);
    res.completion = stats.wall_s;
    finalize_timing(res);
    check_status();
    return res;
  }

  // Device timing of the last execute. The switch span and the K3 figures
  // are computed before execute() returns. The per-batch detail (the batch
  // timeline, per-stream launch time, K1 figures, device times on the PCIe
  // records) costs one cudaEventElapsedTime per event, ~300 per config-2
  // switch and ~1.4 ms in all. On the copy-engine path with grouped checks it
  // is computed only when asked for (batch_trace(); the events stay valid
  // until the next execute), and the records keep their host times (leg
  // start, commit).
  bool detail_pending = false;
  float since_ev0(cudaEvent_t e) {
    float ms = 0;
    NX_CUDA(cudaEventElapsedTime(&ms, ev0, e));
    return ms;
  }
  void finalize_timing(ExecResult& res) {
    std::vector<std::pair<double, double>> k3_spans;
    k3_trace.clear();
    batch_tr.clear();
    const bool fast = grouped && std::all_of(landed.begin(), landed.end(), [](const Batch& B) {
      return B.ce && !B.end_on_side && B.k3ev.empty();
    });
    if (fast) {
      // Batches of a stream start and end in submission order: the span is
      // the first start and the last end of each stream.
      double first = 1e30, last = 0;
      for (int s = 0; s < 2; ++s) {
        const Batch* a = nullptr;
        const Batch* z = nullptr;
        for (const Batch& B : landed)
          if (B.stream == s) {
            if (!a) a = &B;
            z = &B;
          }
        if (!a) continue;
        first = std::min(first, since_ev0(a->ev_start) * 1e-3);
        last = std::max(last, since_ev0(z->ev_end) * 1e-3);
      }
      stats.device_span_s = landed.empty() ? 0.0 : last - first;
      detail_pending = !landed.empty();
    } else {
      batch_detail(&res);
    }
    for (const GroupK3& g : gk3) {
      const double a0 = since_ev0(g.a) * 1e-3, a1 = since_ev0(g.z) * 1e-3;
      stats.k3_s += a1 - a0;
      k3_spans.emplace_back(a0, a1);
      k3_trace.push_back(K3Launch{a0, a1, g.legs, g.lane});
      stats.k3_bytes += static_cast<Bytes>(g.legs) * kBlockBytes;
      ++stats.k3_launches;
    }
    for (const Batch& B : landed) {  // per-batch K3 launches (ungrouped CE path)
      stats.k3_bytes += B.k3_bytes;
      for (const auto& ke : B.k3ev) {
        const double a0 = since_ev0(ke[0]) * 1e-3, a1 = since_ev0(ke[1]) * 1e-3;
        stats.k3_s += a1 - a0;
        k3_spans.emplace_back(a0, a1);
        k3_trace.push_back(K3Launch{a0, a1, static_cast<int>(B.k3_bytes / kBlockBytes / B.k3ev.size()), B.stream});
        ++stats.k3_launches;
      }
    }
    // K3 launches of the two lanes overlap on the device; their busy time is
    // the union of their intervals (bytes / busy = achieved HBM bandwidth).
    std::sort(k3_spans.begin(), k3_spans.end());
    double busy = 0, lo = -1, hi = -1;
    for (const auto& [a, b] : k3_spans) {
      if (a > hi) {
        busy += hi - lo;
        lo = a;
        hi = b;
      } else {
        hi = std::max(hi, b);
      }
    }
    busy += hi - lo;
    stats.k3_busy_s = k3_spans.empty() ? 0.0 : busy;

    // Kernel-only K3 time from the in-kernel %globaltimer stamps (first CTA
    // start .. last CTA end per launch), free of stream/front-end delays.
    if (k3_slots_used > 0) {
      std::vector<unsigned long long> ks(k3_slots_used), ke(k3_slots_used);
      NX_CUDA(cudaMemcpyAsync(ks.data(), ck.kstart, sizeof(unsigned long long) * k3_slots_used, cudaMemcpyDeviceToHost, aux));
      NX_CUDA(cudaMemcpyAsync(ke.data(), ck.kend, sizeof(unsigned long long) * k3_slots_used, cudaMemcpyDeviceToHost, aux));
      NX_CUDA(cudaStreamSynchronize(aux));
      for (std::uint32_t i = 0; i < k3_slots_used; ++i)
        if (ke[i] > ks[i] && ks[i] != ~0ull) stats.k3_kernel_s += (ke[i] - ks[i]) * 1e-9;
    }
  }

  // Per-batch device timing: the batch timeline, per-stream launch time, K1
  // figures, and (when `res` is given) device times on the PCIe records.
  void batch_detail(ExecResult* res) {
    detail_pending = false;
    batch_tr.clear();
    stats.kernel_s[0] = stats.kernel_s[1] = 0;
    stats.k1_s = 0;
    stats.k1_bytes = 0;
    stats.k1_launches = 0;
    double first = 1e30, last = 0;
    for (const Batch& B : landed) {
      const double s0 = since_ev0(B.ev_start) * 1e-3, s1 = since_ev0(B.ev_end) * 1e-3;
      const double c = B.ev_copied != nullptr ? since_ev0(B.ev_copied) * 1e-3 : s1;
      batch_tr.push_back(BatchTrace{B.stream, static_cast<int>(B.legs.size()), B.ce, s0, c, s1, B.host_submit, B.host_done});
      first = std::min(first, s0);
      last = std::max(last, s1);
      stats.kernel_s[B.stream] += s1 - s0;
      if (!B.ce) {
        stats.k1_s += s1 - s0;
        stats.k1_bytes += B.legs.size() * kBlockBytes;
        ++stats.k1_launches;
      }
      if (res)
        for (auto i : B.legs) {
          TransferRecord& r = res->events[legs[i].rec];
          r.start = s0;
          r.end = s1;
        }
    }
    if (res) stats.device_span_s = landed.empty() ? 0.0 : last - first;
  }

  void check_status() {
    NxDevStatus now{};
    NX_CUDA(cudaMemcpyAsync(&now, ck.status, sizeof(now), cudaMemcpyDeviceToHost, aux));
    NX_CUDA(cudaStreamSynchronize(aux));
    stats.verified = now.verified - status_seen.verified;
    stats.unverified = now.unverified - status_seen.unverified;
    stats.mismatches = now.mismatches - status_seen.mismatches;
    const unsigned first_bad = status_seen.n_bad;
    status_seen = now;
    if (stats.mismatches != 0) {
      std::string which;
      for (unsigned k = first_bad; k < now.n_bad && k < 64; ++k) which += " " + std::to_string(now.bad_blocks[k]);
      throw InvariantViolation("restore checksum mismatch on " + std::to_string(stats.mismatches) + " block(s):" + which);
    }
  }
};

// ---- SwapEngine ---------------------------------------------------------------
SwapEngine::SwapEngine(const EngineConfig& cfg) : impl_(std::make_unique<Impl>(cfg)) {}
SwapEngine::~SwapEngine() = default;
const EngineConfig& SwapEngine::config() const { return impl_->cfg; }
MemState& SwapEngine::mem() { return impl_->mem; }
const MemState& SwapEngine::mem() const { return impl_->mem; }
HardwareConfig SwapEngine::hardware() const { return impl_->hw; }
std::vector<ChunkId> SwapEngine::allocate(AppId app, Bytes size, TierId tier) { return impl_->allocate(app, size, tier); }
Bytes SwapEngine::free_chunk(AppId app, ChunkId chunk) { return impl_->free_chunk(app, chunk); }
void SwapEngine::fill_pattern(AppId app, std::uint64_t seed) { impl_->fill_pattern(app, seed); }
std::uint64_t SwapEngine::verify_pattern(AppId app, std::uint64_t seed) { return impl_->verify_pattern(app, seed); }

ExecResult SwapEngine::execute(const MigrationPlan& plan, const PlannerConfig& cfg, cudaStream_t drain,
                               const GateRelease* release) {
  ExecOptions o;
  o.drain = drain;
  if (release != nullptr) {
    o.gate_event = release->event;
    o.gate_callback = release->callback;
    o.gate_ctx = release->ctx;
  }
  return impl_->execute(plan, cfg, o);
}

ExecResult SwapEngine::switch_to(AppId incoming, const PlannerConfig& cfg, cudaStream_t drain) {
  impl_->prefetch_quiesce();  // plan_switch needs a quiescent registry (planner.cpp:132-133)
  const auto t = Clock::now();
  MigrationPlan plan = plan_switch(incoming, impl_->mem, cfg);
  const double plan_s = secs_since(t);
  ExecResult r = execute(plan, cfg, drain);
  impl_->stats.plan_s = plan_s;
  return r;
}

const SwitchStats& SwapEngine::last_stats() const { return impl_->stats; }
const std::array<std::vector<LegTrace>, 6>& SwapEngine::lane_trace() const { return impl_->trace; }
std::uint64_t SwapEngine::total_launches() const { return impl_->launches_total; }
const std::vector<K3Launch>& SwapEngine::k3_launches() const { return impl_->k3_trace; }
const std::vector<BatchTrace>& SwapEngine::batch_trace() const {
  if (impl_->detail_pending) impl_->batch_detail(nullptr);  // events of the last execute are still valid
  return impl_->batch_tr;
}
Bytes SwapEngine::pinned_overhead() const {
  return static_cast<Bytes>(kBounceUnits) * kBlockBytes + impl_->ktab_cap * sizeof(NxLeg) + 2 * impl_->ck_cap * sizeof(std::uint64_t);
}

void* SwapEngine::frame_of(BlockId b) const {
  const Location& loc = impl_->mem.block(b).loc;
  if (!loc.is_resident() || loc.tier != TierId::Gpu) return nullptr;
  return impl_->arena.frame(impl_->unit[b]);
}
const std::uint64_t* SwapEngine::device_frame_table() const { return impl_->d_frames; }

std::int64_t SwapEngine::frame_index(BlockId b) const {
  const Location& loc = impl_->mem.block(b).loc;
  if (!loc.is_resident() || loc.tier != TierId::Gpu) return -1;
  return impl_->unit[b];
}

std::uint32_t SwapEngine::arena_frames() const { return impl_->arena.ring.units(); }
std::uint32_t SwapEngine::arena_grow_slab() { return impl_->arena.grow_slab(); }
void SwapEngine::arena_drop_slab(std::uint32_t slab) { impl_->arena.drop_slab(slab); }
void SwapEngine::set_frame_placer(FramePlacer* placer) { impl_->placer = placer; }
void SwapEngine::prefetch_begin(const MigrationPlan& plan) { impl_->prefetch_begin(plan); }
bool SwapEngine::prefetch_pump() { return impl_->prefetch_pump(); }
void SwapEngine::prefetch_quiesce() { impl_->prefetch_quiesce(); }
void SwapEngine::prefetch_wait() { impl_->prefetch_wait(); }
bool SwapEngine::prefetch_active() const { return !impl_->pf_queue.empty() || !impl_->pf_inflight.empty(); }
Bytes SwapEngine::prefetched_bytes() const { return impl_->pf_committed; }
std::vector<BlockId> SwapEngine::take_prefetch_commits() {
  std::vector<BlockId> out;
  out.swap(impl_->pf_log);
  return out;
}
void SwapEngine::set_progress_hook(std::function<void()> hook) { impl_->progress = std::move(hook); }

int SwapEngine::arena_export_fd(std::uint32_t slab) const {
  const int fd = impl_->arena.export_fd(slab);
  if (fd < 0) throw SimError(Err::InvalidState, "the arena is not exportable (EngineConfig::exportable_arena)");
  return fd;
}

std::uint64_t SwapEngine::block_checksum(BlockId b) const {
  unsigned long long v = 0;
  NX_CUDA(cudaMemcpyAsync(&v, impl_->ck.ck_ref + b, sizeof(v), cudaMemcpyDeviceToHost, impl_->aux));
  NX_CUDA(cudaStreamSynchronize(impl_->aux));
  return v;
}

cudaStream_t SwapEngine::stream(int lane) const { return impl_->st[lane == 0 ? kH2D : kD2H]; }

void SwapEngine::read_block(BlockId b, void* dst) {
  Impl& m = *impl_;
  const Location& loc = m.mem.block(b).loc;
  if (!loc.is_resident()) throw SimError(Err::InvalidState, "block in flight");
  if (loc.tier == TierId::Gpu)
  {
    NX_CUDA(cudaMemcpyAsync(dst, m.arena.frame(m.unit[b]), kBlockBytes, cudaMemcpyDeviceToHost, m.aux));
    NX_CUDA(cudaStreamSynchronize(m.aux));
  }
  else
    std::memcpy(dst, m.host_addr(loc.tier, m.unit[b]), kBlockBytes);
}

void SwapEngine::poke_block(BlockId b, std::uint64_t offset, std::uint8_t value) {
  Impl& m = *impl_;
  const Location& loc = m.mem.block(b).loc;
  if (!loc.is_resident()) throw SimError(Err::InvalidState, "block in flight");
  if (offset >= kBlockBytes) throw SimError(Err::InvalidState, "offset outside the block");
  if (loc.tier == TierId::Gpu)
  {
    NX_CUDA(cudaMemcpyAsync(m.arena.frame(m.unit[b]) + offset, &value, 1, cudaMemcpyHostToDevice, m.aux));
    NX_CUDA(cudaStreamSynchronize(m.aux));
  }
  else
    m.host_addr(loc.tier, m.unit[b])[offset] = value;
}

void SwapEngine::set_auto_table(const std::vector<bool>& sm_faster) { impl_->auto_sm = sm_faster; }

}  // namespace nixie::b200

// ---- host-link probe ----------------------------------------------------------
namespace nixie::b200 {

namespace {
struct ProbeBufs {
  std::uint8_t* dev[2] = {nullptr, nullptr};
  std::uint8_t* host[2] = {nullptr, nullptr};
  ~ProbeBufs() {
    for (auto* p : dev)
      if (p) cudaFree(p);
    for (auto* p : host)
      if (p) cudaFreeHost(p);
  }
};
}  // namespace

// CE and SM-kernel bandwidth of the host link, each direction alone and both
// at once (the bidirectional figure is the roofline denominator of the swap).
PcieProbe SwapEngine::probe_pcie(Bytes bytes, Bytes chunk) {
  Impl& m = *impl_;
  if (chunk < kBlockBytes || chunk % kBlockBytes) chunk = kBlockBytes;
  bytes = std::max<Bytes>(chunk, bytes - bytes % chunk);
  PcieProbe out;
  out.bytes_per_direction = bytes;
  out.chunk_bytes = chunk;
  out.numa_node = m.numa.node;
  ProbeBufs b;
  for (int i = 0; i < 2; ++i) {
    NX_CUDA(cudaMalloc(&b.dev[i], bytes));
    NX_CUDA(cudaMemset(b.dev[i], i, bytes));
    prefer_numa_node(m.numa.node);
    void* h = nullptr;
    const cudaError_t e = cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
    prefer_numa_node(-1);
    NX_CUDA(e);
    b.host[i] = static_cast<std::uint8_t*>(h);
    std::memset(h, 1 + i, bytes);
  }
  const int legs_per_chunk = static_cast<int>(chunk / kBlockBytes);
  // dir 0 = H2D (host[1] -> dev[1]) on st[0], dir 1 = D2H (dev[0] -> host[0]) on st[1].
  auto issue = [&](int dir, bool sm) {
    cudaStream_t s = m.st[dir];
    for (Bytes off = 0; off < bytes; off += chunk) {
      if (!sm) {
        if (dir == 0)
          NX_CUDA(cudaMemcpyAsync(b.dev[1] + off, b.host[1] + off, chunk, cudaMemcpyHostToDevice, s));
        else
          NX_CUDA(cudaMemcpyAsync(b.host[0] + off, b.dev[0] + off, chunk, cudaMemcpyDeviceToHost, s));
        continue;
      }
      std::vector<NxLeg> legs;
      for (int k = 0; k < legs_per_chunk; ++k) {
        const Bytes o = off + static_cast<Bytes>(k) * kBlockBytes;
        if (legs.size() == static_cast<std::size_t>(kMaxLegsPerLaunch)) {
          NX_CUDA(m.sm_copy_launch(legs.data(), dir == 1 ? static_cast<int>(legs.size()) : 0, dir == 0 ? static_cast<int>(legs.size()) : 0,
                                   kNxNoChecksum, m.scratch[dir], s));
          legs.clear();
        }
        if (dir == 0)
          legs.push_back(NxLeg{b.host[1] + o, b.dev[1] + o, 0, 0});
        else
          legs.push_back(NxLeg{b.dev[0] + o, b.host[0] + o, 0, 0});
      }
      NX_CUDA(m.sm_copy_launch(legs.data(), dir == 1 ? static_cast<int>(legs.size()) : 0, dir == 0 ? static_cast<int>(legs.size()) : 0,
                               kNxNoChecksum, m.scratch[dir], s));
      ++m.launches_total;
    }
  };
  cudaEvent_t ev[4];
  for (auto& e : ev) NX_CUDA(cudaEventCreate(&e));
  auto run = [&](bool sm, bool h2d, bool d2h, double* gbs_h2d, double* gbs_d2h, double* gbs_total) {
    double best_h = 0, best_d = 0, best_t = 0;
    for (int rep = 0; rep < 4; ++rep) {
      m.sync_own();
      if (h2d) NX_CUDA(cudaEventRecord(ev[0], m.st[0]));
      if (d2h) NX_CUDA(cudaEventRecord(ev[2], m.st[1]));
      if (h2d) issue(0, sm);
      if (d2h) issue(1, sm);
      if (h2d) NX_CUDA(cudaEventRecord(ev[1], m.st[0]));
      if (d2h) NX_CUDA(cudaEventRecord(ev[3], m.st[1]));
      m.sync_own();
      float th = 0, td = 0, a = 0, z = 0;
      if (h2d) NX_CUDA(cudaEventElapsedTime(&th, ev[0], ev[1]));
      if (d2h) NX_CUDA(cudaEventElapsedTime(&td, ev[2], ev[3]));
      if (rep == 0) continue;  // warm-up
      double total = 0;
      if (h2d && d2h) {
        // span from the earlier start to the later end
        NX_CUDA(cudaEventElapsedTime(&a, ev[0], ev[2]));
        NX_CUDA(cudaEventElapsedTime(&z, ev[0], ev[3]));
        const double span = std::max<double>(th, z) - std::min<double>(0.0, a);
        total = 2.0 * static_cast<double>(bytes) / (span * 1e-3) / 1e9;
      }
      if (h2d) best_h = std::max(best_h, static_cast<double>(bytes) / (th * 1e-3) / 1e9);
      if (d2h) best_d = std::max(best_d, static_cast<double>(bytes) / (td * 1e-3) / 1e9);
      best_t = std::max(best_t, total);
    }
    if (gbs_h2d) *gbs_h2d = best_h;
    if (gbs_d2h) *gbs_d2h = best_d;
    if (gbs_total) *gbs_total = best_t;
  };
  for (int k = 0; k < 2; ++k) {
    const bool sm = k == 1;
    run(sm, true, false, &out.h2d[k], nullptr, nullptr);
    run(sm, false, true, nullptr, &out.d2h[k], nullptr);
    run(sm, true, true, &out.bidir_h2d[k], &out.bidir_d2h[k], &out.bidir_total[k]);
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return out;
}

std::array<double, 3> SwapEngine::probe_pcie_paced(Bytes bytes, Bytes chunk, int lag) {
  Impl& m = *impl_;
  if (chunk < kBlockBytes || chunk % kBlockBytes) chunk = kBlockBytes;
  bytes = std::max<Bytes>(chunk, bytes - bytes % chunk);
  lag = std::max(1, lag);
  ProbeBufs b;
  for (int i = 0; i < 2; ++i) {
    NX_CUDA(cudaMalloc(&b.dev[i], bytes));
    NX_CUDA(cudaMemset(b.dev[i], i, bytes));
    prefer_numa_node(m.numa.node);
    void* h = nullptr;
    const cudaError_t e = cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
    prefer_numa_node(-1);
    NX_CUDA(e);
    b.host[i] = static_cast<std::uint8_t*>(h);
    std::memset(h, 1 + i, bytes);
  }
  const std::size_t n = bytes / chunk;
  std::vector<cudaEvent_t> landed(n);
  for (auto& e : landed) NX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaEvent_t ev[4];
  for (auto& e : ev) NX_CUDA(cudaEventCreate(&e));
  std::array<double, 3> best{0, 0, 0};
  for (int rep = 0; rep < 4; ++rep) {
    m.sync_own();
    NX_CUDA(cudaEventRecord(ev[0], m.st[0]));
    NX_CUDA(cudaEventRecord(ev[2], m.st[1]));
    for (std::size_t i = 0; i < n; ++i) {
      const Bytes off = i * chunk;
      NX_CUDA(cudaMemcpyAsync(b.dev[1] + off, b.host[1] + off, chunk, cudaMemcpyHostToDevice, m.st[0]));
      NX_CUDA(cudaEventRecord(landed[i], m.st[0]));
      if (i >= static_cast<std::size_t>(lag)) NX_CUDA(cudaStreamWaitEvent(m.st[1], landed[i - lag], 0));
      NX_CUDA(cudaMemcpyAsync(b.host[0] + off, b.dev[0] + off, chunk, cudaMemcpyDeviceToHost, m.st[1]));
    }
    NX_CUDA(cudaEventRecord(ev[1], m.st[0]));
    NX_CUDA(cudaEventRecord(ev[3], m.st[1]));
    m.sync_own();
    if (rep == 0) continue;  // warm-up
    float th = 0, td = 0, a = 0, z = 0;
    NX_CUDA(cudaEventElapsedTime(&th, ev[0], ev[1]));
    NX_CUDA(cudaEventElapsedTime(&td, ev[2], ev[3]));
    NX_CUDA(cudaEventElapsedTime(&a, ev[0], ev[2]));
    NX_CUDA(cudaEventElapsedTime(&z, ev[0], ev[3]));
    const double span = std::max<double>(th, z) - std::min<double>(0.0, a);
    const double total = 2.0 * static_cast<double>(bytes) / (span * 1e-3) / 1e9;
    if (total > best[2]) best = {static_cast<double>(bytes) / (th * 1e-3) / 1e9, static_cast<double>(bytes) / (td * 1e-3) / 1e9, total};
  }
  for (auto& e : landed) cudaEventDestroy(e);
  for (auto& e : ev) cudaEventDestroy(e);
  return best;
}

}  // namespace nixie::b200

namespace nixie::b200 {
cudaError_t launch_raw_copy(int variant, void* dst, const void* src, std::uint64_t bytes, int ctas, cudaStream_t stream);
cudaError_t launch_spin(unsigned ns, cudaStream_t stream);

// Raw copy-variant probe (copy_variants.cu): GB/s of H2D alone, D2H alone,
// and the total while both run, `bytes` per direction in one launch each.
std::array<double, 3> SwapEngine::probe_copy_variant(int variant, Bytes bytes, int ctas) {
  Impl& m = *impl_;
  bytes -= bytes % (1 << 20);
  ProbeBufs b;
  for (int i = 0; i < 2; ++i) {
    NX_CUDA(cudaMalloc(&b.dev[i], bytes));
    NX_CUDA(cudaMemset(b.dev[i], i, bytes));
    void* h = nullptr;
    NX_CUDA(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    b.host[i] = static_cast<std::uint8_t*>(h);
    std::memset(h, 1 + i, bytes);
  }
  cudaEvent_t ev[4];
  for (auto& e : ev) NX_CUDA(cudaEventCreate(&e));
  auto go = [&](bool h2d, bool d2h) {
    double best = 0;
    for (int rep = 0; rep < 4; ++rep) {
      m.sync_own();
      if (h2d) NX_CUDA(cudaEventRecord(ev[0], m.st[0]));
      if (d2h) NX_CUDA(cudaEventRecord(ev[2], m.st[1]));
      // variant >= 10 mixes mechanisms: 10 = CE H2D + SM D2H, 11 = SM H2D + CE D2H
      // (SM = variant 0); anything else uses `variant` for both directions.
      const bool ce_h = variant == 10, ce_d = variant == 11;
      const int v = variant >= 10 ? 0 : variant;
      if (h2d) {
        if (ce_h)
          for (Bytes o = 0; o < bytes; o += 64 << 20)
            NX_CUDA(cudaMemcpyAsync(b.dev[1] + o, b.host[1] + o, std::min<Bytes>(64 << 20, bytes - o), cudaMemcpyHostToDevice, m.st[0]));
        else
          NX_CUDA(launch_raw_copy(v, b.dev[1], b.host[1], bytes, ctas, m.st[0]));
      }
      if (d2h) {
        if (ce_d)
          for (Bytes o = 0; o < bytes; o += 64 << 20)
            NX_CUDA(cudaMemcpyAsync(b.host[0] + o, b.dev[0] + o, std::min<Bytes>(64 << 20, bytes - o), cudaMemcpyDeviceToHost, m.st[1]));
        else
          NX_CUDA(launch_raw_copy(v, b.host[0], b.dev[0], bytes, ctas, m.st[1]));
      }
      if (h2d) NX_CUDA(cudaEventRecord(ev[1], m.st[0]));
      if (d2h) NX_CUDA(cudaEventRecord(ev[3], m.st[1]));
      m.sync_own();
      m.launches_total += (h2d ? 1 : 0) + (d2h ? 1 : 0);
      if (rep == 0) continue;
      float t = 0;
      if (h2d && d2h) {
        float a = 0, z = 0, th = 0;
        NX_CUDA(cudaEventElapsedTime(&th, ev[0], ev[1]));
        NX_CUDA(cudaEventElapsedTime(&a, ev[0], ev[2]));
        NX_CUDA(cudaEventElapsedTime(&z, ev[0], ev[3]));
        t = std::max(th, z) - std::min(0.0f, a);
        best = std::max(best, 2.0 * static_cast<double>(bytes) / (t * 1e-3) / 1e9);
      } else {
        NX_CUDA(cudaEventElapsedTime(&t, h2d ? ev[0] : ev[2], h2d ? ev[1] : ev[3]));
        best = std::max(best, static_cast<double>(bytes) / (t * 1e-3) / 1e9);
      }
    }
    return best;
  };
  std::array<double, 3> out{go(true, false), go(false, true), go(true, true)};
  for (auto& e : ev) cudaEventDestroy(e);
  return out;
}
}  // namespace nixie::b200

namespace nixie::b200 {
// Measured per-batch-size choice between the SM swap kernel and the copy
// engines (both directions running, the swap's operating point).
// K3 launch timing for 1, 2, 4 ... 128 legs over a scratch HBM buffer
// (CUDA events, median of 9): microseconds per launch, [0] TMA, [1] LDG.
std::vector<std::array<double, 2>> SwapEngine::probe_checksum_launch(bool under_pcie_load) {
  Impl& m = *impl_;
  constexpr int kMax = 128;
  std::uint8_t* buf = nullptr;
  NX_CUDA(cudaMalloc(&buf, kMax * kBlockBytes));
  NX_CUDA(cudaMemset(buf, 7, kMax * kBlockBytes));
  // Optional background load: both PCIe directions busy on the copy
  // engines (as during a switch) while the K3 launches are timed.
  constexpr std::size_t kLoad = std::size_t{1} << 30;
  std::uint8_t *hload = nullptr, *dload = nullptr;
  if (under_pcie_load) {
    void* h = nullptr;
    NX_CUDA(cudaHostAlloc(&h, 2 * kLoad, cudaHostAllocPortable));
    hload = static_cast<std::uint8_t*>(h);
    NX_CUDA(cudaMalloc(&dload, 2 * kLoad));
    for (int r = 0; r < 16; ++r) {
      NX_CUDA(cudaMemcpyAsync(dload, hload, kLoad, cudaMemcpyHostToDevice, m.st[0]));
      NX_CUDA(cudaMemcpyAsync(hload + kLoad, dload + kLoad, kLoad, cudaMemcpyDeviceToHost, m.st[1]));
    }
  }
  cudaEvent_t a, z;
  NX_CUDA(cudaEventCreate(&a));
  NX_CUDA(cudaEventCreate(&z));
  std::vector<std::array<double, 2>> out;
  for (int n = 1; n <= kMax; n *= 2) {
    std::vector<NxLeg> legs;
    for (int i = 0; i < n; ++i) legs.push_back(NxLeg{buf + static_cast<std::size_t>(i) * kBlockBytes, nullptr, static_cast<std::uint32_t>(i), 0});
    std::array<double, 2> r{};
    // Under load, column 1 is the TMA launch issued as a CUDA graph (event,
    // kernel, event captured once): is the extra latency the launch's trip
    // through host memory?
    cudaGraphExec_t gexec = nullptr;
    if (under_pcie_load) {
      cudaGraph_t graph = nullptr;
      NX_CUDA(cudaStreamBeginCapture(m.aux, cudaStreamCaptureModeThreadLocal));
      NX_CUDA(cudaEventRecord(a, m.aux));
      NX_CUDA(launch_checksum_tma(legs.data(), n, false, 0, m.ck, m.scratch[2], m.sm_count, m.aux));
      NX_CUDA(cudaEventRecord(z, m.aux));
      NX_CUDA(cudaStreamEndCapture(m.aux, &graph));
      NX_CUDA(cudaGraphInstantiate(&gexec, graph, 0));
      NX_CUDA(cudaGraphUpload(gexec, m.aux));
      cudaGraphDestroy(graph);
    }
    for (int variant = 0; variant < 2; ++variant) {
      std::vector<double> t;
      for (int rep = 0; rep < 10; ++rep) {
        NX_CUDA(launch_spin(200000, m.aux));  // host finishes enqueueing before the GPU reaches `a`
        if (variant == 1 && gexec) {
          NX_CUDA(cudaGraphLaunch(gexec, m.aux));
        } else {
          NX_CUDA(cudaEventRecord(a, m.aux));
          if (variant == 0)
            NX_CUDA(launch_checksum_tma(legs.data(), n, false, 0, m.ck, m.scratch[2], m.sm_count, m.aux));
          else
            NX_CUDA(launch_swap(legs.data(), n, 0, 0, m.ck, m.scratch[2], m.k3_ctas, m.aux));
          NX_CUDA(cudaEventRecord(z, m.aux));
        }
        NX_CUDA(cudaEventSynchronize(z));
        float ms = 0;
        NX_CUDA(cudaEventElapsedTime(&ms, a, z));
        if (rep > 0) t.push_back(ms * 1e3);
        ++m.launches_total;
      }
      std::sort(t.begin(), t.end());
      r[variant] = t[t.size() / 2];
    }
    if (gexec) cudaGraphExecDestroy(gexec);
    out.push_back(r);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(z);
  cudaFree(buf);
  if (under_pcie_load) {
    NX_CUDA(cudaStreamSynchronize(m.st[0]));
    NX_CUDA(cudaStreamSynchronize(m.st[1]));
    cudaFree(dload);
    cudaFreeHost(hload);
  }
  return out;
}

void SwapEngine::set_option(const std::string& name, int value) {
  EngineConfig& c = impl_->cfg;
  if (name == "legs_per_launch" && value >= 1) c.legs_per_launch = value;
  else if (name == "first_batch_legs" && value >= 1) c.first_batch_legs = value;
  else if (name == "d2h_commit_legs" && value >= 0) c.d2h_commit_legs = value;
  else if (name == "early_frame_release" && (value == 0 || value == 1)) c.early_frame_release = value != 0;
  else if (name == "k3_verify_group" && value >= 1) c.k3_verify_group = value;
  else if (name == "pace_lag_legs" && value >= -1) c.pace_lag_legs = value;
  else if (name == "fetch_first_pump" && (value == 0 || value == 1)) c.fetch_first_pump = value != 0;
  else if (name == "sm_tma_ctas" && value >= -1) c.sm_tma_ctas = value;
  else if (name == "path" && value >= 0 && value <= 2) c.path = static_cast<CopyPath>(value);  // read per execute
  else if (name == "host_streaming_copy" && (value == 0 || value == 1)) {
    c.host_streaming_copy = value != 0;
    impl_->pool.set_streaming(value != 0);
  }
  else throw SimError(Err::ValidationError, "set_option: unknown option or bad value: " + name + "=" + std::to_string(value));
}

HostCalibration SwapEngine::calibrate_host(Bytes bytes_per_direction) { return impl_->calibrate_host(bytes_per_direction); }
const HostCalibration& SwapEngine::host_calibration() const { return impl_->host_cal; }
int SwapEngine::host_threads() const { return impl_->pool.active(); }

Calibration SwapEngine::calibrate(Bytes bytes_per_direction) {
  Calibration c;
  std::vector<bool> table;
  for (int k = 0; k < 8; ++k) {
    const Bytes chunk = kBlockBytes << k;
    const PcieProbe p = probe_pcie(std::max<Bytes>(bytes_per_direction, 4 * chunk), chunk);
    c.legs.push_back(1 << k);
    c.ce_gbps.push_back(p.bidir_total[0]);
    c.sm_gbps.push_back(p.bidir_total[1]);
    table.push_back(p.bidir_total[1] > p.bidir_total[0]);
  }
  set_auto_table(table);
  return c;
}
}  // namespace nixie::b200
