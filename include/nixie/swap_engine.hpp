// nixie-b200 — the CUDA swap engine: the reference's modeled "memcpy loop"
// (proj/src/transfer.cpp:173-186, occupancy kBlockBytes/bw) replaced by real
// byte movement on one B200, behind the same registry / planner / lane
// semantics.
//
//   tier 0 Gpu        device arena (cudaMalloc of the capped budget), 2 MiB frames
//   tier 1 PinnedHost staging ring: cudaHostAlloc(mapped|portable) of exactly the
//                     pinned budget, 2 MiB slots recycled FIFO; the budget is the
//                     tier capacity, so MemState's back-pressure enforces it
//   tier 2 PagedHost  pageable host memory, 2 MiB units mapped on first use
//   tier 3 Disk       not backed by this engine (no configuration reaches it)
//
// PCIe lanes (pinned<->GPU) run the sm_100a swap kernel (K1, checksum fused)
// or the copy engines (K2, cudaMemcpyAsync, with the K3 checksum kernel
// around it), many legs in flight per direction, one CUDA stream per
// direction. Host lanes (pinned<->paged) run on a NUMA-local thread pool.
// Every arrival on the GPU is checked against the checksum recorded when the
// block left it; a mismatch fails the switch (InvariantViolation).
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "nixie/mem_model.hpp"
#include "nixie/mlfq.hpp"
#include "nixie/planner.hpp"
#include "nixie/transfer.hpp"

typedef struct CUstream_st* cudaStream_t;
typedef struct CUevent_st* cudaEvent_t;

namespace nixie::b200 {

enum class CopyPath : int { Auto = 0, SmKernel = 1, CopyEngine = 2 };

struct EngineConfig {
  int device = 0;
  Bytes gpu_capacity = 32 * kGiB;     // capped device budget (consumer-GPU emulation)
  Bytes pinned_capacity = 16 * kGiB;  // enforced pinned budget
  Bytes paged_capacity = 96 * kGiB;
  CopyPath path = CopyPath::Auto;
  int pcie_legs_in_flight = 1024;     // per direction (x 2 MiB); 1024 measured ~1% faster than 512 (tools/tune_batches.py)
  int legs_per_launch = 128;          // max legs per K1 launch / CE batch (measured best)
  int host_threads = 0;               // pinned<->paged copy workers; 0 = measured at construction (calibrate_host)
  int host_legs_in_flight = 64;       // per host lane
  int max_ctas = 0;                   // K1 grid cap; 0 = 2 x SM count
  // SM copy path kernel: > 0 runs K1T (TMA bulk copies) on this many CTAs per
  // launch, -1 the same on half the SMs (the two directions' launches stay
  // co-resident, one CTA per SM), 0 K1 (LDG/STG). Config 2 on the SM path,
  // paired A/B (profiles/r02_k1t_ab.txt): K1 60.4 GB/s, K1T on 74 CTAs 78.9.
  int sm_tma_ctas = -1;
  bool fused_launch = false;          // both directions in one launch stream (warp-group split)
  bool verify = true;                 // checksum every restore
  bool numa_bind = true;              // pinned ring + workers on the GPU's NUMA node
  int first_batch_legs = 8;           // batch-size ramp start (doubles per batch up to legs_per_launch); 2 vs 8 within 1% either way
  bool k3_tma = true;                 // CE-path checksum pass on the TMA pipeline (else the LDG loop)
  bool k3_one_stream = true;          // both lanes' K3 launches on one stream (no SM contention between them)
  bool k3_grouped = true;             // CE path: one record launch per switch, arrival checks per group
  int k3_verify_group = 4096;         // legs per grouped arrival check (the last group is flushed at the end)
  // CE path, grouped K3: departure batches are cut into groups of this many
  // legs (first_batch_legs-sized groups for the first 32 x first_batch_legs
  // legs of a switch), each ending at its own event (0: whole batches).
  //  * early_frame_release (default): a departure commits when its copy is
  //    queued; a fetch landing in the frame it vacated waits on the device
  //    for that group's event (and the departure record), so the fetch stream
  //    trails the evictions by one group without a host round trip, in
  //    batches as large as the lanes allow. A second hop out of the pinned
  //    slot (pinned -> paged) waits for the landing on the host.
  //  * otherwise each group commits when the host sees its event (measured
  //    on config 2: fetches then run as many small batches, 1.3% slower than
  //    whole-batch commits).
  int d2h_commit_legs = 32;
  bool early_frame_release = true;
  // Early frame release only: a departure group may start once the fetches
  // of the switch have landed up to (its first leg - pace_lag_legs), while
  // fetches remain (-1: no pacing). With both PCIe directions saturated the
  // upstream link carries the D2H data AND the fetches' read requests, so an
  // unpaced D2H runs ahead, H2D slows down and finishes alone; holding D2H a
  // few groups behind the fetches moves more bytes per second in total
  // (tools/pcie_pace.cu: 4+4 GiB in 64 MiB calls, 89 GB/s free vs 97 paced).
  // Config 2, paired A/B (profiles/r02_ab_pace*.txt): lag 64 legs 3.1% faster
  // per switch than none; 48-96 within 0.5%; 0 serialises the two directions
  // (the fetches need the frames the departures vacate) and 128 gains nothing.
  int pace_lag_legs = 64;
  bool fetch_first_pump = true;
  // Host copy pool (pinned <-> paged legs): AVX2 streaming stores. A plain
  // memcpy of a 2 MiB leg reads the destination before writing it; with the
  // two-hop switch host-DRAM-bound that third transfer per byte costs 15-17%
  // of a config-4 switch at 2-4 GiB budgets (profiles/r02_ab_streaming_copy_c4.txt).
  bool host_streaming_copy = true;  // lanes toward the GPU pumped first after a commit (LaneSet::set_fetch_first)
  bool exportable_arena = false;      // GPU tier = exportable VMM slabs shims can import (interposer daemon)
  Bytes arena_slab_bytes = 128 * kMiB; // exportable arena: bytes per physical allocation (a multiple of 2 MiB)
  Bytes gpu_physical = 0;             // arena bytes (0 = gpu_capacity); the registry still enforces gpu_capacity
  Bytes gpu_physical_max = 0;         // exportable arena: virtual space reserved for growth (0 = gpu_physical)
};

// Physical placement of blocks arriving on the GPU tier. Default (no placer):
// any free 2 MiB frame of the arena, FIFO. The interposer daemon installs one
// that keeps each application's 128 MiB virtual slabs backed by whole
// physical slabs (csrc/daemon/daemon.cpp), so a restore maps one slab per
// 64 blocks into the application instead of one frame per block.
class FramePlacer {
 public:
  virtual ~FramePlacer() = default;
  virtual std::uint32_t acquire(BlockId block) = 0;                // frame for a block about to land on the GPU
  virtual void release(BlockId block, std::uint32_t frame) = 0;    // the block left the GPU (or was freed)
};

struct SwitchStats {
  Bytes bytes_in = 0, bytes_out = 0;        // plan totals
  Bytes pcie_h2d_bytes = 0, pcie_d2h_bytes = 0, host_bytes = 0;
  double wall_s = 0;                        // host wall time of execute()
  double plan_s = 0;                        // plan_switch time when run via switch_to()
  double device_span_s = 0;                 // first PCIe launch start -> last end (CUDA events)
  double kernel_s[2] = {0, 0};              // summed launch durations: [0] H2D stream, [1] D2H stream
  int launches[2] = {0, 0};                 // K1/K3 kernel launches per stream
  int ce_batches[2] = {0, 0};               // copy-engine batches per stream
  int host_legs = 0;
  int ce_calls = 0;                         // cudaMemcpyAsync calls (contiguous runs) of the CE batches
  int pace_waits = 0;                       // D2H groups held behind landed fetches (pace_lag_legs)
  // CE runs per direction ([0] H2D, [1] D2H) and why each run ended early:
  // source not contiguous, destination not contiguous (the rest end at a
  // group or batch boundary).
  int ce_calls_dir[2] = {0, 0}, run_breaks_src[2] = {0, 0}, run_breaks_dst[2] = {0, 0};
  std::uint64_t verified = 0, unverified = 0, mismatches = 0;
  // Per kernel kind (CUDA events on the launching stream):
  double k1_s = 0;      // K1 swap launches (SM path): summed durations
  Bytes k1_bytes = 0;   // bytes they moved across PCIe
  int k1_launches = 0;
  double k3_s = 0;      // K3 checksum launches (CE path): summed durations
  double k3_busy_s = 0; // union of K3 launch intervals (both lanes' launches overlap)
  double k3_kernel_s = 0;  // summed in-kernel spans (%globaltimer, first CTA start .. last CTA end)
  Bytes k3_bytes = 0;   // HBM bytes they read
  int k3_launches = 0;
};

// Launch-gate hook of execute(): once the incoming app's last fetch has been
// submitted (and its frame table published), `event` is recorded on the H2D
// stream and `callback(ctx)` runs on the calling thread. A waiter that
// enqueues cudaStreamWaitEvent(app_stream, event) after the callback gets a
// device-side dependency whose producer is already enqueued.
struct GateRelease {
  cudaEvent_t event = nullptr;
  void (*callback)(void* ctx) = nullptr;
  void* ctx = nullptr;
};

// One K3 checksum launch of the last execute (device times from its start).
struct K3Launch {
  double start_s, end_s;
  int legs;
  int lane;  // 0 = arrivals (verify), 1 = departures (record)
};

// One PCIe batch of the last execute: device times (s, from the switch start)
// of its start, of the end of its copies, and of its end (checks included);
// host times (s, from the execute() call) of its submission and of the poll
// that saw it end. The per-switch timeline (tools/timeline.py).
struct BatchTrace {
  int stream;  // 0 = H2D, 1 = D2H
  int legs;
  bool ce;
  double start_s, copied_s, end_s;
  double host_submit_s, host_done_s;
};

struct LegTrace {
  BlockId block;
  TierId src, dst;
};

struct PcieProbe {
  // GB/s (1e9 B/s). [0] CE (cudaMemcpyAsync), [1] SM kernel.
  double h2d[2] = {0, 0};
  double d2h[2] = {0, 0};
  double bidir_h2d[2] = {0, 0};  // H2D rate while D2H runs concurrently
  double bidir_d2h[2] = {0, 0};
  double bidir_total[2] = {0, 0};
  Bytes bytes_per_direction = 0;
  Bytes chunk_bytes = 0;
  int link_gen = 0, link_width = 0, link_gen_max = 0, link_width_max = 0;
  int numa_node = -1;
};

// Host copy pool sizing (the pinned<->paged lanes of the two-hop path): GB/s
// of both directions at once per worker count; `chosen` is installed.
struct HostCalibration {
  std::vector<int> threads;
  std::vector<double> gbps;
  int chosen = 0;
  double peak_gbps = 0;  // best measured: the two-hop path's host-memcpy roofline
};

// Per-batch-size SM-kernel vs copy-engine measurement (bidirectional GB/s).
struct Calibration {
  std::vector<int> legs;
  std::vector<double> sm_gbps, ce_gbps;
};

class SwapEngine {
 public:
  explicit SwapEngine(const EngineConfig& cfg);
  ~SwapEngine();
  SwapEngine(const SwapEngine&) = delete;
  SwapEngine& operator=(const SwapEngine&) = delete;

  const EngineConfig& config() const;
  MemState& mem();
  const MemState& mem() const;
  HardwareConfig hardware() const;  // capacities = budgets; link numbers from the last probe

  // Registry entry points (interposer stand-ins) with physical placement.
  std::vector<ChunkId> allocate(AppId app, Bytes size, TierId tier);
  Bytes free_chunk(AppId app, ChunkId chunk);

  // K4: synthetic working set. fill writes every block of `app` wherever it
  // lives and records its checksum; verify returns the number of 16-byte
  // vectors that differ from the pattern (0 = byte-exact).
  void fill_pattern(AppId app, std::uint64_t seed);
  std::uint64_t verify_pattern(AppId app, std::uint64_t seed);

  // Executes a plan with real copies (same contract as nixie::execute).
  // `drain`: the incumbent's stream; evictions start only after its queued
  // kernels finish (device-side eviction gate).
  ExecResult execute(const MigrationPlan& plan, const PlannerConfig& cfg, cudaStream_t drain = nullptr,
                     const GateRelease* release = nullptr);
  // plan_switch + execute.
  ExecResult switch_to(AppId incoming, const PlannerConfig& cfg, cudaStream_t drain = nullptr);

  // Prefetch: runs a plan_prefetch() plan (paged -> pinned)
  // on the host copy pool in the background. The caller's thread owns the
  // registry: prefetch_pump() commits finished legs and starts queued ones
  // (call it periodically; true while active). prefetch_quiesce() is the
  // reference's cancel_pending + wait-until-quiesced (transfer.cpp:89-113):
  // queued legs are dropped, legs on the pool land. execute() quiesces first.
  void prefetch_begin(const MigrationPlan& plan);
  bool prefetch_pump();
  void prefetch_quiesce();
  void prefetch_wait();  // runs every queued leg to completion
  bool prefetch_active() const;
  Bytes prefetched_bytes() const;  // committed since construction
  // Blocks whose prefetch leg committed (paged -> pinned), in commit order,
  // since the last call (the daemon's --trace replays them on the reference).
  std::vector<BlockId> take_prefetch_commits();

  const SwitchStats& last_stats() const;
  const std::array<std::vector<LegTrace>, 6>& lane_trace() const;  // per lane, start order, last execute
  std::uint64_t total_launches() const;  // kernels this engine has launched (all kinds)
  const std::vector<K3Launch>& k3_launches() const;  // last execute
  const std::vector<BatchTrace>& batch_trace() const;  // last execute
  // Pinned bytes held outside the budgeted staging ring (bounce buffer, leg
  // and frame table stages).
  Bytes pinned_overhead() const;

  // Device pointer of the frame holding a GPU-resident block; device table
  // of frame pointers indexed by BlockId (0 when not on the GPU), refreshed
  // on the H2D stream at the end of every execute.
  void* frame_of(BlockId block) const;
  const std::uint64_t* device_frame_table() const;
  // Frame number (offset / 2 MiB into the arena) of a GPU-resident block, or
  // -1. With EngineConfig::exportable_arena the arena is a row of physical
  // slabs of arena_slab_bytes; arena_export_fd(s) returns a new POSIX
  // descriptor of slab s (caller closes it): a shim imports it and maps it at
  // its own address (frames s * slab_frames ... belong to slab s).
  std::int64_t frame_index(BlockId block) const;
  int arena_export_fd(std::uint32_t slab) const;
  std::uint32_t arena_frames() const;  // physical 2 MiB frames in the arena
  // Exportable arena: one more physical slab (up to gpu_physical_max); returns its index.
  std::uint32_t arena_grow_slab();
  // Exportable arena: unmaps and releases a slab no block uses (its slot is
  // refilled by the next grow).
  void arena_drop_slab(std::uint32_t slab);
  // Not owned; nullptr restores the default. Install before any GPU allocation.
  void set_frame_placer(FramePlacer* placer);
  // Called on the thread running execute() whenever legs have committed (the
  // interposer daemon maps the incoming app's slabs while copies continue).
  // It must not call back into the engine.
  void set_progress_hook(std::function<void()> hook);
  std::uint64_t block_checksum(BlockId block) const;  // last recorded departure checksum
  // Test access to a resident block's bytes wherever it lives.
  void read_block(BlockId block, void* host_dst);
  void poke_block(BlockId block, std::uint64_t offset, std::uint8_t value);

  cudaStream_t stream(int lane) const;  // 0 = H2D lane stream, 1 = D2H lane stream

  // Measures the host link: CE and SM, H2D / D2H alone and both at once.
  PcieProbe probe_pcie(Bytes bytes_per_direction, Bytes chunk_bytes);
  // Both directions at once on the copy engines, D2H chunk i held (on the
  // device) until H2D chunk i - lag_chunks has landed: the paced shape the
  // engine uses (EngineConfig::pace_lag_legs). {H2D, D2H, both} GB/s, best of 3.
  std::array<double, 3> probe_pcie_paced(Bytes bytes_per_direction, Bytes chunk_bytes, int lag_chunks);
  // Raw SM copy variants (csrc/cuda/copy_variants.cu): {H2D, D2H, both} GB/s.
  std::array<double, 3> probe_copy_variant(int variant, Bytes bytes_per_direction, int ctas);
  // Per-batch-size choice for CopyPath::Auto: index k covers launches of
  // 2^k legs; true = SM kernel, false = copy engines.
  void set_auto_table(const std::vector<bool>& sm_faster);
  // Per-switch tunables, changeable between executes (paired A/B runs on
  // one engine, tools/ab_switch.py): legs_per_launch, first_batch_legs,
  // d2h_commit_legs, early_frame_release, k3_verify_group. Throws
  // ValidationError for other names or bad values.
  void set_option(const std::string& name, int value);
  // Measures both mechanisms at 1..128 legs per batch and installs the
  // faster one per size for CopyPath::Auto.
  Calibration calibrate(Bytes bytes_per_direction);
  // Measures the host copy pool (pinned -> paged and paged -> pinned at once,
  // 2 MiB jobs) at 1, 2, 4 ... workers and keeps the fastest count (the
  // smallest within 2% of the best). EngineConfig::host_threads = 0 runs it
  // at construction with a small sample.
  HostCalibration calibrate_host(Bytes bytes_per_direction);
  const HostCalibration& host_calibration() const;  // last measurement (empty if host_threads was fixed)
  int host_threads() const;                         // workers taking jobs now
  // K3 launch duration (us) for 1, 2, 4 ... 128 legs: [0] TMA pipeline, [1] LDG loop.
  // under_pcie_load: while both PCIe directions carry copy-engine traffic.
  std::vector<std::array<double, 2>> probe_checksum_launch(bool under_pcie_load = false);

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

// Kernel-launch gate (§3 steps 1-2 and 6, §4): an app's kernels run
// only while it holds the grant and its working set is GPU-resident.
// Thread-safe: application threads call before_launch while a scheduler
// thread runs context_switch.
//   * before_launch(app, now): a granted, resident app passes (true).
//     Otherwise the app's request is enqueued with the scheduler and the
//     calling thread is held until a switch to the app has submitted its last
//     fetch; the app's stream then waits on the device for that fetch to land
//     and before_launch returns false: the caller's next launch on its
//     stream is ordered after the swap-in.
//   * context_switch(to, now): pauses the incumbent (its later launches are
//     held; its queued kernels drain before any eviction starts, on the
//     device), plans with the scheduler's victim hint, executes with real
//     copies and grants `to`.
class LaunchGate {
 public:
  LaunchGate(SwapEngine& engine, MlfqScheduler& sched, PlannerConfig cfg);
  ~LaunchGate();

  void attach(AppId app, cudaStream_t stream);
  // Returns holding the app's launch lock; call after_launch(app) once the
  // kernel is enqueued (a pause waits for it).
  bool before_launch(AppId app, Seconds now, double timeout_s = 120.0);
  void after_launch(AppId app);
  // Blocking-call brackets and other API activity (idleness, §6.1).
  void api_event(AppId app, Seconds now, ApiEventKind kind);
  ExecResult context_switch(AppId to, Seconds now);
  // One scheduler tick: infer_all, then switch to select_next() if the GPU
  // has no holder, the holder is idle, or should_preempt fires.
  std::optional<AppId> tick(Seconds now);
  std::optional<AppId> select_next(Seconds now);
  std::optional<AppId> granted();
  std::uint64_t switches() const;
  // MLFQ prefetch: when on, every tick that does not switch
  // pumps the engine's prefetch and, when none runs, starts plan_prefetch()
  // for next_prefetch_candidate() (if it is not the holder). A switch
  // quiesces it first.
  void set_prefetch(bool on);
  Bytes prefetched_bytes() const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

}  // namespace nixie::b200
