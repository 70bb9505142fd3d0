/*
 * nixie-b200 C ABI — the drop-in boundary of the B200 swap path.
 *
 * The reference (arxiv 2601.11743 "Nixie", /root/reference/proj) exposes a
 * C++20 API in namespace nixie (proj/include/nixie/ headers) and no FFI. This
 * header is the thin C layer beneath the same C++ API in this repo
 * (include/nixie/ headers): plain pointers and sizes, status codes instead of
 * exceptions, opaque handles. Each entry point names the reference interface
 * it replaces or the paper mechanism it implements.
 *
 * Status codes: NX_OK, or 1 + nixie::Err (errors.hpp:8-21) for a SimError,
 * NX_E_INVARIANT for an InvariantViolation (a bug: overcommit, deadlock, a
 * restore whose checksum differs), NX_E_CUDA for a CUDA failure,
 * NX_E_ARG for a bad argument. nx_last_error() returns the message of the
 * calling thread's last failure.
 */
#ifndef NIXIE_B200_H_
#define NIXIE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NX_OK 0
#define NX_E_INVARIANT 100
#define NX_E_CUDA 200
#define NX_E_ARG 300

/* Tier ids: reference TierId (proj/include/nixie/mem_model.hpp:14). */
#define NX_TIER_GPU 0
#define NX_TIER_PINNED 1
#define NX_TIER_PAGED 2
#define NX_TIER_DISK 3

/* Copy paths for the PCIe lanes. */
#define NX_PATH_AUTO 0   /* per-batch-size choice from nx_set_auto_table */
#define NX_PATH_SM 1     /* K1: sm_100a swap kernel, checksum fused */
#define NX_PATH_CE 2     /* K2: cudaMemcpyAsync copy engines + K3 checksum kernel */

typedef struct nx_engine nx_engine;
typedef struct nx_gate nx_gate;

/* Engine configuration. Replaces HardwareConfig's tier capacities
 * (proj/include/nixie/transfer.hpp:24-37): the GPU capacity becomes the
 * capped device arena, the pinned capacity the enforced pinned budget. */
typedef struct nx_engine_config {
  int device;
  uint64_t gpu_capacity;
  uint64_t pinned_capacity;
  uint64_t paged_capacity;
  int path;
  int pcie_legs_in_flight;
  int legs_per_launch;
  int host_threads;
  int host_legs_in_flight;
  int max_ctas;
  int fused_launch;
  int verify;
  int numa_bind;
  int first_batch_legs;
  int k3_tma;
  int k3_one_stream; /* both lanes' K3 launches on one stream */
  int k3_grouped;    /* CE path: one switch-wide record launch, grouped arrival checks */
  int k3_verify_group; /* legs per grouped arrival check */
  int d2h_commit_legs; /* CE departures are cut into event groups of this many legs (0: whole batches) */
  int early_frame_release; /* departures commit when queued; fetches wait on the device for their frames */
  int pace_lag_legs; /* departure groups wait for fetches landed up to (first leg - lag); -1: off */
  int fetch_first_pump; /* after a commit, lanes toward the GPU are pumped first (concurrent lanes) */
  int host_streaming_copy; /* host copy pool copies with AVX2 streaming stores */
} nx_engine_config;

/* PlannerConfig (proj/include/nixie/planner.hpp:39-43). victim_order may be
 * NULL (n_victims = 0). */
typedef struct nx_planner_config {
  uint64_t streaming_window;
  uint64_t pinned_budget; /* UINT64_MAX = unbounded */
  const uint32_t* victim_order;
  size_t n_victims;
} nx_planner_config;

typedef struct nx_switch_stats {
  uint64_t bytes_in, bytes_out;
  uint64_t pcie_h2d_bytes, pcie_d2h_bytes, host_bytes;
  double wall_s, plan_s, device_span_s;
  double kernel_s_h2d, kernel_s_d2h;
  int launches_h2d, launches_d2h, ce_batches_h2d, ce_batches_d2h, host_legs;
  uint64_t verified, unverified, mismatches;
  /* aggregate_throughput (proj/src/transfer.cpp:7-28) over the switch's
   * GPU<->pinned records, device-timed, in bytes/s */
  double tp_to_gpu, tp_from_gpu, tp_bidir;
  /* per kernel kind: K1 swap (SM path) and K3 checksum (CE path) */
  double k1_s, k3_s;
  uint64_t k1_bytes, k3_bytes;
  int k1_launches, k3_launches;
  double k3_busy_s;   /* union of the K3 launch intervals (CUDA events) */
  double k3_kernel_s; /* summed in-kernel K3 spans (%globaltimer) */
  int ce_calls;       /* cudaMemcpyAsync calls of the CE batches */
  int pace_waits;     /* departure groups held behind landed fetches (pace_lag_legs) */
  int ce_calls_dir[2]; /* CE calls per direction: [0] H2D, [1] D2H */
  int run_breaks_src[2], run_breaks_dst[2]; /* runs ended by a non-contiguous source / destination */
} nx_switch_stats;

typedef struct nx_pcie_probe {
  double h2d[2], d2h[2], bidir_h2d[2], bidir_d2h[2], bidir_total[2]; /* GB/s; [0] CE, [1] SM */
  uint64_t bytes_per_direction, chunk_bytes;
  int numa_node;
} nx_pcie_probe;

typedef struct nx_mlfq_config {
  int levels;
  double base_allotment, base_preemption, idle_threshold, tick;
} nx_mlfq_config;

/* ---- errors / library ---------------------------------------------------- */
const char* nx_last_error(void);
const char* nx_version(void);
int nx_cuda_device_count(int* count);

/* ---- engine lifecycle ---------------------------------------------------- */
void nx_engine_config_default(nx_engine_config* cfg);
void nx_planner_config_default(nx_planner_config* cfg);
/* Creates one per-GPU Nixie instance: device arena, pinned staging ring,
 * paged store, host copy pool, streams. */
int nx_engine_create(const nx_engine_config* cfg, nx_engine** out);
void nx_engine_destroy(nx_engine* e);

/* ---- registry (interposer stand-ins) ------------------------------------ */
/* MemState::allocate (proj/src/mem_model.cpp:48-86) plus physical
 * placement; writes up to cap chunk ids, *n = number created. */
int nx_alloc(nx_engine* e, uint32_t app, uint64_t size, int tier, uint64_t* chunks, size_t cap, size_t* n);
/* MemState::free_chunk (proj/src/mem_model.cpp:88-116). */
int nx_free_chunk(nx_engine* e, uint32_t app, uint64_t chunk, uint64_t* released);
/* MemState::audit (proj/src/mem_model.cpp:274-325). */
int nx_audit(nx_engine* e);
/* MemState::app_bytes_resident for the four tiers. */
int nx_app_resident(nx_engine* e, uint32_t app, uint64_t out[4]);
/* MemState::pinned_physical / pinned_physical_peak (mem_model.cpp:244-247, 270-272). */
int nx_pinned_physical(nx_engine* e, uint64_t* now, uint64_t* peak);
/* Pinned host memory the engine holds OUTSIDE the budgeted staging ring:
 * the 128 MiB bounce buffer for pageable fills/compares (never on the swap
 * path) and the pinned stages of the K3 leg table and the frame table. */
int nx_pinned_overhead(nx_engine* e, uint64_t* bytes);

/* ---- K4 synthetic working set ------------------------------------------- */
int nx_fill_pattern(nx_engine* e, uint32_t app, uint64_t seed);
/* Number of 16-byte vectors of app that differ from the pattern (0 = exact). */
int nx_verify_pattern(nx_engine* e, uint32_t app, uint64_t seed, uint64_t* bad_vectors);
/* Device pointer of a GPU-resident block's frame (NULL otherwise). */
int nx_block_frame(nx_engine* e, uint64_t block, void** frame);
int nx_block_checksum(nx_engine* e, uint64_t block, uint64_t* checksum);
int nx_app_blocks(nx_engine* e, uint32_t app, uint64_t* blocks, size_t cap, size_t* n);
/* Copies the 2 MiB of a resident block, wherever it lives, into host memory. */
int nx_block_read(nx_engine* e, uint64_t block, void* host_dst);
/* Overwrites one byte of a resident block in place (fault injection for the
 * restore-verification tests). */
int nx_block_poke(nx_engine* e, uint64_t block, uint64_t offset, uint8_t value);

/* ---- swap-engine interface ----------------------------------------------- */
/* plan_switch (proj/src/planner.cpp:111-216): the plan's dump()
 * (`block src dst distance kind` lines) is written to dump (NUL-terminated,
 * truncated to cap); *len = full length. */
int nx_plan(nx_engine* e, uint32_t incoming, const nx_planner_config* cfg, char* dump, size_t cap, size_t* len,
            uint64_t* bytes_in, uint64_t* bytes_out);
/* plan_switch + execute (proj/src/transfer.cpp:250-271) with real copies:
 * the modeled leg occupancy (transfer.cpp:173-186) becomes K1/K2 launches
 * and host memcpy legs. drain_stream (cudaStream_t, may be NULL) is the
 * incumbent's stream; evictions wait for its queued kernels on the device. */
int nx_switch(nx_engine* e, uint32_t incoming, const nx_planner_config* cfg, void* drain_stream, nx_switch_stats* out);
/* Prefetch: plan_prefetch(app) (planner.cpp:218-242) started
 * in the background on the host copy pool (*moves = its size, 0 = nothing to
 * do); pump commits finished legs and starts queued ones (*active = 0 when
 * done); quiesce = Orchestrator::cancel_pending + wait until quiesced
 * (transfer.cpp:89-113). nx_switch quiesces first. */
int nx_prefetch_begin(nx_engine* e, uint32_t app, const nx_planner_config* cfg, uint64_t* moves);
int nx_prefetch_pump(nx_engine* e, int* active);
int nx_prefetch_quiesce(nx_engine* e, uint64_t* committed_bytes);
/* Per-lane leg sequence of the last switch (lane = 2*link + (up ? 0 : 1),
 * transfer.cpp:39-45), in start order. */
int nx_lane_trace(nx_engine* e, int lane, uint64_t* blocks, uint8_t* src, uint8_t* dst, size_t cap, size_t* n);
uint64_t nx_total_launches(nx_engine* e);
/* K3 checksum launches of the last switch: device start/end (s, from the
 * switch start), legs per launch, lane (0 arrivals, 1 departures). */
int nx_k3_trace(nx_engine* e, double* start_s, double* end_s, int* legs, int* lane, size_t cap, size_t* n);
/* PCIe batches of the last switch, in landing order (the switch timeline;
 * the reference's per-leg TransferRecord log, transfer.hpp:40-47, at batch
 * granularity): device times (s, from the switch start) of the batch start,
 * copy end and end (checks included), and host times of its submission and
 * of the poll that committed it. */
typedef struct {
  int32_t stream; /* 0 = H2D, 1 = D2H */
  int32_t legs;
  int32_t ce;     /* 1 = copy engines, 0 = K1 */
  int32_t pad;
  double start_s, copied_s, end_s;
  double host_submit_s, host_done_s;
} nx_batch_record;
int nx_batch_trace(nx_engine* e, nx_batch_record* out, size_t cap, size_t* n);
/* Every leg of the last nx_switch (the reference's TransferRecord log,
 * transfer.hpp:40-47), in commit order, times in s from the switch start:
 * host times of the leg's start and commit; on the SM path and with per-batch
 * checks, PCIe legs carry their batch's device start/end instead. */
typedef struct {
  uint64_t block;
  uint8_t src, dst; /* TierId */
  uint8_t pad[6];
  double start_s, end_s;
} nx_leg_record;
int nx_leg_records(nx_engine* e, nx_leg_record* out, size_t cap, size_t* n);
/* cudaStream_t of a PCIe lane: 0 = H2D, 1 = D2H. */
void* nx_lane_stream(nx_engine* e, int lane);

/* ---- host link ------------------------------------------------------------ */
/* CE and SM bandwidth, H2D / D2H alone and simultaneously. */
int nx_probe_pcie(nx_engine* e, uint64_t bytes_per_direction, uint64_t chunk_bytes, nx_pcie_probe* out);
/* Both directions at once on the copy engines, D2H chunk i held on the device
 * until H2D chunk i - lag_chunks has landed (the engine's paced shape,
 * pace_lag_legs): gbs = {H2D, D2H, both}, best of 3. */
int nx_probe_pcie_paced(nx_engine* e, uint64_t bytes_per_direction, uint64_t chunk_bytes, int lag_chunks, double gbs[3]);
/* Where a device sits on the host: PCI bus id, NUMA node
 * (sysfs numa_node; when that reads -1, the node holding most of the
 * device's local_cpulist, node_from_cpus = 1) and the local CPUs this process
 * may use (cpulist, e.g. "0-15,32-47"). This is the placement the engine's
 * pinned ring and host copy pool bind to. */
typedef struct {
  char pci_bus_id[32];
  int32_t numa_node;
  int32_t node_from_cpus;
  int32_t n_cpus;
  char cpulist[256];
} nx_device_info;
int nx_device_info_get(int device, nx_device_info* out);
/* Raw SM copy variant probe: out = {H2D, D2H, bidirectional total} GB/s. */
int nx_probe_copy_variant(nx_engine* e, int variant, uint64_t bytes, int ctas, double out[3]);
/* CopyPath::Auto table: sm_faster[k] for launches of 2^k legs. */
int nx_set_auto_table(nx_engine* e, const int* sm_faster, size_t n);
/* Measures SM kernel vs copy engines, both directions running, for batches of
 * 1, 2, 4 ... 128 legs and installs the faster per size (CopyPath::Auto).
 * Arrays hold 8 entries. */
int nx_calibrate(nx_engine* e, uint64_t bytes_per_direction, double sm_gbps[8], double ce_gbps[8], int sm_faster[8]);
/* Host copy pool sizing: GB/s of pinned->paged + paged->pinned at once for
 * worker counts threads[i] (up to cap entries, *n written), installs the
 * fastest (*chosen; the smallest count within 2% of the best). */
int nx_calibrate_host(nx_engine* e, uint64_t bytes_per_direction, int* threads, double* gbps, size_t cap, size_t* n,
                      int* chosen);
/* Per-switch tunables between executes: legs_per_launch, first_batch_legs,
 * d2h_commit_legs, early_frame_release, k3_verify_group, pace_lag_legs,
 * fetch_first_pump, host_streaming_copy, sm_tma_ctas (SM copy kernel: -1 K1T
 * on half the SMs, the default; > 0 K1T on that many CTAs; 0 K1), path (the
 * copy path, 0 Auto / 1 SmKernel / 2 CopyEngine, read at each execute). */
int nx_engine_set_option(nx_engine* e, const char* name, int value);
/* Workers of the host copy pool taking jobs now. */
int nx_host_threads(nx_engine* e, int* out);
/* K3 checksum launch duration (us) for 1, 2, 4 ... 128 legs; us[2*k] TMA, us[2*k+1] LDG. */
int nx_probe_checksum_launch(nx_engine* e, double us[16]);
/* Same, optionally while both PCIe directions carry copy-engine traffic. */
int nx_probe_checksum_launch_ex(nx_engine* e, int under_pcie_load, double us[16]);

/* ---- scheduler + launch gate (§3, §6) ---------------------------- */
/* MlfqConfig defaults (proj/include/nixie/mlfq.hpp:13-23). */
void nx_mlfq_config_default(nx_mlfq_config* cfg);
int nx_gate_create(nx_engine* e, const nx_mlfq_config* mcfg, const nx_planner_config* pcfg, nx_gate** out);
void nx_gate_destroy(nx_gate* g);
/* MlfqScheduler::register_app (mlfq.cpp:51-57) + the app's CUDA stream. */
int nx_gate_attach(nx_gate* g, uint32_t app, void* stream, double now);
/* Interposed kernel launch (thread-safe): *passed = 1 if the app holds the
 * grant and is resident. Otherwise its request is enqueued (mlfq.cpp:132-138)
 * and the calling thread is held until a switch to the app has submitted its
 * last fetch; the app's stream then waits on the device for that fetch to
 * land (*passed = 0). Fails with InvalidState after timeout_s. */
int nx_gate_before_launch(nx_gate* g, uint32_t app, double now, double timeout_s, int* passed);
/* Must follow every successful nx_gate_before_launch once the kernel is
 * enqueued: releases the app's launch lock (a pause waits for it). */
int nx_gate_after_launch(nx_gate* g, uint32_t app);
/* MlfqScheduler::on_api_event (mlfq.cpp:71-85): 0 NonBlockingReturn,
 * 1 BlockingEnter, 2 BlockingExit. */
int nx_gate_api_event(nx_gate* g, uint32_t app, double now, int kind);
/* One scheduler tick: infer_all, then a switch if the GPU has
 * no holder, the holder is idle or should_preempt fires; *switched_to =
 * UINT32_MAX when nothing switched. */
int nx_gate_tick(nx_gate* g, double now, uint32_t* switched_to);
uint64_t nx_gate_switches(nx_gate* g);
/* MLFQ prefetch (plan_prefetch planner.cpp:218-242,
 * next_prefetch_candidate mlfq.cpp:164-166, cancel_pending transfer.cpp:89-113):
 * ticks that do not switch move the next candidate's pageable blocks to the
 * pinned tier on the host copy pool; a switch quiesces it first. */
int nx_gate_set_prefetch(nx_gate* g, int on);
uint64_t nx_gate_prefetched_bytes(nx_gate* g);
/* Synthetic application kernel: occupies one warp for ~ns on `stream`. */
int nx_launch_busy_kernel(void* stream, uint64_t ns);
/* MlfqScheduler::select_next (mlfq.cpp:144-162); *app = UINT32_MAX if none. */
int nx_gate_select_next(nx_gate* g, double now, uint32_t* app);
/* Pause incumbent, drain, plan, execute, grant `to`, release its gate. */
int nx_gate_switch(nx_gate* g, uint32_t to, double now, nx_switch_stats* out);
int nx_gate_granted(nx_gate* g, uint32_t* app);
/* Test app kernel: sums the checksums of `app`'s blocks, reading them through
 * the device frame table on `stream`; result (device-side) copied to *out
 * after the stream reaches it. */
int nx_gate_app_checksum_async(nx_gate* g, uint32_t app, void* stream, uint64_t* out_pinned);
int nx_stream_sync(void* stream);
/* Plumbing for callers without their own CUDA runtime (tests, bindings). */
int nx_stream_create(void** stream);
void nx_stream_destroy(void* stream);
int nx_stream_query(void* stream, int* done); /* *done = 1 when all queued work finished */
int nx_pinned_alloc(size_t bytes, void** out);
void nx_pinned_free(void* p);

/* ---- workload driver / parity traces -------------------------------------- */
/* Runs a scenario (include/nixie/scenario.hpp grammar) on the virtual clock
 * with reference-identical link timing; no GPU needed. *trace is malloc'ed,
 * free with nx_free. */
int nx_scenario_model(const char* spec, char** trace, size_t* len);
/* Same, with up to legs_per_lane legs in flight per lane (the concurrency the
 * CUDA engine uses); per-lane sequences and placements must not change. */
int nx_scenario_model_lanes(const char* spec, int legs_per_lane, char** trace, size_t* len);
/* Same scenario through the CUDA engine (real copies). Every app is filled
 * with the pattern (seed) up front; after each switch the incoming app is
 * verified byte-exact (`V k app bad` lines) and at the end every app is. */
int nx_scenario_real(const char* spec, const nx_engine_config* cfg, uint64_t seed, char** trace, size_t* len);
/* An MLFQ-driven workload (include/nixie_workload/workload_sim.hpp grammar:
 * interactive / batch apps, launch gate, scheduler ticks) on
 * the virtual clock. Replaces the reference's (absent) workload-sim `run`
 * (SPEC.md:455); its reference twin is oracle/_ref/ref_workload. */
int nx_workload_model(const char* spec, char** trace, size_t* len);
/* Same workload with every planned switch executed by the CUDA engine (real
 * bytes; decisions keep the virtual clock; with `prefetch on` the engine also
 * performs the prefetch moves the model committed before each switch). Adds
 * `H k moves`, `M k differing-blocks`, `V k app bad ...` and final
 * `F app bad` lines. */
int nx_workload_real(const char* spec, const nx_engine_config* cfg, uint64_t seed, char** trace, size_t* len);
/* ---- UVM demand-paging model (the comparator; include/nixie/uvm.hpp) ------
 * UvmSim (proj/include/nixie/uvm.hpp:40-80) behind a handle,
 * for policy comparisons in the CLI (uvm_rr_<W>: round-robin time slices
 * over demand paging, as nvshare does). No GPU. */
typedef struct nx_uvm nx_uvm;
/* UvmSim(gpu_capacity, pcie link, UvmConfig{fault_latency, prefetch_pages}) (uvm.hpp:42-44). */
int nx_uvm_create(uint64_t gpu_capacity, double pcie_up_bw, double pcie_down_bw, int half_duplex,
                  double fault_latency, int prefetch_pages, nx_uvm** out);
/* register_alloc(app, size) (uvm.hpp:46). */
int nx_uvm_register(nx_uvm* h, uint32_t app, uint64_t size);
/* touch_kernel(app, every chunk of app, base, now) (uvm.hpp:55): the kernel's
 * duration including the fault service time. */
int nx_uvm_touch(nx_uvm* h, uint32_t app, double base_duration, double now, double* duration);
/* fault_count, faulted_bytes_total, pinned_mirror_peak (uvm.hpp:58-63); any pointer may be NULL. */
int nx_uvm_stats(const nx_uvm* h, uint64_t* faults, uint64_t* faulted_bytes, uint64_t* mirror_peak);
void nx_uvm_destroy(nx_uvm* h);

void nx_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* NIXIE_B200_H_ */
