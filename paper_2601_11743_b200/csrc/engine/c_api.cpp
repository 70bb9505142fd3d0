// C ABI (include/nixie_b200.h) over the C++ API: exceptions become status
// codes, handles are opaque.
#include "nixie_b200.h"

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <string>

#include "phys.hpp"
#include "nixie/scenario.hpp"
#include "nixie/uvm.hpp"
#include "nixie/workload.hpp"
#include <nixie_workload/workload_sim.hpp>
#include "nixie/swap_engine.hpp"
#include "nixie/uvm.hpp"
#include "nx_kernels.h"
#include "phys.hpp"

using namespace nixie;
using namespace nixie::b200;

struct nx_engine {
  std::unique_ptr<SwapEngine> eng;
  std::vector<TransferRecord> last_legs;  // the last nx_switch's per-leg log
};

struct nx_gate {
  nx_engine* e = nullptr;
  std::unique_ptr<MlfqScheduler> sched;
  std::unique_ptr<LaunchGate> gate;
  unsigned long long* d_out = nullptr;  // [2] per app-checksum launch
  unsigned* d_blocks = nullptr;
  unsigned* h_blocks = nullptr;  // pinned staging of the block list
  std::size_t blocks_cap = 0;
};

namespace {

// A launch gate parks application streams behind a device-side wait. With
// the default 8 hardware work queues, streams share queues and a parked
// stream could stall an engine stream queued behind it; 32 queues give every
// stream of a typical instance its own. Only effective if the process has not
// initialised CUDA before loading this library; an explicit setting wins.
__attribute__((constructor)) void nx_widen_hw_queues() { setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0); }

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return NX_OK;
  } catch (const CudaFailure& e) {
    g_err = e.what();
    return NX_E_CUDA;
  } catch (const SimError& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  } catch (const InvariantViolation& e) {
    g_err = e.what();
    return NX_E_INVARIANT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NX_E_ARG;
  } catch (...) {
    g_err = "unknown exception";
    return NX_E_ARG;
  }
}

void need(const void* p, const char* what) {
  if (p == nullptr) throw std::invalid_argument(std::string("null argument: ") + what);
}

EngineConfig to_cpp(const nx_engine_config& c) {
  EngineConfig o;
  o.device = c.device;
  o.gpu_capacity = c.gpu_capacity;
  o.pinned_capacity = c.pinned_capacity;
  o.paged_capacity = c.paged_capacity;
  o.path = static_cast<CopyPath>(c.path);
  o.pcie_legs_in_flight = c.pcie_legs_in_flight;
  o.legs_per_launch = c.legs_per_launch;
  o.host_threads = c.host_threads;
  o.host_legs_in_flight = c.host_legs_in_flight;
  o.max_ctas = c.max_ctas;
  o.fused_launch = c.fused_launch != 0;
  o.verify = c.verify != 0;
  o.numa_bind = c.numa_bind != 0;
  o.first_batch_legs = c.first_batch_legs;
  o.k3_tma = c.k3_tma != 0;
  o.k3_one_stream = c.k3_one_stream != 0;
  o.k3_grouped = c.k3_grouped != 0;
  o.k3_verify_group = c.k3_verify_group;
  o.d2h_commit_legs = c.d2h_commit_legs;
  o.early_frame_release = c.early_frame_release != 0;
  o.pace_lag_legs = c.pace_lag_legs;
  o.fetch_first_pump = c.fetch_first_pump != 0;
  o.host_streaming_copy = c.host_streaming_copy != 0;
  return o;
}

PlannerConfig to_cpp(const nx_planner_config* c) {
  PlannerConfig p;
  if (c == nullptr) return p;
  p.streaming_window = c->streaming_window;
  p.pinned_budget = c->pinned_budget;
  if (c->victim_order != nullptr) p.eviction_policy.victim_order.assign(c->victim_order, c->victim_order + c->n_victims);
  return p;
}

void fill_stats(const SwapEngine& eng, const ExecResult& r, nx_switch_stats* out) {
  if (out == nullptr) return;
  const SwitchStats& s = eng.last_stats();
  std::memset(out, 0, sizeof(*out));
  out->bytes_in = s.bytes_in;
  out->bytes_out = s.bytes_out;
  out->pcie_h2d_bytes = s.pcie_h2d_bytes;
  out->pcie_d2h_bytes = s.pcie_d2h_bytes;
  out->host_bytes = s.host_bytes;
  out->wall_s = s.wall_s;
  out->plan_s = s.plan_s;
  out->device_span_s = s.device_span_s;
  out->kernel_s_h2d = s.kernel_s[0];
  out->kernel_s_d2h = s.kernel_s[1];
  out->launches_h2d = s.launches[0];
  out->launches_d2h = s.launches[1];
  out->ce_batches_h2d = s.ce_batches[0];
  out->ce_batches_d2h = s.ce_batches[1];
  out->host_legs = s.host_legs;
  out->verified = s.verified;
  out->unverified = s.unverified;
  out->mismatches = s.mismatches;
  out->k1_s = s.k1_s;
  out->k3_s = s.k3_s;
  out->k1_bytes = s.k1_bytes;
  out->k3_bytes = s.k3_bytes;
  out->k1_launches = s.k1_launches;
  out->k3_launches = s.k3_launches;
  out->k3_busy_s = s.k3_busy_s;
  out->k3_kernel_s = s.k3_kernel_s;
  out->ce_calls = s.ce_calls;
  out->pace_waits = s.pace_waits;
  for (int k = 0; k < 2; ++k) {
    out->ce_calls_dir[k] = s.ce_calls_dir[k];
    out->run_breaks_src[k] = s.run_breaks_src[k];
    out->run_breaks_dst[k] = s.run_breaks_dst[k];
  }
  if (s.device_span_s > 0) {
    double lo = 1e30, hi = 0;
    for (const TransferRecord& t : r.events)
      if ((t.src == TierId::Gpu && t.dst == TierId::PinnedHost) || (t.src == TierId::PinnedHost && t.dst == TierId::Gpu)) {
        lo = std::min(lo, t.start);
        hi = std::max(hi, t.end);
      }
    if (hi > lo) {
      const ThroughputSample tp = aggregate_throughput(r.events, lo, hi);
      out->tp_to_gpu = tp.to_gpu;
      out->tp_from_gpu = tp.from_gpu;
      out->tp_bidir = tp.bidirectional;
    }
  }
}

char* dup_out(const std::string& s, size_t* len) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (p == nullptr) throw std::bad_alloc();
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = '\0';
  if (len) *len = s.size();
  return p;
}

}  // namespace

extern "C" {

const char* nx_last_error(void) { return g_err.c_str(); }
const char* nx_version(void) { return "nixie-b200 0.1 (sm_100a)"; }

int nx_cuda_device_count(int* count) {
  return guard([&] {
    need(count, "count");
    *count = 0;
    const cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
      *count = 0;
      cudaGetLastError();
    }
  });
}

void nx_engine_config_default(nx_engine_config* c) {
  if (c == nullptr) return;
  const EngineConfig d;
  c->device = d.device;
  c->gpu_capacity = d.gpu_capacity;
  c->pinned_capacity = d.pinned_capacity;
  c->paged_capacity = d.paged_capacity;
  c->path = static_cast<int>(d.path);
  c->pcie_legs_in_flight = d.pcie_legs_in_flight;
  c->legs_per_launch = d.legs_per_launch;
  c->host_threads = d.host_threads;
  c->host_legs_in_flight = d.host_legs_in_flight;
  c->max_ctas = d.max_ctas;
  c->fused_launch = d.fused_launch;
  c->verify = d.verify;
  c->numa_bind = d.numa_bind;
  c->first_batch_legs = d.first_batch_legs;
  c->k3_tma = d.k3_tma;
  c->k3_one_stream = d.k3_one_stream;
  c->k3_grouped = d.k3_grouped;
  c->k3_verify_group = d.k3_verify_group;
  c->d2h_commit_legs = d.d2h_commit_legs;
  c->early_frame_release = d.early_frame_release;
  c->pace_lag_legs = d.pace_lag_legs;
  c->fetch_first_pump = d.fetch_first_pump;
  c->host_streaming_copy = d.host_streaming_copy;
}

void nx_planner_config_default(nx_planner_config* c) {
  if (c == nullptr) return;
  const PlannerConfig d;
  c->streaming_window = d.streaming_window;
  c->pinned_budget = d.pinned_budget;
  c->victim_order = nullptr;
  c->n_victims = 0;
}

int nx_engine_create(const nx_engine_config* cfg, nx_engine** out) {
  return guard([&] {
    need(cfg, "cfg");
    need(out, "out");
    auto h = std::make_unique<nx_engine>();
    h->eng = std::make_unique<SwapEngine>(to_cpp(*cfg));
    *out = h.release();
  });
}

void nx_engine_destroy(nx_engine* e) { delete e; }

int nx_alloc(nx_engine* e, uint32_t app, uint64_t size, int tier, uint64_t* chunks, size_t cap, size_t* n) {
  return guard([&] {
    need(e, "engine");
    if (tier < 0 || tier >= kTierCount) throw std::invalid_argument("bad tier");
    const std::vector<ChunkId> ids = e->eng->allocate(app, size, static_cast<TierId>(tier));
    if (chunks)
      for (size_t i = 0; i < ids.size() && i < cap; ++i) chunks[i] = ids[i];
    if (n) *n = ids.size();
  });
}

int nx_free_chunk(nx_engine* e, uint32_t app, uint64_t chunk, uint64_t* released) {
  return guard([&] {
    need(e, "engine");
    const Bytes r = e->eng->free_chunk(app, chunk);
    if (released) *released = r;
  });
}

int nx_audit(nx_engine* e) {
  return guard([&] {
    need(e, "engine");
    e->eng->mem().audit();
  });
}

int nx_app_resident(nx_engine* e, uint32_t app, uint64_t out[4]) {
  return guard([&] {
    need(e, "engine");
    need(out, "out");
    for (int d = 0; d < kTierCount; ++d) out[d] = e->eng->mem().app_bytes_resident(app, tier_at_depth(d));
  });
}

int nx_pinned_physical(nx_engine* e, uint64_t* now, uint64_t* peak) {
  return guard([&] {
    need(e, "engine");
    if (now) *now = e->eng->mem().pinned_physical();
    if (peak) *peak = e->eng->mem().pinned_physical_peak();
  });
}

int nx_pinned_overhead(nx_engine* e, uint64_t* bytes) {
  return guard([&] {
    need(e, "engine");
    need(bytes, "bytes");
    *bytes = e->eng->pinned_overhead();
  });
}

int nx_fill_pattern(nx_engine* e, uint32_t app, uint64_t seed) {
  return guard([&] {
    need(e, "engine");
    e->eng->fill_pattern(app, seed);
  });
}

int nx_verify_pattern(nx_engine* e, uint32_t app, uint64_t seed, uint64_t* bad) {
  return guard([&] {
    need(e, "engine");
    const std::uint64_t b = e->eng->verify_pattern(app, seed);
    if (bad) *bad = b;
  });
}

int nx_block_frame(nx_engine* e, uint64_t block, void** frame) {
  return guard([&] {
    need(e, "engine");
    need(frame, "frame");
    *frame = e->eng->frame_of(block);
  });
}

int nx_block_checksum(nx_engine* e, uint64_t block, uint64_t* ck) {
  return guard([&] {
    need(e, "engine");
    need(ck, "checksum");
    *ck = e->eng->block_checksum(block);
  });
}

int nx_app_blocks(nx_engine* e, uint32_t app, uint64_t* blocks, size_t cap, size_t* n) {
  return guard([&] {
    need(e, "engine");
    size_t k = 0;
    const MemState& m = e->eng->mem();
    for (ChunkId c : m.chunks_of(app))
      for (BlockId b : m.chunk(c).blocks) {
        if (blocks && k < cap) blocks[k] = b;
        ++k;
      }
    if (n) *n = k;
  });
}

int nx_block_read(nx_engine* e, uint64_t block, void* host_dst) {
  return guard([&] {
    need(e, "engine");
    need(host_dst, "dst");
    e->eng->read_block(block, host_dst);
  });
}

int nx_block_poke(nx_engine* e, uint64_t block, uint64_t offset, uint8_t value) {
  return guard([&] {
    need(e, "engine");
    e->eng->poke_block(block, offset, value);
  });
}

int nx_plan(nx_engine* e, uint32_t incoming, const nx_planner_config* cfg, char* dump, size_t cap, size_t* len,
            uint64_t* bytes_in, uint64_t* bytes_out) {
  return guard([&] {
    need(e, "engine");
    const MigrationPlan p = plan_switch(incoming, e->eng->mem(), to_cpp(cfg));
    const std::string d = p.dump();
    if (dump && cap > 0) {
      const size_t m = std::min(cap - 1, d.size());
      std::memcpy(dump, d.data(), m);
      dump[m] = '\0';
    }
    if (len) *len = d.size();
    if (bytes_in) *bytes_in = p.bytes_in;
    if (bytes_out) *bytes_out = p.bytes_out;
  });
}

int nx_switch(nx_engine* e, uint32_t incoming, const nx_planner_config* cfg, void* drain, nx_switch_stats* out) {
  return guard([&] {
    need(e, "engine");
    ExecResult r = e->eng->switch_to(incoming, to_cpp(cfg), static_cast<cudaStream_t>(drain));
    fill_stats(*e->eng, r, out);
    e->last_legs = std::move(r.events);
  });
}

int nx_leg_records(nx_engine* e, nx_leg_record* out, size_t cap, size_t* n) {
  return guard([&] {
    need(e, "engine");
    const auto& t = e->last_legs;
    for (size_t i = 0; i < t.size() && i < cap && out; ++i)
      out[i] = nx_leg_record{t[i].block, static_cast<uint8_t>(t[i].src), static_cast<uint8_t>(t[i].dst), {0}, t[i].start,
                             t[i].end};
    if (n) *n = t.size();
  });
}

int nx_prefetch_begin(nx_engine* e, uint32_t app, const nx_planner_config* cfg, uint64_t* moves) {
  return guard([&] {
    need(e, "engine");
    const MigrationPlan plan = plan_prefetch(app, e->eng->mem(), to_cpp(cfg));
    if (moves) *moves = plan.moves.size();
    if (!plan.moves.empty()) e->eng->prefetch_begin(plan);
  });
}

int nx_prefetch_pump(nx_engine* e, int* active) {
  return guard([&] {
    need(e, "engine");
    const bool a = e->eng->prefetch_pump();
    if (active) *active = a ? 1 : 0;
  });
}

int nx_prefetch_quiesce(nx_engine* e, uint64_t* committed_bytes) {
  return guard([&] {
    need(e, "engine");
    e->eng->prefetch_quiesce();
    if (committed_bytes) *committed_bytes = e->eng->prefetched_bytes();
  });
}

int nx_lane_trace(nx_engine* e, int lane, uint64_t* blocks, uint8_t* src, uint8_t* dst, size_t cap, size_t* n) {
  return guard([&] {
    need(e, "engine");
    if (lane < 0 || lane >= 6) throw std::invalid_argument("bad lane");
    const auto& t = e->eng->lane_trace()[lane];
    for (size_t i = 0; i < t.size() && i < cap; ++i) {
      if (blocks) blocks[i] = t[i].block;
      if (src) src[i] = static_cast<uint8_t>(t[i].src);
      if (dst) dst[i] = static_cast<uint8_t>(t[i].dst);
    }
    if (n) *n = t.size();
  });
}

uint64_t nx_total_launches(nx_engine* e) { return e ? e->eng->total_launches() : 0; }

int nx_k3_trace(nx_engine* e, double* start_s, double* end_s, int* legs, int* lane, size_t cap, size_t* n) {
  return guard([&] {
    need(e, "engine");
    const auto& t = e->eng->k3_launches();
    for (size_t i = 0; i < t.size() && i < cap; ++i) {
      if (start_s) start_s[i] = t[i].start_s;
      if (end_s) end_s[i] = t[i].end_s;
      if (legs) legs[i] = t[i].legs;
      if (lane) lane[i] = t[i].lane;
    }
    if (n) *n = t.size();
  });
}
int nx_batch_trace(nx_engine* e, nx_batch_record* out, size_t cap, size_t* n) {
  return guard([&] {
    need(e, "engine");
    const auto& t = e->eng->batch_trace();
    for (size_t i = 0; i < t.size() && i < cap && out; ++i)
      out[i] = nx_batch_record{t[i].stream, t[i].legs, t[i].ce ? 1 : 0, 0, t[i].start_s, t[i].copied_s, t[i].end_s,
                               t[i].host_submit_s, t[i].host_done_s};
    if (n) *n = t.size();
  });
}
void* nx_lane_stream(nx_engine* e, int lane) { return e ? static_cast<void*>(e->eng->stream(lane)) : nullptr; }

int nx_probe_pcie_paced(nx_engine* e, uint64_t bytes, uint64_t chunk, int lag_chunks, double gbs[3]) {
  return guard([&] {
    need(e, "engine");
    need(gbs, "gbs");
    if (lag_chunks < 1) throw SimError(Err::ValidationError, "lag_chunks must be >= 1");
    const auto r = e->eng->probe_pcie_paced(bytes, chunk, lag_chunks);
    for (int k = 0; k < 3; ++k) gbs[k] = r[k];
  });
}

int nx_probe_pcie(nx_engine* e, uint64_t bytes, uint64_t chunk, nx_pcie_probe* out) {
  return guard([&] {
    need(e, "engine");
    need(out, "out");
    const PcieProbe p = e->eng->probe_pcie(bytes, chunk);
    std::memset(out, 0, sizeof(*out));
    for (int k = 0; k < 2; ++k) {
      out->h2d[k] = p.h2d[k];
      out->d2h[k] = p.d2h[k];
      out->bidir_h2d[k] = p.bidir_h2d[k];
      out->bidir_d2h[k] = p.bidir_d2h[k];
      out->bidir_total[k] = p.bidir_total[k];
    }
    out->bytes_per_direction = p.bytes_per_direction;
    out->chunk_bytes = p.chunk_bytes;
    out->numa_node = p.numa_node;
  });
}

int nx_device_info_get(int device, nx_device_info* out) {
  return guard([&] {
    need(out, "out");
    std::memset(out, 0, sizeof(*out));
    const nixie::b200::NumaInfo n = nixie::b200::numa_for_device(device);
    std::snprintf(out->pci_bus_id, sizeof(out->pci_bus_id), "%s", n.pci_bus_id.c_str());
    out->numa_node = n.node;
    out->node_from_cpus = n.node_from_cpus ? 1 : 0;
    out->n_cpus = static_cast<int32_t>(n.cpus.size());
    std::string list;
    for (std::size_t i = 0; i < n.cpus.size();) {  // compress runs: 0-15,32-47
      std::size_t j = i;
      while (j + 1 < n.cpus.size() && n.cpus[j + 1] == n.cpus[j] + 1) ++j;
      if (!list.empty()) list += ",";
      list += std::to_string(n.cpus[i]) + (j > i ? "-" + std::to_string(n.cpus[j]) : "");
      i = j + 1;
    }
    std::snprintf(out->cpulist, sizeof(out->cpulist), "%s", list.c_str());
  });
}

int nx_probe_copy_variant(nx_engine* e, int variant, uint64_t bytes, int ctas, double out[3]) {
  return guard([&] {
    need(e, "engine");
    need(out, "out");
    const auto r = e->eng->probe_copy_variant(variant, bytes, ctas);
    for (int i = 0; i < 3; ++i) out[i] = r[i];
  });
}

int nx_calibrate(nx_engine* e, uint64_t bytes, double sm_gbps[8], double ce_gbps[8], int sm_faster[8]) {
  return guard([&] {
    need(e, "engine");
    const Calibration c = e->eng->calibrate(bytes);
    for (std::size_t k = 0; k < 8 && k < c.legs.size(); ++k) {
      if (sm_gbps) sm_gbps[k] = c.sm_gbps[k];
      if (ce_gbps) ce_gbps[k] = c.ce_gbps[k];
      if (sm_faster) sm_faster[k] = c.sm_gbps[k] > c.ce_gbps[k] ? 1 : 0;
    }
  });
}

int nx_calibrate_host(nx_engine* e, uint64_t bytes, int* threads, double* gbps, size_t cap, size_t* n, int* chosen) {
  return guard([&] {
    need(e, "engine");
    const HostCalibration c = e->eng->calibrate_host(bytes);
    std::size_t k = 0;
    for (; k < c.threads.size() && k < cap; ++k) {
      if (threads) threads[k] = c.threads[k];
      if (gbps) gbps[k] = c.gbps[k];
    }
    if (n) *n = k;
    if (chosen) *chosen = c.chosen;
  });
}

int nx_engine_set_option(nx_engine* e, const char* name, int value) {
  return guard([&] {
    need(e, "engine");
    need(name, "name");
    e->eng->set_option(name, value);
  });
}

int nx_host_threads(nx_engine* e, int* out) {
  return guard([&] {
    need(e, "engine");
    need(out, "out");
    *out = e->eng->host_threads();
  });
}

int nx_probe_checksum_launch(nx_engine* e, double us[16]) { return nx_probe_checksum_launch_ex(e, 0, us); }

int nx_probe_checksum_launch_ex(nx_engine* e, int under_pcie_load, double us[16]) {
  return guard([&] {
    need(e, "engine");
    need(us, "us");
    const auto r = e->eng->probe_checksum_launch(under_pcie_load != 0);
    for (std::size_t k = 0; k < r.size() && k < 8; ++k) {
      us[2 * k] = r[k][0];
      us[2 * k + 1] = r[k][1];
    }
  });
}

int nx_set_auto_table(nx_engine* e, const int* sm_faster, size_t n) {
  return guard([&] {
    need(e, "engine");
    std::vector<bool> t(n);
    for (size_t i = 0; i < n; ++i) t[i] = sm_faster[i] != 0;
    e->eng->set_auto_table(t);
  });
}

void nx_mlfq_config_default(nx_mlfq_config* c) {
  if (c == nullptr) return;
  const MlfqConfig d;
  c->levels = d.levels;
  c->base_allotment = d.base_allotment;
  c->base_preemption = d.base_preemption;
  c->idle_threshold = d.idle_threshold;
  c->tick = d.tick;
}

int nx_gate_create(nx_engine* e, const nx_mlfq_config* mcfg, const nx_planner_config* pcfg, nx_gate** out) {
  return guard([&] {
    need(e, "engine");
    need(out, "out");
    MlfqConfig m;
    if (mcfg) {
      m.levels = mcfg->levels;
      m.base_allotment = mcfg->base_allotment;
      m.base_preemption = mcfg->base_preemption;
      m.idle_threshold = mcfg->idle_threshold;
      m.tick = mcfg->tick;
    }
    auto g = std::make_unique<nx_gate>();
    g->e = e;
    g->sched = std::make_unique<MlfqScheduler>(m);
    g->sched->set_logging(true);
    g->gate = std::make_unique<LaunchGate>(*e->eng, *g->sched, to_cpp(pcfg));
    NX_CUDA(cudaMalloc(&g->d_out, 2 * sizeof(unsigned long long)));
    g->blocks_cap = 1u << 20;  // 2 TiB of 2 MiB blocks: never regrown while streams may be gated
    NX_CUDA(cudaMalloc(&g->d_blocks, sizeof(unsigned) * g->blocks_cap));
    NX_CUDA(cudaHostAlloc(&g->h_blocks, sizeof(unsigned) * g->blocks_cap, cudaHostAllocPortable));
    *out = g.release();
  });
}

void nx_gate_destroy(nx_gate* g) {
  if (g == nullptr) return;
  cudaDeviceSynchronize();
  cudaFree(g->d_out);
  cudaFree(g->d_blocks);
  if (g->h_blocks) cudaFreeHost(g->h_blocks);
  delete g;
}

int nx_gate_attach(nx_gate* g, uint32_t app, void* stream, double now) {
  return guard([&] {
    need(g, "gate");
    if (!g->sched->registered(app)) g->sched->register_app(app, now);
    g->gate->attach(app, static_cast<cudaStream_t>(stream));
  });
}

int nx_gate_before_launch(nx_gate* g, uint32_t app, double now, double timeout_s, int* passed) {
  return guard([&] {
    need(g, "gate");
    const bool ok = g->gate->before_launch(app, now, timeout_s);
    if (passed) *passed = ok ? 1 : 0;
  });
}

int nx_gate_after_launch(nx_gate* g, uint32_t app) {
  return guard([&] {
    need(g, "gate");
    g->gate->after_launch(app);
  });
}

int nx_gate_api_event(nx_gate* g, uint32_t app, double now, int kind) {
  return guard([&] {
    need(g, "gate");
    if (kind < 0 || kind > 2) throw std::invalid_argument("bad api event kind");
    g->gate->api_event(app, now, static_cast<ApiEventKind>(kind));
  });
}

int nx_gate_tick(nx_gate* g, double now, uint32_t* switched_to) {
  return guard([&] {
    need(g, "gate");
    const auto s = g->gate->tick(now);
    if (switched_to) *switched_to = s ? *s : ~uint32_t{0};
  });
}

uint64_t nx_gate_switches(nx_gate* g) { return g ? g->gate->switches() : 0; }

int nx_gate_set_prefetch(nx_gate* g, int on) {
  return guard([&] {
    need(g, "gate");
    g->gate->set_prefetch(on != 0);
  });
}

uint64_t nx_gate_prefetched_bytes(nx_gate* g) { return g ? g->gate->prefetched_bytes() : 0; }

int nx_launch_busy_kernel(void* stream, uint64_t ns) {
  return guard([&] {
    NX_CUDA(launch_spin(static_cast<unsigned>(std::min<uint64_t>(ns, 4000000000ull)), static_cast<cudaStream_t>(stream)));
  });
}

int nx_gate_select_next(nx_gate* g, double now, uint32_t* app) {
  return guard([&] {
    need(g, "gate");
    need(app, "app");
    const auto n = g->gate->select_next(now);
    *app = n ? *n : ~uint32_t{0};
  });
}

int nx_gate_switch(nx_gate* g, uint32_t to, double now, nx_switch_stats* out) {
  return guard([&] {
    need(g, "gate");
    const ExecResult r = g->gate->context_switch(to, now);
    fill_stats(*g->e->eng, r, out);
  });
}

int nx_gate_granted(nx_gate* g, uint32_t* app) {
  return guard([&] {
    need(g, "gate");
    need(app, "app");
    const auto a = g->gate->granted();
    *app = a ? *a : ~uint32_t{0};
  });
}

int nx_gate_app_checksum_async(nx_gate* g, uint32_t app, void* stream, uint64_t* out_pinned) {
  return guard([&] {
    need(g, "gate");
    need(out_pinned, "out");
    const MemState& m = g->e->eng->mem();
    std::vector<unsigned> blocks;
    for (ChunkId c : m.chunks_of(app))
      for (BlockId b : m.chunk(c).blocks) blocks.push_back(static_cast<unsigned>(b));
    auto s = static_cast<cudaStream_t>(stream);
    // No device-wide synchronisation here: `stream` (or another app's
    // stream) may be parked behind a gate that only a later switch opens.
    if (blocks.size() > g->blocks_cap) throw SimError(Err::CapacityExceeded, "app has more blocks than the gate's list");
    // Fully asynchronous: the launch may sit behind a device-side gate. The
    // pinned staging list stays valid until the next call on this gate.
    std::memcpy(g->h_blocks, blocks.data(), sizeof(unsigned) * blocks.size());
    NX_CUDA(cudaMemcpyAsync(g->d_blocks, g->h_blocks, sizeof(unsigned) * blocks.size(), cudaMemcpyHostToDevice, s));
    NX_CUDA(cudaMemsetAsync(g->d_out, 0, 2 * sizeof(unsigned long long), s));
    NX_CUDA(launch_table_checksum(g->e->eng->device_frame_table(), g->d_blocks, static_cast<int>(blocks.size()), g->d_out, s));
    NX_CUDA(cudaMemcpyAsync(out_pinned, g->d_out, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  });
}

int nx_stream_create(void** out) {
  return guard([&] {
    need(out, "out");
    cudaStream_t s = nullptr;
    NX_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    *out = s;
  });
}

void nx_stream_destroy(void* stream) {
  if (stream) cudaStreamDestroy(static_cast<cudaStream_t>(stream));
}

int nx_stream_query(void* stream, int* done) {
  return guard([&] {
    need(done, "done");
    const cudaError_t e = cudaStreamQuery(static_cast<cudaStream_t>(stream));
    if (e == cudaErrorNotReady) {
      *done = 0;
      return;
    }
    NX_CUDA(e);
    *done = 1;
  });
}

int nx_stream_sync(void* stream) {
  return guard([&] { NX_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream))); });
}

int nx_pinned_alloc(size_t bytes, void** out) {
  return guard([&] {
    need(out, "out");
    NX_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocPortable));
    std::memset(*out, 0, bytes);
  });
}

void nx_pinned_free(void* p) {
  if (p) cudaFreeHost(p);
}

int nx_scenario_model(const char* spec, char** trace, size_t* len) {
  return guard([&] {
    need(spec, "spec");
    need(trace, "trace");
    *trace = dup_out(run_scenario_model(parse_scenario(spec)), len);
  });
}

int nx_scenario_model_lanes(const char* spec, int legs_per_lane, char** trace, size_t* len) {
  return guard([&] {
    need(spec, "spec");
    need(trace, "trace");
    *trace = dup_out(run_scenario_model(parse_scenario(spec), legs_per_lane), len);
  });
}

int nx_scenario_real(const char* spec, const nx_engine_config* cfg, uint64_t seed, char** trace, size_t* len) {
  return guard([&] {
    need(spec, "spec");
    need(cfg, "cfg");
    need(trace, "trace");
    const Scenario sc = parse_scenario(spec);
    EngineConfig ec = to_cpp(*cfg);
    ec.gpu_capacity = sc.hw.tier_capacity[0];
    ec.pinned_capacity = sc.hw.tier_capacity[1];
    ec.paged_capacity = sc.hw.tier_capacity[2];
    SwapEngine eng(ec);
    for (const ScenarioApp& a : sc.apps) eng.allocate(a.id, a.size, a.tier);
    for (const ScenarioApp& a : sc.apps) eng.fill_pattern(a.id, seed);
    SwitchRunner runner;
    runner.mem = [&]() -> MemState& { return eng.mem(); };
    runner.virtual_clock = false;
    // The scenario's schedule runs on the virtual clock, as in the reference:
    // a switch completes when the model (on a copy of the registry) says so,
    // not when the real copies end. Otherwise a scenario whose switch times
    // are close together would schedule differently on real hardware (which
    // request arrives before which switch ends feeds the MLFQ's decisions),
    // and the plans of later switches would follow another schedule.
    runner.run = [&](const MigrationPlan& plan, const PlannerConfig& pc, Seconds now,
                     std::array<std::vector<std::array<std::uint64_t, 3>>, 6>& lanes) {
      MemState shadow = eng.mem();
      const ExecResult model = execute(plan, shadow, sc.hw, pc, now);
      eng.execute(plan, pc);
      const auto& t = eng.lane_trace();
      for (int l = 0; l < 6; ++l)
        for (const LegTrace& x : t[l])
          lanes[l].push_back({x.block, static_cast<std::uint64_t>(x.src), static_cast<std::uint64_t>(x.dst)});
      return model.completion;
    };
    runner.after_switch = [&](std::size_t k, AppId incoming, std::string& out) {
      const SwitchStats& s = eng.last_stats();
      out += "V " + std::to_string(k) + " " + std::to_string(incoming) + " " +
             std::to_string(eng.verify_pattern(incoming, seed)) + " verified " + std::to_string(s.verified) + " unverified " +
             std::to_string(s.unverified) + "\n";
    };
    std::string out = drive_scenario(sc, runner);
    for (const ScenarioApp& a : sc.apps)
      out += "F " + std::to_string(a.id) + " " + std::to_string(eng.verify_pattern(a.id, seed)) + "\n";
    *trace = dup_out(out, len);
  });
}

int nx_workload_model(const char* spec, char** trace, size_t* len) {
  return guard([&] {
    need(spec, "spec");
    need(trace, "trace");
    *trace = dup_out(run_workload_model(spec), len);
  });
}

// The workload's decisions follow the virtual clock (the model's completion
// of each switch, computed on a copy of the registry), while the CUDA engine
// moves the bytes of every planned switch; after each switch the engine's
// placement must equal the model's (`M` line) and the incoming app must be
// byte-exact (`V` line).
int nx_workload_real(const char* spec, const nx_engine_config* cfg, uint64_t seed, char** trace, size_t* len) {
  return guard([&] {
    need(spec, "spec");
    need(cfg, "cfg");
    need(trace, "trace");
    const workload::Spec ws = workload::parse(spec);
    EngineConfig ec = to_cpp(*cfg);
    ec.gpu_capacity = ws.hw.tier_capacity[0];
    ec.pinned_capacity = ws.hw.tier_capacity[1];
    ec.paged_capacity = ws.hw.tier_capacity[2];
    SwapEngine eng(ec);
    // The workload engine runs on its own model registry (its prefetch
    // Orchestrator commits there, on the virtual clock); the CUDA engine
    // mirrors it: before each switch it performs, for real, the prefetch
    // moves the model committed, then executes the same plan.
    MemState model_mem;
    ws.hw.apply_to(model_mem);
    std::string extra;
    std::size_t k = 0;
    workload::Runner runner = [&](const MigrationPlan& plan, MemState& mem, const HardwareConfig& hw, const PlannerConfig& pc,
                                  Seconds now, std::array<std::vector<std::array<std::uint64_t, 3>>, 6>& lanes) {
      MigrationPlan pf;
      for (std::size_t b = 0; b < mem.block_count(); ++b) {
        const Block& mb = mem.block(b);
        const Block& eb = eng.mem().block(b);
        if (mb.alive && mb.loc.is_resident() && eb.loc.is_resident() && mb.loc.tier == TierId::PinnedHost &&
            eb.loc.tier == TierId::PagedHost)
          pf.moves.push_back(Move{b, TierId::PagedHost, TierId::PinnedHost, MoveKind::PrefetchToPinned});
      }
      if (!pf.moves.empty()) {
        eng.prefetch_begin(pf);
        eng.prefetch_wait();
        extra += "H " + std::to_string(k) + " " + std::to_string(pf.moves.size()) + "\n";
      }
      const ExecResult m = execute(plan, mem, hw, pc, now);  // the model (decisions, virtual clock)
      eng.execute(plan, pc);                                  // the bytes
      const auto& t = eng.lane_trace();
      for (int l = 0; l < 6; ++l)
        for (const LegTrace& x : t[l])
          lanes[l].push_back({x.block, static_cast<std::uint64_t>(x.src), static_cast<std::uint64_t>(x.dst)});
      std::uint64_t differ = 0;
      for (std::size_t b = 0; b < mem.block_count(); ++b)
        if (mem.block(b).alive && mem.block(b).loc.tier != eng.mem().block(b).loc.tier) ++differ;
      const SwitchStats& s = eng.last_stats();
      AppId incoming = kNoApp;
      for (const Move& mv : plan.moves)
        if (mv.kind == MoveKind::FetchForIncoming) {
          incoming = mem.block(mv.block).app;
          break;
        }
      extra += "M " + std::to_string(k) + " " + std::to_string(differ) + "\n";
      if (incoming != kNoApp)
        extra += "V " + std::to_string(k) + " " + std::to_string(incoming) + " " + std::to_string(eng.verify_pattern(incoming, seed)) +
                 " verified " + std::to_string(s.verified) + " unverified " + std::to_string(s.unverified) + "\n";
      ++k;
      return m.completion;
    };
    workload::Engine we(ws, model_mem, runner);
    const workload::Result r = we.run([&](AppId a, Bytes size, TierId tier) {
      model_mem.allocate(a, size, tier);
      eng.allocate(a, size, tier);
      eng.fill_pattern(a, seed);
    });
    std::string out = r.trace + extra;
    for (const workload::AppSpec& a : ws.apps)
      out += "F " + std::to_string(a.id) + " " + std::to_string(eng.verify_pattern(a.id, seed)) + "\n";
    *trace = dup_out(out, len);
  });
}

// ---- UVM model (include/nixie/uvm.hpp; reference proj/include/nixie/uvm.hpp) ----
struct nx_uvm {
  std::unique_ptr<UvmSim> sim;
};

int nx_uvm_create(uint64_t gpu_capacity, double pcie_up_bw, double pcie_down_bw, int half_duplex,
                  double fault_latency, int prefetch_pages, nx_uvm** out) {
  return guard([&] {
    need(out, "out");
    LinkConfig pcie{pcie_up_bw, pcie_down_bw, half_duplex ? Duplex::HalfDuplex : Duplex::FullDuplex};
    UvmConfig cfg;
    cfg.fault_latency = fault_latency;
    cfg.prefetch_pages = prefetch_pages;
    auto h = std::make_unique<nx_uvm>();
    h->sim = std::make_unique<UvmSim>(gpu_capacity, pcie, cfg);
    *out = h.release();
  });
}

int nx_uvm_register(nx_uvm* h, uint32_t app, uint64_t size) {
  return guard([&] {
    need(h, "uvm");
    h->sim->register_alloc(app, size);
  });
}

int nx_uvm_touch(nx_uvm* h, uint32_t app, double base_duration, double now, double* duration) {
  return guard([&] {
    need(h, "uvm");
    need(duration, "duration");
    *duration = h->sim->touch_kernel(app, h->sim->chunks_of(app), base_duration, now);
  });
}

int nx_uvm_stats(const nx_uvm* h, uint64_t* faults, uint64_t* faulted_bytes, uint64_t* mirror_peak) {
  return guard([&] {
    need(h, "uvm");
    if (faults) *faults = h->sim->fault_count();
    if (faulted_bytes) *faulted_bytes = h->sim->faulted_bytes_total();
    if (mirror_peak) *mirror_peak = h->sim->pinned_mirror_peak();
  });
}

void nx_uvm_destroy(nx_uvm* h) { delete h; }

void nx_free(void* p) { std::free(p); }

}  // extern "C"
