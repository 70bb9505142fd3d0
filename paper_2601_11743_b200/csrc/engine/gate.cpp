// Kernel-launch gate (include/nixie/swap_engine.hpp, LaunchGate).
//
// Paper protocol: (1) an app launches a kernel, (2) the
// shim checks the execution flag and, if the app is not granted, asks the
// daemon to schedule it, (3)-(5) the daemon pauses the incumbent, drains its
// kernels and migrates memory, (6) the app is granted and its launch
// proceeds. Here the "execution flag" is a per-app 64-bit gate word in device
// memory holding the app's grant epoch: an ungranted launch enqueues a
// device-side wait for epoch+1 on the app's stream, and the engine writes
// that epoch on its H2D stream right after the last fetch of the switch that
// grants the app. Reference anchors: grant = MlfqScheduler::on_grant_start
// (proj/src/mlfq.cpp:188-194), drain = the eviction gate
// (proj/src/transfer.cpp:82-87, 126-129).
#include <cuda_runtime.h>

#include <map>

#include "gate_ops.hpp"
#include "nixie/swap_engine.hpp"
#include "phys.hpp"

namespace nixie::b200 {

struct LaunchGate::Impl {
  SwapEngine& eng;
  MlfqScheduler& sched;
  PlannerConfig cfg;
  std::map<AppId, cudaStream_t> streams;
  std::map<AppId, std::size_t> slot;
  std::map<AppId, std::uint64_t> epoch;
  std::map<AppId, cudaEvent_t> landed;  // fallback gate (no stream memory ops)
  std::uint64_t* words = nullptr;
  std::size_t cap = 1024;
  bool memops = false;

  Impl(SwapEngine& e, MlfqScheduler& s, PlannerConfig c) : eng(e), sched(s), cfg(std::move(c)) {
    memops = gate_mem_ops_available();
    NX_CUDA(cudaMalloc(&words, sizeof(std::uint64_t) * cap));
    NX_CUDA(cudaMemset(words, 0, sizeof(std::uint64_t) * cap));
  }
  ~Impl() {
    for (auto& kv : landed) cudaEventDestroy(kv.second);
    cudaFree(words);
  }
};

LaunchGate::LaunchGate(SwapEngine& engine, MlfqScheduler& sched, PlannerConfig cfg)
    : impl_(std::make_unique<Impl>(engine, sched, std::move(cfg))) {}
LaunchGate::~LaunchGate() = default;

bool LaunchGate::stream_mem_ops() const { return impl_->memops; }

void LaunchGate::attach(AppId app, cudaStream_t stream) {
  Impl& g = *impl_;
  if (!g.slot.count(app)) {
    if (g.slot.size() == g.cap) throw SimError(Err::CapacityExceeded, "launch gate: too many apps");
    g.slot[app] = g.slot.size();
    g.epoch[app] = 0;
    cudaEvent_t ev;
    NX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    g.landed[app] = ev;
  }
  g.streams[app] = stream;
}

bool LaunchGate::before_launch(AppId app, Seconds now) {
  Impl& g = *impl_;
  auto it = g.streams.find(app);
  if (it == g.streams.end()) throw SimError(Err::UnknownApp, "launch gate: app " + std::to_string(app) + " not attached");
  g.sched.on_api_event(app, now, ApiEventKind::NonBlockingReturn);
  if (g.sched.granted() == app && g.eng.mem().app_fully_resident(app, TierId::Gpu)) return true;
  g.sched.enqueue_request(app, now);
  if (g.memops) {
    auto* word = g.words + g.slot[app];
    if (gate_wait_geq(reinterpret_cast<CUstream>(it->second), reinterpret_cast<CUdeviceptr>(word), g.epoch[app] + 1) !=
        CUDA_SUCCESS)
      throw SimError(Err::IoError, "cuStreamWaitValue64 failed");
  }
  return false;
}

ExecResult LaunchGate::context_switch(AppId to, Seconds now) {
  Impl& g = *impl_;
  if (!g.streams.count(to)) throw SimError(Err::UnknownApp, "launch gate: app " + std::to_string(to) + " not attached");
  const std::optional<AppId> incumbent = g.sched.granted();
  if (incumbent == to) return ExecResult{};
  cudaStream_t drain = nullptr;
  if (incumbent) {
    g.sched.on_grant_end(*incumbent, now);  // pause: its next launches are gated
    auto it = g.streams.find(*incumbent);
    if (it != g.streams.end()) drain = it->second;
  }
  g.cfg.eviction_policy.victim_order = g.sched.victim_hint();
  const MigrationPlan plan = plan_switch(to, g.eng.mem(), g.cfg);
  GateRelease rel;
  if (g.memops) {
    rel.device_word = g.words + g.slot[to];
    rel.value = g.epoch[to] + 1;
  } else {
    rel.event = g.landed[to];
  }
  ExecResult r = g.eng.execute(plan, g.cfg, drain, &rel);
  g.epoch[to] += 1;
  if (!g.memops) NX_CUDA(cudaStreamWaitEvent(g.streams[to], g.landed[to], 0));
  g.sched.clear_request(to);
  g.sched.on_grant_start(to, now + r.completion);
  return r;
}

}  // namespace nixie::b200
