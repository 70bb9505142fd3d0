// Kernel-launch gate (include/nixie/swap_engine.hpp, LaunchGate).
//
// Paper protocol: (1) an app launches a kernel, (2) the
// shim checks the execution flag and, if the app is not granted, asks the
// daemon to schedule it and holds the launch, (3)-(5) the daemon pauses the
// incumbent, drains its kernels and migrates memory, (6) the app is granted
// and its launch proceeds.
//
// B200 version: the launching thread is held only until the switch that
// grants its app has SUBMITTED its last fetch (not until it completes); the
// app's stream then waits, on the device, for an event recorded right after
// that fetch. The app's kernel therefore starts the moment its data lands,
// without a host round trip. The event wait is enqueued after the work that
// completes it, so it cannot deadlock through a shared hardware queue (a
// value-wait enqueued before the producer can). The incumbent drain is
// likewise device-side: the engine's D2H stream waits for an event recorded
// on the incumbent's stream. Reference anchors: grant =
// MlfqScheduler::on_grant_start (proj/src/mlfq.cpp:188-194), drain = the
// eviction gate (proj/src/transfer.cpp:82-87, 126-129).
#include <cuda_runtime.h>

#include <chrono>
#include <condition_variable>
#include <map>
#include <mutex>

#include "nixie/swap_engine.hpp"
#include "phys.hpp"

namespace nixie::b200 {

struct LaunchGate::Impl {
  SwapEngine& eng;
  MlfqScheduler& sched;
  PlannerConfig cfg;
  std::mutex mu;  // guards the scheduler and the maps below
  std::condition_variable cv;
  std::map<AppId, cudaStream_t> streams;
  std::map<AppId, cudaEvent_t> landed;          // recorded after an app's last fetch
  std::map<AppId, std::uint64_t> released;      // swap-ins submitted (grant epochs)

  Impl(SwapEngine& e, MlfqScheduler& s, PlannerConfig c) : eng(e), sched(s), cfg(std::move(c)) {}
  ~Impl() {
    for (auto& kv : landed) cudaEventDestroy(kv.second);
  }

  static void on_release(void* ctx) {
    auto* p = static_cast<std::pair<Impl*, AppId>*>(ctx);
    {
      std::lock_guard<std::mutex> lk(p->first->mu);
      p->first->released[p->second] += 1;
    }
    p->first->cv.notify_all();
  }
};

LaunchGate::LaunchGate(SwapEngine& engine, MlfqScheduler& sched, PlannerConfig cfg)
    : impl_(std::make_unique<Impl>(engine, sched, std::move(cfg))) {}
LaunchGate::~LaunchGate() = default;

void LaunchGate::attach(AppId app, cudaStream_t stream) {
  Impl& g = *impl_;
  std::lock_guard<std::mutex> lk(g.mu);
  if (!g.landed.count(app)) {
    cudaEvent_t ev;
    NX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    g.landed[app] = ev;
    g.released[app] = 0;
  }
  g.streams[app] = stream;
}

bool LaunchGate::before_launch(AppId app, Seconds now, double timeout_s) {
  Impl& g = *impl_;
  std::unique_lock<std::mutex> lk(g.mu);
  auto it = g.streams.find(app);
  if (it == g.streams.end()) throw SimError(Err::UnknownApp, "launch gate: app " + std::to_string(app) + " not attached");
  g.sched.on_api_event(app, now, ApiEventKind::NonBlockingReturn);
  if (g.sched.granted() == app && g.eng.mem().app_fully_resident(app, TierId::Gpu)) return true;
  g.sched.enqueue_request(app, now);
  const std::uint64_t ticket = g.released[app];
  const bool ok = g.cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return g.released[app] > ticket; });
  if (!ok) throw SimError(Err::InvalidState, "launch gate: app " + std::to_string(app) + " was not scheduled within the timeout");
  NX_CUDA(cudaStreamWaitEvent(it->second, g.landed[app], 0));
  return false;
}

ExecResult LaunchGate::context_switch(AppId to, Seconds now) {
  Impl& g = *impl_;
  MigrationPlan plan;
  cudaStream_t drain = nullptr;
  GateRelease rel;
  std::pair<Impl*, AppId> ctx{&g, to};
  {
    std::lock_guard<std::mutex> lk(g.mu);
    if (!g.streams.count(to)) throw SimError(Err::UnknownApp, "launch gate: app " + std::to_string(to) + " not attached");
    const std::optional<AppId> incumbent = g.sched.granted();
    if (incumbent == to) return ExecResult{};
    if (incumbent) {
      g.sched.on_grant_end(*incumbent, now);  // pause: its next launches are held
      auto it = g.streams.find(*incumbent);
      if (it != g.streams.end()) drain = it->second;
    }
    g.cfg.eviction_policy.victim_order = g.sched.victim_hint();
    plan = plan_switch(to, g.eng.mem(), g.cfg);
    rel.event = g.landed[to];
    rel.callback = &Impl::on_release;
    rel.ctx = &ctx;
  }
  ExecResult r = g.eng.execute(plan, g.cfg, drain, &rel);
  std::lock_guard<std::mutex> lk(g.mu);
  g.sched.clear_request(to);
  g.sched.on_grant_start(to, now + r.completion);
  return r;
}

std::optional<AppId> LaunchGate::select_next(Seconds now) {
  std::lock_guard<std::mutex> lk(impl_->mu);
  return impl_->sched.select_next(now);
}

std::optional<AppId> LaunchGate::granted() {
  std::lock_guard<std::mutex> lk(impl_->mu);
  return impl_->sched.granted();
}

}  // namespace nixie::b200
