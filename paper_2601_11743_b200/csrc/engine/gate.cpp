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
// value-wait enqueued before the producer can). Check-and-launch is atomic
// w.r.t. a pause: before_launch returns holding the app's launch lock until
// after_launch, and a pause takes that lock before it records the drain event
// the evictions wait for (the shim's "blocks new launches and synchronizes
// outstanding kernels"). Reference anchors: grant =
// MlfqScheduler::on_grant_start (proj/src/mlfq.cpp:188-194), drain = the
// eviction gate (proj/src/transfer.cpp:82-87, 126-129), tick = SPEC.md:354.
#include <cuda_runtime.h>

#include <chrono>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>

#include "nixie/swap_engine.hpp"
#include "phys.hpp"

namespace nixie::b200 {

struct LaunchGate::Impl {
  SwapEngine& eng;
  MlfqScheduler& sched;
  PlannerConfig cfg;
  std::mutex switch_mu;  // one context switch at a time (the engine has a single control loop)
  std::mutex mu;         // guards the scheduler and the maps below; taken after a launch lock
  std::condition_variable cv;
  std::map<AppId, cudaStream_t> streams;
  std::map<AppId, cudaEvent_t> landed;                 // recorded after an app's last fetch
  std::map<AppId, cudaEvent_t> drained;                // recorded on the app's stream at pause
  std::map<AppId, std::uint64_t> released;             // swap-ins submitted (grant epochs)
  std::map<AppId, std::unique_ptr<std::mutex>> launch; // check-and-launch atomicity
  std::uint64_t switches = 0;
  AppId incoming = kNoApp;  // swap-in submitted, grant not yet recorded
  bool prefetch = false;

  Impl(SwapEngine& e, MlfqScheduler& s, PlannerConfig c) : eng(e), sched(s), cfg(std::move(c)) {}
  ~Impl() {
    for (auto& kv : landed) cudaEventDestroy(kv.second);
    for (auto& kv : drained) cudaEventDestroy(kv.second);
  }

  static void on_release(void* ctx) {
    auto* p = static_cast<std::pair<Impl*, AppId>*>(ctx);
    {
      std::lock_guard<std::mutex> lk(p->first->mu);
      p->first->released[p->second] += 1;
      p->first->incoming = p->second;
    }
    p->first->cv.notify_all();
  }

  std::mutex& launch_lock(AppId app) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = launch.find(app);
    if (it == launch.end()) throw SimError(Err::UnknownApp, "launch gate: app " + std::to_string(app) + " not attached");
    return *it->second;
  }
};

LaunchGate::LaunchGate(SwapEngine& engine, MlfqScheduler& sched, PlannerConfig cfg)
    : impl_(std::make_unique<Impl>(engine, sched, std::move(cfg))) {}
LaunchGate::~LaunchGate() = default;

void LaunchGate::attach(AppId app, cudaStream_t stream) {
  Impl& g = *impl_;
  std::lock_guard<std::mutex> lk(g.mu);
  if (!g.landed.count(app)) {
    cudaEvent_t a, b;
    NX_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    NX_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    g.landed[app] = a;
    g.drained[app] = b;
    g.released[app] = 0;
    g.launch[app] = std::make_unique<std::mutex>();
  }
  g.streams[app] = stream;
}

bool LaunchGate::before_launch(AppId app, Seconds now, double timeout_s) {
  Impl& g = *impl_;
  std::mutex& lmu = g.launch_lock(app);
  lmu.lock();  // held until after_launch: a pause cannot slip between check and launch
  try {
    std::unique_lock<std::mutex> lk(g.mu);
    g.sched.on_api_event(app, now, ApiEventKind::NonBlockingReturn);
    if (g.sched.granted() == app && g.eng.mem().app_fully_resident(app, TierId::Gpu)) return true;
    if (g.incoming == app) {  // its swap-in is submitted: order the launch after it lands
      NX_CUDA(cudaStreamWaitEvent(g.streams[app], g.landed[app], 0));
      return false;
    }
    g.sched.enqueue_request(app, now);
    const std::uint64_t ticket = g.released[app];
    const bool ok = g.cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return g.released[app] > ticket; });
    if (!ok) throw SimError(Err::InvalidState, "launch gate: app " + std::to_string(app) + " was not scheduled within the timeout");
    NX_CUDA(cudaStreamWaitEvent(g.streams[app], g.landed[app], 0));
    return false;
  } catch (...) {
    lmu.unlock();
    throw;
  }
}

void LaunchGate::after_launch(AppId app) { impl_->launch_lock(app).unlock(); }

void LaunchGate::api_event(AppId app, Seconds now, ApiEventKind kind) {
  std::lock_guard<std::mutex> lk(impl_->mu);
  impl_->sched.on_api_event(app, now, kind);
}

ExecResult LaunchGate::context_switch(AppId to, Seconds now) {
  Impl& g = *impl_;
  std::lock_guard<std::mutex> serial(g.switch_mu);
  MigrationPlan plan;
  GateRelease rel;
  std::pair<Impl*, AppId> ctx{&g, to};
  std::optional<AppId> incumbent;
  {
    std::lock_guard<std::mutex> lk(g.mu);
    if (!g.streams.count(to)) throw SimError(Err::UnknownApp, "launch gate: app " + std::to_string(to) + " not attached");
    incumbent = g.sched.granted();
    if (incumbent == to) return ExecResult{};
  }
  if (incumbent) {
    // Pause: no launch of the incumbent is in progress while its grant ends
    // and the drain point is recorded on its stream.
    std::lock_guard<std::mutex> launch_guard(g.launch_lock(*incumbent));
    std::lock_guard<std::mutex> lk(g.mu);
    g.sched.on_grant_end(*incumbent, now);
    auto it = g.streams.find(*incumbent);
    if (it != g.streams.end()) {
      NX_CUDA(cudaEventRecord(g.drained[*incumbent], it->second));
      for (int lane = 0; lane < 2; ++lane) NX_CUDA(cudaStreamWaitEvent(g.eng.stream(lane), g.drained[*incumbent], 0));
    }
  }
  {
    std::lock_guard<std::mutex> lk(g.mu);
    g.eng.prefetch_quiesce();  // cancel_pending + quiesced: plan_switch needs a quiescent registry
    g.cfg.eviction_policy.victim_order = g.sched.victim_hint();
    plan = plan_switch(to, g.eng.mem(), g.cfg);
    rel.event = g.landed[to];
    rel.callback = &Impl::on_release;
    rel.ctx = &ctx;
  }
  ExecResult r = g.eng.execute(plan, g.cfg, nullptr, &rel);
  std::lock_guard<std::mutex> lk(g.mu);
  g.sched.clear_request(to);
  g.sched.on_grant_start(to, now + r.completion);
  g.incoming = kNoApp;
  ++g.switches;
  return r;
}

// One scheduler tick (MlfqConfig::tick): Algorithm-1 inference
// for every app, then a switch to select_next() when the GPU has no holder,
// when the holder has gone idle (no API activity and not blocked in a call
// for > idle_threshold) while others wait, or when should_preempt fires.
std::optional<AppId> LaunchGate::tick(Seconds now) {
  Impl& g = *impl_;
  std::optional<AppId> next;
  {
    std::lock_guard<std::mutex> serial(g.switch_mu);
    std::lock_guard<std::mutex> lk(g.mu);
    g.sched.infer_all(now);
    next = g.sched.select_next(now);
    const std::optional<AppId> holder = g.sched.granted();
    const bool go = next && (!holder || g.sched.is_idle(*holder, now) || g.sched.should_preempt(*holder, now));
    if (!go) {
      if (g.prefetch && !g.eng.prefetch_pump()) {
        const std::optional<AppId> cand = g.sched.next_prefetch_candidate(now);
        if (cand && cand != holder) {
          const MigrationPlan pf = plan_prefetch(*cand, g.eng.mem(), g.cfg);
          if (!pf.moves.empty()) g.eng.prefetch_begin(pf);
        }
      }
      return std::nullopt;
    }
  }
  context_switch(*next, now);
  return next;
}

void LaunchGate::set_prefetch(bool on) {
  std::lock_guard<std::mutex> serial(impl_->switch_mu);
  impl_->prefetch = on;
  if (!on) {
    std::lock_guard<std::mutex> lk(impl_->mu);
    impl_->eng.prefetch_quiesce();
  }
}

Bytes LaunchGate::prefetched_bytes() const { return impl_->eng.prefetched_bytes(); }

std::optional<AppId> LaunchGate::select_next(Seconds now) {
  std::lock_guard<std::mutex> lk(impl_->mu);
  return impl_->sched.select_next(now);
}

std::optional<AppId> LaunchGate::granted() {
  std::lock_guard<std::mutex> lk(impl_->mu);
  return impl_->sched.granted();
}

std::uint64_t LaunchGate::switches() const { return impl_->switches; }

}  // namespace nixie::b200
