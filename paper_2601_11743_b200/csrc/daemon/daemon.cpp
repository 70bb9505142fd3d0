// nixied — the Nixie daemon for unmodified CUDA applications (PAPER.md:114-116,
// "a centralized system service ... performs global coordination and
// enforces multiplexing policies").
//
// One daemon per GPU. It owns:
//   * the allocation registry (MemState, proj/src/mem_model.cpp) and the GPU
//     tier as a row of exportable VMM slabs (csrc/engine/vmm.hpp); each
//     application's shim imports the slabs it is handed and maps them under
//     the stable virtual range it reserved, one physical slab
//     per virtual slab that holds resident blocks (SlabPlacer);
//   * the MLFQ scheduler (proj/src/mlfq.cpp) fed from the shims' control
//     pages (launch counts, blocking calls: PAPER.md §6.1);
//   * the swap engine (csrc/engine/engine.cpp): a context switch is
//     plan_switch (proj/src/planner.cpp:111-216) executed with real copies,
//     both PCIe directions at once, every restore checksum-verified.
//
// A context switch (PAPER.md:116 steps 3-6):
//   Pause(incumbent)   its shim clears the execution flag, waits for
//                      launches in progress, synchronises its context,
//                      acks Drained
//   plan_switch        victim order = the scheduler's hint; victim blocks
//                      slab by slab (SlabPlacer::slab_victims)
//   execute            the swap engine: evictions and fetches at once; slabs
//                      newly assigned to the incoming app are mapped in its
//                      shim while the copies run (Map, from the progress hook)
//   Grant(incoming)    the remaining mapping changes; the shim applies them,
//                      sets the execution flag, acks Granted
//   after the grant    victims unmap the slabs they lost, unless stale
//                      mappings are kept (two apps, or --keep-stale-maps);
//                      grown slabs beyond the slack are dropped
// The daemon loop is single-threaded: every decision and
// registry mutation happens here, in arrival order.
#include <fcntl.h>
#include <poll.h>
#include <signal.h>
#include <sys/mman.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <deque>
#include <utility>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <optional>
#include <set>
#include <string>
#include <vector>

#include "nixie/swap_engine.hpp"
#include "nixie_ipc.hpp"
#include "slab_placer.hpp"

using namespace nixie;
using namespace nixie::b200;
namespace ipc = nixie::ipc;

namespace {

volatile sig_atomic_t g_stop = 0;
void on_signal(int) { g_stop = 1; }

struct Options {
  std::string socket_path = "/tmp/nixie.sock";
  std::string log_path;
  std::string trace_path;          // registry + plan trace for the reference replay (oracle/ref_replay.cpp)
  EngineConfig eng;
  PlannerConfig planner;
  MlfqConfig mlfq;
  Bytes min_bytes = kBlockBytes;  // smaller allocations pass through
  double ack_timeout_s = 60.0;
  int exit_after_apps = 0;         // exit once this many apps have come and gone (tests)
  int phys_slack_slabs = -1;       // physical slabs beyond the budget (partly resident slabs); -1: max(4, 2 GiB worth)
  std::uint32_t slab_blocks = 0;   // 0: 512 MiB for budgets >= 16 GiB, else 128 MiB
  bool prefetch = false;           // MLFQ prefetch of the next candidate
  bool reference_victims = false;  // the planner's own victim blocks instead of slab-aligned ones
  int keep_stale_maps = -1;        // victims keep mappings of lost slabs until their next Grant: 1 always, 0 never
                                   // (--isolate-victims), -1 while exactly two apps hold memory
};

Bytes parse_size(const char* s) {
  char* end = nullptr;
  const double v = std::strtod(s, &end);
  std::string u = end ? end : "";
  double mul = 1;
  if (u == "K" || u == "KiB") mul = 1024.0;
  else if (u == "M" || u == "MiB") mul = 1024.0 * 1024;
  else if (u == "G" || u == "GiB" || u.empty()) mul = 1024.0 * 1024 * 1024;
  return static_cast<Bytes>(v * mul);
}

void usage() {
  std::fprintf(stderr,
               "usage: nixied [--socket PATH] [--device N] [--gpu SIZE] [--pinned SIZE] [--paged SIZE]\n"
               "              [--window SIZE] [--min-bytes SIZE] [--path auto|ce|sm] [--host-threads N]\n"
               "              [--tick-ms X] [--idle-ms X] [--allot-s X] [--preempt-s X] [--log FILE] [--trace FILE]\n"
               "              [--phys-slack SLABS] [--slab-mib 2..1024, power of 2] [--prefetch] [--exit-after-apps N]\n              [--reference-victims] [--keep-stale-maps | --isolate-victims] [--pace-lag LEGS (-1: off)]\n"
               "sizes take a K/M/G suffix (GiB when bare). The daemon serves LD_PRELOAD=libnixie_shim.so apps\n"
               "that set NIXIE_SOCKET=PATH.\n");
}

bool parse_args(int argc, char** argv, Options& o) {
  o.eng.gpu_capacity = 32 * kGiB;
  o.eng.pinned_capacity = 16 * kGiB;
  o.eng.paged_capacity = 96 * kGiB;
  o.eng.path = CopyPath::CopyEngine;
  o.eng.exportable_arena = true;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&]() -> const char* {
      if (i + 1 >= argc) throw SimError(Err::ParseError, "missing value for " + a);
      return argv[++i];
    };
    if (a == "--socket") o.socket_path = val();
    else if (a == "--device") o.eng.device = std::atoi(val());
    else if (a == "--gpu") o.eng.gpu_capacity = parse_size(val()) / kBlockBytes * kBlockBytes;
    else if (a == "--pinned") o.eng.pinned_capacity = parse_size(val()) / kBlockBytes * kBlockBytes;
    else if (a == "--paged") o.eng.paged_capacity = parse_size(val()) / kBlockBytes * kBlockBytes;
    else if (a == "--window") o.planner.streaming_window = parse_size(val());
    else if (a == "--min-bytes") o.min_bytes = parse_size(val());
    else if (a == "--host-threads") o.eng.host_threads = std::atoi(val());
    else if (a == "--tick-ms") o.mlfq.tick = std::atof(val()) / 1000.0;
    else if (a == "--idle-ms") o.mlfq.idle_threshold = std::atof(val()) / 1000.0;
    else if (a == "--allot-s") o.mlfq.base_allotment = std::atof(val());
    else if (a == "--preempt-s") o.mlfq.base_preemption = std::atof(val());
    else if (a == "--log") o.log_path = val();
    else if (a == "--trace") o.trace_path = val();
    else if (a == "--exit-after-apps") o.exit_after_apps = std::atoi(val());
    else if (a == "--phys-slack") o.phys_slack_slabs = std::atoi(val());
    else if (a == "--slab-mib") {
      // Validated as given (a truncating division would turn 1 into "default" and 3 into 2).
      char* end = nullptr;
      const char* v = val();
      const long mib = std::strtol(v, &end, 10);
      if (!end || *end != 0 || mib < 2 || mib > 1024 || (mib & (mib - 1)) != 0)
        throw SimError(Err::ValidationError, std::string("--slab-mib must be a power of two between 2 and 1024, got ") + v);
      o.slab_blocks = static_cast<std::uint32_t>(mib / 2);
    }
    else if (a == "--prefetch") o.prefetch = true;
    else if (a == "--pace-lag") {
      char* end = nullptr;
      const char* v = val();
      const long lag = std::strtol(v, &end, 10);
      if (!end || *end != 0 || lag < -1) throw SimError(Err::ValidationError, std::string("--pace-lag must be >= -1, got ") + v);
      o.eng.pace_lag_legs = static_cast<int>(lag);
    }
    else if (a == "--reference-victims") o.reference_victims = true;
    else if (a == "--keep-stale-maps") o.keep_stale_maps = 1;
    else if (a == "--isolate-victims") o.keep_stale_maps = 0;
    else if (a == "--path") {
      const std::string p = val();
      o.eng.path = p == "sm" ? CopyPath::SmKernel : p == "auto" ? CopyPath::Auto : CopyPath::CopyEngine;
    } else if (a == "-h" || a == "--help") {
      usage();
      std::exit(0);
    } else {
      usage();
      return false;
    }
  }
  o.mlfq.validate();
  // Larger slabs mean fewer driver mappings per switch (each costs ~1 ms
  // whatever its size); smaller ones waste less physical memory on partly
  // resident slabs, which matters on small budgets.
  if (o.slab_blocks == 0) o.slab_blocks = o.eng.gpu_capacity >= 16 * kGiB ? ipc::kDefaultSlabBlocks : 64;
  if (o.slab_blocks < 1 || (o.slab_blocks & (o.slab_blocks - 1)) != 0 || o.slab_blocks > 512)
    throw SimError(Err::ValidationError, "--slab-mib must be a power of two between 2 and 1024");
  const Bytes slab = static_cast<Bytes>(o.slab_blocks) * kBlockBytes;
  if (o.phys_slack_slabs < 0) o.phys_slack_slabs = static_cast<int>(std::max<Bytes>(4, 2 * kGiB / slab));  // 2 GiB
  o.eng.arena_slab_bytes = slab;
  o.eng.gpu_physical = (o.eng.gpu_capacity + slab - 1) / slab * slab + static_cast<Bytes>(std::max(o.phys_slack_slabs, 0)) * slab;
  o.eng.gpu_physical_max = 2 * o.eng.gpu_physical;  // room to grow when partly resident slabs use up the slack
  return true;
}

class Daemon {
 public:
  explicit Daemon(const Options& o)
      : opt_(o), eng_(o.eng), sched_(o.mlfq), placer_(eng_.arena_frames() / o.slab_blocks, o.slab_blocks) {
    eng_.set_frame_placer(&placer_);
    placer_.set_grow([this] { return grow_arena(); });
    if (!o.reference_victims)
      victims_ = [this](const MemState& st, const std::vector<AppId>& order, Bytes want) {
        return placer_.slab_victims(st, order, want);
      };
    eng_.set_progress_hook([this] { send_maps(); });
    sched_.set_logging(true);
    t0_ = ipc::mono_ns();
    if (!o.log_path.empty()) {
      log_ = std::fopen(o.log_path.c_str(), "w");
      if (!log_) throw SimError(Err::IoError, "cannot open log " + o.log_path);
    }
    if (!o.trace_path.empty()) {
      trace_ = std::fopen(o.trace_path.c_str(), "w");
      if (!trace_) throw SimError(Err::IoError, "cannot open trace " + o.trace_path);
      trace_header();
    }
  }
  ~Daemon() {
    for (auto& [id, a] : apps_) close_app(a);
    for (int fd : pending_) ::close(fd);
    if (listen_fd_ >= 0) ::close(listen_fd_);
    ::unlink(opt_.socket_path.c_str());
    if (log_) std::fclose(log_);
    if (trace_) std::fclose(trace_);
  }

  void listen_on() {
    listen_fd_ = ::socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    sockaddr_un addr{};
    addr.sun_family = AF_UNIX;
    if (opt_.socket_path.size() >= sizeof(addr.sun_path)) throw SimError(Err::ValidationError, "socket path too long");
    std::strcpy(addr.sun_path, opt_.socket_path.c_str());
    ::unlink(opt_.socket_path.c_str());
    if (::bind(listen_fd_, reinterpret_cast<sockaddr*>(&addr), sizeof(addr)) != 0 || ::listen(listen_fd_, 64) != 0)
      throw SimError(Err::IoError, "cannot listen on " + opt_.socket_path + ": " + std::strerror(errno));
    std::fprintf(stderr, "[nixied] listening on %s  gpu %.1f GiB (physical %.1f GiB)  pinned %.1f GiB  path %s\n",
                 opt_.socket_path.c_str(), double(opt_.eng.gpu_capacity) / kGiB, double(opt_.eng.gpu_physical) / kGiB,
                 double(opt_.eng.pinned_capacity) / kGiB,
                 opt_.eng.path == CopyPath::SmKernel ? "sm" : opt_.eng.path == CopyPath::Auto ? "auto" : "ce");
    std::fflush(stderr);
  }

  int run() {
    Seconds next_tick = now() + opt_.mlfq.tick;
    while (!g_stop) {
      std::vector<pollfd> fds;
      fds.push_back({listen_fd_, POLLIN, 0});
      for (int fd : pending_) fds.push_back({fd, POLLIN, 0});
      for (auto& [id, a] : apps_) {
        if (!a.alive) continue;
        fds.push_back({a.rpc, POLLIN, 0});
        if (a.ev >= 0) fds.push_back({a.ev, POLLIN, 0});
      }
      const int wait_ms = std::max(0, static_cast<int>((next_tick - now()) * 1000.0));
      const int n = ::poll(fds.data(), fds.size(), wait_ms);
      if (n < 0 && errno != EINTR) throw SimError(Err::IoError, std::string("poll: ") + std::strerror(errno));
      if (n > 0) {
        for (const pollfd& p : fds) {
          if (!p.revents) continue;
          if (p.fd == listen_fd_) {
            const int c = ::accept4(listen_fd_, nullptr, nullptr, SOCK_CLOEXEC);
            if (c >= 0) pending_.push_back(c);
          } else if (std::find(pending_.begin(), pending_.end(), p.fd) != pending_.end()) {
            on_pending(p.fd);
          } else {
            on_app_fd(p.fd);
          }
        }
      }
      reap();
      if (now() >= next_tick) {
        tick();
        next_tick = now() + opt_.mlfq.tick;
      }
      if (opt_.exit_after_apps > 0 && gone_ >= opt_.exit_after_apps && live_apps() == 0) break;
    }
    write_summary();
    return 0;
  }

 private:
  struct App {
    AppId id = 0;
    int rpc = -1, ev = -1;
    int pid = 0;
    std::string name;
    int ctl_fd = -1;
    ipc::CtlPage* ctl = nullptr;
    bool alive = true;
    std::uint64_t seen_launches = 0;
    bool seen_blocking = false;
    std::uint64_t active_launch_mark = 0;
    std::vector<std::uint32_t> gen_rpc, gen_ev;  // slab generation whose descriptor each socket carried (0: none)
  };

  Seconds now() const { return static_cast<double>(ipc::mono_ns() - t0_) * 1e-9; }
  Seconds to_daemon_time(std::uint64_t ns) const { return ns > t0_ ? static_cast<double>(ns - t0_) * 1e-9 : 0.0; }

  int live_apps() const {
    int n = 0;
    for (const auto& kv : apps_) n += kv.second.alive ? 1 : 0;
    return n;
  }

  void close_app(App& a) {
    if (a.rpc >= 0) ::close(a.rpc);
    if (a.ev >= 0) ::close(a.ev);
    if (a.ctl) ::munmap(a.ctl, 4096);
    if (a.ctl_fd >= 0) ::close(a.ctl_fd);
    a.rpc = a.ev = a.ctl_fd = -1;
    a.ctl = nullptr;
  }

  App* app_by_fd(int fd) {
    for (auto& [id, a] : apps_)
      if (a.alive && (a.rpc == fd || a.ev == fd)) return &a;
    return nullptr;
  }

  // ---- connections ---------------------------------------------------------
  void on_pending(int fd) {
    pending_.erase(std::find(pending_.begin(), pending_.end(), fd));
    ipc::Msg type;
    std::vector<std::uint8_t> body;
    if (!ipc::recv_msg(fd, type, body)) {
      ::close(fd);
      return;
    }
    ipc::Reader r{body};
    if (type == ipc::Msg::Hello) {
      const auto req = r.get<ipc::HelloReq>();
      if (!r.ok) {
        ::close(fd);
        return;
      }
      hello(fd, req);
    } else if (type == ipc::Msg::EventHello) {
      const auto req = r.get<ipc::EventHelloReq>();
      auto it = apps_.find(req.app);
      if (!r.ok || it == apps_.end() || it->second.ev >= 0) {
        ::close(fd);
        return;
      }
      it->second.ev = fd;
    } else {
      ::close(fd);
    }
  }

  void hello(int fd, const ipc::HelloReq& req) {
    App a;
    a.id = next_app_++;
    a.rpc = fd;
    a.pid = req.pid;
    a.name.assign(req.name, strnlen(req.name, sizeof(req.name)));
    a.ctl_fd = ::memfd_create("nixie-ctl", MFD_CLOEXEC);
    if (a.ctl_fd < 0 || ::ftruncate(a.ctl_fd, 4096) != 0) throw SimError(Err::IoError, "memfd_create for the control page");
    void* p = ::mmap(nullptr, 4096, PROT_READ | PROT_WRITE, MAP_SHARED, a.ctl_fd, 0);
    if (p == MAP_FAILED) throw SimError(Err::IoError, "mmap control page");
    a.ctl = new (p) ipc::CtlPage();
    sched_.register_app(a.id, now());
    ipc::HelloRep rep{};
    rep.status = req.device == opt_.eng.device ? 0 : 1;
    rep.app = a.id;
    rep.gpu_budget = opt_.eng.gpu_capacity;
    rep.block_bytes = kBlockBytes;
    rep.min_bytes = opt_.min_bytes;
    rep.device = opt_.eng.device;
    const std::uint32_t slabs = placer_.base();  // grown slabs follow lazily (send_new_slabs)
    rep.slabs = slabs;
    rep.slab_bytes = static_cast<std::uint64_t>(opt_.slab_blocks) * kBlockBytes;
    rep.arena_bytes = rep.slabs * rep.slab_bytes;
    bool ok = ipc::send_msg(fd, ipc::Msg::Hello, &rep, sizeof(rep)) && ipc::send_fds(fd, &a.ctl_fd, 1);
    std::vector<int> batch;
    for (std::uint32_t f = 0; f < slabs && ok; f += ipc::kFdBatch) {
      const std::uint32_t n = std::min<std::uint32_t>(ipc::kFdBatch, slabs - f);
      batch.clear();
      for (std::uint32_t k = 0; k < n; ++k) batch.push_back(eng_.arena_export_fd(f + k));
      ok = ipc::send_fds(fd, batch.data(), static_cast<int>(n));
      for (int x : batch) ::close(x);
    }
    a.gen_rpc.assign(slabs, 1);  // imported at start-up, before the listener runs
    a.gen_ev = a.gen_rpc;
    apps_[a.id] = a;
    if (!ok) apps_[a.id].alive = false;
    note("{\"t\": %.6f, \"event\": \"hello\", \"app\": %u, \"pid\": %d, \"name\": \"%s\"}", now(), a.id, a.pid, a.name.c_str());
  }

  void on_app_fd(int fd) {
    App* a = app_by_fd(fd);
    if (!a) return;
    ipc::Msg type;
    std::vector<std::uint8_t> body;
    if (!ipc::recv_msg(fd, type, body)) {
      a->alive = false;  // reaped below
      return;
    }
    if (fd == a->ev) {  // unsolicited event-socket traffic outside a switch: protocol error
      a->alive = false;
      return;
    }
    serve(*a, type, body);
  }

  void serve(App& app, ipc::Msg type, const std::vector<std::uint8_t>& body) {
    App* a = &app;
    try {
      rpc(*a, type, body);
    } catch (const InvariantViolation&) {
      throw;
    } catch (const std::exception& e) {
      // The request failed (e.g. a tier is full): answer with the reply type
      // the shim waits for, carrying an error status (cudaMalloc then
      // returns cudaErrorMemoryAllocation).
      std::fprintf(stderr, "[nixied] app %u: %s\n", a->id, e.what());
      const auto* se = dynamic_cast<const SimError*>(&e);
      const std::int32_t code = 100 + (se ? static_cast<std::int32_t>(se->code()) : 0);
      if (type == ipc::Msg::Alloc) {
        ipc::AllocRep rep{};
        rep.status = code;
        rep.epoch = ++epoch_;
        ipc::send_msg(a->rpc, ipc::Msg::Alloc, &rep, sizeof(rep));
      } else if (type == ipc::Msg::Free) {
        ipc::FreeRep rep{code, 0, ++epoch_};
        ipc::send_msg(a->rpc, ipc::Msg::Free, &rep, sizeof(rep));
      } else {
        ipc::StatusRep st{code, 0};
        ipc::send_msg(a->rpc, type == ipc::Msg::Stats ? ipc::Msg::Stats : ipc::Msg::Status, &st, sizeof(st));
      }
    }
  }

  // Apps whose sockets closed: their memory returns to the registry.
  void reap() {
    for (auto& [id, a] : apps_) {
      if (a.alive || a.rpc < 0) continue;
      if (sched_.granted() == id) sched_.on_grant_end(id, now());
      sched_.clear_request(id);
      eng_.prefetch_quiesce();
      const std::vector<ChunkId> chunks = eng_.mem().chunks_of(id);
      for (ChunkId c : chunks) {
        eng_.free_chunk(id, c);
        trace_free(id, c);
      }
      placer_.take_released();  // its slabs return to the pool; nobody to unmap them
      std::uint64_t launches = 0, table = 0, blas = 0, waits = 0, wait_ns = 0, drain_ns = 0, map_ns = 0;
      std::uint64_t small = 0, implicit = 0, captured = 0;
      if (a.ctl) {
        launches = a.ctl->launches.load();
        table = a.ctl->table_launches.load();
        blas = a.ctl->blas_calls.load();
        waits = a.ctl->gate_waits.load();
        wait_ns = a.ctl->gate_wait_ns.load();
        drain_ns = a.ctl->drain_ns.load();
        map_ns = a.ctl->map_ns.load();
        small = a.ctl->small_bytes.load();
        implicit = a.ctl->implicit_bytes.load();
        captured = a.ctl->captured_launches.load();
      }
      close_app(a);
      ++gone_;
      note("{\"t\": %.6f, \"event\": \"bye\", \"app\": %u, \"chunks_freed\": %zu, \"gated_calls\": %" PRIu64
           ", \"table_launches\": %" PRIu64 ", \"blas_calls\": %" PRIu64 ", \"gate_waits\": %" PRIu64 ", \"gate_wait_ms\": %.3f, \"drain_ms\": %.3f"
           ", \"map_ms\": %.3f, \"small_bytes\": %" PRIu64 ", \"implicit_bytes\": %" PRIu64 ", \"captured_launches\": %" PRIu64 "}",
           now(), id, chunks.size(), launches, table, blas, waits, wait_ns * 1e-6, drain_ns * 1e-6, map_ns * 1e-6, small, implicit,
           captured);
    }
  }

  // ---- requests --------------------------------------------------------------
  void rpc(App& a, ipc::Msg type, const std::vector<std::uint8_t>& body) {
    ipc::Reader r{body};
    if (type == ipc::Msg::Alloc || type == ipc::Msg::Free) eng_.prefetch_quiesce();  // registry changes: no legs in flight
    switch (type) {
      case ipc::Msg::Alloc: {
        const auto req = r.get<ipc::AllocReq>();
        alloc(a, req.bytes, req.va_block);
        break;
      }
      case ipc::Msg::Free: {
        const auto n = r.get<std::uint32_t>();
        int status = 0;
        for (std::uint32_t i = 0; i < n && r.ok; ++i) {
          const auto c = r.get<std::uint32_t>();
          try {
            eng_.free_chunk(a.id, c);
            trace_free(a.id, c);
          } catch (const SimError&) {
            status = 1;
          }
        }
        // Slabs the free emptied: the shim unmaps them (its reply carries them).
        std::vector<std::uint32_t> mine;
        for (const auto& k : placer_.take_released()) {
          if (k.first != a.id) throw InvariantViolation("free released another app's slab");
          mine.push_back(k.second);
          placer_.set_mapped(k, ipc::kNoFrame);
        }
        ipc::FreeRep rep{status, static_cast<std::uint32_t>(mine.size()), ++epoch_};
        ipc::Writer w;
        w.put(rep);
        w.put_u32s(mine);
        ipc::send_msg(a.rpc, ipc::Msg::Free, w.buf);
        break;
      }
      case ipc::Msg::Acquire: {
        ipc::StatusRep st{0, 0};
        ipc::send_msg(a.rpc, ipc::Msg::Status, &st, sizeof(st));
        if (sched_.granted() != a.id) {
          sched_.enqueue_request(a.id, now());
          decide(now());
        }
        break;
      }
      case ipc::Msg::Stats: {
        ipc::StatsRep s{switches_, bytes_in_, bytes_out_, mismatches_, verified_};
        ipc::send_msg(a.rpc, ipc::Msg::Stats, &s, sizeof(s));
        break;
      }
      default:
        a.alive = false;
    }
  }

  // Device memory an app holds outside the registry: passthrough allocations
  // below min_bytes and what implicitly allocating APIs took (shim control page).
  static Bytes unmanaged(const App& a) {
    return a.ctl ? a.ctl->small_bytes.load(std::memory_order_relaxed) + a.ctl->implicit_bytes.load(std::memory_order_relaxed) : 0;
  }

  // cudaMalloc >= min_bytes (MemState::allocate, proj/src/mem_model.cpp:48-86).
  // Placement: the GPU when it has room; otherwise the holder's allocation
  // is brought in by an in-place plan (other apps' blocks are evicted), and
  // a waiting app's allocation starts in pageable memory (its next grant
  // fetches it). An app's footprint may not exceed the GPU budget
  // (the planner's precondition), counting the app's
  // unmanaged device memory too (implicit allocations count).
  void alloc(App& a, Bytes bytes, std::uint64_t va_block) {
    MemState& mem = eng_.mem();
    const Bytes fp = footprint_for(bytes);
    ipc::AllocRep rep{};
    if (bytes == 0 || mem.app_footprint(a.id) + fp + unmanaged(a) > opt_.eng.gpu_capacity) {
      rep.status = 2;
      ipc::send_msg(a.rpc, ipc::Msg::Alloc, &rep, sizeof(rep));
      return;
    }
    const bool holder = sched_.granted() == a.id;
    TierId tier = TierId::Gpu;
    if (mem.tier(TierId::Gpu).free_bytes() < fp) {
      tier = mem.tier(TierId::PagedHost).free_bytes() >= fp ? TierId::PagedHost : TierId::PinnedHost;
      if (mem.tier(tier).free_bytes() < fp) {
        rep.status = 2;
        ipc::send_msg(a.rpc, ipc::Msg::Alloc, &rep, sizeof(rep));
        return;
      }
    }
    const std::uint64_t nblk = fp / kBlockBytes;
    placer_.expect(mem.block_count(), nblk, a.id, va_block);
    const std::vector<ChunkId> chunks = eng_.allocate(a.id, bytes, tier);
    trace_alloc(a.id, bytes, tier, chunks);
    if (holder && tier != TierId::Gpu) fetch_in_place(a.id);
    std::vector<std::uint32_t> ids;
    for (ChunkId c : chunks) ids.push_back(static_cast<std::uint32_t>(c));
    std::vector<ipc::SlabMap> slabs;
    for (std::uint64_t v = va_block / opt_.slab_blocks; v <= (va_block + nblk - 1) / opt_.slab_blocks; ++v) {
      slabs.push_back(placer_.map_of(a.id, static_cast<std::uint32_t>(v)));
      placer_.set_mapped({a.id, static_cast<std::uint32_t>(v)}, slabs.back().phys);
    }
    rep.n_chunks = static_cast<std::uint32_t>(ids.size());
    rep.n_slabs = static_cast<std::uint32_t>(slabs.size());
    rep.footprint = fp;
    send_new_slabs(a, true);
    rep.epoch = ++epoch_;
    ipc::Writer w;
    w.put(rep);
    w.put_u32s(ids);
    for (const auto& m : slabs) w.put(m);
    ipc::send_msg(a.rpc, ipc::Msg::Alloc, w.buf);
  }

  // ---- activity (the shims' control pages) -> MLFQ inputs ---------------------
  void poll_activity(Seconds t, Seconds dt) {
    for (auto& [id, a] : apps_) {
      if (!a.alive || !a.ctl) continue;
      const std::uint64_t launches = a.ctl->launches.load(std::memory_order_acquire);
      const bool blocking = a.ctl->blocking.load(std::memory_order_acquire) > 0;
      const Seconds t_api = std::min(t, to_daemon_time(a.ctl->last_api_ns.load(std::memory_order_acquire)));
      const Seconds t_blk = std::min(t, to_daemon_time(a.ctl->last_block_ns.load(std::memory_order_acquire)));
      if (blocking && !a.seen_blocking) sched_.on_api_event(id, t_blk, ApiEventKind::BlockingEnter);
      if (!blocking && a.seen_blocking) sched_.on_api_event(id, t_blk, ApiEventKind::BlockingExit);
      if (launches != a.seen_launches) sched_.on_api_event(id, t_api, ApiEventKind::NonBlockingReturn);
      // The holder's busy time drives demotion (t_a in Algorithm 1).
      if (dt > 0 && sched_.granted() == id && (blocking || launches != a.active_launch_mark)) sched_.add_execution(id, dt);
      a.active_launch_mark = launches;
      a.seen_launches = launches;
      a.seen_blocking = blocking;
    }
  }

  void tick() {
    const Seconds t = now();
    poll_activity(t, last_tick_ > 0 ? t - last_tick_ : 0.0);
    last_tick_ = t;
    decide(t);
  }

  // SPEC.md:354 tick rule (as LaunchGate::tick): switch to select_next() when
  // nobody holds the GPU, when the holder has gone idle, or when
  // should_preempt fires.
  void decide(Seconds t) {
    poll_activity(t, 0.0);
    sched_.infer_all(t);
    const std::optional<AppId> next = sched_.select_next(t);
    const std::optional<AppId> holder = sched_.granted();
    const bool go = next && (!holder || sched_.is_idle(*holder, t) || sched_.should_preempt(*holder, t));
    if (go) {
      context_switch(*next, t);
      return;
    }
    if (opt_.prefetch && !eng_.prefetch_pump()) {  // the queue head is likely next
      const std::optional<AppId> cand = sched_.next_prefetch_candidate(t);
      if (cand && cand != holder) {
        const MigrationPlan pf = plan_prefetch(*cand, eng_.mem(), opt_.planner);
        if (!pf.moves.empty()) {
          trace_prefetch(*cand, pf);
          eng_.prefetch_begin(pf);
          note("{\"t\": %.6f, \"event\": \"prefetch\", \"app\": %u, \"moves\": %zu}", t, *cand, pf.moves.size());
        }
      }
    }
  }

  // ---- acks on the event socket ------------------------------------------------
  // The shim acks from its listener thread while the application's own
  // threads keep running: one of them may be inside cudaMalloc during a
  // stream capture, which the pause waits out, so its Alloc/Free RPCs are
  // served while the ack is awaited (otherwise both sides wait on each other
  // until the ack timeout). An Acquire is answered and queued for after the
  // switch (no scheduling decision inside a switch).
  bool wait_ack(App& a, ipc::Msg want, std::vector<std::uint8_t>& body) {
    if (!a.alive || a.ev < 0) return false;
    const std::uint64_t deadline = ipc::mono_ns() + static_cast<std::uint64_t>(opt_.ack_timeout_s * 1e9);
    ipc::Msg type;
    while (a.alive) {
      const std::uint64_t t = ipc::mono_ns();
      if (t >= deadline) break;
      pollfd p[2] = {{a.ev, POLLIN, 0}, {a.rpc, POLLIN, 0}};
      const int n = ::poll(p, 2, static_cast<int>(std::min<std::uint64_t>((deadline - t) / 1000000 + 1, 1000)));
      if (n < 0 && errno != EINTR) break;
      if (n <= 0) continue;
      if (p[0].revents) {
        if (!ipc::recv_msg(a.ev, type, body) || type != want) break;
        return true;
      }
      if (p[1].revents) {
        std::vector<std::uint8_t> req;
        if (!ipc::recv_msg(a.rpc, type, req)) break;
        if (type == ipc::Msg::Acquire) {
          ipc::StatusRep st{0, 0};
          ipc::send_msg(a.rpc, ipc::Msg::Status, &st, sizeof(st));
          deferred_acquires_.push_back(a.id);
        } else {
          ++rpcs_in_switch_;
          note("{\"t\": %.6f, \"event\": \"rpc_in_switch\", \"app\": %u, \"type\": \"%s\"}", now(), a.id,
               type == ipc::Msg::Alloc ? "alloc" : type == ipc::Msg::Free ? "free" : "other");
          serve(a, type, req);
        }
      }
    }
    std::fprintf(stderr, "[nixied] app %u: no %u ack (dropping the app)\n", a.id, static_cast<unsigned>(want));
    a.alive = false;
    return false;
  }

  // Acquires that arrived during a switch: queued now (decided at the next tick).
  void take_deferred_acquires() {
    for (AppId id : deferred_acquires_) {
      auto it = apps_.find(id);
      if (it != apps_.end() && it->second.alive && sched_.granted() != id) sched_.enqueue_request(id, now());
    }
    deferred_acquires_.clear();
  }

  // While a plan runs: the incoming app maps the slabs its blocks are landing
  // in (it cannot launch until the Grant, so the bytes need not be there yet),
  // and victims drop released ones, overlapping the driver's per-mapping
  // cost with the copies. A slab is reassigned only after its release, and
  // every message to one shim is ordered on its event socket.
  void send_maps() {
    std::map<AppId, std::vector<ipc::SlabMap>> per_app;
    for (const auto& k : placer_.take_assigned()) {
      const ipc::SlabMap m = placer_.map_of(k.first, k.second);
      if (m.phys == ipc::kNoFrame || placer_.mapped(k) == m.phys) continue;  // already mapped there (affinity)
      placer_.set_mapped(k, m.phys);
      per_app[k.first].push_back(m);
    }
    // A vslab that lost its slab keeps its (stale) mapping for now: its owner
    // cannot run before its next Grant. cuMemUnmap while the copy engines
    // move data costs up to ~80 ms per slab on these hosts (it waits on the
    // GPU), so the owners drop their stale mappings after the switch, when
    // the link is quiet (flush_unmaps).
    for (const auto& k : placer_.take_released()) stale_.insert(k);
    for (auto& [app, ms] : per_app) {
      auto it = apps_.find(app);
      if (it == apps_.end() || !it->second.alive || it->second.ev < 0) continue;
      send_new_slabs(it->second, false);
      ipc::Writer w;
      w.put(ipc::SlabsMsg{++epoch_, static_cast<std::uint32_t>(ms.size()), 0});
      for (const auto& m : ms) w.put(m);
      if (!ipc::send_msg(it->second.ev, ipc::Msg::Map, w.buf)) it->second.alive = false;
    }
  }

  // A new physical slab when partly resident slabs used up the slack. Shims
  // learn about it lazily: before any message on a socket that may name it
  // (send_new_slabs), so each socket delivers the descriptor first.
  std::uint32_t grow_arena() {
    const std::uint32_t s = eng_.arena_grow_slab();
    placer_.revive(s);
    note("{\"t\": %.6f, \"event\": \"slab_grow\", \"slab\": %u, \"partial_slabs\": %" PRIu64 "}", now(), s, placer_.partial());
    return s;
  }

  // Sends the app every live slab generation it has not received on this
  // socket yet (Slab message + descriptor each).
  void send_new_slabs(App& a, bool on_rpc) {
    std::vector<std::uint32_t>& known = on_rpc ? a.gen_rpc : a.gen_ev;
    const int sock = on_rpc ? a.rpc : a.ev;
    if (known.size() < placer_.slabs()) known.resize(placer_.slabs(), 0);
    for (std::uint32_t f = 0; f < placer_.slabs() && a.alive && sock >= 0; ++f) {
      if (placer_.dropped(f) || known[f] == placer_.gen(f)) continue;
      const int fd = eng_.arena_export_fd(f);
      ipc::SlabFdMsg m{f, placer_.gen(f)};
      const bool ok = ipc::send_msg(sock, ipc::Msg::Slab, &m, sizeof(m)) && ipc::send_fds(sock, &fd, 1);
      ::close(fd);
      if (!ok) a.alive = false;
      known[f] = placer_.gen(f);
    }
  }

  // Between switches: grown slabs beyond the slack that no block uses are
  // released again, in the daemon and in every shim that imported them, so
  // physical use returns to budget + slack (growth is only transient).
  void shrink_arena() {
    const std::vector<std::uint32_t> drop = placer_.take_droppable(static_cast<std::size_t>(opt_.phys_slack_slabs));
    for (std::uint32_t f : drop) {
      const std::uint32_t gen = placer_.gen(f);
      eng_.arena_drop_slab(f);
      for (auto& [id, a] : apps_) {
        const bool has = (f < a.gen_ev.size() && a.gen_ev[f] == gen) || (f < a.gen_rpc.size() && a.gen_rpc[f] == gen);
        if (f < a.gen_ev.size()) a.gen_ev[f] = 0;
        if (f < a.gen_rpc.size()) a.gen_rpc[f] = 0;
        if (!has || !a.alive || a.ev < 0) continue;
        ipc::DropMsg m{++epoch_, f, gen};
        if (!ipc::send_msg(a.ev, ipc::Msg::Drop, &m, sizeof(m))) a.alive = false;
      }
      note("{\"t\": %.6f, \"event\": \"slab_drop\", \"slab\": %u}", now(), f);
    }
  }

  // After a switch: victims unmap the slabs they lost, off the critical path.
  // A vslab that got a slab back meanwhile is skipped (mapped there again).
  // A paused victim may keep mapping slabs another app now uses (its next
  // Grant remaps what changed), so a vslab that gets its old slab back costs
  // no driver call. Nixie's threat model is one user's applications, which
  // already share the pinned pool. That pays off when two
  // apps alternate: the descending eviction order (plan_moves) hands every
  // vslab its old slab back. With more apps the slabs rotate, a kept mapping
  // must be unmapped during a later switch, and cuMemUnmap then waits on the
  // copies (up to 600 ms per switch in config 3, measured), so by default
  // stale mappings are kept only while exactly two apps hold memory.
  bool keep_stale() const {
    return opt_.keep_stale_maps > 0 || (opt_.keep_stale_maps < 0 && eng_.mem().apps().size() == 2);
  }

  void flush_unmaps() {
    if (keep_stale()) return;  // kept in stale_: unmapped if a third app arrives
    std::map<AppId, std::vector<std::uint32_t>> per_app;
    for (const auto& k : stale_) {
      if (placer_.map_of(k.first, k.second).phys != ipc::kNoFrame) continue;  // backed again
      if (placer_.mapped(k) == ipc::kNoFrame) continue;
      placer_.set_mapped(k, ipc::kNoFrame);
      per_app[k.first].push_back(k.second);
    }
    stale_.clear();
    for (auto& [app, vs] : per_app) {
      auto it = apps_.find(app);
      if (it == apps_.end() || !it->second.alive || it->second.ev < 0 || sched_.granted() == app) continue;
      ipc::Writer w;
      w.put(ipc::SlabsMsg{++epoch_, static_cast<std::uint32_t>(vs.size()), 0});
      w.put_u32s(vs);
      if (!ipc::send_msg(it->second.ev, ipc::Msg::Unmap, w.buf)) it->second.alive = false;
    }
  }

  // plan_switch; with stale mappings kept and slab-aligned victims, each run of
  // evictions in descending virtual-slab order. The engine starts legs in plan order
  // and fetches run ascending, so a victim's vslab empties before the
  // incoming vslab that had its slab asks for one, and the same slabs go to
  // the same vslabs at every switch (tools/slab_sim.cpp: 13-18 remaps per
  // switch in plan order, 0 descending).
  MigrationPlan plan_moves(AppId app, const PlannerConfig& cfg) {
    MigrationPlan plan = plan_switch(app, eng_.mem(), cfg);
    if (!victims_ || !keep_stale()) return plan;
    auto& mv = plan.moves;
    for (std::size_t i = 0; i < mv.size();) {
      std::size_t j = i + 1;
      if (mv[i].kind == MoveKind::EvictFromGpu)
        while (j < mv.size() && mv[j].kind == MoveKind::EvictFromGpu && mv[j].dst == mv[i].dst) ++j;
      // whole vslabs in descending order, blocks ascending inside each one
      // (adjacent frames stay adjacent for the copy batches: reversing the
      // blocks cost 15% of the copy rate, measured)
      std::stable_sort(mv.begin() + static_cast<std::ptrdiff_t>(i), mv.begin() + static_cast<std::ptrdiff_t>(j),
                       [&](const Move& a, const Move& b) { return placer_.vslab_of(a.block) > placer_.vslab_of(b.block); });
      i = j;
    }
    return plan;
  }

  void account(const ExecResult&) {
    const SwitchStats& s = eng_.last_stats();
    bytes_in_ += s.pcie_h2d_bytes;
    bytes_out_ += s.pcie_d2h_bytes;
    verified_ += s.verified;
    mismatches_ += s.mismatches;
  }

  // The holder allocated past the GPU's free space: its new blocks come in
  // and other apps' blocks go out; the holder keeps running (its resident
  // blocks do not move: plan_switch never evicts the incoming app).
  void fetch_in_place(AppId app) {
    PlannerConfig cfg = opt_.planner;
    cfg.eviction_policy.victim_order = sched_.victim_hint();
    cfg.gpu_victims = victims_;
    eng_.prefetch_quiesce();
    const MigrationPlan plan = plan_moves(app, cfg);
    const ExecResult r = eng_.execute(plan, cfg);
    trace_plan("inplace", app, cfg, plan);
    send_maps();
    account(r);
    flush_unmaps();
    shrink_arena();
    note("{\"t\": %.6f, \"event\": \"fetch_in_place\", \"app\": %u, \"bytes_in\": %" PRIu64 ", \"bytes_out\": %" PRIu64 "}",
         now(), app, plan.bytes_in, plan.bytes_out);
  }

  void context_switch(AppId to, Seconds t) {
    App& in = apps_.at(to);
    if (!in.alive || in.ev < 0) {
      sched_.clear_request(to);
      return;
    }
    const std::uint64_t t_start = ipc::mono_ns();
    const std::optional<AppId> holder = sched_.granted();
    std::vector<std::uint8_t> body;
    // (3) pause the incumbent and drain its kernels.
    if (holder) {
      App& h = apps_.at(*holder);
      ipc::EpochMsg pm{++epoch_};
      if (h.alive && h.ev >= 0 && ipc::send_msg(h.ev, ipc::Msg::Pause, &pm, sizeof(pm))) wait_ack(h, ipc::Msg::Drained, body);
      sched_.on_grant_end(*holder, t);
    }
    const std::uint64_t t_drained = ipc::mono_ns();
    // (4) plan + real copies, victims unmapping concurrently.
    PlannerConfig cfg = opt_.planner;
    cfg.eviction_policy.victim_order = sched_.victim_hint();
    cfg.gpu_victims = victims_;
    eng_.prefetch_quiesce();  // cancel_pending + quiesced (transfer.cpp:89-113)
    const MigrationPlan plan = plan_moves(to, cfg);
    const std::uint64_t t_planned = ipc::mono_ns();
    const ExecResult r = eng_.execute(plan, cfg);
    const std::uint64_t t_copied = ipc::mono_ns();
    trace_plan("switch", to, cfg, plan);
    send_maps();
    account(r);
    const std::uint64_t t_unmapped = ipc::mono_ns();
    // (5) grant: the incoming shim maps its slabs and sets its flag.
    const std::vector<ipc::SlabMap> slabs = placer_.backed(to);
    placer_.granted(to);
    ipc::Writer w;
    w.put(ipc::SlabsMsg{++epoch_, static_cast<std::uint32_t>(slabs.size()), 0});
    for (const auto& m : slabs) w.put(m);
    if (!eng_.mem().app_fully_resident(to, TierId::Gpu))
      throw InvariantViolation("grant: app " + std::to_string(to) + " is not GPU-resident after its switch");
    ipc::GrantedMsg gm{};
    send_new_slabs(in, false);
    const std::uint64_t t_grant_sent = ipc::mono_ns();
    if (ipc::send_msg(in.ev, ipc::Msg::Grant, w.buf) && wait_ack(in, ipc::Msg::Granted, body) && body.size() >= sizeof(gm))
      std::memcpy(&gm, body.data(), sizeof(gm));
    const std::uint64_t t_end = ipc::mono_ns();
    sched_.clear_request(to);
    const Seconds granted_at = t + static_cast<double>(t_end - t_start) * 1e-9;
    sched_.on_grant_start(to, granted_at);
    sched_.on_api_event(to, granted_at, ApiEventKind::NonBlockingReturn);  // its held launch resumes now
    flush_unmaps();
    shrink_arena();
    take_deferred_acquires();
    ++switches_;
    const SwitchStats& s = eng_.last_stats();
    auto ms = [](std::uint64_t a, std::uint64_t b) { return static_cast<double>(b - a) * 1e-6; };
    note("{\"t\": %.6f, \"event\": \"switch\", \"from\": %d, \"to\": %u, \"bytes_in\": %" PRIu64 ", \"bytes_out\": %" PRIu64
         ", \"pcie_h2d\": %" PRIu64 ", \"pcie_d2h\": %" PRIu64 ", \"host_bytes\": %" PRIu64
         ", \"pause_ms\": %.3f, \"plan_ms\": %.3f, \"copy_ms\": %.3f, \"unmap_wait_ms\": %.3f, \"grant_ms\": %.3f"
         ", \"map_ms\": %.3f, \"map_calls\": %" PRIu64 ", \"unmap_calls\": %" PRIu64 ", \"grant_recv_ms\": %.3f"
         ", \"premap_ms\": %.3f, \"premap_calls\": %" PRIu64 ", \"premap_unmap_ms\": %.3f, \"total_ms\": %.3f"
         ", \"device_span_ms\": %.3f"
         ", \"verified\": %" PRIu64 ", \"unverified\": %" PRIu64 ", \"mismatches\": %" PRIu64
         ", \"partial_slabs\": %" PRIu64 ", \"free_slabs\": %zu, \"live_slabs\": %zu, \"ce_calls\": %d, \"pace_waits\": %d"
         ", \"ce_calls_dir\": [%d, %d], \"run_breaks_src\": [%d, %d], \"run_breaks_dst\": [%d, %d]}",
         t, holder ? static_cast<int>(*holder) : -1, to, plan.bytes_in, plan.bytes_out, s.pcie_h2d_bytes, s.pcie_d2h_bytes,
         s.host_bytes, ms(t_start, t_drained), ms(t_drained, t_planned), ms(t_planned, t_copied), ms(t_copied, t_unmapped),
         ms(t_unmapped, t_end), static_cast<double>(gm.map_ns) * 1e-6, gm.map_calls, gm.unmap_calls,
         gm.recv_ns > t_grant_sent ? ms(t_grant_sent, gm.recv_ns) : 0.0, static_cast<double>(gm.premap_ns) * 1e-6, gm.premap_calls,
         static_cast<double>(gm.premap_unmap_ns) * 1e-6, ms(t_start, t_end),
         s.device_span_s * 1e3, s.verified, s.unverified, s.mismatches, placer_.partial(), placer_.free_slabs(),
         placer_.live_slabs(), s.ce_calls, s.pace_waits, s.ce_calls_dir[0], s.ce_calls_dir[1], s.run_breaks_src[0],
         s.run_breaks_src[1], s.run_breaks_dst[0], s.run_breaks_dst[1]);
  }

  // ---- reference replay trace (--trace) ---------------------------------------
  // Every registry mutation and executed plan in the order this single thread
  // performed them. oracle/ref_replay.cpp replays the allocations and frees on
  // the unmodified reference MemState (proj/src/mem_model.cpp:48-116),
  // recomputes plan_switch for each plan (proj/src/planner.cpp:111-216) and
  // executes the daemon's plan on the reference Orchestrator
  // (proj/src/transfer.cpp:250-271) for its per-lane leg sequences, so the
  // interposer path is checked against the reference switch by switch.
  void trace_header() {
    std::fprintf(trace_, "capacity gpu %" PRIu64 "\ncapacity pinned %" PRIu64 "\ncapacity paged %" PRIu64 "\n",
                 opt_.eng.gpu_capacity, opt_.eng.pinned_capacity, opt_.eng.paged_capacity);
    std::fprintf(trace_, "window %" PRIu64 "\nbudget %" PRIu64 "\nvictims %s\n", opt_.planner.streaming_window,
                 opt_.planner.pinned_budget, opt_.reference_victims ? "reference" : "slab");
    std::fflush(trace_);
  }
  // Prefetch legs commit inside the engine (its pump runs wherever the
  // registry must be quiescent): their commits are written ahead of the next
  // trace line, which is where they happened relative to it.
  void trace_pcommits() {
    if (!trace_) return;
    for (BlockId b : eng_.take_prefetch_commits()) std::fprintf(trace_, "pcommit %" PRIu64 "\n", static_cast<std::uint64_t>(b));
  }
  void trace_prefetch(AppId app, const MigrationPlan& plan) {
    if (!trace_) return;
    trace_pcommits();
    const std::uint64_t k = prefetches_++;
    std::fprintf(trace_, "prefetch %" PRIu64 " %u moves %zu\n", k, app, plan.moves.size());
    std::string dump = plan.dump();
    for (std::size_t i = 0; i < dump.size();) {
      const std::size_t j = dump.find('\n', i);
      std::fprintf(trace_, "Q %" PRIu64 " %s\n", k, dump.substr(i, j - i).c_str());
      i = j == std::string::npos ? dump.size() : j + 1;
    }
    std::fflush(trace_);
  }
  void trace_alloc(AppId app, Bytes bytes, TierId tier, const std::vector<ChunkId>& chunks) {
    if (!trace_) return;
    trace_pcommits();
    std::fprintf(trace_, "alloc %u %" PRIu64 " %s", app, bytes, tier_name(tier));
    for (ChunkId c : chunks) std::fprintf(trace_, " %u", static_cast<unsigned>(c));
    std::fputc('\n', trace_);
    std::fflush(trace_);
  }
  void trace_free(AppId app, ChunkId c) {
    if (!trace_) return;
    trace_pcommits();
    std::fprintf(trace_, "free %u %u\n", app, static_cast<unsigned>(c));
    std::fflush(trace_);
  }
  void trace_plan(const char* kind, AppId app, const PlannerConfig& cfg, const MigrationPlan& plan) {
    if (!trace_) return;
    trace_pcommits();
    const std::uint64_t k = plans_++;
    std::fprintf(trace_, "plan %" PRIu64 " %s %u in %" PRIu64 " out %" PRIu64 " victims", k, kind, app, plan.bytes_in, plan.bytes_out);
    for (AppId v : cfg.eviction_policy.victim_order) std::fprintf(trace_, " %u", v);
    std::fputc('\n', trace_);
    std::string dump = plan.dump();
    for (std::size_t i = 0; i < dump.size();) {
      const std::size_t j = dump.find('\n', i);
      std::fprintf(trace_, "P %" PRIu64 " %s\n", k, dump.substr(i, j - i).c_str());
      i = j == std::string::npos ? dump.size() : j + 1;
    }
    const auto& lanes = eng_.lane_trace();
    for (int l = 0; l < 6; ++l)
      for (const LegTrace& x : lanes[l])
        std::fprintf(trace_, "L %" PRIu64 " %d %" PRIu64 " %s %s\n", k, l, static_cast<std::uint64_t>(x.block), tier_name(x.src), tier_name(x.dst));
    std::fflush(trace_);
  }

  template <typename... A>
  void note(const char* fmt, A... args) {
    if (!log_) return;
    std::fprintf(log_, fmt, args...);
    std::fputc('\n', log_);
    std::fflush(log_);
  }

  void write_summary() {
    note("{\"event\": \"summary\", \"switches\": %" PRIu64 ", \"pcie_bytes_in\": %" PRIu64 ", \"pcie_bytes_out\": %" PRIu64
         ", \"verified\": %" PRIu64 ", \"mismatches\": %" PRIu64 ", \"apps\": %u, \"rpcs_in_switch\": %" PRIu64 "}",
         switches_, bytes_in_, bytes_out_, verified_, mismatches_, next_app_, rpcs_in_switch_);
    for (const SchedLogRow& row : sched_.log())
      note("{\"event\": \"sched\", \"t\": %.6f, \"app\": %u, \"what\": \"%s\", \"level\": %d}", row.time, row.app,
           row.event.c_str(), row.level);
  }

  Options opt_;
  SwapEngine eng_;
  MlfqScheduler sched_;
  SlabPlacer placer_;
  std::function<std::vector<BlockId>(const MemState&, const std::vector<AppId>&, Bytes)> victims_;
  int listen_fd_ = -1;
  std::vector<int> pending_;
  std::set<SlabPlacer::Key> stale_;  // released vslabs whose owners may still map their old slab
  std::map<AppId, App> apps_;
  AppId next_app_ = 0;
  int gone_ = 0;
  std::uint64_t epoch_ = 0;
  std::uint64_t t0_ = 0;
  Seconds last_tick_ = 0;
  std::uint64_t switches_ = 0, bytes_in_ = 0, bytes_out_ = 0, verified_ = 0, mismatches_ = 0;
  std::FILE* log_ = nullptr;
  std::FILE* trace_ = nullptr;
  std::uint64_t plans_ = 0;             // plans written to the trace
  std::uint64_t prefetches_ = 0;        // prefetch plans written to the trace
  std::vector<AppId> deferred_acquires_;
  std::uint64_t rpcs_in_switch_ = 0;    // requests served while awaiting an ack
};

}  // namespace

int main(int argc, char** argv) {
  Options opt;
  try {
    if (!parse_args(argc, argv, opt)) return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "nixied: %s\n", e.what());
    return 1;
  }
  signal(SIGINT, on_signal);
  signal(SIGTERM, on_signal);
  signal(SIGPIPE, SIG_IGN);
  try {
    Daemon d(opt);
    d.listen_on();
    return d.run();
  } catch (const InvariantViolation& e) {
    std::fprintf(stderr, "nixied: invariant violation: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "nixied: %s\n", e.what());
    return 1;
  }
}
