// Shim <-> daemon protocol of the interposer path (internal header, shared by
// csrc/shim/shim.cpp and csrc/daemon/daemon.cpp).
//
// a per-application shim interposes the CUDA runtime and
// talks to a central daemon over a UNIX domain socket; the daemon owns the
// scheduler (MLFQ) and the memory system, the shim gates its application's
// launches on an execution flag. Here the daemon also owns the GPU tier (one
// exportable VMM arena) and drives every copy itself, both directions at once
// (the swap engine); the shims only map/unmap arena frames under their
// applications' stable virtual ranges and gate launches.
//
// Transport: two SOCK_STREAM connections per application, length-prefixed
// messages (Header + payload).
//   rpc   app thread -> daemon request, daemon -> app reply (Hello, Alloc,
//         Free, Acquire); serialised by a mutex in the shim.
//   event daemon -> shim command, shim -> daemon ack (Unmap, Pause, Grant);
//         served by the shim's listener thread, so the daemon can pause an
//         application whose threads are blocked inside an rpc.
// Activity (launch counts, blocking calls; the MLFQ's idleness input,
// PAPER.md §6.1) is published lock-free in a shared control page the daemon
// reads on its tick, so a granted application's launch never does IPC
// ("App 1 only executes step 1 and 6, bypassing IPC").
#pragma once

#include <sys/socket.h>
#include <sys/uio.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace nixie::ipc {

constexpr std::uint32_t kMagic = 0x4E585831;  // "NXX1"
constexpr std::uint32_t kNoFrame = 0xFFFFFFFFu;
constexpr int kFdBatch = 250;  // SCM_RIGHTS carries at most 253 descriptors

enum class Msg : std::uint32_t {
  Hello = 1,     // rpc  shim->d : HelloReq   reply HelloRep, fd [ctl], then the arena slabs' fds in
                 //                            batches of kFdBatch (slab order)
  EventHello,    // event shim->d: EventHelloReq (no reply)
  Alloc,         // rpc  shim->d : AllocReq   reply AllocRep + u32 chunk ids + SlabMap[n_slabs]
  Free,          // rpc  shim->d : u32 n + u32 chunk ids; reply FreeRep + u32 released vslabs
  Acquire,       // rpc  shim->d : (empty)    reply Status (queued; a Grant follows on the event socket)
  Status,        // reply: StatusRep
  Pause,         // event d->shim: EpochMsg -> shim stops launches, drains, acks Drained
  Drained,       // event shim->d: EpochMsg
  Unmap,         // event d->shim: SlabsMsg + u32 vslabs (their physical slab was released; no ack)
  Grant,         // event d->shim: SlabsMsg + SlabMap[n] (every mapped vslab of the app) -> ack Granted
  Granted,       // event shim->d: GrantedMsg
  Stats,         // rpc  shim->d : (empty)    reply StatsRep
  Map,           // event d->shim: SlabsMsg + SlabMap[n] (slabs placed while the switch runs; no ack)
  Slab,          // rpc or event d->shim: SlabFdMsg, then 1 fd: a (re)created slab to import (no ack)
  Drop,          // event d->shim: DropMsg: the daemon released a grown slab; unmap and release it (no ack)
};

struct SlabFdMsg {
  std::uint32_t slab;
  std::uint32_t gen;  // creation count of that slot (a dropped slot can be created again)
};
struct DropMsg {
  std::uint64_t epoch;
  std::uint32_t slab;
  std::uint32_t gen;
};

// Virtual slabs: a shim reserves one large virtual range and places its
// managed allocations in it at 2 MiB granularity; vslab k is the 128 MiB
// (slab_blocks frames, announced in HelloRep) window k of that range. The daemon backs every vslab
// that holds a GPU-resident block with one physical slab of its arena, so the
// shim maps whole slabs (one mapping per 64 blocks), and block j of an
// allocation placed at range block v lives in frame phys * slab_blocks +
// (v + j) % slab_blocks. The daemon picks the slab size (--slab-mib); every
// mapping costs the same whatever its size (profiles/r01_vmm_probe*.txt).
constexpr std::uint32_t kDefaultSlabBlocks = 256;  // 512 MiB (budgets >= 16 GiB; 128 MiB below)

struct SlabMap {
  std::uint32_t vslab;
  std::uint32_t phys;  // kNoFrame: not backed
};

struct Header {
  std::uint32_t magic;
  std::uint32_t type;
  std::uint64_t bytes;  // payload bytes after the header
};

struct HelloReq {
  std::int32_t pid;
  std::int32_t device;
  char name[64];
};
struct HelloRep {
  std::int32_t status;  // 0 ok
  std::uint32_t app;
  std::uint64_t gpu_budget;    // bytes the app may see as device memory (cudaMemGetInfo total)
  std::uint64_t block_bytes;   // 2 MiB
  std::uint64_t arena_bytes;   // physical bytes of the arena (slabs x slab_bytes)
  std::uint64_t slabs;         // exported slab allocations that follow
  std::uint64_t slab_bytes;
  std::uint64_t min_bytes;     // allocations below this pass through to cudaMalloc
  std::int32_t device;
  std::int32_t pad;
};
struct EventHelloReq {
  std::uint32_t app;
  std::uint32_t pad;
};
struct AllocReq {
  std::uint64_t bytes;
  std::uint64_t va_block;  // placement in the shim's range, in 2 MiB blocks
};
struct AllocRep {
  std::int32_t status;  // 0 ok, 2 out of memory, other: SimError code + 100
  std::uint32_t n_chunks;
  std::uint32_t n_slabs;  // SlabMap entries that follow the chunk ids
  std::uint32_t pad;
  std::uint64_t footprint;  // bytes charged (2 MiB rounded)
  std::uint64_t epoch;      // daemon message sequence at reply time (orders it
                            // against Unmap/Grant already sent on the event socket)
};
struct StatusRep {
  std::int32_t status;
  std::int32_t pad;
};
struct EpochMsg {
  std::uint64_t epoch;
};
struct SlabsMsg {
  std::uint64_t epoch;
  std::uint32_t n;
  std::uint32_t pad;
};
struct FreeRep {
  std::int32_t status;
  std::uint32_t n;  // released vslabs that follow
  std::uint64_t epoch;
};
struct GrantedMsg {
  std::uint64_t epoch;
  std::uint64_t map_ns;       // shim-side mapping time
  std::uint64_t map_calls;    // cuMemMap calls made
  std::uint64_t unmap_calls;  // cuMemUnmap calls made
  std::uint64_t recv_ns;      // CLOCK_MONOTONIC when the listener took the Grant off the socket
  std::uint64_t premap_ns;    // time spent on Map messages since the previous Grant
  std::uint64_t premap_calls; // cuMemMap calls they made
  std::uint64_t premap_unmap_ns;  // of premap_ns: cuMemUnmap of the slabs' previous mappings
};
struct StatsRep {
  std::uint64_t switches;
  std::uint64_t bytes_in, bytes_out;
  std::uint64_t mismatches, verified;
};

// Shared control page (memfd, one per application): written by the shim,
// read by the daemon's tick. Times are CLOCK_MONOTONIC nanoseconds.
struct alignas(64) CtlPage {
  std::atomic<std::uint64_t> launches;        // gated launches/copies issued
  std::atomic<std::uint64_t> last_api_ns;     // last API return
  std::atomic<std::uint32_t> blocking;        // threads inside a blocking call
  std::atomic<std::uint32_t> granted;         // mirror of the execution flag
  std::atomic<std::uint64_t> last_block_ns;   // last blocking enter/exit
  std::atomic<std::uint64_t> gate_waits;      // launches held by the gate
  std::atomic<std::uint64_t> gate_wait_ns;    // total time held
  std::atomic<std::uint64_t> map_ns;          // total mapping time
  std::atomic<std::uint64_t> unmap_ns;        // total unmapping time
  std::atomic<std::uint64_t> drain_ns;        // total pause-drain time
  std::atomic<std::uint64_t> blas_calls;      // gated library calls (cuBLAS / cuBLASLt GEMMs, cuDNN executes)
  std::atomic<std::uint64_t> table_launches;  // gated calls that came through cuGetProcAddress entry
                                              // points directly (not via an interposed runtime call)
  std::atomic<std::uint64_t> small_bytes;     // passthrough allocations below min_bytes (live)
  std::atomic<std::uint64_t> implicit_bytes;  // device memory taken by implicitly allocating APIs
                                              // (stream/handle creation, limits, graph instantiation), live
  std::atomic<std::uint64_t> captured_launches;  // launches recorded into stream captures (activity, not gated)
};
static_assert(sizeof(CtlPage) <= 4096, "control page fits one page");

inline std::uint64_t mono_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return static_cast<std::uint64_t>(ts.tv_sec) * 1000000000ull + static_cast<std::uint64_t>(ts.tv_nsec);
}

// ---- framing (return false on EOF / error) ----------------------------------
inline bool write_all(int fd, const void* p, std::size_t n) {
  const auto* c = static_cast<const std::uint8_t*>(p);
  while (n) {
    const ssize_t w = ::send(fd, c, n, MSG_NOSIGNAL);
    if (w < 0 && errno == EINTR) continue;
    if (w <= 0) return false;
    c += w;
    n -= static_cast<std::size_t>(w);
  }
  return true;
}

inline bool read_all(int fd, void* p, std::size_t n) {
  auto* c = static_cast<std::uint8_t*>(p);
  while (n) {
    const ssize_t r = ::recv(fd, c, n, 0);
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) return false;
    c += r;
    n -= static_cast<std::size_t>(r);
  }
  return true;
}

inline bool send_msg(int fd, Msg type, const void* payload, std::size_t bytes) {
  Header h{kMagic, static_cast<std::uint32_t>(type), bytes};
  if (!write_all(fd, &h, sizeof(h))) return false;
  return bytes == 0 || write_all(fd, payload, bytes);
}

inline bool send_msg(int fd, Msg type, const std::vector<std::uint8_t>& payload) {
  return send_msg(fd, type, payload.data(), payload.size());
}

// Reads one message; payload is resized to its length.
inline bool recv_msg(int fd, Msg& type, std::vector<std::uint8_t>& payload) {
  Header h{};
  if (!read_all(fd, &h, sizeof(h)) || h.magic != kMagic || h.bytes > (1ull << 30)) return false;
  type = static_cast<Msg>(h.type);
  payload.resize(h.bytes);
  return h.bytes == 0 || read_all(fd, payload.data(), h.bytes);
}

// Descriptor passing (SCM_RIGHTS) alongside a one-byte marker.
inline bool send_fds(int sock, const int* fds, int n) {
  char byte = 'F';
  iovec iov{&byte, 1};
  std::vector<char> ctrl(CMSG_SPACE(sizeof(int) * n));
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctrl.data();
  m.msg_controllen = ctrl.size();
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  c->cmsg_level = SOL_SOCKET;
  c->cmsg_type = SCM_RIGHTS;
  c->cmsg_len = CMSG_LEN(sizeof(int) * n);
  std::memcpy(CMSG_DATA(c), fds, sizeof(int) * n);
  for (;;) {
    const ssize_t w = ::sendmsg(sock, &m, MSG_NOSIGNAL);
    if (w < 0 && errno == EINTR) continue;
    return w == 1;
  }
}

inline bool recv_fds(int sock, int* fds, int n) {
  char byte = 0;
  iovec iov{&byte, 1};
  std::vector<char> ctrl(CMSG_SPACE(sizeof(int) * n));
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctrl.data();
  m.msg_controllen = ctrl.size();
  ssize_t r;
  do {
    r = ::recvmsg(sock, &m, MSG_CMSG_CLOEXEC);
  } while (r < 0 && errno == EINTR);
  if (r != 1) return false;
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  if (!c || c->cmsg_type != SCM_RIGHTS || c->cmsg_len != CMSG_LEN(sizeof(int) * n)) return false;
  std::memcpy(fds, CMSG_DATA(c), sizeof(int) * n);
  return true;
}

// Little payload builder / reader.
struct Writer {
  std::vector<std::uint8_t> buf;
  template <typename T>
  void put(const T& v) {
    const auto* p = reinterpret_cast<const std::uint8_t*>(&v);
    buf.insert(buf.end(), p, p + sizeof(T));
  }
  void put_u32s(const std::vector<std::uint32_t>& v) {
    const auto* p = reinterpret_cast<const std::uint8_t*>(v.data());
    buf.insert(buf.end(), p, p + v.size() * sizeof(std::uint32_t));
  }
};

struct Reader {
  const std::vector<std::uint8_t>& buf;
  std::size_t off = 0;
  bool ok = true;
  template <typename T>
  T get() {
    T v{};
    if (off + sizeof(T) > buf.size()) {
      ok = false;
      return v;
    }
    std::memcpy(&v, buf.data() + off, sizeof(T));
    off += sizeof(T);
    return v;
  }
};

}  // namespace nixie::ipc
