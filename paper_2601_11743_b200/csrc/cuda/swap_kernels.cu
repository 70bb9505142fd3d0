// sm_100a kernels of the swap path.
//
//   K1 nx_swap_kernel     bidirectional HBM <-> mapped-pinned copy of 2 MiB
//                         legs with the per-block checksum fused in (records
//                         it on departure, verifies it on arrival)
//   K3 (same kernel)      checksum-only legs (dst == nullptr): used around the
//                         copy-engine variant, which cannot checksum
//   K4 nx_fill_kernel / nx_compare_kernel
//                         synthetic working-set pattern fill and byte compare
//
// Design (B200, PCIe-bound path, no tensor cores):
//   * A CTA is two 128-thread warp groups. With both directions in one launch
//     group 0 moves D2H legs and group 1 H2D legs, so every SM issues both
//     PCIe writes (posted, D2H) and PCIe reads (non-posted, H2D) and the two
//     link directions fill at once. With one direction per launch (the
//     engine's default two-stream mode: one launch stream per direction) both
//     groups serve it.
//   * Each thread keeps 8 independent 16-byte loads in flight
//     (ld.global.nc.L1::no_allocate.v4), i.e. 16 KiB per warp group: a few
//     hundred groups cover the PCIe bandwidth-delay product many times over.
//     Stores are st.global.L1::no_allocate.v4; a warp touches 512 contiguous
//     bytes per instruction.
//   * A leg can be split into 2^k parts so a small launch still spreads over
//     all 148 SMs; part checksums are combined by the last finisher
//     (threadfence + counter), which also resets the counter.
//   * Legs travel in the kernel parameter block (__grid_constant__, <= 256
//     legs, ~6 KB): no descriptor copy precedes a launch.
#include <cuda_runtime.h>

#include "nx_common.cuh"
#include "nx_kernels.h"
#include "nx_tma.cuh"

namespace nixie::b200 {

namespace {

// K3 over a device-resident leg table (any number of legs): one launch can
// cover a whole switch's departures or a group of arrival batches.
struct SwapParamsTable {
  NxCkTables ck;
  NxScratch scratch;
  std::uint32_t n_d2h;
  std::uint32_t n_h2d;
  std::uint32_t parts_log2;
  std::uint32_t flags;
  std::uint32_t clock_slot;
  const NxLeg* legs;  // device memory
};

// Kernel parameter block sized for up to N legs. Launches pick the smallest
// N that fits: the block is copied into every launch, so a 6 KB block for a
// 1-leg launch is pure overhead.
template <int N>
struct SwapParamsT {
  NxCkTables ck;
  NxScratch scratch;
  std::uint32_t n_d2h;
  std::uint32_t n_h2d;
  std::uint32_t parts_log2;
  std::uint32_t flags;
  std::uint32_t clock_slot;  // kNoClockSlot: no device-clock stamps
  NxLeg legs[N];
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
using SwapParams = SwapParamsT<kMaxLegsPerLaunch>;

struct FillParams {
  NxLeg legs[kMaxLegsPerLaunch];
  NxCkTables ck;
  unsigned long long* mismatches;
  std::uint64_t seed;
  std::uint32_t n;
};

constexpr int kUnroll = 8;
constexpr int kGroupThreads = 128;

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void st_stream(uint4* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Named barrier of one 128-thread warp group (ids 1 and 2; id 0 is __syncthreads).
// Immediate ids keep ptxas from reserving all 16 barriers.
__device__ __forceinline__ void group_barrier(int group) {
  if (group == 0)
    asm volatile("bar.sync 1, 128;" ::: "memory");
  else
    asm volatile("bar.sync 2, 128;" ::: "memory");
}

__device__ __forceinline__ std::uint64_t ck16(const uint4& v, std::uint64_t vec_index) {
  const std::uint64_t w0 = static_cast<std::uint64_t>(v.x) | (static_cast<std::uint64_t>(v.y) << 32);
  const std::uint64_t w1 = static_cast<std::uint64_t>(v.z) | (static_cast<std::uint64_t>(v.w) << 32);
  return ck_term(w0, 2 * vec_index) + ck_term(w1, 2 * vec_index + 1);
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Streams `nvec` vectors src -> dst (dst may be null: checksum only) with
// kUnroll loads in flight per thread; returns this thread's checksum share.
template <bool kChecksum>
__device__ __forceinline__ std::uint64_t stream_part(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                     std::uint64_t nvec, std::uint64_t j0, int gt) {
  // Position key of word 2*idx is 2*idx*golden; keys advance by constants
  // instead of a multiply per word (vector idx = j0 + b + u*kGroupThreads).
  constexpr std::uint64_t kKeyStepU = 2ull * kGroupThreads * kGolden;
  std::uint64_t key = 2ull * (j0 + static_cast<std::uint64_t>(gt)) * kGolden;
  std::uint64_t acc = 0;
  for (std::uint64_t b = gt; b < nvec; b += kGroupThreads * kUnroll) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream(src + b + u * kGroupThreads);
    if (dst != nullptr) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) st_stream(dst + b + u * kGroupThreads, v[u]);
    }
    if (kChecksum) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const std::uint64_t w0 = static_cast<std::uint64_t>(v[u].x) | (static_cast<std::uint64_t>(v[u].y) << 32);
        const std::uint64_t w1 = static_cast<std::uint64_t>(v[u].z) | (static_cast<std::uint64_t>(v[u].w) << 32);
        const std::uint64_t k = key + u * kKeyStepU;
        acc += ck_term_keyed(w0, k) + ck_term_keyed(w1, k + kGolden);
      }
      key += kUnroll * kKeyStepU;
    }
  }
  return acc;
}

// Final checksum of leg `li` (all parts summed): record on departure, check
// on arrival.
template <class P>
__device__ void finish_leg(const P& p, std::uint32_t li, unsigned long long sum, bool arriving) {
  const std::uint32_t blk = p.legs[li].block;
  if (!arriving) {
    p.ck.ck_ref[blk] = sum;
    p.ck.ck_valid[blk] = 1u;
    return;
  }
  p.ck.ck_seen[blk] = sum;
  if (!(p.flags & kNxVerify)) return;
  if (p.ck.ck_valid[blk] == 0u) {
    atomicAdd(&p.ck.status->unverified, 1ull);
    return;
  }
  atomicAdd(&p.ck.status->verified, 1ull);
  if (sum != p.ck.ck_ref[blk]) {
    atomicAdd(&p.ck.status->mismatches, 1ull);
    const unsigned slot = atomicAdd(&p.ck.status->n_bad, 1u);
    if (slot < 64u) p.ck.status->bad_blocks[slot] = blk;
  }
}

template <bool kChecksum, class P>
__global__ void __launch_bounds__(2 * kGroupThreads) nx_swap_kernel(const __grid_constant__ P p) {
  __shared__ unsigned long long red[2][4];
  const int group = threadIdx.x / kGroupThreads;
  const int gt = threadIdx.x % kGroupThreads;
  const bool fused = p.n_d2h != 0 && p.n_h2d != 0;
  // Role: 0 = departing (D2H / checksum-record), 1 = arriving (H2D / verify).
  const int role = fused ? group : (p.n_d2h != 0 ? 0 : 1);
  const std::uint32_t first = fused ? blockIdx.x : blockIdx.x * 2 + group;
  const std::uint32_t stride = fused ? gridDim.x : gridDim.x * 2;
  const std::uint32_t base = role == 0 ? 0u : p.n_d2h;
  const std::uint32_t n_items = (role == 0 ? p.n_d2h : p.n_h2d) << p.parts_log2;
  const std::uint64_t part_vecs = kVecsPerBlock >> p.parts_log2;
  const std::uint32_t part_mask = (1u << p.parts_log2) - 1u;

  for (std::uint32_t item = first; item < n_items; item += stride) {
    const std::uint32_t li = base + (item >> p.parts_log2);
    const std::uint32_t part = item & part_mask;
    const NxLeg leg = p.legs[li];
    const std::uint64_t off = static_cast<std::uint64_t>(part) * part_vecs;
    const uint4* src = static_cast<const uint4*>(leg.src) + off;
    uint4* dst = leg.dst != nullptr ? static_cast<uint4*>(leg.dst) + off : nullptr;
    std::uint64_t acc = stream_part<kChecksum>(src, dst, part_vecs, off, gt);
    if (!kChecksum) continue;

    acc = warp_sum(acc);
    if ((gt & 31) == 0) red[group][gt >> 5] = acc;
    group_barrier(group);
    if (gt == 0) {
      const unsigned long long part_sum = red[group][0] + red[group][1] + red[group][2] + red[group][3];
      if (p.parts_log2 == 0) {
        finish_leg(p, li, part_sum, role == 1);
      } else {
        p.scratch.part_sums[(li << kMaxPartsLog2) + part] = part_sum;
        __threadfence();
        const unsigned done = atomicAdd(&p.scratch.part_count[li], 1u);
        if (done == part_mask) {  // last part of this leg
          __threadfence();
          unsigned long long total = 0;
          for (std::uint32_t q = 0; q <= part_mask; ++q) total += __ldcg(&p.scratch.part_sums[(li << kMaxPartsLog2) + q]);
          p.scratch.part_count[li] = 0u;
          finish_leg(p, li, total, role == 1);
        }
      }
    }
    group_barrier(group);
  }
}

// K4: one CTA per leg, 256 threads. Fill writes the pattern and records the
// checksum; compare counts mismatching 16-byte vectors.
template <bool kFill>
__global__ void __launch_bounds__(256) nx_pattern_kernel(const __grid_constant__ FillParams p) {
  __shared__ unsigned long long red[8];
  const NxLeg leg = p.legs[blockIdx.x];
  const std::uint64_t blk = leg.block;
  unsigned long long acc = 0;
  for (std::uint64_t j = threadIdx.x; j < kVecsPerBlock; j += blockDim.x) {
    const std::uint64_t w0 = pattern_word(p.seed, leg.tag, blk, 2 * j);
    const std::uint64_t w1 = pattern_word(p.seed, leg.tag, blk, 2 * j + 1);
    if (kFill) {
      uint4 v;
      v.x = static_cast<unsigned>(w0);
      v.y = static_cast<unsigned>(w0 >> 32);
      v.z = static_cast<unsigned>(w1);
      v.w = static_cast<unsigned>(w1 >> 32);
      st_stream(static_cast<uint4*>(leg.dst) + j, v);
      acc += ck_term(w0, 2 * j) + ck_term(w1, 2 * j + 1);
    } else {
      const uint4 v = ld_stream(static_cast<const uint4*>(leg.src) + j);
      const std::uint64_t g0 = static_cast<std::uint64_t>(v.x) | (static_cast<std::uint64_t>(v.y) << 32);
      const std::uint64_t g1 = static_cast<std::uint64_t>(v.z) | (static_cast<std::uint64_t>(v.w) << 32);
      acc += (g0 != w0 || g1 != w1) ? 1ull : 0ull;
    }
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long total = 0;
    for (int w = 0; w < 8; ++w) total += red[w];
    if (kFill) {
      p.ck.ck_ref[blk] = total;
      p.ck.ck_valid[blk] = 1u;
    } else {
      p.mismatches[blockIdx.x] += total;
    }
  }
}

// K3 on the TMA pipeline. The chunks of all legs form one sequence; CTA b
// takes the contiguous, balanced range [total*b/grid, total*(b+1)/grid), so
// every SM gets the same bytes whatever the leg count. The last warp's lane 0
// is the producer (bulk loads into a kStages ring, full/empty mbarriers); the
// consume. A leg split across CTAs is combined by the CTA that completes its
// chunk count (threadfence + counter, accumulator reset for the next launch).
constexpr int kTmaChunk = 32 << 10;
constexpr int kTmaStages = 6;
constexpr int kTmaConsumers = 512;  // 16 consumer warps: the checksum must keep up with ~23 B/clk/SM of HBM
constexpr std::uint32_t kTmaChunksPerLeg = kBlockBytesDev / kTmaChunk;

template <class P>
__device__ void tma_flush(const P& p, std::uint32_t base, std::uint32_t leg, std::uint32_t chunks,
                          unsigned long long acc, bool arriving, unsigned long long* red) {
  acc = warp_sum(acc);
  const int warp = threadIdx.x / 32;
  if ((threadIdx.x & 31) == 0) red[warp] = acc;
  asm volatile("bar.sync 1, %0;" ::"n"(kTmaConsumers) : "memory");
  if (threadIdx.x == 0) {
    unsigned long long part = 0;
    for (int w = 0; w < kTmaConsumers / 32; ++w) part += red[w];
    atomicAdd(&p.scratch.leg_acc[base + leg], part);
    __threadfence();
    const unsigned before = atomicAdd(&p.scratch.part_count[base + leg], chunks);
    if (before + chunks == kTmaChunksPerLeg) {
      __threadfence();
      const unsigned long long total = atomicExch(&p.scratch.leg_acc[base + leg], 0ull);
      p.scratch.part_count[base + leg] = 0u;
      finish_leg(p, base + leg, total, arriving);
    }
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kTmaConsumers) : "memory");
}

template <class P>
__global__ void __launch_bounds__(kTmaConsumers + 32, 1) nx_checksum_tma_kernel(const __grid_constant__ P p) {
  extern __shared__ __align__(1024) std::uint8_t ring[];
  __shared__ __align__(8) std::uint64_t full[kTmaStages];
  __shared__ __align__(8) std::uint64_t empty[kTmaStages];
  __shared__ unsigned long long red[kTmaConsumers / 32];
  const bool arriving = p.n_h2d != 0;
  const std::uint32_t base = arriving ? p.n_d2h : 0u;
  const std::uint64_t total = static_cast<std::uint64_t>(arriving ? p.n_h2d : p.n_d2h) * kTmaChunksPerLeg;
  const std::uint64_t c0 = total * blockIdx.x / gridDim.x;
  const std::uint64_t c1 = total * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaConsumers / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (c0 >= c1) return;
  if (threadIdx.x == 0 && p.clock_slot != kNoClockSlot) atomicMin(&p.ck.kstart[p.clock_slot], global_ns());
  const std::uint64_t n = c1 - c0;
  const int warp = threadIdx.x / 32;

  if (warp == kTmaConsumers / 32) {  // producer warp
    if ((threadIdx.x & 31) == 0) {
      for (std::uint64_t i = 0; i < n; ++i) {
        const int s = static_cast<int>(i % kTmaStages);
        if (i >= static_cast<std::uint64_t>(kTmaStages))
          mbar_wait(&empty[s], static_cast<unsigned>((i / kTmaStages - 1) & 1));
        const std::uint64_t c = c0 + i;
        const auto* src = static_cast<const std::uint8_t*>(p.legs[base + c / kTmaChunksPerLeg].src) +
                          (c % kTmaChunksPerLeg) * static_cast<std::uint64_t>(kTmaChunk);
        mbar_expect_tx(&full[s], kTmaChunk);
        bulk_load(ring + s * kTmaChunk, src, kTmaChunk, &full[s]);
      }
    }
    return;
  }

  // Consumers: thread t reads vectors t, t+256, ... of each 32 KiB chunk.
  constexpr int kVecsPerThread = kTmaChunk / 16 / kTmaConsumers;
  constexpr std::uint64_t kKeyStep = 2ull * kTmaConsumers * kGolden;
  std::uint32_t leg = static_cast<std::uint32_t>(c0 / kTmaChunksPerLeg);
  std::uint32_t seg_chunks = 0;
  unsigned long long acc = 0;
  for (std::uint64_t i = 0; i < n; ++i) {
    const std::uint64_t c = c0 + i;
    const auto li = static_cast<std::uint32_t>(c / kTmaChunksPerLeg);
    if (li != leg) {
      tma_flush(p, base, leg, seg_chunks, acc, arriving, red);
      leg = li;
      seg_chunks = 0;
      acc = 0;
    }
    const int s = static_cast<int>(i % kTmaStages);
    mbar_wait(&full[s], static_cast<unsigned>((i / kTmaStages) & 1));
    const uint4* v = reinterpret_cast<const uint4*>(ring + s * kTmaChunk);
    const std::uint64_t vbase = (c % kTmaChunksPerLeg) * static_cast<std::uint64_t>(kTmaChunk / 16);
    std::uint64_t key = 2ull * (vbase + threadIdx.x) * kGolden;
#pragma unroll
    for (int k = 0; k < kVecsPerThread; ++k) {
      const uint4 x = v[threadIdx.x + k * kTmaConsumers];
      const std::uint64_t w0 = static_cast<std::uint64_t>(x.x) | (static_cast<std::uint64_t>(x.y) << 32);
      const std::uint64_t w1 = static_cast<std::uint64_t>(x.z) | (static_cast<std::uint64_t>(x.w) << 32);
      acc += ck_term_keyed(w0, key) + ck_term_keyed(w1, key + kGolden);
      key += kKeyStep;
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
    ++seg_chunks;
  }
  tma_flush(p, base, leg, seg_chunks, acc, arriving, red);  // ends with a consumer barrier
  if (threadIdx.x == 0 && p.clock_slot != kNoClockSlot) atomicMax(&p.ck.kend[p.clock_slot], global_ns());
}

// K1T: the swap copy on the TMA pipeline (round 2). Same chunk sequence and
// balanced CTA ranges as K3, over the legs' sources (pinned host memory for
// fetches, HBM frames for departures). The producer thread bulk-loads a chunk
// into a 4-stage ring, bulk-stores it to the leg's destination as soon as it
// landed, and refills a stage once its store has read shared memory and the
// consumer warps have checksummed it (record on departure, verify on arrival,
// as K1). Few CTAs suffice: one CTA keeps 128 KiB in flight per direction,
// and a sweep of grid sizes (tools/sm_inflight_sweep.py) put the best
// bidirectional rate at 8-74 CTAs per direction, not at a full grid.
constexpr int kSwapTmaStages = 4;

template <class P>
__global__ void __launch_bounds__(kTmaConsumers + 32, 1) nx_swap_tma_kernel(const __grid_constant__ P p) {
  extern __shared__ __align__(1024) std::uint8_t ring[];
  __shared__ __align__(8) std::uint64_t full[kSwapTmaStages];
  __shared__ __align__(8) std::uint64_t empty[kSwapTmaStages];
  __shared__ unsigned long long red[kTmaConsumers / 32];
  const std::uint64_t total = static_cast<std::uint64_t>(p.n_d2h + p.n_h2d) * kTmaChunksPerLeg;
  const std::uint64_t c0 = total * blockIdx.x / gridDim.x;
  const std::uint64_t c1 = total * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSwapTmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaConsumers / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (c0 >= c1) return;
  const std::uint64_t n = c1 - c0;
  const int warp = threadIdx.x / 32;
  const bool checksum = (p.flags & kNxNoChecksum) == 0u;
  auto chunk_ptr = [&](std::uint64_t c, bool dst) {
    const NxLeg& l = p.legs[c / kTmaChunksPerLeg];
    return static_cast<std::uint8_t*>(dst ? l.dst : const_cast<void*>(l.src)) +
           (c % kTmaChunksPerLeg) * static_cast<std::uint64_t>(kTmaChunk);
  };

  if (warp == kTmaConsumers / 32) {  // producer warp: loads and stores
    if ((threadIdx.x & 31) == 0) {
      const std::uint64_t pre = n < kSwapTmaStages ? n : kSwapTmaStages;
      for (std::uint64_t i = 0; i < pre; ++i) {
        mbar_expect_tx(&full[i], kTmaChunk);
        bulk_load(ring + i * kTmaChunk, chunk_ptr(c0 + i, false), kTmaChunk, &full[i]);
      }
      for (std::uint64_t j = 0; j < n; ++j) {
        const int s = static_cast<int>(j % kSwapTmaStages);
        mbar_wait(&full[s], static_cast<unsigned>((j / kSwapTmaStages) & 1));
        bulk_store(chunk_ptr(c0 + j, true), ring + s * kTmaChunk, kTmaChunk);
        // Refill the stage of chunk j-1 (store j stays in flight meanwhile).
        if (j >= 1 && j - 1 + kSwapTmaStages < n) {
          bulk_wait_read<1>();
          const int r = static_cast<int>((j - 1) % kSwapTmaStages);
          mbar_wait(&empty[r], static_cast<unsigned>(((j - 1) / kSwapTmaStages) & 1));
          mbar_expect_tx(&full[r], kTmaChunk);
          bulk_load(ring + r * kTmaChunk, chunk_ptr(c0 + j - 1 + kSwapTmaStages, false), kTmaChunk, &full[r]);
        }
      }
      bulk_wait_all();  // every store written before the kernel (and its completion event) ends
    }
    return;
  }

  constexpr int kVecsPerThread = kTmaChunk / 16 / kTmaConsumers;
  constexpr std::uint64_t kKeyStep = 2ull * kTmaConsumers * kGolden;
  std::uint32_t leg = static_cast<std::uint32_t>(c0 / kTmaChunksPerLeg);
  std::uint32_t seg_chunks = 0;
  unsigned long long acc = 0;
  for (std::uint64_t i = 0; i < n; ++i) {
    const std::uint64_t c = c0 + i;
    const auto li = static_cast<std::uint32_t>(c / kTmaChunksPerLeg);
    if (li != leg) {
      if (checksum) tma_flush(p, 0u, leg, seg_chunks, acc, leg >= p.n_d2h, red);
      leg = li;
      seg_chunks = 0;
      acc = 0;
    }
    const int s = static_cast<int>(i % kSwapTmaStages);
    mbar_wait(&full[s], static_cast<unsigned>((i / kSwapTmaStages) & 1));
    if (checksum) {
      const uint4* v = reinterpret_cast<const uint4*>(ring + s * kTmaChunk);
      const std::uint64_t vbase = (c % kTmaChunksPerLeg) * static_cast<std::uint64_t>(kTmaChunk / 16);
      std::uint64_t key = 2ull * (vbase + threadIdx.x) * kGolden;
#pragma unroll
      for (int k = 0; k < kVecsPerThread; ++k) {
        const uint4 x = v[threadIdx.x + k * kTmaConsumers];
        const std::uint64_t w0 = static_cast<std::uint64_t>(x.x) | (static_cast<std::uint64_t>(x.y) << 32);
        const std::uint64_t w1 = static_cast<std::uint64_t>(x.z) | (static_cast<std::uint64_t>(x.w) << 32);
        acc += ck_term_keyed(w0, key) + ck_term_keyed(w1, key + kGolden);
        key += kKeyStep;
      }
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
    ++seg_chunks;
  }
  if (checksum) tma_flush(p, 0u, leg, seg_chunks, acc, leg >= p.n_d2h, red);
}

int parts_log2_for(int n_legs, int groups_wanted) {
  int k = 0;
  while (k < kMaxPartsLog2 && (n_legs << k) < groups_wanted) ++k;
  return k;
}

}  // namespace

int device_sm_count(int device) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  return sms;
}

namespace {

template <int N>
cudaError_t launch_swap_n(const NxLeg* legs, int n_d2h, int n_h2d, std::uint32_t flags, const NxCkTables& ck,
                          const NxScratch& scratch, int max_ctas, cudaStream_t stream) {
  SwapParamsT<N> p;
  for (int i = 0; i < n_d2h + n_h2d; ++i) p.legs[i] = legs[i];
  p.ck = ck;
  p.scratch = scratch;
  p.n_d2h = static_cast<std::uint32_t>(n_d2h);
  p.n_h2d = static_cast<std::uint32_t>(n_h2d);
  p.flags = flags;
  p.clock_slot = kNoClockSlot;
  const bool fused = n_d2h > 0 && n_h2d > 0;
  // Aim for one work item per warp group of the capped grid.
  const int groups = fused ? max_ctas : 2 * max_ctas;
  const int n_dir = fused ? (n_d2h > n_h2d ? n_d2h : n_h2d) : n_d2h + n_h2d;
  p.parts_log2 = static_cast<std::uint32_t>(parts_log2_for(n_dir, groups));
  const int items = n_dir << p.parts_log2;
  int ctas = fused ? items : (items + 1) / 2;
  if (ctas > max_ctas) ctas = max_ctas;
  if (ctas < 1) ctas = 1;
  if (flags & kNxNoChecksum)
    nx_swap_kernel<false, SwapParamsT<N>><<<ctas, 2 * kGroupThreads, 0, stream>>>(p);
  else
    nx_swap_kernel<true, SwapParamsT<N>><<<ctas, 2 * kGroupThreads, 0, stream>>>(p);
  return cudaGetLastError();
}

template <int N>
cudaError_t launch_checksum_tma_n(const NxLeg* legs, int n, bool arriving, std::uint32_t flags, const NxCkTables& ck,
                                  const NxScratch& scratch, int ctas, cudaStream_t stream, std::uint32_t clock_slot) {
  static bool configured = false;
  constexpr int kSmem = kTmaStages * kTmaChunk;
  if (!configured) {
    const cudaError_t e =
        cudaFuncSetAttribute(nx_checksum_tma_kernel<SwapParamsT<N>>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  SwapParamsT<N> p;
  for (int i = 0; i < n; ++i) p.legs[i] = legs[i];
  p.ck = ck;
  p.scratch = scratch;
  p.n_d2h = arriving ? 0u : static_cast<std::uint32_t>(n);
  p.n_h2d = arriving ? static_cast<std::uint32_t>(n) : 0u;
  p.parts_log2 = 0;
  p.clock_slot = (ck.kstart != nullptr && ck.kend != nullptr) ? clock_slot : kNoClockSlot;
  p.flags = flags;
  const int chunks = n * static_cast<int>(kTmaChunksPerLeg);
  if (ctas > chunks) ctas = chunks;
  nx_checksum_tma_kernel<SwapParamsT<N>><<<ctas, kTmaConsumers + 32, kSmem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_swap(const NxLeg* legs, int n_d2h, int n_h2d, std::uint32_t flags, const NxCkTables& ck,
                        const NxScratch& scratch, int max_ctas, cudaStream_t stream) {
  if (n_d2h < 0 || n_h2d < 0 || n_d2h + n_h2d > kMaxLegsPerLaunch) return cudaErrorInvalidValue;
  const int n = n_d2h + n_h2d;
  if (n == 0) return cudaSuccess;
  if (n <= 8) return launch_swap_n<8>(legs, n_d2h, n_h2d, flags, ck, scratch, max_ctas, stream);
  if (n <= 32) return launch_swap_n<32>(legs, n_d2h, n_h2d, flags, ck, scratch, max_ctas, stream);
  if (n <= 128) return launch_swap_n<128>(legs, n_d2h, n_h2d, flags, ck, scratch, max_ctas, stream);
  return launch_swap_n<kMaxLegsPerLaunch>(legs, n_d2h, n_h2d, flags, ck, scratch, max_ctas, stream);
}

template <int N>
cudaError_t launch_swap_tma_n(const NxLeg* legs, int n_d2h, int n_h2d, std::uint32_t flags, const NxCkTables& ck,
                              const NxScratch& scratch, int ctas, cudaStream_t stream) {
  static bool configured = false;
  constexpr int kSmem = kSwapTmaStages * kTmaChunk;
  if (!configured) {
    const cudaError_t e =
        cudaFuncSetAttribute(nx_swap_tma_kernel<SwapParamsT<N>>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  SwapParamsT<N> p;
  for (int i = 0; i < n_d2h + n_h2d; ++i) p.legs[i] = legs[i];
  p.ck = ck;
  p.scratch = scratch;
  p.n_d2h = static_cast<std::uint32_t>(n_d2h);
  p.n_h2d = static_cast<std::uint32_t>(n_h2d);
  p.parts_log2 = 0;
  p.flags = flags;
  p.clock_slot = kNoClockSlot;
  // no more CTAs than chunks: every CTA gets at least one
  const int chunks = (n_d2h + n_h2d) * static_cast<int>(kTmaChunksPerLeg);
  nx_swap_tma_kernel<SwapParamsT<N>><<<ctas < chunks ? ctas : chunks, kTmaConsumers + 32, kSmem, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_swap_tma(const NxLeg* legs, int n_d2h, int n_h2d, std::uint32_t flags, const NxCkTables& ck,
                            const NxScratch& scratch, int ctas, cudaStream_t stream) {
  if (n_d2h < 0 || n_h2d < 0 || n_d2h + n_h2d > kMaxLegsPerLaunch || ctas < 1) return cudaErrorInvalidValue;
  const int n = n_d2h + n_h2d;
  if (n == 0) return cudaSuccess;
  if (n <= 8) return launch_swap_tma_n<8>(legs, n_d2h, n_h2d, flags, ck, scratch, ctas, stream);
  if (n <= 32) return launch_swap_tma_n<32>(legs, n_d2h, n_h2d, flags, ck, scratch, ctas, stream);
  if (n <= 128) return launch_swap_tma_n<128>(legs, n_d2h, n_h2d, flags, ck, scratch, ctas, stream);
  return launch_swap_tma_n<kMaxLegsPerLaunch>(legs, n_d2h, n_h2d, flags, ck, scratch, ctas, stream);
}

cudaError_t launch_checksum_tma(const NxLeg* legs, int n, bool arriving, std::uint32_t flags, const NxCkTables& ck,
                                const NxScratch& scratch, int ctas, cudaStream_t stream, std::uint32_t slot) {
  if (n <= 0) return cudaSuccess;
  if (n > kMaxLegsPerLaunch) return cudaErrorInvalidValue;
  if (n <= 8) return launch_checksum_tma_n<8>(legs, n, arriving, flags, ck, scratch, ctas, stream, slot);
  if (n <= 32) return launch_checksum_tma_n<32>(legs, n, arriving, flags, ck, scratch, ctas, stream, slot);
  if (n <= 128) return launch_checksum_tma_n<128>(legs, n, arriving, flags, ck, scratch, ctas, stream, slot);
  return launch_checksum_tma_n<kMaxLegsPerLaunch>(legs, n, arriving, flags, ck, scratch, ctas, stream, slot);
}

cudaError_t launch_checksum_tma_table(const NxLeg* d_legs, int n, bool arriving, std::uint32_t flags, const NxCkTables& ck,
                                      const NxScratch& scratch, int ctas, cudaStream_t stream, std::uint32_t clock_slot) {
  if (n <= 0) return cudaSuccess;
  static bool configured = false;
  constexpr int kSmem = kTmaStages * kTmaChunk;
  if (!configured) {
    const cudaError_t e =
        cudaFuncSetAttribute(nx_checksum_tma_kernel<SwapParamsTable>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  SwapParamsTable p;
  p.legs = d_legs;
  p.ck = ck;
  p.scratch = scratch;
  p.n_d2h = arriving ? 0u : static_cast<std::uint32_t>(n);
  p.n_h2d = arriving ? static_cast<std::uint32_t>(n) : 0u;
  p.parts_log2 = 0;
  p.clock_slot = (ck.kstart != nullptr && ck.kend != nullptr) ? clock_slot : kNoClockSlot;
  p.flags = flags;
  const long long chunks = static_cast<long long>(n) * kTmaChunksPerLeg;
  if (ctas > chunks) ctas = static_cast<int>(chunks);
  nx_checksum_tma_kernel<SwapParamsTable><<<ctas, kTmaConsumers + 32, kSmem, stream>>>(p);
  return cudaGetLastError();
}

__global__ void nx_table_upload_kernel(std::uint64_t* __restrict__ dst, const std::uint64_t* __restrict__ src, std::uint32_t words) {
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < words; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

cudaError_t launch_table_upload(NxLeg* d_dst, const NxLeg* h_src, int n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  static_assert(sizeof(NxLeg) % 8 == 0, "descriptor is a whole number of words");
  const auto words = static_cast<std::uint32_t>(static_cast<std::size_t>(n) * sizeof(NxLeg) / 8);
  const int ctas = static_cast<int>(std::min<std::uint32_t>(32u, (words + 255u) / 256u));
  nx_table_upload_kernel<<<ctas, 256, 0, stream>>>(reinterpret_cast<std::uint64_t*>(d_dst),
                                                     reinterpret_cast<const std::uint64_t*>(h_src), words);
  return cudaGetLastError();
}

cudaError_t launch_fill(const NxLeg* legs, int n, std::uint64_t seed, const NxCkTables& ck, cudaStream_t stream) {
  for (int done = 0; done < n; done += kMaxLegsPerLaunch) {
    FillParams p;
    const int m = n - done < kMaxLegsPerLaunch ? n - done : kMaxLegsPerLaunch;
    for (int i = 0; i < m; ++i) p.legs[i] = legs[done + i];
    p.ck = ck;
    p.mismatches = nullptr;
    p.seed = seed;
    p.n = static_cast<std::uint32_t>(m);
    nx_pattern_kernel<true><<<m, 256, 0, stream>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_compare(const NxLeg* legs, int n, std::uint64_t seed, unsigned long long* mismatches,
                           cudaStream_t stream) {
  for (int done = 0; done < n; done += kMaxLegsPerLaunch) {
    FillParams p;
    const int m = n - done < kMaxLegsPerLaunch ? n - done : kMaxLegsPerLaunch;
    for (int i = 0; i < m; ++i) p.legs[i] = legs[done + i];
    p.ck = NxCkTables{};
    p.mismatches = mismatches + done;
    p.seed = seed;
    p.n = static_cast<std::uint32_t>(m);
    nx_pattern_kernel<false><<<m, 256, 0, stream>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace nixie::b200

// ---- launch-gate test kernel ---------------------------------------------------
// An "application kernel": checksums the app's blocks by reading them through
// the engine's device frame table (the stable-address stand-in). A missing
// frame is counted, never dereferenced.
namespace nixie::b200 {
namespace {
__global__ void __launch_bounds__(256) nx_table_checksum_kernel(const unsigned long long* __restrict__ table,
                                                                const unsigned* __restrict__ blocks, int n,
                                                                unsigned long long* out) {
  __shared__ unsigned long long red[8];
  const unsigned blk = blocks[blockIdx.x];
  const unsigned long long frame = table[blk];
  if (frame == 0ull) {
    if (threadIdx.x == 0) atomicAdd(out + 1, 1ull);
    return;
  }
  const uint4* src = reinterpret_cast<const uint4*>(frame);
  unsigned long long acc = 0;
  for (std::uint64_t j = threadIdx.x; j < kVecsPerBlock; j += blockDim.x) acc += ck16(ld_stream(src + j), j);
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < 8; ++w) t += red[w];
    atomicAdd(out, t);
  }
}
}  // namespace

cudaError_t launch_table_checksum(const std::uint64_t* table, const unsigned* blocks, int n, unsigned long long* out,
                                  cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  nx_table_checksum_kernel<<<n, 256, 0, stream>>>(reinterpret_cast<const unsigned long long*>(table), blocks, n, out);
  return cudaGetLastError();
}
}  // namespace nixie::b200
