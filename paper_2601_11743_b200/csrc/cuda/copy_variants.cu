// Raw host-link copy variants, used by the probe to pick the SM copy
// mechanism (development + calibration; no checksum):
//   0  LDG/STG 16-byte vectors, 8 in flight per thread (the K1 inner loop)
//   1  same with the .L2::256B prefetch-size hint on the loads
//   2  TMA bulk copies: cp.async.bulk global->shared (mbarrier complete_tx)
//      then shared->global (bulk_group), 4-stage ring of 32 KiB per CTA
//   3  as 2 with 64 KiB stages (2 stages... 4 x 48 KiB ring)
#include <cuda_runtime.h>

#include <cstdint>

#include "nx_common.cuh"
#include "nx_tma.cuh"

namespace nixie::b200 {

namespace {

template <bool kHint>
__global__ void __launch_bounds__(256) nx_raw_ldg_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                         std::uint64_t nvec) {
  constexpr int U = 8;
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x * U;
  for (std::uint64_t b = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x * U + threadIdx.x; b < nvec; b += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint4* p = src + b + u * blockDim.x;
      if (b + u * blockDim.x < nvec) {
        if (kHint)
          asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                       : "l"(p));
        else
          asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                       : "l"(p));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (b + u * blockDim.x < nvec)
        asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst + b + u * blockDim.x), "r"(v[u].x),
                     "r"(v[u].y), "r"(v[u].z), "r"(v[u].w)
                     : "memory");
  }
}

// One thread per CTA drives a kStages-deep ring of kChunk-byte stages over the
// CTA's contiguous share of [src, src + bytes).
template <int kChunk, int kStages>
__global__ void __launch_bounds__(32) nx_raw_tma_kernel(const std::uint8_t* __restrict__ src, std::uint8_t* __restrict__ dst,
                                                        std::uint64_t bytes) {
  extern __shared__ __align__(128) std::uint8_t ring[];
  __shared__ __align__(8) std::uint64_t full[kStages];
  const std::uint64_t nchunks = bytes / kChunk;
  const std::uint64_t per = (nchunks + gridDim.x - 1) / gridDim.x;
  const std::uint64_t c0 = static_cast<std::uint64_t>(blockIdx.x) * per;
  const std::uint64_t c1 = c0 + per < nchunks ? c0 + per : nchunks;
  if (threadIdx.x != 0 || c0 >= c1) return;
  for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
  mbar_fence_init();
  const std::uint64_t n = c1 - c0;
  for (std::uint64_t i = 0; i < n && i < static_cast<std::uint64_t>(kStages); ++i) {
    mbar_expect_tx(&full[i], kChunk);
    bulk_load(ring + i * kChunk, src + (c0 + i) * kChunk, kChunk, &full[i]);
  }
  for (std::uint64_t i = 0; i < n; ++i) {
    const int s = static_cast<int>(i % kStages);
    mbar_wait(&full[s], static_cast<unsigned>((i / kStages) & 1));
    bulk_store(dst + (c0 + i) * kChunk, ring + s * kChunk, kChunk);
    // Refill the stage of chunk i-1 once its store has read shared memory.
    if (i >= 1 && i - 1 + kStages < n) {
      bulk_wait_read<1>();
      const int r = static_cast<int>((i - 1) % kStages);
      mbar_expect_tx(&full[r], kChunk);
      bulk_load(ring + r * kChunk, src + (c0 + i - 1 + kStages) * kChunk, kChunk, &full[r]);
    }
  }
  // The last refill opportunity is skipped for i == 0; handle kStages == n edge by construction.
  bulk_wait_all();
}

__global__ void nx_spin_kernel(unsigned ns) {
  const unsigned long long t0 = clock64();
  (void)t0;
  for (unsigned waited = 0; waited < ns; waited += 1000) __nanosleep(1000);
}

}  // namespace

// Keeps a stream busy for ~ns so that events recorded after it time the next
// kernel alone, not the host's launch latency (timing probes only).
cudaError_t launch_spin(unsigned ns, cudaStream_t stream) {
  nx_spin_kernel<<<1, 32, 0, stream>>>(ns);
  return cudaGetLastError();
}

cudaError_t launch_raw_copy(int variant, void* dst, const void* src, std::uint64_t bytes, int ctas, cudaStream_t stream) {
  switch (variant) {
    case 0:
      nx_raw_ldg_kernel<false><<<ctas, 256, 0, stream>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst), bytes / 16);
      break;
    case 1:
      nx_raw_ldg_kernel<true><<<ctas, 256, 0, stream>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst), bytes / 16);
      break;
    case 2: {
      constexpr int C = 32 << 10, S = 4;
      static bool set = false;
      if (!set) {
        cudaFuncSetAttribute(nx_raw_tma_kernel<C, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, C * S);
        set = true;
      }
      nx_raw_tma_kernel<C, S><<<ctas, 32, C * S, stream>>>(static_cast<const std::uint8_t*>(src), static_cast<std::uint8_t*>(dst), bytes);
      break;
    }
    case 3: {
      constexpr int C = 48 << 10, S = 4;
      static bool set = false;
      if (!set) {
        cudaFuncSetAttribute(nx_raw_tma_kernel<C, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, C * S);
        set = true;
      }
      nx_raw_tma_kernel<C, S><<<ctas, 32, C * S, stream>>>(static_cast<const std::uint8_t*>(src), static_cast<std::uint8_t*>(dst), bytes);
      break;
    }
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace nixie::b200
