// Launch interface of the sm_100a kernels (implemented in swap_kernels.cu),
// callable from host C++ compiled by g++.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace nixie::b200 {

// One 2 MiB leg. src/dst are device-visible addresses: HBM frames or mapped
// pinned-host slots (UVA). For checksum-only legs dst is null; for fill /
// compare legs `tag` carries the app id.
struct NxLeg {
  const void* src;
  void* dst;
  std::uint32_t block;
  std::uint32_t tag;
};

inline constexpr int kMaxLegsPerLaunch = 256;  // d2h + h2d legs in one launch (kernel-parameter resident)
inline constexpr int kMaxPartsLog2 = 4;        // a leg splits into at most 16 parts

// Device-resident counters, read back once per switch.
struct NxDevStatus {
  unsigned long long mismatches;   // restores whose checksum differed from the departure checksum
  unsigned long long verified;     // restores checked
  unsigned long long unverified;   // restores of blocks with no recorded checksum
  unsigned int n_bad;
  unsigned int bad_blocks[64];
};

// Per-block checksum state (device arrays indexed by BlockId) plus the
// per-stream scratch used to combine parts of a split leg.
struct NxCkTables {
  unsigned long long* ck_ref;   // checksum recorded when the block last left the GPU (or was filled)
  unsigned long long* ck_seen;  // checksum observed at the last arrival on the GPU
  unsigned int* ck_valid;       // 1 if ck_ref is meaningful
  NxDevStatus* status;
  // Device-clock span of each K3 launch (%globaltimer ns): first CTA start
  // (atomicMin, preset to ~0) and last CTA end (atomicMax, preset to 0).
  unsigned long long* kstart;
  unsigned long long* kend;
};

inline constexpr std::uint32_t kNoClockSlot = 0xFFFFFFFFu;
inline constexpr int kClockSlots = 8192;

struct NxScratch {
  unsigned long long* part_sums;  // [kMaxLegsPerLaunch << kMaxPartsLog2]
  unsigned int* part_count;       // [kMaxLegsPerLaunch], self-resetting
  unsigned long long* leg_acc;    // [kMaxLegsPerLaunch], zero at rest (TMA checksum), self-resetting
};

enum NxSwapFlags : std::uint32_t {
  kNxVerify = 1u,      // compare arrival checksums with ck_ref
  kNxNoChecksum = 2u,  // raw copy (probe only)
};

// K1: bidirectional swap. Legs [0, n_d2h) leave the GPU (their checksum is
// recorded), legs [n_d2h, n_d2h + n_h2d) arrive (their checksum is checked).
// With both lists non-empty every CTA runs one D2H warp group and one H2D
// warp group; with one list, both groups serve it. Legs with dst == nullptr
// are checksum-only (K3). Returns the launch error.
cudaError_t launch_swap(const NxLeg* legs, int n_d2h, int n_h2d, std::uint32_t flags, const NxCkTables& ck,
                        const NxScratch& scratch, int max_ctas, cudaStream_t stream);

// K1T: the same swap (same legs, checksum record/verify, every dst non-null)
// on the TMA pipeline: `ctas` CTAs each stream a balanced range of 32 KiB
// chunks through a 4-stage shared-memory ring with cp.async.bulk loads and
// stores; 16 consumer warps checksum each stage. kNxNoChecksum: copy only.
cudaError_t launch_swap_tma(const NxLeg* legs, int n_d2h, int n_h2d, std::uint32_t flags, const NxCkTables& ck,
                            const NxScratch& scratch, int ctas, cudaStream_t stream);

// K3 on the TMA pipeline: checksum-only pass over `n` legs of HBM frames
// (legs[i].src), recorded (arriving = false) or verified (arriving = true).
// One CTA per SM: a producer thread streams 32 KiB cp.async.bulk chunks into
// a 6-stage shared-memory ring, 16 consumer warps checksum from shared memory.
cudaError_t launch_checksum_tma(const NxLeg* legs, int n, bool arriving, std::uint32_t flags, const NxCkTables& ck,
                                const NxScratch& scratch, int ctas, cudaStream_t stream,
                                std::uint32_t clock_slot = kNoClockSlot);

// Same pass over a DEVICE-resident leg table of any length (d_legs[0..n)).
// `scratch` must hold n entries (part_count and leg_acc zero at rest). One
// launch covers a whole switch's departures or a group of arrival batches:
// under PCIe load every launch pays a fixed ~30 us on the GPU's launch path
// (tools/k3_probe.py), so fewer, larger launches run closer to HBM speed.
cudaError_t launch_checksum_tma_table(const NxLeg* d_legs, int n, bool arriving, std::uint32_t flags, const NxCkTables& ck,
                                      const NxScratch& scratch, int ctas, cudaStream_t stream,
                                      std::uint32_t clock_slot = kNoClockSlot);

// Copies `n` leg descriptors from pinned host memory into the device table
// with SM loads (one small launch on the K3 stream). A cudaMemcpyAsync would
// queue on the host->device copy engine behind the switch's own fetch copies
// and hold every arrival check until the last fetch landed.
cudaError_t launch_table_upload(NxLeg* d_dst, const NxLeg* h_src, int n, cudaStream_t stream);

// K4: pattern fill (records checksums, marks them valid) and compare (adds
// the number of mismatching 16-byte vectors per leg into mismatches[i]).
cudaError_t launch_fill(const NxLeg* legs, int n, std::uint64_t seed, const NxCkTables& ck, cudaStream_t stream);
cudaError_t launch_compare(const NxLeg* legs, int n, std::uint64_t seed, unsigned long long* mismatches,
                           cudaStream_t stream);

// Number of SMs and the resident-CTA count used to size grids.
int device_sm_count(int device);

}  // namespace nixie::b200

namespace nixie::b200 {
// Launch-gate test kernel: out[0] += sum of block checksums read through the
// frame table, out[1] += number of blocks with no frame.
// One warp busy for ~ns (timing probes; synthetic application kernels).
cudaError_t launch_spin(unsigned ns, cudaStream_t stream);
cudaError_t launch_table_checksum(const std::uint64_t* table, const unsigned* blocks, int n, unsigned long long* out,
                                  cudaStream_t stream);
}  // namespace nixie::b200
