// Shared by the sm_100a kernels and the engine's host code: the synthetic
// working-set pattern and the per-block checksum.
//
// Checksum of a 2 MiB block = sum over its 64-bit words w_i (i = word index
// within the block) of ck_term(w_i, i) (below), mod 2^64. It is a sum, so any
// split of the block over warps, CTAs or launches reduces to the same value,
// and the position term catches swapped or misplaced words. The swap kernel
// computes it while the bytes stream through registers (no extra HBM pass).
// oracle/swap_oracle.c restates both functions in C as the checker.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define NX_HD __host__ __device__ __forceinline__
#else
#define NX_HD inline
#endif

namespace nixie::b200 {

inline constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ull;
inline constexpr std::uint64_t kBlockBytesDev = 2ull << 20;
inline constexpr std::uint64_t kVecsPerBlock = kBlockBytesDev / 16;  // 131072 16-byte vectors

NX_HD std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// First output of splitmix64 seeded with x.
NX_HD std::uint64_t splitmix64(std::uint64_t x) { return mix64(x + kGolden); }

// Word `w` (0 .. 262143) of block `block` of app `app` in the synthetic
// working set.
NX_HD std::uint64_t pattern_word(std::uint64_t seed, std::uint32_t app, std::uint64_t block, std::uint64_t w) {
  return splitmix64(seed ^ (static_cast<std::uint64_t>(app) << 48) ^ (block << 20) ^ w);
}

// Checksum term of the 64-bit word at word index `index` of its block:
// (word ^ index*golden) * kCkMul, xor-folded. Multiplying by an odd constant
// and the fold are bijections, so any change to a word changes its term; the
// position key makes swapped words change the sum. One 64-bit multiply per
// word keeps the checksum well below the HBM roofline's instruction budget.
inline constexpr std::uint64_t kCkMul = 0xD6E8FEB86659FD93ull;
NX_HD std::uint64_t ck_term_keyed(std::uint64_t word, std::uint64_t key) {
  const std::uint64_t t = (word ^ key) * kCkMul;
  return t ^ (t >> 32);
}
NX_HD std::uint64_t ck_term(std::uint64_t word, std::uint64_t index) { return ck_term_keyed(word, index * kGolden); }

}  // namespace nixie::b200
