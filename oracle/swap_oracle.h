/* TEST INFRASTRUCTURE ONLY (oracle/): CPU restatement of the byte-level
 * functions of the swap path, used by tests/ and bench.py's cpu_baseline leg
 * as the checker. The reference models no data contents, so
 * byte parity is pinned by this self-oracle: the synthetic pattern
 * (splitmix64(seed ^ app<<48 ^ block<<20 ^ word)) and the
 * per-block checksum the CUDA kernels compute
 * (paper_2601_11743_b200/csrc/cuda/nx_common.cuh). splitmix64 itself is
 * pinned by its published first output for seed 0 (0xE220A8397B1DCDAF). */
#ifndef SWAP_ORACLE_H_
#define SWAP_ORACLE_H_
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
uint64_t so_mix64(uint64_t z);
uint64_t so_splitmix64(uint64_t x);
uint64_t so_pattern_word(uint64_t seed, uint32_t app, uint64_t block, uint64_t word);
/* Fills a 2 MiB block with the pattern. */
void so_fill_block(uint64_t* dst, uint64_t seed, uint32_t app, uint64_t block);
/* Checksum of `nwords` 64-bit words (word index restarts at 0 per block):
 * sum of t ^ (t >> 32), t = (w_i ^ i*0x9E3779B97F4A7C15) * 0xD6E8FEB86659FD93. */
uint64_t so_checksum(const uint64_t* words, size_t nwords);
/* Checksum of the pattern block without materialising it. */
uint64_t so_pattern_block_checksum(uint64_t seed, uint32_t app, uint64_t block);
/* Number of 16-byte vectors of a 2 MiB block that differ from the pattern. */
uint64_t so_compare_block(const uint64_t* words, uint64_t seed, uint32_t app, uint64_t block);
/* CPU swap baseline: memcpy `n` 2 MiB blocks src[i] -> dst[i] on `threads`
 * threads; returns seconds. */
double so_copy_blocks(void** dst, void** src, size_t n, int threads);
#ifdef __cplusplus
}
#endif
#endif
