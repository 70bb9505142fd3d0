/* TEST INFRASTRUCTURE ONLY (oracle/). See swap_oracle.h. */
#define _GNU_SOURCE
#include "swap_oracle.h"

#include <pthread.h>
#include <string.h>
#include <time.h>

#define SO_GOLDEN 0x9E3779B97F4A7C15ull
#define SO_BLOCK_WORDS (2u * 1024u * 1024u / 8u)
#define SO_CK_MUL 0xD6E8FEB86659FD93ull

/* Checksum term of word w at word index i (paper_2601_11743_b200/csrc/cuda/nx_common.cuh). */
static uint64_t so_ck_term(uint64_t w, uint64_t i) {
  uint64_t t = (w ^ (i * SO_GOLDEN)) * SO_CK_MUL;
  return t ^ (t >> 32);
}

uint64_t so_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t so_splitmix64(uint64_t x) { return so_mix64(x + SO_GOLDEN); }

uint64_t so_pattern_word(uint64_t seed, uint32_t app, uint64_t block, uint64_t word) {
  return so_splitmix64(seed ^ ((uint64_t)app << 48) ^ (block << 20) ^ word);
}

void so_fill_block(uint64_t* dst, uint64_t seed, uint32_t app, uint64_t block) {
  for (uint64_t w = 0; w < SO_BLOCK_WORDS; ++w) dst[w] = so_pattern_word(seed, app, block, w);
}

uint64_t so_checksum(const uint64_t* words, size_t nwords) {
  uint64_t s = 0;
  for (size_t i = 0; i < nwords; ++i) s += so_ck_term(words[i], (uint64_t)(i % SO_BLOCK_WORDS));
  return s;
}

uint64_t so_pattern_block_checksum(uint64_t seed, uint32_t app, uint64_t block) {
  uint64_t s = 0;
  for (uint64_t w = 0; w < SO_BLOCK_WORDS; ++w) s += so_ck_term(so_pattern_word(seed, app, block, w), w);
  return s;
}

uint64_t so_compare_block(const uint64_t* words, uint64_t seed, uint32_t app, uint64_t block) {
  uint64_t bad = 0;
  for (uint64_t v = 0; v < SO_BLOCK_WORDS / 2; ++v)
    bad += (words[2 * v] != so_pattern_word(seed, app, block, 2 * v) ||
            words[2 * v + 1] != so_pattern_word(seed, app, block, 2 * v + 1));
  return bad;
}

struct so_job {
  void** dst;
  void** src;
  size_t lo, hi;
};

static void* so_worker(void* p) {
  struct so_job* j = (struct so_job*)p;
  for (size_t i = j->lo; i < j->hi; ++i) memcpy(j->dst[i], j->src[i], 2u * 1024u * 1024u);
  return NULL;
}

double so_copy_blocks(void** dst, void** src, size_t n, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  struct so_job jobs[256];
  struct timespec a, b;
  clock_gettime(CLOCK_MONOTONIC, &a);
  for (int t = 0; t < threads; ++t) {
    jobs[t].dst = dst;
    jobs[t].src = src;
    jobs[t].lo = n * (size_t)t / (size_t)threads;
    jobs[t].hi = n * (size_t)(t + 1) / (size_t)threads;
    pthread_create(&tid[t], NULL, so_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  clock_gettime(CLOCK_MONOTONIC, &b);
  return (double)(b.tv_sec - a.tv_sec) + 1e-9 * (double)(b.tv_nsec - a.tv_nsec);
}
