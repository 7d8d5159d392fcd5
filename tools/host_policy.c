/* The e2e leg's host policy (bench.py): for every agent, a uniform legal action
 * from its returned 5-byte action mask -- the same rule as the device's random
 * policy (vecenv.cpp:125-134: the j-th legal action, j = floor(u * #legal)), on
 * its own splitmix64 stream. Harness code (a stand-in for the caller's policy),
 * not part of the product; padding agents with no legal action get 0.
 *
 *   gcc -O3 -shared -fPIC -fopenmp -o tools/_lib/libhost_policy.so tools/host_policy.c
 */
#include <stdint.h>

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* masks: n_agents x 5 bytes (0/1); actions: n_agents int32; *counter advances
 * by n_agents per call (the stream position); n_threads: the host threads this
 * rank may use (the node's cores split over its ranks). */
static int32_t kth[32][5];
static int kth_ready = 0;

static void kth_init(void) {
  for (unsigned c = 0; c < 32; ++c) {
    int n = 0;
    for (int b = 0; b < 5; ++b)
      if ((c >> b) & 1u) kth[c][n++] = b;
  }
  kth_ready = 1;
}

void host_policy(const uint8_t* masks, int64_t n_agents, int32_t* actions, uint64_t seed, uint64_t* counter,
                 int n_threads) {
  const uint64_t base = *counter;
  if (!kth_ready) kth_init();
#pragma omp parallel for schedule(static) num_threads(n_threads)
  for (int64_t i = 0; i < n_agents; ++i) {
    const uint8_t* m = masks + 5 * i;
    const unsigned code = (unsigned)m[0] | (unsigned)m[1] << 1 | (unsigned)m[2] << 2 | (unsigned)m[3] << 3 |
                          (unsigned)m[4] << 4;
    const unsigned nl = (unsigned)__builtin_popcount(code);
    const uint32_t r = (uint32_t)(splitmix64(seed ^ (base + (uint64_t)i)) >> 32);
    const unsigned j = (unsigned)(((uint64_t)r * nl) >> 32); /* floor(u * #legal) */
    const int32_t a = kth[code][j];                            /* branch-free: the j-th set bit */
    actions[i] = a;
  }
  *counter = base + (uint64_t)n_agents;
}
