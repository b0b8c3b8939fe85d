/*
 * eh_synth.c -- seeded synthetic edge-list generators (RMAT, Erdos-Renyi).
 *
 * This module is the ONLY code shared by the CPU oracle (oracle/) and the
 * CUDA product path (paper_1503_02368_b200/): both consume the edge lists it
 * writes.  It holds none of the method's arithmetic (no canonicalisation,
 * dedup, ordering, trie, intersection or counting): it only draws tuples.
 *
 * The paper measures on public graphs (Table `table:datasets`,
 * PAPER.md:681-700) that are not available here; BASELINE.json's five
 * configs name RMAT / ER stand-ins.  The recipe (SURVEY.md §8(c) reading
 * c19):
 *
 *   RMAT (Graph500 quadrant rule, no noise): edge e, level l draws
 *     r = rng(seed, e, l) in [0, 2^53); quadrant a -> (0,0), b -> (0,1),
 *     c -> (1,0), d -> (1,1); u, v accumulate one bit per level (MSB first).
 *     Ids are then passed through a seeded bijection of [0, 2^scale) so that
 *     vertex id does not correlate with degree.  n_in = edge_factor * 2^scale.
 *   ER G(n, p): every pair i < j is kept iff rng(seed, pair) < p, emitted once
 *     as (i, j) or (j, i) by one further bit of the same draw.
 *
 * rng is a counter-based splitmix64 finaliser chain, so every tuple is a pure
 * function of (seed, index) and the generator parallelises trivially.
 */
#include <stdint.h>
#include <stddef.h>
#include <pthread.h>
#include <stdlib.h>

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* Counter-based draw: stream key from the seed, then one finaliser per counter. */
static inline uint64_t draw(uint64_t key, uint64_t ctr) { return mix64(key ^ mix64(ctr)); }

/* Probability -> 53-bit integer threshold (r53 < thr  <=>  U[0,1) < p). */
static uint64_t thr53(double p) {
  if (p <= 0.0) return 0;
  if (p >= 1.0) return 1ull << 53;
  return (uint64_t)(p * 9007199254740992.0); /* 2^53 */
}

/* Seeded bijection of [0, 2^scale): odd multiply, xorshift, odd multiply, add. */
static inline uint32_t scramble(uint64_t x, uint32_t scale, uint64_t k1, uint64_t k2, uint64_t k3) {
  const uint64_t mask = (scale >= 64) ? ~0ull : ((1ull << scale) - 1ull);
  const uint32_t s = scale / 2u;
  x = (x * (k1 | 1ull)) & mask;
  if (s) x ^= x >> s;
  x = (x * (k2 | 1ull)) & mask;
  if (s) x ^= x >> s;
  x = (x + k3) & mask;
  return (uint32_t)x;
}

typedef struct {
  uint32_t scale;
  uint64_t begin, end;
  uint64_t key, ta, tab, tabc;
  uint64_t k1, k2, k3;
  int do_scramble;
  uint32_t *src, *dst;
} rmat_job;

static void* rmat_worker(void* arg) {
  rmat_job* j = (rmat_job*)arg;
  for (uint64_t e = j->begin; e < j->end; ++e) {
    const uint64_t ek = mix64(j->key ^ (e * 0xD1B54A32D192ED03ull));
    uint64_t u = 0, v = 0;
    for (uint32_t l = 0; l < j->scale; ++l) {
      const uint64_t r = mix64(ek + (uint64_t)l * 0x9E3779B97F4A7C15ull) >> 11;
      const uint64_t bu = (r >= j->tab);                 /* c or d: row bit 1 */
      const uint64_t bv = (r >= j->ta && r < j->tab) | (r >= j->tabc); /* b or d */
      u = (u << 1) | bu;
      v = (v << 1) | bv;
    }
    if (j->do_scramble) {
      u = scramble(u, j->scale, j->k1, j->k2, j->k3);
      v = scramble(v, j->scale, j->k1, j->k2, j->k3);
    }
    j->src[e] = (uint32_t)u;
    j->dst[e] = (uint32_t)v;
  }
  return NULL;
}

/*
 * Fill src[0..n_edges), dst[0..n_edges) with RMAT tuples.
 * scale in [1, 32]; a + b + c <= 1 (d = 1 - a - b - c).  threads <= 0 -> 1.
 * Returns 0 on success, -1 on bad arguments.
 */
int eh_synth_rmat(uint32_t scale, uint64_t n_edges, double a, double b, double c,
                  uint64_t seed, int do_scramble, uint32_t* src, uint32_t* dst, int threads) {
  if (scale < 1 || scale > 32 || (!src && n_edges) || (!dst && n_edges)) return -1;
  if (a < 0 || b < 0 || c < 0 || a + b + c > 1.0 + 1e-12) return -1;
  if (threads <= 0) threads = 1;
  if ((uint64_t)threads > n_edges / 4096 + 1) threads = (int)(n_edges / 4096 + 1);
  const uint64_t key = mix64(seed ^ 0x5EED5EED5EED5EEDull);
  rmat_job* jobs = (rmat_job*)calloc((size_t)threads, sizeof(rmat_job));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  if (!jobs || !tids) { free(jobs); free(tids); return -1; }
  for (int t = 0; t < threads; ++t) {
    rmat_job* j = &jobs[t];
    j->scale = scale;
    j->begin = n_edges * (uint64_t)t / (uint64_t)threads;
    j->end = n_edges * (uint64_t)(t + 1) / (uint64_t)threads;
    j->key = key;
    j->ta = thr53(a);
    j->tab = thr53(a + b);
    j->tabc = thr53(a + b + c);
    j->k1 = mix64(key ^ 1);
    j->k2 = mix64(key ^ 2);
    j->k3 = mix64(key ^ 3);
    j->do_scramble = do_scramble;
    j->src = src;
    j->dst = dst;
  }
  for (int t = 1; t < threads; ++t) pthread_create(&tids[t], NULL, rmat_worker, &jobs[t]);
  rmat_worker(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tids[t], NULL);
  free(jobs);
  free(tids);
  return 0;
}

/*
 * Erdos-Renyi G(n, p): pairs i < j in lexicographic order, kept iff
 * draw < p; direction from bit 0 of the draw.  If src == NULL only counts.
 * Writes at most cap tuples.  Returns the number of kept pairs.
 */
uint64_t eh_synth_er(uint32_t n, double p, uint64_t seed, uint32_t* src, uint32_t* dst, uint64_t cap) {
  const uint64_t key = mix64(seed ^ 0xE7E7E7E7E7E7E7E7ull);
  const uint64_t tp = thr53(p);
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; ++i) {
    for (uint64_t jj = i + 1; jj < n; ++jj) {
      const uint64_t r = draw(key, i * (uint64_t)n + jj);
      if ((r >> 11) < tp) {
        if (src && k < cap) {
          if (r & 1ull) { src[k] = (uint32_t)jj; dst[k] = (uint32_t)i; }
          else          { src[k] = (uint32_t)i;  dst[k] = (uint32_t)jj; }
        }
        ++k;
      }
    }
  }
  return k;
}

/* 64-bit FNV-1a-style checksum of an edge list (recorded next to counts). */
uint64_t eh_synth_checksum(const uint32_t* src, const uint32_t* dst, uint64_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < n; ++i) {
    h = (h ^ src[i]) * 0x100000001b3ull;
    h = (h ^ dst[i]) * 0x100000001b3ull;
  }
  return h;
}
