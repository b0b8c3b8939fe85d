/*
 * eh_oracle.c -- the CPU ORACLE for the EmptyHeaded (arXiv 1503.02368) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` legs may load, call or link this file.  The
 * product path (paper_1503_02368_b200/, include/eh.h) never does, and the two
 * share no code: no headers, helpers, constants or pre/post-processing.
 *
 * It is a plain, slow, obviously correct implementation of what the path
 * computes, written from PAPER.md in the paper's order:
 *
 *   ingest    ("Dictionary Encoding", "Column (Index) Order";
 *              PAPER.md:799-800 pruning "src_id > dst_id and id's are assigned
 *              based upon the degree of the node")
 *     1. each input pair (u, v), u != v, becomes the canonical key (min, max);
 *        qsort + unique give the distinct undirected edges ("sets of distinct
 *        values").  Self-loops dropped (reading c5).
 *     2. deg(v) = number of distinct neighbours (reading c4).
 *     3. total order  u < v  iff  (deg u, u) < (deg v, v), u, v ORIGINAL ids
 *        (readings c2, c3).
 *     4. E+ = {(u, v) : {u, v} an edge, u < v}; every out-list N+(u) is sorted
 *        by ORIGINAL id -- deliberately not the rank space the CUDA path uses.
 *   triangle (Generic-Join of Alg. `fig:worst_case`,
 *             PAPER.md:172-192, with R = S = T = E+):
 *        for x in pi_X R  cap  pi_X T
 *          for y in R[x]  cap  pi_Y S
 *            Q += | S[y]  cap  T[x] |          (scalar two-pointer merge)
 *   4-clique (PAPER.md:217 4Clique(x,y,z,w) :- R(x,y),S(y,z),T(x,z),U(x,w),
 *             V(y,w),Q(z,w); Generic-Join in attribute order x, y, z, w):
 *        for x in pi_X R cap pi_X T cap pi_X U
 *          for y in R[x] cap pi_Y S cap pi_Y V
 *            P = S[y] cap T[x]      (= U[x] cap V[y]: the same two sets)
 *            for z in P cap pi_Z Q
 *              K += | P cap Q[z] |          (two scalar merges in total)
 *   COUNT(*) is a uint64 sum ("w:long"; reading c9).
 *   Rank ranges: both nests with x restricted to the vertices whose rank (their
 *   position in the order of step 3) lies in [r0, r1) -- sampled outputs for
 *   sizes where the full count is out of the oracle's reach.
 *   NEXT-1 / NEXT-2: per-vertex counts + Lollipop / Barbell,
 *   and the unpruned nests on the symmetric data -- see their sections below.
 *   intersect (Table `lst:eh_operators`): sorted merge.
 *
 * Parallelism: only the outermost x loop is split over pthreads, with one
 * uint64 partial sum per thread; integer addition makes the result identical
 * at every thread count.
 *
 * Pins (tests/test_oracle_*.py, run with -m "not gpu"): brute-force O(n^3) /
 * O(n^4) enumeration, trace(A^3)/6, C(n,3) / C(n,4) on K_n, e3 / e4 of the part
 * sizes on complete r-partite graphs, 0 on bipartite graphs, wheel W_k -> k,
 * the worked examples W1-W3 (tests/golden/), invariances.  No function here is
 * "parity unpinned".
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint64_t n_input;  /* input tuples */
  uint64_t m;        /* distinct undirected edges (no self-loops) */
  uint64_t nv;       /* non-isolated vertices */
  uint64_t max_out;  /* max |N+(x)| */
  uint32_t* vid;     /* [nv] sorted distinct original ids */
  uint32_t* deg;     /* [nv] degree */
  uint64_t* off;     /* [nv+1] out-list offsets */
  uint32_t* adj;     /* [m] out-neighbours (original ids), sorted per list */
  uint64_t* soff;    /* NEXT-2, built on first use: [nv+1] offsets of the full neighbour lists */
  uint32_t* sadj;    /* [2m] all neighbours (original ids), sorted per list */
} oracle_graph;

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}
static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

/* index of original id v in g->vid (v must be present) */
static uint64_t vindex(const oracle_graph* g, uint32_t v) {
  const uint32_t* p = (const uint32_t*)bsearch(&v, g->vid, g->nv, sizeof(uint32_t), cmp_u32);
  return (uint64_t)(p - g->vid);
}

/* u precedes v in the (degree, original id) order */
static int precedes(const oracle_graph* g, uint64_t iu, uint64_t iv) {
  if (g->deg[iu] != g->deg[iv]) return g->deg[iu] < g->deg[iv];
  return g->vid[iu] < g->vid[iv];
}

void oracle_free(oracle_graph* g) {
  if (!g) return;
  free(g->vid); free(g->deg); free(g->off); free(g->adj); free(g->soff); free(g->sadj); free(g);
}

oracle_graph* oracle_build(const uint32_t* src, const uint32_t* dst, uint64_t n) {
  oracle_graph* g = (oracle_graph*)calloc(1, sizeof(oracle_graph));
  if (!g) return NULL;
  g->n_input = n;
  /* 1. canonical keys, sort, unique */
  uint64_t* key = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  if (!key) { free(g); return NULL; }
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t u = src[i], v = dst[i];
    if (u == v) continue;
    if (u > v) { uint32_t t = u; u = v; v = t; }
    key[k++] = ((uint64_t)u << 32) | v;
  }
  qsort(key, k, sizeof(uint64_t), cmp_u64);
  uint64_t m = 0;
  for (uint64_t i = 0; i < k; ++i)
    if (i == 0 || key[i] != key[i - 1]) key[m++] = key[i];
  g->m = m;
  /* 2. vertices and degrees: each distinct edge adds one to each endpoint */
  uint32_t* ends = (uint32_t*)malloc((2 * m ? 2 * m : 1) * sizeof(uint32_t));
  if (!ends) { free(key); free(g); return NULL; }
  for (uint64_t i = 0; i < m; ++i) {
    ends[2 * i] = (uint32_t)(key[i] >> 32);
    ends[2 * i + 1] = (uint32_t)key[i];
  }
  qsort(ends, 2 * m, sizeof(uint32_t), cmp_u32);
  uint64_t nv = 0;
  for (uint64_t i = 0; i < 2 * m; ++i)
    if (i == 0 || ends[i] != ends[i - 1]) ++nv;
  g->nv = nv;
  g->vid = (uint32_t*)malloc((nv ? nv : 1) * sizeof(uint32_t));
  g->deg = (uint32_t*)calloc(nv ? nv : 1, sizeof(uint32_t));
  g->off = (uint64_t*)calloc(nv + 1, sizeof(uint64_t));
  g->adj = (uint32_t*)malloc((m ? m : 1) * sizeof(uint32_t));
  if (!g->vid || !g->deg || !g->off || !g->adj) { free(ends); free(key); oracle_free(g); return NULL; }
  for (uint64_t i = 0, j = 0; i < 2 * m; ++i) {
    if (i == 0 || ends[i] != ends[i - 1]) g->vid[j++] = ends[i];
    g->deg[j - 1] += 1;
  }
  free(ends);
  /* 3.-4. orient each edge from the earlier to the later vertex of the order */
  uint64_t* fill = (uint64_t*)calloc(nv + 1, sizeof(uint64_t));
  if (!fill) { free(key); oracle_free(g); return NULL; }
  for (uint64_t i = 0; i < m; ++i) {
    const uint64_t iu = vindex(g, (uint32_t)(key[i] >> 32)), iv = vindex(g, (uint32_t)key[i]);
    g->off[(precedes(g, iu, iv) ? iu : iv) + 1] += 1;
  }
  for (uint64_t i = 0; i < nv; ++i) g->off[i + 1] += g->off[i];
  for (uint64_t i = 0; i < m; ++i) {
    const uint32_t u = (uint32_t)(key[i] >> 32), v = (uint32_t)key[i];
    const uint64_t iu = vindex(g, u), iv = vindex(g, v);
    if (precedes(g, iu, iv)) g->adj[g->off[iu] + fill[iu]++] = v;
    else                     g->adj[g->off[iv] + fill[iv]++] = u;
  }
  free(fill);
  free(key);
  for (uint64_t i = 0; i < nv; ++i) {
    const uint64_t d = g->off[i + 1] - g->off[i];
    if (d > g->max_out) g->max_out = d;
    qsort(g->adj + g->off[i], d, sizeof(uint32_t), cmp_u32);
  }
  return g;
}

/* |a cap b| by the scalar two-pointer merge */
static uint64_t merge_count(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb) {
  uint64_t i = 0, j = 0, c = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j]) ++i;
    else if (a[i] > b[j]) ++j;
    else { ++c; ++i; ++j; }
  }
  return c;
}

/* a cap b written to out (if non-NULL); returns the count */
static uint64_t merge_into(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb, uint32_t* out) {
  uint64_t i = 0, j = 0, c = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j]) ++i;
    else if (a[i] > b[j]) ++j;
    else { if (out) out[c] = a[i]; ++c; ++i; ++j; }
  }
  return c;
}

int64_t oracle_intersect(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb, uint32_t* out) {
  return (int64_t)merge_into(a, na, b, nb, out);
}

#define OUT(g, i) ((g)->adj + (g)->off[i])
#define DOUT(g, i) ((g)->off[(i) + 1] - (g)->off[i])

/* Triangle loop nest for x in vertex-index range [x0, x1);
 * with ord != NULL, x runs over ord[x0 .. x1) instead (rank ranges, below). */
static uint64_t tri_range(const oracle_graph* g, uint64_t x0, uint64_t x1, const uint64_t* ord) {
  uint64_t q = 0;
  for (uint64_t p = x0; p < x1; ++p) {
    const uint64_t x = ord ? ord[p] : p;
    if (DOUT(g, x) == 0) continue;                  /* x in pi_X R cap pi_X T */
    for (uint64_t e = g->off[x]; e < g->off[x + 1]; ++e) {
      const uint64_t y = vindex(g, g->adj[e]);      /* y in R[x] */
      if (DOUT(g, y) == 0) continue;                /* y in pi_Y S */
      q += merge_count(OUT(g, y), DOUT(g, y), OUT(g, x), DOUT(g, x)); /* S[y] cap T[x] */
    }
  }
  return q;
}

/* 4-clique loop nest for x in [x0, x1), attribute order x, y, z, w. */
static uint64_t k4_range(const oracle_graph* g, uint64_t x0, uint64_t x1, uint32_t* P, const uint64_t* ord) {
  uint64_t k = 0;
  for (uint64_t p = x0; p < x1; ++p) {
    const uint64_t x = ord ? ord[p] : p;
    if (DOUT(g, x) == 0) continue;
    for (uint64_t e = g->off[x]; e < g->off[x + 1]; ++e) {
      const uint64_t y = vindex(g, g->adj[e]);
      if (DOUT(g, y) == 0) continue;
      const uint64_t np = merge_into(OUT(g, y), DOUT(g, y), OUT(g, x), DOUT(g, x), P);
      for (uint64_t t = 0; t < np; ++t) {
        const uint64_t z = vindex(g, P[t]);
        if (DOUT(g, z) == 0) continue;              /* z in pi_Z Q */
        k += merge_count(P, np, OUT(g, z), DOUT(g, z));
      }
    }
  }
  return k;
}

/*
 * NEXT-2: the same Generic-Join on the UNPRUNED data -- the
 * symmetric Edge relation, every undirected edge in both directions, no
 * symmetry breaking ("Default" vs "Symmetrically
 * Filtered").  Every binding is an ordered tuple, so the results are 6T and
 * 24 K4 ("a multiple of the former").
 *   triangle: for x, for y in N(x): Q += |N(y) cap N(x)|
 *   4-clique: for x, for y in N(x): P = N(y) cap N(x); for z in P: K += |P cap N(z)|
 */
#define NB(g, i) ((g)->sadj + (g)->soff[i])
#define DN(g, i) ((g)->soff[(i) + 1] - (g)->soff[i])

/* Full neighbour lists N(v) (sorted by original id) from E+; idempotent. */
static int build_symmetric(oracle_graph* g) {
  if (g->soff) return 0;
  uint64_t* soff = (uint64_t*)calloc(g->nv + 1, sizeof(uint64_t));
  uint32_t* sadj = (uint32_t*)malloc((2 * g->m ? 2 * g->m : 1) * sizeof(uint32_t));
  uint64_t* fill = (uint64_t*)calloc(g->nv + 1, sizeof(uint64_t));
  if (!soff || !sadj || !fill) { free(soff); free(sadj); free(fill); return -1; }
  for (uint64_t i = 0; i < g->nv; ++i) soff[i + 1] = soff[i] + g->deg[i];
  for (uint64_t x = 0; x < g->nv; ++x)
    for (uint64_t e = g->off[x]; e < g->off[x + 1]; ++e) {
      const uint64_t y = vindex(g, g->adj[e]);
      sadj[soff[x] + fill[x]++] = g->adj[e];
      sadj[soff[y] + fill[y]++] = g->vid[x];
    }
  for (uint64_t i = 0; i < g->nv; ++i) qsort(sadj + soff[i], soff[i + 1] - soff[i], sizeof(uint32_t), cmp_u32);
  free(fill);
  g->sadj = sadj;
  g->soff = soff;
  return 0;
}

static uint64_t tri_unpruned_range(const oracle_graph* g, uint64_t x0, uint64_t x1) {
  uint64_t q = 0;
  for (uint64_t x = x0; x < x1; ++x)
    for (uint64_t e = g->soff[x]; e < g->soff[x + 1]; ++e) {
      const uint64_t y = vindex(g, g->sadj[e]);
      q += merge_count(NB(g, y), DN(g, y), NB(g, x), DN(g, x));
    }
  return q;
}

static uint64_t k4_unpruned_range(const oracle_graph* g, uint64_t x0, uint64_t x1, uint32_t* P) {
  uint64_t k = 0;
  for (uint64_t x = x0; x < x1; ++x)
    for (uint64_t e = g->soff[x]; e < g->soff[x + 1]; ++e) {
      const uint64_t y = vindex(g, g->sadj[e]);
      const uint64_t np = merge_into(NB(g, y), DN(g, y), NB(g, x), DN(g, x), P);
      for (uint64_t t = 0; t < np; ++t) {
        const uint64_t z = vindex(g, P[t]);
        k += merge_count(P, np, NB(g, z), DN(g, z));
      }
    }
  return k;
}

typedef struct {
  const oracle_graph* g;
  uint64_t x0, x1;
  volatile uint64_t* next;
  pthread_mutex_t* mu;
  int query; /* 0 = triangles, 1 = 4-cliques, 2 / 3 = the same, unpruned (NEXT-2) */
  const uint64_t* ord; /* NULL, or the vertex index of each position (rank ranges) */
  uint64_t sum;
  int err;
} job_t;

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  uint32_t* P = NULL;
  if (j->query == 1 || j->query == 3) {
    uint64_t cap = j->g->max_out;
    if (j->query == 3)
      for (uint64_t i = 0; i < j->g->nv; ++i) cap = cap > j->g->deg[i] ? cap : j->g->deg[i];
    P = (uint32_t*)malloc((cap ? cap : 1) * sizeof(uint32_t));
    if (!P) { j->err = 1; return NULL; }
  }
  const uint64_t chunk = 64;
  for (;;) {
    pthread_mutex_lock(j->mu);
    const uint64_t a = *j->next;
    *j->next = a + chunk;
    pthread_mutex_unlock(j->mu);
    if (a >= j->x1) break;
    const uint64_t b = (a + chunk < j->x1) ? a + chunk : j->x1;
    j->sum += j->query == 0 ? tri_range(j->g, a, b, j->ord)
            : j->query == 1 ? k4_range(j->g, a, b, P, j->ord)
            : j->query == 2 ? tri_unpruned_range(j->g, a, b)
                            : k4_unpruned_range(j->g, a, b, P);
  }
  free(P);
  return NULL;
}

static uint64_t run_ord(const oracle_graph* g, uint64_t x0, uint64_t x1, int threads, int query,
                        const uint64_t* ord) {
  if (!g) return UINT64_MAX;
  if (x1 > g->nv) x1 = g->nv;
  if (x0 >= x1) return 0;
  if (threads <= 0) threads = 1;
  job_t* jobs = (job_t*)calloc((size_t)threads, sizeof(job_t));
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  volatile uint64_t next = x0;
  if (!jobs || !tid) { free(jobs); free(tid); return UINT64_MAX; }
  for (int t = 0; t < threads; ++t) {
    jobs[t].g = g; jobs[t].x0 = x0; jobs[t].x1 = x1; jobs[t].next = &next;
    jobs[t].mu = &mu; jobs[t].query = query; jobs[t].ord = ord;
  }
  for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, worker, &jobs[t]);
  worker(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
  uint64_t s = 0;
  int err = 0;
  for (int t = 0; t < threads; ++t) { s += jobs[t].sum; err |= jobs[t].err; }
  free(jobs); free(tid);
  return err ? UINT64_MAX : s;
}

static uint64_t run(const oracle_graph* g, uint64_t x0, uint64_t x1, int threads, int query) {
  return run_ord(g, x0, x1, threads, query, NULL);
}

uint64_t oracle_count_triangles(const oracle_graph* g, int threads) { return run(g, 0, UINT64_MAX, threads, 0); }
/* NEXT-2: unpruned (ordered-binding) counts on the symmetric data; UINT64_MAX on allocation failure. */
uint64_t oracle_count_triangles_unpruned(oracle_graph* g, int threads) {
  if (!g || build_symmetric(g)) return UINT64_MAX;
  return run(g, 0, UINT64_MAX, threads, 2);
}
uint64_t oracle_count_4cliques_unpruned(oracle_graph* g, int threads) {
  if (!g || build_symmetric(g)) return UINT64_MAX;
  return run(g, 0, UINT64_MAX, threads, 3);
}
uint64_t oracle_count_4cliques(const oracle_graph* g, int threads) { return run(g, 0, UINT64_MAX, threads, 1); }

/* Partial sums over the outer loop, x restricted to vertex indices [x0, x1)
 * of the sorted original-id list (bounded CPU-baseline samples). */
uint64_t oracle_count_triangles_range(const oracle_graph* g, uint64_t x0, uint64_t x1, int threads) {
  return run(g, x0, x1, threads, 0);
}
uint64_t oracle_count_4cliques_range(const oracle_graph* g, uint64_t x0, uint64_t x1, int threads) {
  return run(g, x0, x1, threads, 1);
}

/* Triangles whose earliest vertex (in the degree order) has original id x. */
uint64_t oracle_triangles_at(const oracle_graph* g, uint32_t x) {
  const uint32_t* p = (const uint32_t*)bsearch(&x, g->vid, g->nv, sizeof(uint32_t), cmp_u32);
  if (!p) return 0;
  const uint64_t i = (uint64_t)(p - g->vid);
  return tri_range(g, i, i + 1, NULL);
}

/*
 * Rank ranges: the counts restricted to the cliques whose EARLIEST vertex (the
 * x of the loop nest, PAPER.md:538-542 / 217 on the pruned data) has a rank in
 * [r0, r1), the rank of a vertex being its position in the total order of step
 * 3 above -- ascending (degree, original id).  A partition of [0, nv) into
 * ranges partitions the cliques, so the range counts sum to the full count.
 * (These are the sampled outputs against which the CUDA path's
 * eh_count_*_range are checked at sizes where the full oracle count is out of
 * reach, e.g. 4-cliques of C5.)  UINT64_MAX on allocation failure.
 */
static uint64_t* rank_order(const oracle_graph* g) {
  uint64_t* key = (uint64_t*)malloc((g->nv ? g->nv : 1) * sizeof(uint64_t));
  if (!key) return NULL;
  for (uint64_t i = 0; i < g->nv; ++i) key[i] = ((uint64_t)g->deg[i] << 32) | g->vid[i];
  qsort(key, g->nv, sizeof(uint64_t), cmp_u64);
  for (uint64_t r = 0; r < g->nv; ++r) key[r] = vindex(g, (uint32_t)key[r]);  /* rank -> vertex index */
  return key;
}

static uint64_t rank_range(const oracle_graph* g, uint64_t r0, uint64_t r1, int threads, int query) {
  if (!g) return UINT64_MAX;
  uint64_t* ord = rank_order(g);
  if (!ord) return UINT64_MAX;
  const uint64_t q = run_ord(g, r0, r1, threads, query, ord);
  free(ord);
  return q;
}

uint64_t oracle_count_triangles_rank_range(const oracle_graph* g, uint64_t r0, uint64_t r1, int threads) {
  return rank_range(g, r0, r1, threads, 0);
}
uint64_t oracle_count_4cliques_rank_range(const oracle_graph* g, uint64_t r0, uint64_t r1, int threads) {
  return rank_range(g, r0, r1, threads, 1);
}

/* The original id of every rank (ord[r] = vid of rank r), for tests. */
int oracle_rank_ids(const oracle_graph* g, uint32_t* ids) {
  uint64_t* ord = rank_order(g);
  if (!ord) return -1;
  for (uint64_t r = 0; r < g->nv; ++r) ids[r] = g->vid[ord[r]];
  free(ord);
  return 0;
}

/*
 * NEXT-1: Lollipop L3,1 and Barbell B3,1 COUNT(*) by the
 * paper's two-phase GHD plan (PAPER.md:379-416 Example `ex:barbell`,
 * PAPER.md:545-567 "Across Nodes": Yannakakis bottom-up pass).  Both queries
 * run on the UNDIRECTED (symmetric) data:
 *   Lollipop(x,y,z,w) :- R(x,y),S(y,z),T(x,z),U(x,w).
 *   Barbell(x,y,z,x',y',z') :- R(x,y),S(y,z),T(x,z),U(x,x'),R'(x',y'),
 *                              S'(y',z'),T'(x',z').
 * Child GHD node {x,y,z}: the triangle nest, aggregated (COUNT) and projected
 * onto x -- on symmetric data every triangle containing x yields the 2 ordered
 * bindings (y,z), so the projected count is 2 t(x), t(x) = #triangles with x.
 * Root node: Lollipop joins it with U(x,w): sum_x 2 t(x) deg(x); Barbell joins
 * the two children through U(x,x'): sum over ORDERED edges (x,x') of
 * (2 t(x)) (2 t(x')).  Counts can exceed 2^64 (Barbell), so they are returned
 * as 128-bit values (lo, hi).
 */

/* t(v) for every vertex index: each triangle x<y<z of the oriented nest adds 1
 * to x, y and z (the merge reports the matching z). */
void oracle_triangles_per_vertex(const oracle_graph* g, uint64_t* t) {
  memset(t, 0, g->nv * sizeof(uint64_t));
  uint32_t* P = (uint32_t*)malloc((g->max_out ? g->max_out : 1) * sizeof(uint32_t));
  if (!P) return;
  for (uint64_t x = 0; x < g->nv; ++x) {
    if (DOUT(g, x) == 0) continue;
    for (uint64_t e = g->off[x]; e < g->off[x + 1]; ++e) {
      const uint64_t y = vindex(g, g->adj[e]);
      if (DOUT(g, y) == 0) continue;
      const uint64_t np = merge_into(OUT(g, y), DOUT(g, y), OUT(g, x), DOUT(g, x), P);
      t[x] += np;
      t[y] += np;
      for (uint64_t k = 0; k < np; ++k) t[vindex(g, P[k])] += 1;
    }
  }
  free(P);
}

static void add128(uint64_t* lo, uint64_t* hi, unsigned __int128 v) {
  unsigned __int128 s = ((unsigned __int128)*hi << 64 | *lo) + v;
  *lo = (uint64_t)s;
  *hi = (uint64_t)(s >> 64);
}

/* out2 = {lo, hi} of the Lollipop COUNT(*); returns 0 or -1 on allocation failure. */
int oracle_count_lollipop(const oracle_graph* g, uint64_t* out2) {
  uint64_t* t = (uint64_t*)malloc((g->nv ? g->nv : 1) * sizeof(uint64_t));
  if (!t) return -1;
  oracle_triangles_per_vertex(g, t);
  out2[0] = out2[1] = 0;
  for (uint64_t x = 0; x < g->nv; ++x) add128(&out2[0], &out2[1], (unsigned __int128)2 * t[x] * g->deg[x]);
  free(t);
  return 0;
}

int oracle_count_barbell(const oracle_graph* g, uint64_t* out2) {
  uint64_t* t = (uint64_t*)malloc((g->nv ? g->nv : 1) * sizeof(uint64_t));
  if (!t) return -1;
  oracle_triangles_per_vertex(g, t);
  out2[0] = out2[1] = 0;
  /* each undirected edge {x, x'} appears once in E+ and twice as an ordered pair */
  for (uint64_t x = 0; x < g->nv; ++x)
    for (uint64_t e = g->off[x]; e < g->off[x + 1]; ++e) {
      const uint64_t y = vindex(g, g->adj[e]);
      add128(&out2[0], &out2[1], (unsigned __int128)8 * t[x] * t[y]);
    }
  free(t);
  return 0;
}

/* stats: [n_input, m, nv, max_out] */
void oracle_stats(const oracle_graph* g, uint64_t* out4) {
  out4[0] = g->n_input; out4[1] = g->m; out4[2] = g->nv; out4[3] = g->max_out;
}

/* Copy the oriented trie out: vid[nv], deg[nv], off[nv+1], adj[m] (any may be NULL). */
void oracle_export(const oracle_graph* g, uint32_t* vid, uint32_t* deg, uint64_t* off, uint32_t* adj) {
  if (vid) memcpy(vid, g->vid, g->nv * sizeof(uint32_t));
  if (deg) memcpy(deg, g->deg, g->nv * sizeof(uint32_t));
  if (off) memcpy(off, g->off, (g->nv + 1) * sizeof(uint64_t));
  if (adj) memcpy(adj, g->adj, g->m * sizeof(uint32_t));
}
