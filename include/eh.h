/*
 * eh.h -- C ABI of the B200-native EmptyHeaded hot path (arXiv 1503.02368).
 *
 * The library (paper_1503_02368_b200/lib/libeh.so, CUDA sm_100a) implements
 * the worst-case-optimal Generic-Join over a trie of the Edge relation
 * (Alg. `fig:worst_case`) for two COUNT(*) queries:
 *
 *   Triangle(x,y,z) :- R(x,y),S(y,z),T(x,z).
 *   4Clique(x,y,z,w) :- R(x,y),S(y,z),T(x,z),U(x,w),V(y,w),Q(z,w). PAPER.md:217
 *
 * with R = S = ... = the symmetrically pruned Edge relation
 * and COUNT(*) aggregated as `w:long`, plus (SURVEY.md §8(f)
 * NEXT-1) per-vertex triangle counts and the Lollipop / Barbell COUNT(*) by the
 * two-phase GHD plan.  Everything below this
 * header runs on one GPU as hand-written CUDA kernels; there is no CPU
 * fallback: every entry point fails (returns an error) when no CUDA device is
 * usable.
 *
 * Conventions for every function:
 *  - fixed-width integers only; no C++ types cross the boundary;
 *  - synchronous with respect to the calling host thread;
 *  - errors are reported by the return value (NULL, EH_COUNT_ERROR or a
 *    negative EH_E* code) and detailed by eh_last_status() / eh_last_error(),
 *    which are thread-local and valid until the next call on that thread;
 *  - a graph handle is immutable after load and may be counted repeatedly;
 *    concurrent calls on ONE handle from several threads are not supported.
 */
#ifndef EH_H_
#define EH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct eh_graph eh_graph; /* opaque; owns all device memory of one loaded graph */

enum {
  EH_OK = 0,
  EH_EINVAL = -1,     /* bad argument (NULL pointer with n > 0, bad flags, ...) */
  EH_ENOMEM = -2,     /* device allocation failed (or the allocator hook returned NULL) */
  EH_ECUDA = -3,      /* a CUDA runtime error (no device, launch failure, ...) */
  EH_EUNSORTED = -4   /* eh_intersect input not strictly increasing */
};

/* Unreachable as a count: T <= (sqrt(2)/3) m^1.5 and K4 < C(sqrt(2m)+1, 4) << 2^64. */
#define EH_COUNT_ERROR UINT64_MAX

#define EH_INPUT_ON_DEVICE 0x1u /* src/dst are device pointers (else host memory, pageable or pinned) */
#define EH_SET_DEVICE      0x2u /* use cfg->device instead of the current device */
#define EH_ALL_UINT        0x4u /* relation-level layout, the paper's "-R" ablation: no bitsets */
#define EH_BLOCK_LAYOUT    0x10u /* NEXT-3 block-level (composite) layout for eh_count_triangles:
                                    every set is split into 128-id blocks; blocks with >= 4 elements are bitset
                                    blocks, the rest stay uint (the set-level layouts serve the other queries) */
#define EH_FORCE_SEARCH    0x20u /* ablation / microbenchmark: EH_ALL_UINT and every uint cap uint row takes the
                                   * galloping (binary-search) side, whatever the cardinalities -- the opposite of
                                   * EH_NO_ALGO; with both, EH_NO_ALGO wins (Fig. `fig:card_skew2`) */
#define EH_NO_ALGO         0x8u /* the paper's "-RA" ablation (NEXT-3): EH_ALL_UINT and no
                                   intersection-algorithm choice (every uint cap uint streams, no galloping) */

/* Load-time configuration.  A zero-initialised struct means "defaults". */
typedef struct {
  /* Set-level layout optimizer: a set S becomes a bitset iff
   * span(S) = max - min + 1 < bitset_tau * |S| (strict; u64 arithmetic).
   * 0 -> 128 (tuned on B200, reading c10; the paper's AVX register
   * is tau = 256).  Counts do not depend on tau. */
  uint32_t bitset_tau;
  int32_t device; /* CUDA ordinal, honoured only with EH_SET_DEVICE */
  /* cudaStream_t used for all work of the handle; NULL -> a library-owned stream
   * created WITHOUT cudaStreamNonBlocking, i.e. ordered after the work pending on
   * the legacy default stream.  Ordering contract for EH_INPUT_ON_DEVICE inputs and
   * device outputs: they must be ready (written) in the order of `stream` -- pass
   * the stream that produced them, or produce them on the legacy default stream. */
  void* stream;
  /* Optional device allocator (e.g. the PyTorch caching allocator).  Both or
   * neither must be set.  dev_alloc returning NULL makes the call fail with EH_ENOMEM. */
  void* (*dev_alloc)(size_t bytes, void* stream, void* ctx);
  void (*dev_free)(void* ptr, void* stream, void* ctx);
  void* alloc_ctx;
  uint32_t flags;          /* EH_INPUT_ON_DEVICE | EH_SET_DEVICE | EH_ALL_UINT | EH_NO_ALGO | EH_BLOCK_LAYOUT | EH_FORCE_SEARCH */
  /* Count-kernel work classes by d = |N+(x)|: 0 = [2, bin_small_max], 1 = up to
   * bin_large_min - 1, 2 = the rest.  Triangle / per-vertex kernels: class 0 warp-per-x,
   * classes 1-2 CTA-per-x; 4-clique kernels: classes 0-1 warp-per-x, class 2 CTA-per-x.
   * 0 -> tuned defaults (64, 129).  Both are clamped to the warp
   * kernels' capacity (d <= 128): bin_small_max = UINT32_MAX puts every d <= 128 into
   * class 0, bin_large_min = 1 puts every vertex into class 2.  Counts do not depend on them. */
  uint32_t bin_small_max;
  uint32_t bin_large_min;
  uint32_t min_bitset_card;/* bitset only if |S| >= this (reading c15); 0 -> 2 */
  /* NEXT-4 node ordering = the id assignment that orients (prunes) the edges
   * (PAPER.md:1065-1153); counts never depend on it.  EH_ORDER_* below;
   * 0 = EH_ORDER_DEGREE, the paper's default. */
  uint32_t order;
  /* a7 thread class: the x with 2 <= |N+(x)| <= bin_thread_max (within class 0) run
   * one THREAD per x in the triangle count (their <= C(d, 2) probes are too few to
   * occupy a warp).  0 -> 12 (16 above 2^19 active ids, 4 above 2^24); 1 disables the class; clamped to
   * bin_small_max and to 16.  Counts do not depend on it. */
  uint32_t bin_thread_max;
} eh_config;

/* Node orderings (readings in DESIGN.md c20).  Each names the
 * paper's labelling; edges are kept from the later to the earlier label (the
 * mirror of "src_id > dst_id"). */
enum {
  EH_ORDER_DEGREE = 0,     /* descending degree (ties by id) -- the default */
  EH_ORDER_REV_DEGREE = 1, /* ascending degree */
  EH_ORDER_RANDOM = 2,     /* a fixed pseudo-random permutation of the ids */
  EH_ORDER_BFS = 3,        /* breadth-first from the highest-degree vertex (level, then id) */
  EH_ORDER_HYBRID = 4,     /* BFS labels, then stably sorted by descending degree */
  EH_ORDER_SHINGLE = 5,    /* by neighbourhood min-hash (shingle), then id */
  EH_ORDER_ID = 6          /* the ids as given: ranks ascend by (dictionary-encoded) input id, edges point low -> high
                            * id.  Not one of the paper's orderings: it lets a caller fix the orientation, which the
                            * intersection microbenchmarks (tools/intersect_bench.py) use
                            * to build rows |A cap B| of chosen cardinality, range and layout. */
};

/* eh_stats: filled by eh_graph_stats (bench / tests). */
typedef struct {
  uint64_t n_input;        /* input tuples */
  uint64_t m_undirected;   /* distinct undirected edges without self-loops = |E+| */
  uint64_t n_active;       /* non-isolated vertices (the rank space is [0, n_active)) */
  uint64_t max_out_degree; /* max |N+(x)| */
  uint64_t n_bitset_sets;  /* sets stored with the bitset layout */
  uint64_t bitset_words;   /* 32-bit words in the bitset pool */
  uint64_t device_bytes;   /* device memory owned by the handle */
  uint64_t alg_bytes_tri;  /* B_tri(tau) of SURVEY.md §8(d): 8(n+1) + sum_x bytes(N+(x)) + sum_(x,y) bytes(N+(y)) */
  uint64_t wedge_work;     /* sum over (x,y) in E+ of |N+(x) after y| (min-property side) */
} eh_stats;

/*
 * eh_load_edges / eh_load_edges_ex -- build the trie of the Edge relation.
 *
 * PAPER.md:281-285 (dictionary encoding to 32-bit ids; sets of distinct values
 * grouped by parent), PAPER.md:799-800 (symmetric pruning, ids by degree),
 * PAPER.md:730 (set-level uint/bitset layout).
 *
 *  src, dst : n undirected pairs (src[i], dst[i]); any uint32 value is a valid id,
 *             0xFFFFFFFF included.  Self-loops are dropped; duplicates and
 *             reversed pairs collapse.  Host pointers unless cfg->flags has
 *             EH_INPUT_ON_DEVICE.  Borrowed for the call only (copied).
 *  n        : number of pairs; n = 0 gives a valid empty graph (counts 0).
 *  cfg      : may be NULL (defaults).
 * Returns a handle owning all device memory until eh_free, or NULL on error
 * (EH_EINVAL: NULL src/dst with n > 0, one allocator hook without the other;
 *  EH_ENOMEM; EH_ECUDA).
 */
eh_graph* eh_load_edges(const uint32_t* src, const uint32_t* dst, uint64_t n);
eh_graph* eh_load_edges_ex(const uint32_t* src, const uint32_t* dst, uint64_t n, const eh_config* cfg);

/*
 * eh_count_batch -- the whole path (eh_load_edges + the COUNT(*) of `query` +
 * eh_free) for k independent edge lists, with the upload of list i+1 (a copy
 * engine, on a separate stream) overlapping the trie build and count of list i
 * on the SMs.  Same semantics per list as eh_load_edges_ex (with cfg) followed
 * by eh_count_triangles / eh_count_4cliques.
 *  src[i], dst[i], n[i] : list i in HOST memory (page-locked memory is needed for
 *                         the overlap; pageable memory works, serialised)
 *  query                : EH_QUERY_TRIANGLES or EH_QUERY_4CLIQUES
 *  cfg                  : may be NULL; EH_INPUT_ON_DEVICE is rejected; cfg->stream
 *                         (else a library-owned blocking stream) runs the compute
 *  counts[k]            : caller-owned host array, receives the k counts
 * Without cfg->stream, batches of small lists (<= 2^23 edges) run in two lanes
 * (library host threads and streams, alternate lists).  Two device input buffers
 * of 8 max(n) bytes per lane are held for the call.  Returns
 * EH_OK, EH_EINVAL, EH_ENOMEM or EH_ECUDA (counts of lists before a failure are
 * written).
 */
#define EH_QUERY_TRIANGLES 0u
#define EH_QUERY_4CLIQUES 1u
int eh_count_batch(const uint32_t* const* src, const uint32_t* const* dst, const uint64_t* n, uint64_t k,
                   uint32_t query, const eh_config* cfg, uint64_t* counts);

/*
 * eh_count_triangles -- COUNT(*) of Triangle(x,y,z) on the pruned relation:
 * the number of 3-vertex sets whose three pairs are edges (each counted once).
 * Generic-Join loop nest PAPER.md:538-542.  Returns EH_COUNT_ERROR on error
 * (EH_EINVAL for g == NULL, EH_ECUDA).
 */
uint64_t eh_count_triangles(eh_graph* g);

/*
 * eh_count_4cliques -- COUNT(*) of 4Clique(x,y,z,w):
 * the number of 4-vertex sets whose six pairs are edges, each counted once.
 * Returns EH_COUNT_ERROR on error.
 */
uint64_t eh_count_4cliques(eh_graph* g);

/*
 * eh_count_triangles_range / eh_count_4cliques_range -- the same COUNT(*)s
 * with the outermost attribute x of the loop nest (PAPER.md:538-542 for the
 * triangle, PAPER.md:217 for the 4-clique, on pruned data every clique is
 * bound once, at its EARLIEST vertex x) restricted to the ranks [r0, r1).  The
 * rank of a vertex is its position in the handle's node ordering (the default
 * EH_ORDER_DEGREE: ascending (degree, original id); rank r has original id
 * eh_graph_export's orig_id[r]).  Ranks run over [0, n_active); r1 is clamped
 * to n_active and r0 >= r1 gives 0.  Any partition of [0, n_active) into
 * ranges partitions the cliques, so the range counts add up to the full count:
 * this is the unit by which the path shards and the sampled
 * output the tests check against the CPU oracle where the full oracle count is
 * out of reach (4-cliques of C5).  The same kernels and launch shapes as the
 * full counts run over the restricted work lists.  Returns EH_COUNT_ERROR on
 * error (EH_EINVAL for g == NULL, EH_ENOMEM, EH_ECUDA).
 */
uint64_t eh_count_triangles_range(eh_graph* g, uint64_t r0, uint64_t r1);
uint64_t eh_count_4cliques_range(eh_graph* g, uint64_t r0, uint64_t r1);

/*
 * eh_alg_bytes_k4 -- B_K4(tau = 32) of SURVEY.md §8(d): the algorithmic bytes
 * of the 4-clique Generic-Join, B_tri(32) + sum over triangles x < y < z of
 * bytes_32(N+(z)), bytes_32(S) = 4 |S| for a uint set or 4 x (32-bit words
 * spanned) for a tau = 32 bitset (the roofline denominator of the K4 bench
 * line).  Computed on the first call by a statistics kernel (one binary search
 * per wedge; not part of any count) and cached in the handle.  Returns
 * EH_COUNT_ERROR on error.
 */
uint64_t eh_alg_bytes_k4(eh_graph* g);

/*
 * eh_triangles_per_vertex -- t(v) = the number of triangles containing v, for
 * every non-isolated vertex: the GROUP BY x aggregate
 * of the triangle node of the Lollipop/Barbell GHDs (Example `ex:barbell`,
 * PAPER.md:379-416, bottom-up pass PAPER.md:545-567; per x the projection
 * counts 2 t(x) ordered (y, z) pairs on symmetric data).
 *  t [n_active] : caller-owned uint64, host memory or device memory of g's
 *                 device (detected); t[r] belongs to the vertex of rank r,
 *                 whose original id is eh_graph_export's orig_id[r].
 * Returns EH_OK, EH_EINVAL (NULL argument, output on another device), EH_ENOMEM, EH_ECUDA.
 */
int eh_triangles_per_vertex(eh_graph* g, uint64_t* t);

/*
 * eh_count_lollipop / eh_count_barbell -- COUNT(*) of
 *   Lollipop(x,y,z,w) :- R(x,y),S(y,z),T(x,z),U(x,w).
 *   Barbell(x,y,z,x',y',z') :- R(x,y),S(y,z),T(x,z),U(x,x'),R'(x',y'),S'(y',z'),T'(x',z').
 * on the UNDIRECTED (symmetric) Edge relation, as the paper runs them
 * (PAPER.md:877-878), by the two-phase GHD plan: L3,1 = sum_v 2 t(v) deg(v),
 * B3,1 = sum over ordered edges (x, x') of 2 t(x) 2 t(x').  The counts can
 * exceed 2^64, so out[0] / out[1] receive the low / high 64 bits (host memory).
 * Returns EH_OK, EH_EINVAL (NULL argument), EH_ENOMEM, EH_ECUDA.
 */
int eh_count_lollipop(eh_graph* g, uint64_t out[2]);
int eh_count_barbell(eh_graph* g, uint64_t out[2]);

/*
 * eh_count_triangles_unpruned -- NEXT-2: the triangle
 * Generic-Join on the UNPRUNED data, i.e. the symmetric Edge relation (every
 * undirected edge in both directions, ids by degree, no symmetry breaking:
 * the "Default" rows of PAPER.md:1155-1236).  COUNT(*) then counts ordered
 * bindings: 6 T ("a multiple of the former").  The
 * symmetric trie (full sorted neighbour lists with their own set layouts, same
 * tau) is built on the first call and kept by the handle (eh_symmetric_stats
 * reports it).  Returns EH_COUNT_ERROR on error (EH_EINVAL, EH_ENOMEM, EH_ECUDA).
 */
uint64_t eh_count_triangles_unpruned(eh_graph* g);

/*
 * eh_count_4cliques_unpruned -- NEXT-2: the 4-clique Generic-Join on the
 * unpruned (symmetric) data, attribute order x, y, z, w: 24 K4.  Same
 * symmetric trie.  Lists above 1024 elements (the hubs) take one CTA per row
 * (x, y): P = N(x) cap N(y) is built on chip and every z in P picks the
 * cheapest of probe / stream / bitset AND (DESIGN.md NEXT-2).  Returns
 * EH_COUNT_ERROR on error.
 */
uint64_t eh_count_4cliques_unpruned(eh_graph* g);

/*
 * eh_symmetric_stats -- statistics of the symmetric trie (building it if
 * needed): m_undirected = |E|, max_out_degree = max degree, alg_bytes_tri =
 * B_tri of the unpruned nest (same formula over N(x)), device_bytes = its
 * memory (not counted by eh_graph_stats).  Returns EH_OK or EH_E*.
 */
int eh_symmetric_stats(eh_graph* g, eh_stats* out);

/*
 * eh_intersect -- the set operation "xs cap ys" of Table `lst:eh_operators`
 * (PAPER.md:515-516), with the paper's layout-dependent algorithms
 * (PAPER.md:628-642): each input gets the set-level layout (uint or bitset,
 * tau = 32); uint cap uint uses a merge when the cardinality ratio is <= 32
 * and binary search (galloping) otherwise; uint cap bitset probes the bitset;
 * bitset cap bitset ANDs the overlapping words.
 *
 *  a[0..na), b[0..nb) : strictly increasing uint32 (host or device memory,
 *                       detected per pointer).  Validated in O(na + nb).
 *  out                : NULL (count only) or caller-owned room for
 *                       min(na, nb) uint32 (host or device memory); receives
 *                       the intersection in increasing order.
 * Returns |a cap b| >= 0, or EH_EINVAL (NULL with n > 0), EH_EUNSORTED,
 * EH_ENOMEM, EH_ECUDA.
 */
int64_t eh_intersect(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb, uint32_t* out);

/* Statistics of a loaded graph.  Returns EH_OK or EH_EINVAL. */
int eh_graph_stats(const eh_graph* g, eh_stats* out);

/*
 * eh_graph_export -- copy the oriented trie to HOST memory (tests, debugging).
 *  row_ptr [n_active+1] : out-list offsets (unpadded, in elements)
 *  col     [m]          : out-neighbours in rank space, each list strictly increasing
 *  orig_id [n_active]   : original uint32 id of each rank
 *  is_bitset[n_active]  : 1 if the set N+(rank) uses the bitset layout
 * Any pointer may be NULL.  Returns EH_OK, EH_EINVAL or EH_ECUDA.
 */
int eh_graph_export(const eh_graph* g, uint64_t* row_ptr, uint32_t* col, uint32_t* orig_id, uint8_t* is_bitset);

/* Release a handle and all its device memory.  NULL-safe.  With the default
 * allocation path (no allocator hook) the memory returns to the library's
 * private pool and its large-block cache, which keep it for the next load
 * (re-mapping device memory costs ~100 ms per load at C3 size, seconds at C5). */
void eh_free(eh_graph* g);

/* Give the device memory the library keeps idle (freed large blocks of its
 * cache, unused memory of its private stream-ordered pools on every device)
 * back to the driver, e.g. before another allocator needs it.  Waits for the
 * pending work that last used each block.  Memory of live handles is not
 * touched.  Also done automatically, once, when a device allocation fails. */
void eh_release_cached_memory(void);

/* Number of CUDA kernels this library has launched in this process (diagnostics; bench.py). */
uint64_t eh_launch_count(void);

int eh_last_status(void);        /* thread-local status of the last call (EH_OK or EH_E*) */
const char* eh_last_error(void); /* thread-local message, "" if none */

#ifdef __cplusplus
}
#endif
#endif /* EH_H_ */
