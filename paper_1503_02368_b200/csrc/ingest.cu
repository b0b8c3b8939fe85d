// ingest.cu -- SURVEY.md §8(a) rows a1-a5: upload, canonicalise + dedup (=
// symmetrisation to a simple undirected graph) + degree by the bucketed pass of
// dedup.cu (or, as an ablation and for 32-bit id spaces, the radix sort of the
// canonical keys), (degree, id) rank (dictionary encoding), orientation
// (symmetric pruning) and CSR.
//
//  PAPER.md:281-282  dictionary encoding of values to 32-bit ids; "the order of
//                    dictionary ID assignment affects the density of the sets"
//  PAPER.md:284      values "grouped into sets of distinct values based on their
//                    parent attribute"
//  PAPER.md:799-800  pruning: "each undirected edge is pruned such that
//                    src_id > dst_id and id's are assigned based upon the degree"
//  Readings: c2 ascending (deg, id) rank, orient low -> high (a mirror
//  of the paper's convention; any strict order gives the same counts), c3 ties by
//  original id, c4 degree = distinct neighbours, c5 self-loops dropped, c6 dedup,
//  c7 (u,v) == (v,u), c16 any uint32 is a valid id.
#include "eh_internal.cuh"
#include "primitives.cuh"

#include <algorithm>
#include <cstring>

namespace eh {

namespace {

__global__ void k_max_id(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst, uint64_t n,
                         uint32_t* __restrict__ out) {
  uint32_t mx = 0;
  const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  uint64_t done = 0;
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {  // 128-bit loads
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    const uint4* d4 = reinterpret_cast<const uint4*>(dst);
    for (uint64_t i = t0; i < n / 4; i += nt) {
      const uint4 a = __ldg(s4 + i), b = __ldg(d4 + i);
      mx = max(mx, max(max(max(a.x, a.y), max(a.z, a.w)), max(max(b.x, b.y), max(b.z, b.w))));
    }
    done = n / 4 * 4;
  }
  for (uint64_t i = done + t0; i < n; i += nt) mx = max(mx, max(src[i], dst[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

// Dictionary path: map each id to its index in the sorted distinct id list.
__global__ void k_dict_map(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t n,
                           const uint32_t* __restrict__ dict, uint64_t nd) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = in[i];
    uint64_t lo = 0, hi = nd;  // lower_bound
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (dict[mid] < v) lo = mid + 1; else hi = mid;
    }
    out[i] = (uint32_t)lo;
  }
}

// a1-a3 fused: canonical key (min << b) | max of every non-loop pair inserted
// into an open-addressing hash set (linear probing; read before CAS, so the
// duplicates that are already present cost no atomic).  Empty slot = all ones,
// which no canonical key of a non-loop pair can equal.
__global__ void k_hash_insert(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst, uint64_t n,
                              uint32_t b, unsigned long long* __restrict__ tab, uint32_t tbits) {
  const unsigned long long kEmpty = ~0ull;
  const uint64_t mask = (1ull << tbits) - 1ull;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = src[i], v = dst[i];
    if (u == v) continue;
    const unsigned long long key = ((uint64_t)min(u, v) << b) | (uint64_t)max(u, v);
    uint64_t h = (key * 0x9E3779B97F4A7C15ull) >> (64 - tbits);
    for (;;) {
      unsigned long long cur = __ldcg(tab + h);
      if (cur == key) break;
      if (cur == kEmpty) {
        cur = atomicCAS(tab + h, kEmpty, key);
        if (cur == kEmpty || cur == key) break;
      }
      h = (h + 1) & mask;
    }
  }
}

struct OccupiedPred {
  const unsigned long long* t;
  __device__ bool operator()(uint64_t i) const { return t[i] != ~0ull; }
};
struct CopySlotEmit {
  const unsigned long long* t;
  uint64_t* out;
  __device__ void operator()(uint64_t pos, uint64_t i) const { out[pos] = t[i]; }
};

struct UniqueU32Pred {
  const uint32_t* k;
  __device__ bool operator()(uint64_t i) const { return i == 0 || k[i] != k[i - 1]; }
};
struct CopyU32Emit {
  const uint32_t* k;
  uint32_t* out;
  __device__ void operator()(uint64_t pos, uint64_t i) const { out[pos] = k[i]; }
};

// The sorted key array is consumed in place (no compaction): an entry counts
// iff it is the first of its run of equal keys and not the self-loop sentinel
// (all ones, sorted last).  The hash path's keys are distinct, so the same
// test accepts all of them.
__device__ __forceinline__ bool key_head(const uint64_t* __restrict__ keys, uint64_t i, uint64_t sentinel,
                                         uint64_t& k) {
  k = keys[i];
  return k != sentinel && (i == 0 || keys[i - 1] != k);
}

// a4: degree = number of distinct neighbours.
// Keys are sorted by the low end u, so u-side counts are run lengths inside a
// warp (one atomic per run); v-side atomics are aggregated over equal v in the
// warp (hubs would otherwise serialise thousands of atomics on one address).
__global__ void k_degree(const uint64_t* __restrict__ keys, uint64_t nk, uint32_t b, uint64_t sentinel,
                         uint32_t* __restrict__ deg, unsigned long long* __restrict__ m_out) {
  const uint64_t mask = (1ull << b) - 1ull;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t heads = 0;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < nk; base += stride) {
    const uint64_t i = base + lane;
    uint64_t k = 0;
    const bool valid = i < nk && key_head(keys, i, sentinel, k);
    heads += valid;
    const uint32_t u = valid ? (uint32_t)(k >> b) : 0xFFFFFFFFu;
    const uint32_t v = valid ? (uint32_t)(k & mask) : 0xFFFFFFFFu;
    const unsigned pu = __match_any_sync(kFull, u);  // keys sorted by u: long runs in a warp
    if (valid && (pu & lt) == 0) atomicAdd(&deg[u], (uint32_t)__popc(pu));
    const unsigned pv = __match_any_sync(kFull, v);
    if (valid && (pv & lt) == 0) atomicAdd(&deg[v], (uint32_t)__popc(pv));
  }
  heads = warp_sum(heads);
  if (lane == 0 && heads) atomicAdd(m_out, (unsigned long long)heads);
}

struct ActivePred {
  const uint32_t* deg;
  __device__ bool operator()(uint64_t i) const { return deg[i] != 0; }
};
struct RankKeyEmit {  // (primary << b) | id, sorted ascending = the rank order (primary = deg by default)
  const uint64_t* prim;  // nullptr: primary = deg
  const uint32_t* deg;
  uint32_t b;
  uint64_t* out;
  __device__ void operator()(uint64_t pos, uint64_t i) const {
    out[pos] = ((prim ? prim[i] : (uint64_t)deg[i]) << b) | i;
  }
};

__global__ void k_rank(const uint64_t* __restrict__ sorted, uint64_t n_act, uint32_t b, uint32_t* __restrict__ deg_rank_id,
                       uint32_t* __restrict__ orig, const uint32_t* __restrict__ dict, uint32_t* __restrict__ deg_rank) {
  // deg_rank_id holds deg[id] on entry and rank[id] on exit (one thread per id: read, then write)
  const uint64_t mask = (1ull << b) - 1ull;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_act; r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t key = sorted[r];
    const uint32_t id = (uint32_t)(key & mask);
    deg_rank[r] = deg_rank_id[id];
    deg_rank_id[id] = (uint32_t)r;
    orig[r] = dict ? dict[id] : id;
  }
}

// ---- NEXT-4 node orderings (reading c20) ------
// Each ordering gives every id a primary key; ranks ascend by (primary, id) and
// edges point low -> high rank, the mirror of the paper's labels with
// "src_id > dst_id", so primary = the REVERSE of the paper's label order.
__device__ __forceinline__ uint32_t hash32(uint32_t x) {  // splitmix-style finaliser
  x ^= 0x9E3779B9u;
  x ^= x >> 16; x *= 0x7FEB352Du;
  x ^= x >> 15; x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}

__global__ void k_prim_simple(const uint32_t* __restrict__ deg, uint64_t n, uint32_t order, uint32_t max_deg,
                              const uint32_t* __restrict__ aux, uint32_t aux_max, uint32_t aux_bits,
                              uint64_t* __restrict__ prim) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t p = 0;
    if (order == EH_ORDER_REV_DEGREE) p = max_deg - deg[i];
    else if (order == EH_ORDER_RANDOM) p = hash32((uint32_t)i);
    else if (order == EH_ORDER_SHINGLE) p = 0xFFFFFFFFu - aux[i];  // aux = min-hash of N(i)
    else if (order == EH_ORDER_BFS) p = aux_max - aux[i];           // aux = BFS level (aux_max: unreached)
    else if (order == EH_ORDER_HYBRID) p = ((uint64_t)deg[i] << aux_bits) | (aux_max - aux[i]);
    prim[i] = p;
  }
}

__global__ void k_shingle(const uint64_t* __restrict__ keys, uint64_t m, uint32_t b, uint64_t sentinel,
                          uint32_t* __restrict__ sh) {
  const uint64_t mask = (1ull << b) - 1ull;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t k;
    if (!key_head(keys, i, sentinel, k)) continue;
    const uint32_t u = (uint32_t)(k >> b), v = (uint32_t)(k & mask);
    atomicMin(&sh[u], hash32(v));
    atomicMin(&sh[v], hash32(u));
  }
}

// undirected adjacency by id for the BFS orderings
__global__ void k_adj_fill(const uint64_t* __restrict__ keys, uint64_t m, uint32_t b, uint64_t sentinel,
                           const uint64_t* __restrict__ off, uint32_t* __restrict__ cur, uint32_t* __restrict__ adj) {
  const uint64_t mask = (1ull << b) - 1ull;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t k;
    if (!key_head(keys, i, sentinel, k)) continue;
    const uint32_t u = (uint32_t)(k >> b), v = (uint32_t)(k & mask);
    adj[off[u] + atomicAdd(&cur[u], 1u)] = v;
    adj[off[v] + atomicAdd(&cur[v], 1u)] = u;
  }
}

__global__ void k_bfs_root(const uint32_t* __restrict__ deg, uint64_t n, unsigned long long* __restrict__ best) {
  unsigned long long b = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    b = max(b, ((unsigned long long)deg[i] << 32) | (0xFFFFFFFFull - i));  // max degree, then smallest id
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) b = max(b, __shfl_xor_sync(kFull, b, o));
  if ((threadIdx.x & 31) == 0) atomicMax(best, b);
}

// one level: warp per frontier vertex, lanes over its neighbours
__global__ void k_bfs_step(const uint32_t* __restrict__ frontier, uint32_t nf, const uint64_t* __restrict__ off,
                           const uint32_t* __restrict__ adj, uint32_t* __restrict__ level, uint32_t next_level,
                           uint32_t* __restrict__ next, uint32_t* __restrict__ nnext) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t k = warp; k < nf; k += nw) {
    const uint32_t v = frontier[k];
    for (uint64_t e = off[v] + lane; e < off[v + 1]; e += 32) {
      const uint32_t u = adj[e];
      if (level[u] == 0xFFFFFFFFu && atomicCAS(&level[u], 0xFFFFFFFFu, next_level) == 0xFFFFFFFFu)
        next[atomicAdd(nnext, 1u)] = u;
    }
  }
}

__global__ void k_level_fix(uint32_t* __restrict__ level, uint64_t n, uint32_t unreached) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (level[i] == 0xFFFFFFFFu) level[i] = unreached;
}

// a5: counting-sort scatter of the high end into the low end's list (slot order
// within a list is arbitrary; the segmented sort orders it).  One cursor atomic
// per group of equal low ends in the warp.  kElem: list x starts at element
// off[x] (the degree-capacity lists of build_trie, cursors end as |N+(x)|);
// else at off[x] * 4 (padded 16-B offsets).
template <bool kElem>
__global__ void k_scatter_col(const uint64_t* __restrict__ keys, uint64_t m, uint32_t b, uint64_t sentinel,
                              const uint32_t* __restrict__ rank, const uint64_t* __restrict__ off16,
                              uint32_t* __restrict__ cursor, uint32_t* __restrict__ col) {
  const uint64_t mask = (1ull << b) - 1ull;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < m; base += stride) {
    const uint64_t i = base + lane;
    uint32_t lo = 0xFFFFFFFFu, hi = 0;
    uint64_t k = 0;
    if (i < m && key_head(keys, i, sentinel, k)) {
      const uint32_t ru = rank[k >> b], rv = rank[k & mask];
      lo = min(ru, rv);
      hi = max(ru, rv);
    }
    const unsigned peers = __match_any_sync(kFull, lo);
    const int leader = __ffs(peers) - 1;
    uint32_t p0 = 0;
    if (lo != 0xFFFFFFFFu && lane == leader) p0 = atomicAdd(&cursor[lo], (uint32_t)__popc(peers));
    p0 = __shfl_sync(peers, p0, leader);
    EH_DASSERT(lo == 0xFFFFFFFFu || !kElem || off16[lo] + p0 + __popc(peers & lt) < off16[lo + 1]);
    if (lo != 0xFFFFFFFFu) col[off16[lo] * (kElem ? 1 : 4) + p0 + __popc(peers & lt)] = hi;
  }
}

__global__ void k_pad4(const uint32_t* __restrict__ d, uint64_t n, uint32_t* __restrict__ p4) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    p4[i] = (d[i] + 3u) >> 2;
}

__global__ void k_desc_base(const uint64_t* __restrict__ off16, const uint32_t* __restrict__ dplus, uint64_t n_act,
                            uint64_t total16, uint4* __restrict__ desc) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n_act; v += (uint64_t)gridDim.x * blockDim.x) {
    if (v < n_act) desc[v] = make_uint4((uint32_t)off16[v], dplus[v], 0u, 0u);
    else desc[v] = make_uint4((uint32_t)total16, 0u, 0u, 0u);
  }
}

// max and number of non-zero entries (n_act = ids with a neighbour)
__global__ void k_deg_stats(const uint32_t* __restrict__ a, uint64_t n, unsigned long long* __restrict__ out) {
  uint32_t mx = 0, nz = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = a[i];
    mx = max(mx, v);
    nz += (v != 0);
  }
  mx = __reduce_max_sync(kFull, mx);
  nz = __reduce_add_sync(kFull, nz);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&out[0], (unsigned long long)mx);
    if (nz) atomicAdd(&out[1], (unsigned long long)nz);
  }
}

__global__ void k_max_u32(const uint32_t* __restrict__ a, uint64_t n, uint32_t* __restrict__ out) {
  uint32_t mx = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    mx = max(mx, a[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

}  // namespace

// BFS levels from the highest-degree id over the undirected simple graph of the
// distinct keys; ids not reached get the returned value (max level + 1).
static uint32_t bfs_levels(const uint64_t* keys, uint64_t nk, uint64_t m, uint32_t b, uint64_t sentinel,
                           const uint32_t* deg, uint64_t n_ids, uint32_t* level, Allocator& al, cudaStream_t s) {
  const unsigned TB = 256;
  DBuf<uint64_t> off(al, n_ids + 1), tot(al, 1);
  scan_exclusive_u32(deg, off.p, n_ids, tot.p, al, s);
  EH_CUDA(cudaMemcpyAsync(off.p + n_ids, tot.p, 8, cudaMemcpyDeviceToDevice, s));  // off[n] = 2m
  DBuf<uint32_t> cur(al, n_ids), adj(al, std::max<uint64_t>(1, 2 * m)), fa(al, n_ids), fb(al, n_ids), cnt(al, 1);
  EH_CUDA(cudaMemsetAsync(cur.p, 0, n_ids * 4, s));
  k_adj_fill<<<grid_for(nk, TB * 4), TB, 0, s>>>(keys, nk, b, sentinel, off.p, cur.p, adj.p);
  EH_LAUNCH("k_adj_fill");
  DBuf<unsigned long long> best(al, 1);
  EH_CUDA(cudaMemsetAsync(best.p, 0, 8, s));
  k_bfs_root<<<grid_for(n_ids, TB * 8), TB, 0, s>>>(deg, n_ids, best.p);
  EH_LAUNCH("k_bfs_root");
  const uint32_t root = (uint32_t)(0xFFFFFFFFull - (read_scalar(best.p, s) & 0xFFFFFFFFull));
  EH_CUDA(cudaMemsetAsync(level, 0xFF, n_ids * 4, s));
  const uint32_t zero = 0;
  EH_CUDA(cudaMemcpyAsync(level + root, &zero, 4, cudaMemcpyHostToDevice, s));
  EH_CUDA(cudaMemcpyAsync(fa.p, &root, 4, cudaMemcpyHostToDevice, s));
  uint32_t nf = 1, l = 0;
  uint32_t* f = fa.p;
  uint32_t* nx = fb.p;
  while (nf) {
    EH_CUDA(cudaMemsetAsync(cnt.p, 0, 4, s));
    k_bfs_step<<<grid_for((uint64_t)nf * 32, TB), TB, 0, s>>>(f, nf, off.p, adj.p, level, l + 1, nx, cnt.p);
    EH_LAUNCH("k_bfs_step");
    nf = read_scalar(cnt.p, s);
    std::swap(f, nx);
    ++l;
  }
  const uint32_t unreached = l;  // levels used: 0 .. l-1
  // ids never reached (other components, isolated ids) get `unreached`
  k_level_fix<<<grid_for(n_ids, TB * 4), TB, 0, s>>>(level, n_ids, unreached);
  EH_LAUNCH("k_level_fix");
  return unreached;
}

void build_trie(eh_graph* g, const uint32_t* d_src, const uint32_t* d_dst, uint64_t n, PhaseTimer* tm) {
  auto mark = [&](const char* p) { if (tm) tm->mark(p); };
  Allocator& al = g->alloc;
  cudaStream_t s = g->stream;
  const unsigned TB = 256;
  g->n_input = n;
  if (n == 0) {
    g->desc = (uint4*)g->own(sizeof(uint4));
    EH_CUDA(cudaMemsetAsync(g->desc, 0, sizeof(uint4), s));
    g->col = (uint32_t*)g->own(16);
    g->orig_id = (uint32_t*)g->own(16);
    return;
  }
  // ---- a1: id space; dictionary-encode if ids are spread out
  DBuf<uint32_t> dmax(al, 1);
  EH_CUDA(cudaMemsetAsync(dmax.p, 0, 4, s));
  k_max_id<<<grid_for(n, TB * 8), TB, 0, s>>>(d_src, d_dst, n, dmax.p);
  EH_LAUNCH("k_max_id");
  const uint32_t max_id = read_scalar(dmax.p, s);
  mark("max_id");
  uint64_t n_ids = (uint64_t)max_id + 1;
  DBuf<uint32_t> dict, msrc, mdst;
  const uint32_t* usrc = d_src;
  const uint32_t* udst = d_dst;
  if (n_ids > 8 * n + (1ull << 20)) {
    DBuf<uint32_t> ends(al, 2 * n), alt(al, 2 * n);
    EH_CUDA(cudaMemcpyAsync(ends.p, d_src, n * 4, cudaMemcpyDeviceToDevice, s));
    EH_CUDA(cudaMemcpyAsync(ends.p + n, d_dst, n * 4, cudaMemcpyDeviceToDevice, s));
    uint32_t* sorted = radix_sort_u32(ends.p, alt.p, 2 * n, bitlen(max_id), al, s);
    DBuf<uint32_t> d(al, 2 * n);
    n_ids = select_if(2 * n, UniqueU32Pred{sorted}, CopyU32Emit{sorted, d.p}, al, s);
    dict = std::move(d);
    msrc = DBuf<uint32_t>(al, n);
    mdst = DBuf<uint32_t>(al, n);
    k_dict_map<<<grid_for(n, TB * 4), TB, 0, s>>>(d_src, msrc.p, n, dict.p, n_ids);
    EH_LAUNCH("k_dict_map");
    k_dict_map<<<grid_for(n, TB * 4), TB, 0, s>>>(d_dst, mdst.p, n, dict.p, n_ids);
    EH_LAUNCH("k_dict_map");
    usrc = msrc.p;
    udst = mdst.p;
  }
  const uint32_t b = std::max<uint32_t>(1, bitlen(n_ids - 1));
  const uint64_t sentinel = (b >= 32) ? ~0ull : ((1ull << (2 * b)) - 1ull);

  // ---- a1-a4: canonical keys, deduplicated, and the degree of every id.
  // Default: the bucketed pass of dedup.cu (one MSD radix digit of the low end, an
  // on-chip hash set per bucket; the degrees come out of the same pass).  Test hook
  // EH_TEST_DEDUP=sort: LSD radix sort over the 2b significant bits, unique adjacent
  // keys, degrees from the sorted runs (round-1 default, kept as an ablation and as
  // the path for ids of 32 bits); EH_TEST_DEDUP=hash: one global hash set.
  const int dd_mode = [] {  // read on every load: a test hook set after the first load must take effect
    const char* e = getenv("EH_TEST_DEDUP");
    return !e ? 0 : (strcmp(e, "sort") == 0 ? 1 : (strcmp(e, "hash") == 0 ? 2 : 0));
  }();
  uint64_t m = 0, nk = 0;  // nk key entries; m of them are distinct non-loop edges
  DBuf<uint64_t> keys, alt;
  uint64_t* ukeys = nullptr;
  DBuf<uint32_t> deg(al, n_ids);
  EH_CUDA(cudaMemsetAsync(deg.p, 0, n_ids * 4, s));
  DBuf<unsigned long long> dm(al, 3);  // {m, max degree, n_act}: one host read
  EH_CUDA(cudaMemsetAsync(dm.p, 0, 24, s));
  const bool bucketed = dd_mode == 0 && bucket_dedup_ok(b, n);
  if (bucketed) {
    keys = DBuf<uint64_t>(al, n);  // m <= n distinct keys, compact
    bucket_dedup(usrc, udst, n, b, deg.p, dm.p, keys.p, g, tm);
    ukeys = keys.p;
    mark("dedup");
  } else if (dd_mode != 2) {
    keys = DBuf<uint64_t>(al, n);
    alt = DBuf<uint64_t>(al, n);
    // a1 canonicalisation fused into the sort's histogram and first pass; the
    // sorted keys are consumed in place (key_head), no compaction
    ukeys = radix_sort_canon(usrc, udst, n, b, keys.p, alt.p, al, s);
    nk = n;
    mark("sort1");
  } else {
    uint32_t tbits = 10;
    while ((1ull << tbits) < n + n / 2 + n / 10) ++tbits;
    DBuf<unsigned long long> tab(al, 1ull << tbits);
    EH_CUDA(cudaMemsetAsync(tab.p, 0xFF, tab.bytes(), s));
    k_hash_insert<<<grid_for(n, TB * 4), TB, 0, s>>>(usrc, udst, n, b, tab.p, tbits);
    EH_LAUNCH("k_hash_insert");
    mark("hash_insert");
    // m <= n: compact into an n-sized buffer
    keys = DBuf<uint64_t>(al, std::max<uint64_t>(1, n));
    nk = select_if(1ull << tbits, OccupiedPred{tab.p}, CopySlotEmit{tab.p, keys.p}, al, s);
    ukeys = keys.p;
  }
  msrc.reset();
  mdst.reset();
  if (!bucketed) mark("dedup");

  // ---- a4: degree + (degree, id) rank
  if (nk && !bucketed) {
    k_degree<<<grid_for(nk, TB * 4), TB, 0, s>>>(ukeys, nk, b, sentinel, deg.p, dm.p);
    EH_LAUNCH("k_degree");
  }
  k_deg_stats<<<grid_for(n_ids, TB * 8), TB, 0, s>>>(deg.p, n_ids, dm.p + 1);
  EH_LAUNCH("k_deg_stats");
  unsigned long long hm[3];
  EH_CUDA(cudaMemcpyAsync(hm, dm.p, 24, cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaStreamSynchronize(s));
  m = hm[0];
  g->m = m;
  if (bucketed) nk = m;
  const uint32_t max_deg = (uint32_t)hm[1];
  const uint64_t n_act = hm[2];
  // NEXT-4: the primary rank key of the chosen node ordering (default: degree)
  DBuf<uint64_t> prim;
  uint32_t pbits = bitlen(max_deg);
  if (g->order != EH_ORDER_DEGREE && m) {
    prim = DBuf<uint64_t>(al, n_ids);
    DBuf<uint32_t> aux;
    uint32_t aux_max = 0, aux_bits = 0;
    if (g->order == EH_ORDER_SHINGLE) {
      aux = DBuf<uint32_t>(al, n_ids);
      EH_CUDA(cudaMemsetAsync(aux.p, 0xFF, n_ids * 4, s));
      k_shingle<<<grid_for(nk, TB * 4), TB, 0, s>>>(ukeys, nk, b, sentinel, aux.p);
      EH_LAUNCH("k_shingle");
      pbits = 32;
    } else if (g->order == EH_ORDER_BFS || g->order == EH_ORDER_HYBRID) {
      aux = DBuf<uint32_t>(al, n_ids);
      aux_max = bfs_levels(ukeys, nk, m, b, sentinel, deg.p, n_ids, aux.p, al, s);  // level of unreached ids
      aux_bits = bitlen(aux_max);
      pbits = (g->order == EH_ORDER_BFS) ? aux_bits : bitlen(max_deg) + aux_bits;
    } else if (g->order == EH_ORDER_RANDOM) {
      pbits = 32;
    } else if (g->order == EH_ORDER_ID) {
      pbits = 1;  // primary 0 everywhere: ranks ascend by id
    }
    if (b + pbits > 64) fail(EH_EINVAL, "node ordering key needs %u bits", b + pbits);
    k_prim_simple<<<grid_for(n_ids, TB * 4), TB, 0, s>>>(deg.p, n_ids, g->order, max_deg, aux.p, aux_max, aux_bits,
                                                         prim.p);
    EH_LAUNCH("k_prim_simple");
  }
  DBuf<uint64_t> rkeys(al, std::max<uint64_t>(1, std::min<uint64_t>(n_ids, 2 * m))),
      ralt(al, std::max<uint64_t>(1, std::min<uint64_t>(n_ids, 2 * m)));
  select_emit(n_ids, ActivePred{deg.p}, RankKeyEmit{prim.p, deg.p, b, rkeys.p}, al, s);  // n_act known
  g->n_act = n_act;
  // select_if emits the ids in ascending order and LSD radix passes are stable:
  // sorting by the primary bits alone gives the (primary, id) order
  uint64_t* rsorted = radix_sort_u64(rkeys.p, ralt.p, n_act, b + pbits, al, s, b);
  prim.reset();
  DBuf<uint32_t>& rank = deg;  // k_rank turns deg[id] into rank[id] (and records deg per rank)
  g->orig_id = (uint32_t*)g->own(std::max<uint64_t>(1, n_act) * 4);
  g->deg_rank = (uint32_t*)g->own(std::max<uint64_t>(1, n_act) * 4);
  if (n_act) {
    k_rank<<<grid_for(n_act, TB * 4), TB, 0, s>>>(rsorted, n_act, b, rank.p, g->orig_id, dict.p, g->deg_rank);
    EH_LAUNCH("k_rank");
  }
  rkeys.reset();
  ralt.reset();
  mark("degree_rank");

  // ---- a5: orient + CSR (padded to 16 B per list)
  // The high end (in rank order) of every edge is scattered into a temporary list
  // of its low end with the low end's DEGREE as capacity (deg_rank, known since
  // k_rank: no orientation pass has to count |N+(x)| first); the cursors end as
  // |N+(x)|, which give the padded 16-B offsets of the final lists, and the
  // segmented sort moves each list into place, in order (segsort.cu).
  DBuf<uint64_t> toff(al, n_act + 1), tot(al, 1);
  scan_exclusive_u32(g->deg_rank, toff.p, n_act, tot.p, al, s);
  EH_CUDA(cudaMemcpyAsync(toff.p + n_act, tot.p, 8, cudaMemcpyDeviceToDevice, s));  // toff[n_act] = 2m
  DBuf<uint32_t> dplus(al, std::max<uint64_t>(1, n_act));
  EH_CUDA(cudaMemsetAsync(dplus.p, 0, std::max<uint64_t>(1, n_act) * 4, s));
  DBuf<uint32_t> tmp(al, std::max<uint64_t>(1, 2 * m));
  if (m) {
    k_scatter_col<true><<<grid_for(nk, TB * 4), TB, 0, s>>>(ukeys, nk, b, sentinel, rank.p, toff.p, dplus.p, tmp.p);
    EH_LAUNCH("k_scatter_col");
  }
  mark("scatter");
  deg.reset();
  keys.reset();  // the sorted keys are consumed
  alt.reset();
  DBuf<uint64_t> off16(al, n_act + 1);
  DBuf<uint32_t> p4(al, std::max<uint64_t>(1, n_act));
  k_pad4<<<grid_for(n_act, TB * 4), TB, 0, s>>>(dplus.p, n_act, p4.p);
  EH_LAUNCH("k_pad4");
  scan_exclusive_u32(p4.p, off16.p, n_act, tot.p, al, s);
  // max |N+(x)| depends only on dplus: read it with the padded total (one host read)
  DBuf<unsigned long long> totmax(al, 2);
  EH_CUDA(cudaMemsetAsync(totmax.p, 0, 16, s));
  EH_CUDA(cudaMemcpyAsync(totmax.p, tot.p, 8, cudaMemcpyDeviceToDevice, s));
  k_max_u32<<<grid_for(n_act, TB * 8), TB, 0, s>>>(dplus.p, n_act, reinterpret_cast<uint32_t*>(totmax.p + 1));
  EH_LAUNCH("k_max_u32");
  unsigned long long htm[2];
  EH_CUDA(cudaMemcpyAsync(htm, totmax.p, 16, cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaStreamSynchronize(s));
  const uint64_t total16 = htm[0];
  g->max_dplus = htm[1];
  if (total16 >= (1ull << 32)) fail(EH_EINVAL, "graph too large: %llu padded 16-B list blocks", (unsigned long long)total16);
  g->col_elems = total16 * 4;
  g->col = (uint32_t*)g->own(std::max<uint64_t>(16, total16 * 16));
  EH_CUDA(cudaMemsetAsync(g->col, 0xFF, std::max<uint64_t>(16, total16 * 16), s));
  mark("orient");
  segmented_sort_u32_into(tmp.p, toff.p, g->col, off16.p, dplus.p, n_act, (uint32_t)g->max_dplus, al, s, g);
  mark("segsort");
  g->desc = (uint4*)g->own((n_act + 1) * sizeof(uint4));
  k_desc_base<<<grid_for(n_act + 1, TB * 4), TB, 0, s>>>(off16.p, dplus.p, n_act, total16, g->desc);
  EH_LAUNCH("k_desc_base");
  mark("csr");
}

}  // namespace eh
