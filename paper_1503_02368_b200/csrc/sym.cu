// sym.cu -- SURVEY.md §8(f) NEXT-2: the symmetric (unpruned) trie.
//
// The paper's "Default" data: every undirected edge in
// both directions, ids assigned by degree, no symmetry breaking; the
// Generic-Join then binds ordered tuples (6T, 24 K4).
// Built lazily from the oriented trie of the same handle: in rank space every
// in-neighbour of v precedes v and every out-neighbour follows it, so the full
// list N(v) is the sorted in-list followed by N+(v) -- a scatter of the reverse
// edges, an on-chip sort of the in-parts (segsort.cu), a copy of the out-parts.
// The result is a second eh_graph (same device, stream and allocator) whose
// "N+(v)" is N(v), with its own set layouts (trie.cu, same tau) and work
// classes, so the layout and count machinery applies unchanged.
#include "eh_internal.cuh"
#include "primitives.cuh"

#include <algorithm>

namespace eh {

namespace {

// in-degree of every rank: one atomic per oriented edge (x, y) on y
__global__ void k_in_degree(const uint4* __restrict__ desc, const uint32_t* __restrict__ col, uint64_t n,
                            uint32_t* __restrict__ din) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t x = warp; x < n; x += nw) {
    const uint4 d = __ldg(desc + x);
    for (uint32_t k = lane; k < d.y; k += 32) atomicAdd(&din[__ldg(col + (uint64_t)d.x * 4 + k)], 1u);
  }
}

__global__ void k_sym_len(const uint4* __restrict__ desc, const uint32_t* __restrict__ din, uint64_t n,
                          uint32_t* __restrict__ deg, uint32_t* __restrict__ p4) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t d = din[v] + desc[v].y;
    deg[v] = d;
    p4[v] = (d + 3u) >> 2;
  }
}

// out-part copied in order after the in-part; in-part scattered (cursor per y)
__global__ void k_sym_fill(const uint4* __restrict__ desc, const uint32_t* __restrict__ col, uint64_t n,
                           const uint64_t* __restrict__ off16, const uint32_t* __restrict__ din,
                           uint32_t* __restrict__ cursor, uint32_t* __restrict__ scol) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t x = warp; x < n; x += nw) {
    const uint4 d = __ldg(desc + x);
    uint32_t* out = scol + off16[x] * 4 + din[x];
    for (uint32_t k = lane; k < d.y; k += 32) {
      const uint32_t y = __ldg(col + (uint64_t)d.x * 4 + k);
      out[k] = y;
      scol[off16[y] * 4 + atomicAdd(&cursor[y], 1u)] = (uint32_t)x;
    }
  }
}

__global__ void k_sym_desc(const uint64_t* __restrict__ off16, const uint32_t* __restrict__ deg, uint64_t n,
                           uint64_t total16, uint4* __restrict__ desc) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n; v += (uint64_t)gridDim.x * blockDim.x)
    desc[v] = (v < n) ? make_uint4((uint32_t)off16[v], deg[v], 0u, 0u) : make_uint4((uint32_t)total16, 0u, 0u, 0u);
}

__global__ void k_max_u32_sym(const uint32_t* __restrict__ a, uint64_t n, uint32_t* __restrict__ out) {
  uint32_t mx = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    mx = max(mx, a[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

}  // namespace

static void build_symmetric(eh_graph* g, eh_graph* h);

eh_graph* symmetric_trie(eh_graph* g) {
  if (g->sym) return g->sym;
  eh_graph* h = new eh_graph();
  try {
    build_symmetric(g, h);
  } catch (...) {
    cudaStreamSynchronize(h->stream);
    for (void* p : h->owned) h->alloc.release(p);
    delete h;
    throw;
  }
  g->sym = h;  // owned by g from here on (destroy() frees it)
  return h;
}

static void build_symmetric(eh_graph* g, eh_graph* h) {
  h->device = g->device;
  h->stream = g->stream;
  h->own_stream = false;
  h->alloc = g->alloc;
  h->flags = g->flags;
  h->tau = g->tau;
  h->min_bitset_card = g->min_bitset_card;
  h->bin_small_max = g->bin_small_max;
  h->bin_large_min = g->bin_large_min;
  h->n_input = g->n_input;
  h->m = g->m;
  h->n_act = g->n_act;
  Allocator& al = h->alloc;
  cudaStream_t s = h->stream;
  const uint64_t n = h->n_act;
  const unsigned TB = 256;
  h->d_counter = (unsigned long long*)h->own(8 * sizeof(unsigned long long));
  if (n == 0) {
    h->desc = (uint4*)h->own(sizeof(uint4));
    EH_CUDA(cudaMemsetAsync(h->desc, 0, sizeof(uint4), s));
    h->col = (uint32_t*)h->own(16);
    build_layouts(h);
    build_worklists(h);
    return;
  }
  DBuf<uint32_t> din(al, n), deg(al, n), p4(al, n), dmax(al, 2);
  EH_CUDA(cudaMemsetAsync(din.p, 0, n * 4, s));
  k_in_degree<<<grid_for(n * 32, TB), TB, 0, s>>>(g->desc, g->col, n, din.p);
  EH_LAUNCH("k_in_degree");
  k_sym_len<<<grid_for(n, TB * 4), TB, 0, s>>>(g->desc, din.p, n, deg.p, p4.p);
  EH_LAUNCH("k_sym_len");
  DBuf<uint64_t> off16(al, n + 1), tot(al, 1);
  scan_exclusive_u32(p4.p, off16.p, n, tot.p, al, s);
  EH_CUDA(cudaMemsetAsync(dmax.p, 0, 8, s));
  k_max_u32_sym<<<grid_for(n, TB * 8), TB, 0, s>>>(deg.p, n, dmax.p);
  EH_LAUNCH("k_max_u32_sym");
  k_max_u32_sym<<<grid_for(n, TB * 8), TB, 0, s>>>(din.p, n, dmax.p + 1);
  EH_LAUNCH("k_max_u32_sym");
  uint64_t total16 = 0;
  uint32_t mx[2] = {0, 0};
  EH_CUDA(cudaMemcpyAsync(&total16, tot.p, 8, cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaMemcpyAsync(mx, dmax.p, 8, cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaStreamSynchronize(s));
  if (total16 >= (1ull << 32)) fail(EH_EINVAL, "symmetric trie too large: %llu padded 16-B list blocks",
                                    (unsigned long long)total16);
  h->max_dplus = mx[0];
  h->col_elems = total16 * 4;
  h->col = (uint32_t*)h->own(std::max<uint64_t>(16, total16 * 16));
  EH_CUDA(cudaMemsetAsync(h->col, 0xFF, std::max<uint64_t>(16, total16 * 16), s));
  EH_CUDA(cudaMemsetAsync(p4.p, 0, n * 4, s));  // reuse as cursors
  k_sym_fill<<<grid_for(n * 32, TB), TB, 0, s>>>(g->desc, g->col, n, off16.p, din.p, p4.p, h->col);
  EH_LAUNCH("k_sym_fill");
  segmented_sort_u32(h->col, off16.p, din.p, n, mx[1], al, s);  // the in-parts
  h->desc = (uint4*)h->own((n + 1) * sizeof(uint4));
  k_sym_desc<<<grid_for(n + 1, TB * 4), TB, 0, s>>>(off16.p, deg.p, n, total16, h->desc);
  EH_LAUNCH("k_sym_desc");
  build_layouts(h);
  build_worklists(h);
}

}  // namespace eh
