// trie.cu -- SURVEY.md §8(a) rows a6 (set-level layout) and a7 (work classes).
//
// Set-level optimizer: "selects the bitset layout when each value
// in the set consumes at most as much space as a SIMD (AVX) register and the uint
// layout otherwise ... with a block size equal to the range of the data in the
// set".  Reading c10/c11: bitset iff span < tau * |S| with
// span = max - min + 1, tau = 32 by default (256 reproduces the paper's AVX
// register); the span is stored as whole 128-bit chunks at ABSOLUTE positions
// (chunk c holds ids [128c, 128c + 128)), so any two bitsets -- and a bitset and
// a staged bitmap -- AND chunk-to-chunk without shifting.  The uint layout
// is the padded `col` segment, kept for every set because the
// loop nests iterate it ("for x in xs", Table `lst:eh_operators`).
#include "eh_internal.cuh"
#include "primitives.cuh"
#include "rows.cuh"

namespace eh {

namespace {

// Per vertex: layout decision, chunk count, first chunk and B_tri bytes(S).
__global__ void k_layout(const uint4* __restrict__ desc, const uint32_t* __restrict__ col, uint64_t n_act,
                         uint32_t tau, uint32_t min_card, bool all_uint, uint32_t* __restrict__ nchunks,
                         uint32_t* __restrict__ chunk0, uint32_t* __restrict__ bytes_tau) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n_act; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 d = desc[v];
    uint32_t nc = 0, c0 = 0, by = 4u * d.y;
    if (d.y > 0) {
      const uint32_t first = col[(uint64_t)d.x * 4], last = col[(uint64_t)d.x * 4 + d.y - 1];
      const uint64_t span = (uint64_t)last - first + 1;
      if (!all_uint && d.y >= min_card && span < (uint64_t)tau * d.y) {
        c0 = first >> 7;
        nc = (last >> 7) - c0 + 1;
      }
      // B_tri's bytes(S) is defined at tau = 32 whatever layout the kernels use
      // (SURVEY.md §8(d)): words spanned for a tau=32 bitset, else 4|S|.
      if (span < 32ull * d.y) by = 4u * ((last >> 5) - (first >> 5) + 1);
    }
    nchunks[v] = nc;
    chunk0[v] = c0;
    bytes_tau[v] = by;
  }
}

// no_algo (EH_NO_ALGO, the "-RA" ablation): every set is uint and its first-chunk
// field carries kNoAlgo, which the row dispatch reads as "never gallop".
__global__ void k_desc_layout(uint4* __restrict__ desc, const uint64_t* __restrict__ bs_off,
                              const uint32_t* __restrict__ chunk0, uint64_t n_act, uint64_t total, bool no_algo) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n_act; v += (uint64_t)gridDim.x * blockDim.x) {
    desc[v].z = (uint32_t)(v < n_act ? bs_off[v] : total);
    desc[v].w = (v < n_act) ? (no_algo ? kNoAlgo : chunk0[v]) : 0u;
  }
}

// Fill the bitset pool: one warp per set, lanes over elements.
__global__ void k_fill_bitsets(const uint4* __restrict__ desc, const uint32_t* __restrict__ col, uint64_t n_act,
                               uint32_t* __restrict__ bs) {
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint64_t v = warp; v < n_act; v += nwarps) {
    const uint4 d = desc[v];
    const uint32_t nc = desc[v + 1].z - d.z;
    if (nc == 0) continue;
    const uint64_t base = (uint64_t)d.z * 4;  // pool word of absolute word 4 * chunk0
    for (uint32_t i = lane; i < d.y; i += 32) {
      const uint32_t e = col[(uint64_t)d.x * 4 + i];
      atomicOr(&bs[base + ((e >> 5) - 4ull * d.w)], 1u << (e & 31));
    }
  }
}

// B_tri(tau) pieces and the wedge work sum_(x,y) |N+(x) after y| = sum_x C(d,2).
__global__ void k_stats(const uint4* __restrict__ desc, const uint32_t* __restrict__ col, uint64_t n_act,
                        const uint32_t* __restrict__ bytes_tau, unsigned long long* __restrict__ out) {
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  unsigned long long ysum = 0, xsum = 0, wedge = 0, nbs = 0;
  for (uint64_t v = warp; v < n_act; v += nwarps) {
    const uint4 d = desc[v];
    if (lane == 0) {
      xsum += bytes_tau[v];
      wedge += (unsigned long long)d.y * (d.y - (d.y > 0)) / 2;
      nbs += (desc[v + 1].z != d.z);
    }
    for (uint32_t i = lane; i < d.y; i += 32) ysum += bytes_tau[col[(uint64_t)d.x * 4 + i]];
  }
  ysum = warp_sum(ysum);
  if (lane == 0) {
    atomicAdd(&out[0], ysum);
    atomicAdd(&out[1], xsum);
    atomicAdd(&out[2], wedge);
    atomicAdd(&out[3], nbs);
  }
}

// Work lists: vertices with |N+(x)| >= 2 (others close no triangle) by class.
struct WorkPred {
  const uint4* desc;
  uint32_t lo, hi;  // lo <= d < hi (hi unbounded if open)
  bool open;
  __device__ bool operator()(uint64_t v) const {
    const uint32_t d = desc[v].y;
    return d >= lo && (open || d < hi);
  }
};
struct WorkEmit {
  uint32_t* out;
  __device__ void operator()(uint64_t pos, uint64_t v) const { out[pos] = (uint32_t)v; }
};

}  // namespace

void build_layouts(eh_graph* g) {
  Allocator& al = g->alloc;
  cudaStream_t s = g->stream;
  const uint64_t n = g->n_act;
  const unsigned TB = 256;
  if (n == 0) {
    g->bs = (uint32_t*)g->own(16);
    return;
  }
  DBuf<uint32_t> nch(al, n), c0(al, n);
  g->bytes32 = (uint32_t*)g->own(n * 4);  // kept for the on-demand statistics (compute_stats)
  k_layout<<<grid_for(n, TB * 4), TB, 0, s>>>(g->desc, g->col, n, g->tau, g->min_bitset_card,
                                              (g->flags & EH_ALL_UINT) != 0, nch.p, c0.p, g->bytes32);
  EH_LAUNCH("k_layout");
  DBuf<uint64_t> off(al, n), tot(al, 1);
  scan_exclusive_u32(nch.p, off.p, n, tot.p, al, s);
  const uint64_t total = read_scalar(tot.p, s);
  if (total >= (1ull << 32)) fail(EH_EINVAL, "bitset pool too large (%llu chunks)", (unsigned long long)total);
  k_desc_layout<<<grid_for(n + 1, TB * 4), TB, 0, s>>>(g->desc, off.p, c0.p, n, total, (g->flags & EH_NO_ALGO) != 0);
  EH_LAUNCH("k_desc_layout");
  g->bs_words = total * 4;
  g->bs = (uint32_t*)g->own(std::max<uint64_t>(16, total * 16));
  EH_CUDA(cudaMemsetAsync(g->bs, 0, std::max<uint64_t>(16, total * 16), s));
  if (total) {
    k_fill_bitsets<<<grid_for(n * 32, TB), TB, 0, s>>>(g->desc, g->col, n, g->bs);
    EH_LAUNCH("k_fill_bitsets");
  }
}

// Statistics that are not needed by the counts (B_tri, wedge work, number of
// bitset sets) are computed on the first eh_graph_stats call, off the load path.
void compute_stats(eh_graph* g) {
  if (g->stats_ready) return;
  const uint64_t n = g->n_act;
  if (n) {
    cudaStream_t s = g->stream;
    const unsigned TB = 256;
    DBuf<unsigned long long> st(g->alloc, 4);
    EH_CUDA(cudaMemsetAsync(st.p, 0, 4 * sizeof(unsigned long long), s));
    k_stats<<<grid_for(n * 32, TB), TB, 0, s>>>(g->desc, g->col, n, g->bytes32, st.p);
    EH_LAUNCH("k_stats");
    unsigned long long h[4];
    EH_CUDA(cudaMemcpyAsync(h, st.p, sizeof h, cudaMemcpyDeviceToHost, s));
    EH_CUDA(cudaStreamSynchronize(s));
    g->alg_bytes_tri = 8ull * (n + 1) + h[1] + h[0];
    g->wedge_work = h[2];
    g->n_bitsets = h[3];
  } else {
    g->alg_bytes_tri = 8;
  }
  g->stats_ready = true;
}

void build_worklists(eh_graph* g) {
  // Three classes by d = |N+(x)| (d >= 2 only): 0 = [2, small_max], 1 = (small_max, large_min),
  // 2 = [large_min, inf).  The triangle and per-vertex kernels run class 0 warp-per-x and
  // classes 1-2 CTA-per-x; the 4-clique kernels run classes 0-1 warp-per-x and class 2
  // CTA-per-x.  The warp kernels stage N+(x) in a fixed shared-memory slot, so d above
  // their capacity always lands in class 2 whatever the configuration asks for.
  Allocator& al = g->alloc;
  cudaStream_t s = g->stream;
  const uint64_t n = g->n_act;
  const uint64_t cap = (uint64_t)tri_warp_max_degree() + 1;
  const uint64_t large_min = std::min<uint64_t>(g->bin_large_min ? g->bin_large_min : cap, cap);
  const uint64_t small_max = std::min<uint64_t>(g->bin_small_max ? g->bin_small_max : 64, large_min - 1);
  g->work = (uint32_t*)g->own(std::max<uint64_t>(1, n) * 4);
  uint64_t lo[3], hi[3];  // class c holds lo[c] <= d < hi[c]
  lo[0] = 2;
  hi[0] = std::max<uint64_t>(2, small_max + 1);
  lo[1] = hi[0];
  hi[1] = std::max<uint64_t>(lo[1], large_min);
  lo[2] = hi[1];
  hi[2] = 1ull << 33;
  uint64_t pos = 0;
  for (int c = 0; c < 3; ++c) {
    const uint32_t l = (uint32_t)std::min<uint64_t>(lo[c], 0xFFFFFFFFull);
    const uint32_t h = (uint32_t)std::min<uint64_t>(hi[c], 0xFFFFFFFFull);
    const uint64_t k = (n == 0 || lo[c] >= hi[c]) ? 0
                       : select_if(n, WorkPred{g->desc, l, h, hi[c] > 0xFFFFFFFFull},
                                   WorkEmit{g->work + pos}, al, s);
    g->n_work[c] = k;
    pos += k;
  }
}

}  // namespace eh
