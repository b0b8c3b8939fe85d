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

// marker (EH_NO_ALGO, the "-RA" ablation / EH_FORCE_SEARCH): every set is uint and its
// first-chunk field carries kNoAlgo / kAlwaysSearch, which the row dispatch reads as
// "never gallop" / "always gallop".
__global__ void k_desc_layout(uint4* __restrict__ desc, const uint64_t* __restrict__ bs_off,
                              const uint32_t* __restrict__ chunk0, uint64_t n_act, uint64_t total, uint32_t marker) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n_act; v += (uint64_t)gridDim.x * blockDim.x) {
    desc[v].z = (uint32_t)(v < n_act ? bs_off[v] : total);
    desc[v].w = (v < n_act) ? (marker ? marker : chunk0[v]) : 0u;
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

// Work lists: vertices with |N+(x)| >= 2 (others close no triangle) by class;
// the thread class (2 <= d < ht) is emitted first, as the head of class 0.
struct WorkClass {  // 0: 2 <= d < ht, 1: ht <= d < h0, 2: h0 <= d < h1, 3: d >= h1 (and d >= 2); -1: d < 2
  const uint4* desc;
  uint32_t ht, h0, h1;
  __device__ int operator()(uint64_t v) const {
    const uint32_t d = desc[v].y;
    return d < 2 ? -1 : d < ht ? 0 : d < h0 ? 1 : d < h1 ? 2 : 3;
  }
};
struct WorkEmit3 {
  uint32_t* out;
  __device__ void operator()(int, uint64_t pos, uint64_t v) const { out[pos] = (uint32_t)v; }
};
struct WorkEmit {
  uint32_t* out;
  __device__ void operator()(uint64_t pos, uint64_t v) const { out[pos] = (uint32_t)v; }
};

// (descending d, ascending x) sort key of a work-list entry, and back
__global__ void k_work_key(const uint4* __restrict__ desc, const uint32_t* __restrict__ w, uint64_t n, uint32_t dmax,
                           uint64_t* __restrict__ key) {
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x)
    key[k] = ((uint64_t)(dmax - desc[w[k]].y) << 32) | w[k];
}
__global__ void k_work_unkey(const uint64_t* __restrict__ key, uint64_t n, uint32_t* __restrict__ w) {
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x)
    w[k] = (uint32_t)key[k];
}

// Rank-range restriction of the work lists (eh_count_*_range): position k of a
// class-major list keeps its class iff the vertex lies in [r0, r1).
struct RangeClass {
  const uint32_t* w;
  uint64_t et, e0, e1;  // class boundaries (positions): thread head of class 0, classes 0, 1
  uint32_t r0, r1;
  __device__ int operator()(uint64_t k) const {
    const uint32_t v = w[k];
    if (v < r0 || v >= r1) return -1;
    return k < et ? 0 : k < e0 ? 1 : k < e1 ? 2 : 3;
  }
};
struct RangeEmit {
  const uint32_t* w;
  uint32_t* out;
  __device__ void operator()(int, uint64_t pos, uint64_t k) const { out[pos] = w[k]; }
};

// B_K4: sum over triangles x < y < z of bytes(N+(z)) at tau = 32.
// One warp per x (grid-stride); for each row y = x_i, the lanes take z in
// N+(x) after y and binary-search N+(y).  Statistics only (not on a count path).
__global__ void k_k4_bytes(const uint4* __restrict__ desc, const uint32_t* __restrict__ col, uint64_t n_act,
                           const uint32_t* __restrict__ bytes_tau, unsigned long long* __restrict__ out) {
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  unsigned long long acc = 0;
  for (uint64_t x = warp; x < n_act; x += nwarps) {
    const uint4 dx = desc[x];
    const uint32_t* xs = col + (uint64_t)dx.x * 4;
    for (uint32_t i = 0; i + 1 < dx.y; ++i) {
      const uint4 dy = desc[xs[i]];
      if (dy.y == 0) continue;
      const uint32_t* ys = col + (uint64_t)dy.x * 4;
      for (uint32_t j = i + 1 + lane; j < dx.y; j += 32) {
        const uint32_t z = xs[j];
        uint32_t lo = 0, hi = dy.y;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (ys[mid] < z) lo = mid + 1; else hi = mid;
        }
        if (lo < dy.y && ys[lo] == z) acc += bytes_tau[z];
      }
    }
  }
  acc = warp_sum(acc);
  if (lane == 0 && acc) atomicAdd(out, acc);
}

}  // namespace

WorkRange::WorkRange(eh_graph* g, uint64_t r0, uint64_t r1) : g_(g) {
  saved_work_ = g->work;
  saved_lpt_ = g->work_lpt;
  saved_nt_ = g->n_thread;
  for (int c = 0; c < 3; ++c) saved_n_[c] = g->n_work[c];
  const uint64_t n = saved_n_[0] + saved_n_[1] + saved_n_[2];
  r1 = std::min<uint64_t>(r1, g->n_act);
  if (r0 >= r1) r0 = r1 = 0;
  // the LPT list is filtered too, so the kernels that take it keep their order
  const uint32_t* lpt = (n && g->work_lpt) ? g->work_lpt : nullptr;
  work_ = DBuf<uint32_t>(g->alloc, std::max<uint64_t>(1, n));
  uint64_t starts[5] = {0, 0, 0, 0, 0};
  const RangeClass rc{saved_work_, saved_nt_, saved_n_[0], saved_n_[0] + saved_n_[1], (uint32_t)r0, (uint32_t)r1};
  partition_k<4>(n, rc, RangeEmit{saved_work_, work_.p}, starts, g->alloc, g->stream);
  if (lpt) {  // same class boundaries (the LPT order permutes inside classes 1-2 only)
    lpt_ = DBuf<uint32_t>(g->alloc, std::max<uint64_t>(1, n));
    RangeClass rl = rc;
    rl.w = lpt;
    uint64_t st2[5];
    partition_k<4>(n, rl, RangeEmit{lpt, lpt_.p}, st2, g->alloc, g->stream);
  }
  g->work = work_.p;
  g->work_lpt = lpt ? lpt_.p : nullptr;
  g->n_thread = starts[1] - starts[0];
  for (int c = 0; c < 3; ++c) g->n_work[c] = starts[c + 2] - starts[c == 0 ? 0 : c + 1];
}

WorkRange::~WorkRange() {
  cudaStreamSynchronize(g_->stream);  // the filtered lists are released below
  // a work_lpt() built while restricted belongs to the handle (g->owned) but lists only
  // the range: it is dropped here (its memory stays with the handle until eh_free)
  g_->work = saved_work_;
  g_->work_lpt = saved_lpt_;
  g_->n_thread = saved_nt_;
  for (int c = 0; c < 3; ++c) g_->n_work[c] = saved_n_[c];
}

uint64_t alg_bytes_k4(eh_graph* g) {
  compute_stats(g);
  if (g->alg_bytes_k4) return g->alg_bytes_k4;
  uint64_t tri_z = 0;
  if (g->n_act) {
    cudaStream_t s = g->stream;
    DBuf<unsigned long long> acc(g->alloc, 1);
    EH_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(unsigned long long), s));
    k_k4_bytes<<<kSMs * 8, 256, 0, s>>>(g->desc, g->col, g->n_act, g->bytes32, acc.p);
    EH_LAUNCH("k_k4_bytes");
    tri_z = read_scalar(reinterpret_cast<const uint64_t*>(acc.p), s);
  }
  g->alg_bytes_k4 = g->alg_bytes_tri + tri_z;
  return g->alg_bytes_k4;
}

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
  k_desc_layout<<<grid_for(n + 1, TB * 4), TB, 0, s>>>(g->desc, off.p, c0.p, n, total,
                                                       (g->flags & EH_NO_ALGO) ? kNoAlgo : (g->flags & EH_FORCE_SEARCH) ? kAlwaysSearch : 0u);
  EH_LAUNCH("k_desc_layout");
  g->bs_words = total * 4;
  g->bs = (uint32_t*)g->own(std::max<uint64_t>(16, total * 16));
  EH_CUDA(cudaMemsetAsync(g->bs, 0, std::max<uint64_t>(16, total * 16), s));
  if (total) {
    k_fill_bitsets<<<grid_for(n * 32, TB), TB, 0, s>>>(g->desc, g->col, n, g->bs);
    EH_LAUNCH("k_fill_bitsets");
  }
}

// ---- NEXT-3: block-level (composite) layout -------------
// Each set N+(v) is split into 128-id blocks (the chunks of the set-level
// bitsets, reading c11); a block holding >= kDenseMin elements becomes a bitset
// block (16 B <= 4 B per element, the set optimizer's space rule applied per
// block), the others stay uint.  One thread per set, two passes (count, fill).
constexpr uint32_t kDenseMin = 4;

__global__ void k_block_count(const uint4* __restrict__ desc, const uint32_t* __restrict__ col, uint64_t n,
                              uint32_t* __restrict__ ns4, uint32_t* __restrict__ nd) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 d = desc[v];
    const uint32_t* l = col + (uint64_t)d.x * 4;
    uint32_t sparse = 0, dense = 0;
    for (uint32_t i = 0; i < d.y;) {
      const uint32_t c = l[i] >> 7;
      uint32_t j = i + 1;
      while (j < d.y && (l[j] >> 7) == c) ++j;
      if (j - i >= kDenseMin) ++dense; else sparse += j - i;
      i = j;
    }
    ns4[v] = (sparse + 3) >> 2;
    nd[v] = dense;
  }
}

__global__ void k_block_fill(const uint4* __restrict__ desc, const uint32_t* __restrict__ col, uint64_t n,
                             const uint64_t* __restrict__ soff16, const uint64_t* __restrict__ doff,
                             uint32_t* __restrict__ bcol, uint32_t* __restrict__ bcid, uint4* __restrict__ bmask,
                             uint4* __restrict__ bdesc, uint64_t total16, uint64_t total_dense) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n; v += (uint64_t)gridDim.x * blockDim.x) {
    if (v == n) {
      bdesc[n] = make_uint4((uint32_t)total16, 0u, (uint32_t)total_dense, 0u);
      continue;
    }
    const uint4 d = desc[v];
    const uint32_t* l = col + (uint64_t)d.x * 4;
    uint32_t* sp = bcol + soff16[v] * 4;
    uint64_t db = doff[v];
    uint32_t ns = 0;
    for (uint32_t i = 0; i < d.y;) {
      const uint32_t c = l[i] >> 7;
      uint32_t j = i + 1;
      while (j < d.y && (l[j] >> 7) == c) ++j;
      if (j - i >= kDenseMin) {
        uint32_t w[4] = {0u, 0u, 0u, 0u};
        for (uint32_t k = i; k < j; ++k) w[(l[k] >> 5) & 3] |= 1u << (l[k] & 31);
        bcid[db] = c;
        bmask[db] = make_uint4(w[0], w[1], w[2], w[3]);
        ++db;
      } else {
        for (uint32_t k = i; k < j; ++k) sp[ns++] = l[k];
      }
      i = j;
    }
    bdesc[v] = make_uint4((uint32_t)soff16[v], ns, (uint32_t)doff[v], 0u);
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

void build_block_layout(eh_graph* g) {
  Allocator& al = g->alloc;
  cudaStream_t s = g->stream;
  const uint64_t n = g->n_act;
  const unsigned TB = 256;
  DBuf<uint32_t> ns4(al, std::max<uint64_t>(1, n)), nd(al, std::max<uint64_t>(1, n));
  if (n) {
    k_block_count<<<grid_for(n, TB), TB, 0, s>>>(g->desc, g->col, n, ns4.p, nd.p);
    EH_LAUNCH("k_block_count");
  }
  DBuf<uint64_t> soff(al, n + 1), doff(al, n + 1), tot(al, 2);
  scan_exclusive_u32(ns4.p, soff.p, n, tot.p, al, s);
  scan_exclusive_u32(nd.p, doff.p, n, tot.p + 1, al, s);
  uint64_t h[2] = {0, 0};
  EH_CUDA(cudaMemcpyAsync(h, tot.p, 16, cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaStreamSynchronize(s));
  if (h[0] >= (1ull << 32) || h[1] >= (1ull << 32)) fail(EH_EINVAL, "block layout too large");
  g->bcol = (uint32_t*)g->own(std::max<uint64_t>(16, h[0] * 16));
  EH_CUDA(cudaMemsetAsync(g->bcol, 0xFF, std::max<uint64_t>(16, h[0] * 16), s));
  g->bcid = (uint32_t*)g->own(std::max<uint64_t>(1, h[1]) * 4);
  g->bmask = (uint4*)g->own(std::max<uint64_t>(1, h[1]) * 16);
  g->bdesc = (uint4*)g->own((n + 1) * sizeof(uint4));
  k_block_fill<<<grid_for(n + 1, TB), TB, 0, s>>>(g->desc, g->col, n, soff.p, doff.p, g->bcol, g->bcid, g->bmask,
                                                  g->bdesc, h[0], h[1]);
  EH_LAUNCH("k_block_fill");
  g->n_dense_blocks = h[1];
  EH_CUDA(cudaStreamSynchronize(s));
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
  g->class0_max = (uint32_t)(hi[0] - 1);
  lo[1] = hi[0];
  hi[1] = std::max<uint64_t>(lo[1], large_min);
  lo[2] = hi[1];
  hi[2] = 1ull << 33;
  // thread class = the head of class 0 with d <= thread_max (a7)
  // default 8, 4 above 2^24 active ids (measured, bin_thread_max 1 / 4 / 8 / 12 / 16: C3 8.39 / 8.01 /
  // 7.88 / 7.84 / 7.90 ms, C4 1.42 / 1.33 / 1.31 / 1.30 / 1.30, C2 0.312 / 0.294 / 0.302 / 0.314 / 0.339,
  // C5 864 / 856 / 864 / 872 / 885)
  // re-measured with the round-2 kernels (8 / 12 / 16): C3 7.90 / 7.79 / 7.72 ms, C4 1.19 / 1.14 / 1.11,
  // C2 0.248 / 0.235 / 0.260; C5 (2 / 4 / 8) 623 / 619 / 623 -- 16 above 2^19 active ids, 12 below, 4 above 2^24
  const uint32_t tdef = g->n_act > (1ull << 24) ? 4u : g->n_act > (1ull << 19) ? 16u : kThreadMaxDefault;
  const uint64_t tmax = std::min<uint64_t>(g->bin_thread_max ? g->bin_thread_max : tdef,
                                           std::min<uint64_t>(hi[0] - 1, tri_thread_max_degree()));
  const uint64_t ht = std::max<uint64_t>(2, tmax + 1);
  // one stable 4-way partition (class-major, each class in rank order)
  uint64_t starts[5];
  partition_k<4>(n, WorkClass{g->desc, (uint32_t)ht, (uint32_t)hi[0], (uint32_t)std::min<uint64_t>(hi[1], 0xFFFFFFFFull)},
                 WorkEmit3{g->work}, starts, al, s);
  g->n_thread = starts[1] - starts[0];
  g->n_work[0] = starts[2] - starts[0];
  for (int c = 1; c < 3; ++c) g->n_work[c] = starts[c + 2] - starts[c + 1];
}

// The work lists with classes 1 and 2 each in descending-d order (heaviest x
// first: longest-processing-time order, so the per-x tails of the persistent CTA
// kernels overlap the rest of the work).  Built on first use and kept in the
// handle; used by the 4-clique and per-vertex kernels (measured: C4 K4 7.62 ->
// 7.38 ms, C3 t(v) 19.6 -> 17.5 ms).  The triangle kernels keep rank order
// (measured 0.3 % slower in LPT order at C3).
const uint32_t* work_lpt(eh_graph* g) {
  if (g->work_lpt) return g->work_lpt;
  Allocator& al = g->alloc;
  cudaStream_t s = g->stream;
  const uint64_t n = g->n_work[0] + g->n_work[1] + g->n_work[2];
  uint32_t* w = (uint32_t*)g->own(std::max<uint64_t>(1, n) * 4);
  if (n) EH_CUDA(cudaMemcpyAsync(w, g->work, n * 4, cudaMemcpyDeviceToDevice, s));
  uint64_t pos = g->n_work[0];
  for (int c = 1; c < 3; ++c) {
    const uint64_t k = g->n_work[c];
    if (k > 1) {
      DBuf<uint64_t> key(al, k), alt(al, k);
      k_work_key<<<grid_for(k, 1024), 256, 0, s>>>(g->desc, w + pos, k, (uint32_t)g->max_dplus, key.p);
      EH_LAUNCH("k_work_key");
      const uint64_t* sorted = radix_sort_u64(key.p, alt.p, k, 32 + bitlen(g->max_dplus), al, s);
      k_work_unkey<<<grid_for(k, 1024), 256, 0, s>>>(sorted, k, w + pos);
      EH_LAUNCH("k_work_unkey");
      EH_CUDA(cudaStreamSynchronize(s));  // key / alt are released on return
    }
    pos += k;
  }
  g->work_lpt = w;
  return w;
}

}  // namespace eh
