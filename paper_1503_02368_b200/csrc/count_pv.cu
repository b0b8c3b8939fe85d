// count_pv.cu -- SURVEY.md §8(f) NEXT-1: per-vertex triangle counts and the
// Lollipop L3,1 / Barbell B3,1 COUNT(*) by the paper's two-phase GHD plan.
//
//   Lollipop(x,y,z,w) :- R(x,y),S(y,z),T(x,z),U(x,w).
//   Barbell(x,y,z,x',y',z') :- R(x,y),S(y,z),T(x,z),U(x,x'),R'(x',y'),S'(y',z'),T'(x',z').
// Both run on the UNDIRECTED data.  GHD plan (Example
// `ex:barbell`; Yannakakis bottom-up): the
// triangle node(s) are aggregated and projected onto x -- on symmetric data
// every triangle containing x gives 2 ordered (y, z), so the projection is
// 2 t(x) with t(x) = #triangles containing x -- then the root joins with U:
//   L3,1 = sum_x 2 t(x) deg(x)        B3,1 = sum over ordered edges (x,x') of 2 t(x) * 2 t(x')
// The counts can exceed 2^64, so they are accumulated in 128 bits.
//
// t(v): the oriented triangle nest of count_tri.cu with
// every found triangle x<y<z credited to its three vertices.  x gets its row
// sums, y gets one atomic per row, and z is credited through a per-x shared
// counter indexed by z's LOCAL position in N+(x) (z is always in N+(x)), flushed
// once per x -- so hub vertices do not serialise one global atomic per triangle.
// Rows use the uint cap bitset probe, the galloping binary search, or a stream
// of N+(y) against a shared-memory hash of N+(x) that returns the local index.
#include "eh_internal.cuh"
#include "primitives.cuh"
#include "rows.cuh"

namespace eh {

namespace {

constexpr int kG = 8;
constexpr int kPvWarpMaxD = 128;  // must equal tri_warp_max_degree(): the work classes are shared
constexpr int kPvWHash = 512;     // >= 4 d
constexpr int kPvWarps = 8;
constexpr int kPvCtaXCap = 4096;
constexpr int kPvCHash = 16384;   // >= 4 d
constexpr int kPvCtaWarps = 16;
constexpr uint32_t kEmptyP = 0xFFFFFFFFu;

struct IdxHash {  // N+(x) -> local index; idx == nullptr: binary search in xs instead
  const uint32_t* keys;
  const uint16_t* idx;
  const uint32_t* xs;
  uint32_t d, shift, mask, amin, amax;
  __device__ __forceinline__ int lookup(uint32_t e) const {
    if (e < amin || e > amax) return -1;
    if (idx) {
      uint32_t s = (e * 2654435761u) >> shift;
      for (;;) {
        const uint32_t v = keys[s];
        if (v == e) return idx[s];
        if (v == kEmptyP) return -1;
        s = (s + 1) & mask;
      }
    }
    uint32_t lo = 0, len = d;
    while (len > 0) {
      const uint32_t h = len >> 1;
      if (xs[lo + h] < e) { lo += h + 1; len -= h + 1; } else { len = h; }
    }
    return (lo < d && xs[lo] == e) ? (int)lo : -1;
  }
};

template <bool kCta>
__device__ __forceinline__ IdxHash build_idx_hash(uint32_t* keys, uint16_t* idx, const uint32_t* xs, uint32_t d,
                                                  bool staged, int tid, int nt) {
  IdxHash H{keys, staged ? idx : nullptr, xs, d, 0, 0, xs[0], xs[d - 1]};
  if (!staged) return H;
  uint32_t hbits = 5;
  while ((1u << hbits) < 4 * d) ++hbits;
  H.shift = 32 - hbits;
  H.mask = (1u << hbits) - 1u;
  for (uint32_t k = tid; k <= H.mask; k += nt) keys[k] = kEmptyP;
  if (kCta) __syncthreads(); else __syncwarp();
  for (uint32_t k = tid; k < d; k += nt) {
    const uint32_t e = xs[k];
    uint32_t h = (e * 2654435761u) >> H.shift;
    while (atomicCAS(&keys[h], kEmptyP, e) != kEmptyP) h = (h + 1) & H.mask;
    idx[h] = (uint16_t)k;
  }
  return H;
}

// Credit one hit z = x_j: local counter if staged, else a direct global atomic.
__device__ __forceinline__ void credit(uint32_t* lc, unsigned long long* t, const uint32_t* xs, int j) {
  if (lc) atomicAdd(&lc[j], 1u);
  else atomicAdd(&t[xs[j]], 1ull);
}

// Row (x, y) with y = xs[i] on an 8-lane group; returns this lane's hit count.
__device__ __forceinline__ uint32_t pv_row(const YInfo& y, const uint32_t* xs, uint32_t d, uint32_t i,
                                           const IdxHash& H, uint32_t* lc, unsigned long long* t,
                                           const uint32_t* __restrict__ col, const uint32_t* __restrict__ bs,
                                           uint32_t gl) {
  const uint32_t a = d - 1 - i;
  uint32_t c = 0;
  if (a == 0 || y.len == 0) return 0;
  if (y.c1 > y.c0) {  // uint cap bitset probe
    for (uint32_t j = i + 1 + gl; j < d; j += kG)
      if (probe_bits(bs, y, xs[j])) { credit(lc, t, xs, (int)j); ++c; }
    return c;
  }
  const uint32_t lg = 32 - __clz(y.len);
  if ((uint64_t)a * lg * 4 < y.len) {  // galloping side: A's elements binary-search N+(y)
    for (uint32_t j = i + 1 + gl; j < d; j += kG)
      if (gmem_search(col + (uint64_t)y.list * 4, y.len, xs[j])) { credit(lc, t, xs, (int)j); ++c; }
    return c;
  }
  const uint4* yl = reinterpret_cast<const uint4*>(col) + y.list;  // stream N+(y)
  for (uint32_t k = gl; k * 4 < y.len; k += kG) {
    const uint4 v = __ldg(yl + k);
    const uint32_t e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (k * 4 + q >= y.len) break;
      const int j = H.lookup(e[q]);
      if (j >= 0) { credit(lc, t, xs, j); ++c; }
    }
  }
  return c;
}

__device__ __forceinline__ uint32_t group_sum(uint32_t v, uint32_t lane) {
  const unsigned gmask = 0xFFu << (lane & ~7u);
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) v += __shfl_xor_sync(gmask, v, o, kG);
  return v;
}

struct __align__(16) PvWarpSmem {
  uint32_t xs[kPvWarpMaxD];
  uint32_t lc[kPvWarpMaxD];
  uint32_t keys[kPvWHash];
  uint16_t idx[kPvWHash];
};

__global__ void __launch_bounds__(kPvWarps * 32) k_pv_warp(const uint4* __restrict__ desc,
                                                          const uint32_t* __restrict__ col,
                                                          const uint32_t* __restrict__ bs,
                                                          const uint32_t* __restrict__ work, uint64_t nwork,
                                                          unsigned long long* __restrict__ t,
                                                          unsigned long long* __restrict__ ctr) {
  __shared__ PvWarpSmem sm_all[kPvWarps];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, grp = lane / kG, gl = lane % kG;
  PvWarpSmem& sm = sm_all[w];
  for (;;) {
    unsigned long long wi = 0;
    if (lane == 0) wi = atomicAdd(&ctr[1], 1ull);
    wi = __shfl_sync(kFull, wi, 0);
    if (wi >= nwork) break;
    const uint32_t x = __ldg(work + wi);
    const uint4 dx = __ldg(desc + x);
    const uint32_t d = dx.y;  // 2 <= d <= kPvWarpMaxD
    const uint32_t* xg = col + (uint64_t)dx.x * 4;
    for (uint32_t k = lane; k < (d + 3) / 4; k += 32)
      reinterpret_cast<uint4*>(sm.xs)[k] = __ldg(reinterpret_cast<const uint4*>(xg) + k);
    for (uint32_t k = lane; k < d; k += 32) sm.lc[k] = 0u;
    __syncwarp();
    const IdxHash H = build_idx_hash<false>(sm.keys, sm.idx, sm.xs, d, true, lane, 32);
    __syncwarp();
    uint32_t cx = 0;
    for (uint32_t i = grp; i + 1 < d; i += 32 / kG) {
      const YInfo y = yinfo(desc, sm.xs[i]);
      const uint32_t c = group_sum(pv_row(y, sm.xs, d, i, H, sm.lc, t, col, bs, gl), lane);
      if (gl == 0 && c) atomicAdd(&t[sm.xs[i]], (unsigned long long)c);
      if (gl == 0) cx += c;
    }
    __syncwarp();
    cx = warp_sum(cx);
    if (lane == 0 && cx) atomicAdd(&t[x], (unsigned long long)cx);
    for (uint32_t k = lane; k < d; k += 32)
      if (sm.lc[k]) atomicAdd(&t[sm.xs[k]], (unsigned long long)sm.lc[k]);
    __syncwarp();
  }
}

__global__ void __launch_bounds__(kPvCtaWarps * 32) k_pv_cta(const uint4* __restrict__ desc,
                                                            const uint32_t* __restrict__ col,
                                                            const uint32_t* __restrict__ bs,
                                                            const uint32_t* __restrict__ work, uint64_t nwork,
                                                            unsigned long long* __restrict__ t,
                                                            unsigned long long* __restrict__ ctr) {
  extern __shared__ __align__(16) uint32_t dsm_pv[];
  uint32_t* xs_s = dsm_pv;                  // kPvCtaXCap
  uint32_t* lc_s = xs_s + kPvCtaXCap;       // kPvCtaXCap
  uint32_t* keys = lc_s + kPvCtaXCap;       // kPvCHash
  uint16_t* idx = reinterpret_cast<uint16_t*>(keys + kPvCHash);  // kPvCHash
  __shared__ unsigned long long s_wi;
  __shared__ uint32_t s_cx;
  constexpr uint32_t kGroups = kPvCtaWarps * 32 / kG;
  const uint32_t lane = threadIdx.x & 31, gid = threadIdx.x / kG, gl = threadIdx.x % kG;
  for (;;) {
    if (threadIdx.x == 0) {
      s_wi = atomicAdd(&ctr[2], 1ull);
      s_cx = 0;
    }
    __syncthreads();
    const unsigned long long wi = s_wi;
    if (wi >= nwork) break;
    const uint32_t x = __ldg(work + wi);
    const uint4 dx = __ldg(desc + x);
    const uint32_t d = dx.y;
    const uint32_t* xg = col + (uint64_t)dx.x * 4;
    const bool staged = d <= (uint32_t)kPvCtaXCap;
    const uint32_t* xs = staged ? xs_s : xg;
    uint32_t* lc = staged ? lc_s : nullptr;  // d > kPvCtaXCap: credit z with global atomics
    if (staged) {
      for (uint32_t k = threadIdx.x; k < (d + 3) / 4; k += blockDim.x)
        reinterpret_cast<uint4*>(xs_s)[k] = __ldg(reinterpret_cast<const uint4*>(xg) + k);
      for (uint32_t k = threadIdx.x; k < d; k += blockDim.x) lc_s[k] = 0u;
    }
    __syncthreads();
    const IdxHash H = build_idx_hash<true>(keys, idx, xs, d, staged, threadIdx.x, blockDim.x);
    __syncthreads();
    uint32_t cx = 0;
    for (uint32_t i = gid; i + 1 < d; i += kGroups) {
      const YInfo y = yinfo(desc, xs[i]);
      const uint32_t c = group_sum(pv_row(y, xs, d, i, H, lc, t, col, bs, gl), lane);
      if (gl == 0 && c) atomicAdd(&t[xs[i]], (unsigned long long)c);
      if (gl == 0) cx += c;
    }
    cx = warp_sum(cx);
    if (lane == 0 && cx) atomicAdd(&s_cx, cx);
    __syncthreads();
    if (threadIdx.x == 0 && s_cx) atomicAdd(&t[x], (unsigned long long)s_cx);
    if (staged)
      for (uint32_t k = threadIdx.x; k < d; k += blockDim.x)
        if (lc_s[k]) atomicAdd(&t[xs_s[k]], (unsigned long long)lc_s[k]);
    __syncthreads();
  }
}

constexpr size_t kPvCtaSmem = (size_t)(2 * kPvCtaXCap + kPvCHash) * 4 + (size_t)kPvCHash * 2;

// ---- 128-bit reductions for the root GHD node ----
__device__ __forceinline__ void add_u128_atomic(unsigned long long* out2, unsigned long long lo,
                                                unsigned long long hi) {
  const unsigned long long old = atomicAdd(&out2[0], lo);
  if (old + lo < old) ++hi;  // carry out of the low word
  if (hi) atomicAdd(&out2[1], hi);
}

__device__ __forceinline__ void warp_add_u128(unsigned long long& lo, unsigned long long& hi) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long l2 = __shfl_xor_sync(kFull, lo, o), h2 = __shfl_xor_sync(kFull, hi, o);
    const unsigned long long s = lo + l2;
    hi += h2 + (s < lo);
    lo = s;
  }
}

// L3,1 = sum_v 2 t(v) deg(v)
__global__ void k_lollipop(const unsigned long long* __restrict__ t, const uint32_t* __restrict__ deg, uint64_t n,
                           unsigned long long* __restrict__ out2) {
  unsigned __int128 acc = 0;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
    acc += (unsigned __int128)2 * t[v] * deg[v];
  unsigned long long lo = (unsigned long long)acc, hi = (unsigned long long)(acc >> 64);
  warp_add_u128(lo, hi);
  if ((threadIdx.x & 31) == 0 && (lo | hi)) add_u128_atomic(out2, lo, hi);
}

// B3,1 = sum over ordered edges (x, x') of 2 t(x) 2 t(x') = 8 sum_{(x,y) in E+} t(x) t(y)
__global__ void k_barbell(const uint4* __restrict__ desc, const uint32_t* __restrict__ col, uint64_t n,
                          const unsigned long long* __restrict__ t, unsigned long long* __restrict__ out2) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned __int128 acc = 0;
  for (uint64_t x = warp; x < n; x += nw) {
    const uint4 dx = __ldg(desc + x);
    const unsigned long long tx = t[x];
    if (tx == 0) continue;
    for (uint32_t k = lane; k < dx.y; k += 32)
      acc += (unsigned __int128)8 * tx * t[__ldg(col + (uint64_t)dx.x * 4 + k)];
  }
  unsigned long long lo = (unsigned long long)acc, hi = (unsigned long long)(acc >> 64);
  warp_add_u128(lo, hi);
  if (lane == 0 && (lo | hi)) add_u128_atomic(out2, lo, hi);
}

}  // namespace

void triangles_per_vertex(eh_graph* g, unsigned long long* d_t) {
  cudaStream_t s = g->stream;
  const uint64_t n = g->n_act;
  EH_CUDA(cudaMemsetAsync(d_t, 0, std::max<uint64_t>(1, n) * 8, s));
  EH_CUDA(cudaMemsetAsync(g->d_counter, 0, 4 * sizeof(unsigned long long), s));
  const uint64_t nsmall = g->n_work[0] + g->n_work[1];
  const uint64_t nlarge = g->n_work[2];
  if (nlarge) {
    EH_CUDA(cudaFuncSetAttribute(k_pv_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPvCtaSmem));
    const unsigned grid = (unsigned)std::min<uint64_t>(nlarge, (uint64_t)kSMs);
    k_pv_cta<<<grid, kPvCtaWarps * 32, kPvCtaSmem, s>>>(g->desc, g->col, g->bs, g->work + nsmall, nlarge, d_t,
                                                         g->d_counter);
    EH_LAUNCH("k_pv_cta");
  }
  if (nsmall) {
    const unsigned grid = (unsigned)std::min<uint64_t>((nsmall + kPvWarps - 1) / kPvWarps, (uint64_t)kSMs * 8);
    k_pv_warp<<<grid, kPvWarps * 32, 0, s>>>(g->desc, g->col, g->bs, g->work, nsmall, d_t, g->d_counter);
    EH_LAUNCH("k_pv_warp");
  }
}

void count_lollipop_barbell(eh_graph* g, bool barbell, uint64_t out2[2]) {
  cudaStream_t s = g->stream;
  const uint64_t n = g->n_act;
  out2[0] = out2[1] = 0;
  if (n == 0) return;
  DBuf<unsigned long long> t(g->alloc, n), acc(g->alloc, 2);
  triangles_per_vertex(g, t.p);  // bottom-up: the triangle GHD node aggregated onto x
  EH_CUDA(cudaMemsetAsync(acc.p, 0, 16, s));
  if (barbell) {
    k_barbell<<<grid_for(n * 32, 256), 256, 0, s>>>(g->desc, g->col, n, t.p, acc.p);
    EH_LAUNCH("k_barbell");
  } else {
    k_lollipop<<<grid_for(n, 256), 256, 0, s>>>(t.p, g->deg_rank, n, acc.p);
    EH_LAUNCH("k_lollipop");
  }
  unsigned long long h[2];
  EH_CUDA(cudaMemcpyAsync(h, acc.p, 16, cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaStreamSynchronize(s));
  out2[0] = h[0];
  out2[1] = h[1];
}

}  // namespace eh
