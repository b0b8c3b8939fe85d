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
// t(v): the oriented triangle nest of count_tri.cu (its row
// kinds PROBE / STREAM / SEARCH, same work classes) with every found triangle
// x<y<z credited to its three vertices.  y and z are both elements of
// N+(x), so their credits go to a per-x shared-memory counter indexed by the
// LOCAL position in N+(x) (row totals for y, one increment per hit for z), and
// are flushed with one global atomic per element of N+(x); x gets its row sum.
// The membership structure of x therefore also returns that position: an exact
// bitmap plus, per 32-bit word, the position of its first element (positions
// within a word by popcount), or a hash table with a position per slot, or a
// binary search of the sorted list.  (No AND rows: see row_kind.)  Tuned on
// C2-C4 (DESIGN.md NEXT-1): 8-warp CTAs, staging sized to max |N+(x)| (C3: 20 KB).
#include "eh_internal.cuh"
#include "primitives.cuh"
#include "rows.cuh"

namespace eh {

namespace {

constexpr int kG = 8;
constexpr int kWarpMaxD = 128;       // must equal tri_warp_max_degree(): the work classes are shared
constexpr int kWarpTabWords = 256;   // warp-kernel x structure: bitmap of 8192 ids or 256-slot hash
constexpr int kWarps = 8;
constexpr int kCtaWarps = 8;
constexpr uint32_t kCtaXCapMax = 16384;   // N+(x) staged and counted locally up to max |N+(x)| rounded to 256, clamped
constexpr int kCtaTabWords = 2048;   // CTA x structure: bitmap of 65536 ids, or a hash of <= 2048 slots
constexpr uint32_t kEmpty = 0xFFFFFFFFu;

enum RowKind : uint8_t { kSkip = 0, kProbe = 1, kStream = 2, kSearch = 3 };
enum XMode : uint32_t { kBitmap = 0, kHash = 1, kSorted = 2 };

// N+(x) with local positions.  Bitmap: pos[w] = position of the first element
// in word w (only read for words that hold an element).  Hash: pos[slot].
struct XIdx {
  uint32_t* tab;
  uint16_t* pos;
  const uint32_t* xs;
  uint32_t mode, lo, nbits, hshift, hmask, d, amin, amax;

  __device__ __forceinline__ int index_of(uint32_t e) const {
    if (mode == kBitmap) {
      const uint32_t o = e - lo;
      if (o >= nbits) return -1;
      const uint32_t w = tab[o >> 5], b = o & 31;
      if (!((w >> b) & 1u)) return -1;
      return pos[o >> 5] + __popc(w & ((1u << b) - 1u));
    }
    if (e < amin || e > amax) return -1;
    if (mode == kHash) {
      uint32_t s = (e * 2654435761u) >> hshift;
      for (;;) {
        const uint32_t v = tab[s];
        if (v == e) return pos[s];
        if (v == kEmpty) return -1;
        s = (s + 1) & hmask;
      }
    }
    uint32_t l = 0, len = d;
    while (len > 0) {
      const uint32_t h = len >> 1;
      if (xs[l + h] < e) { l += h + 1; len -= h + 1; } else { len = h; }
    }
    return (l < d && xs[l] == e) ? (int)l : -1;
  }
};

__device__ __forceinline__ XIdx plan_x(uint32_t* tab, uint16_t* pos, uint32_t tab_words, const uint32_t* xs,
                                       uint32_t d) {
  XIdx s;
  s.tab = tab;
  s.pos = pos;
  s.xs = xs;
  s.d = d;
  s.amin = xs[0];
  s.amax = xs[d - 1];
  const uint32_t lo = (s.amin >> 7) << 7;
  const uint64_t span_bits = (uint64_t)(((s.amax >> 7) + 1) << 7) - lo;
  uint32_t hbits = 5;
  while ((1u << hbits) < 8 * d && (2u << hbits) <= tab_words) ++hbits;
  s.lo = s.nbits = s.hshift = s.hmask = 0;
  if (span_bits <= 32ull * tab_words) {
    s.mode = kBitmap;
    s.lo = lo;
    s.nbits = (uint32_t)span_bits;
  } else if ((1u << hbits) <= tab_words && (1u << hbits) >= 2 * d) {
    s.mode = kHash;
    s.hshift = 32 - hbits;
    s.hmask = (1u << hbits) - 1u;
  } else {
    s.mode = kSorted;
  }
  return s;
}

template <bool kCta>
__device__ __forceinline__ void fill_x(const XIdx& s, int tid, int nt) {
  if (s.mode == kBitmap) {
    for (uint32_t k = tid; k < s.nbits / 32; k += nt) s.tab[k] = 0u;
  } else if (s.mode == kHash) {
    for (uint32_t k = tid; k <= s.hmask; k += nt) s.tab[k] = kEmpty;
  }
  if (kCta) __syncthreads(); else __syncwarp();
  if (s.mode == kBitmap) {
    for (uint32_t k = tid; k < s.d; k += nt) {
      const uint32_t o = s.xs[k] - s.lo;
      atomicOr(&s.tab[o >> 5], 1u << (o & 31));
      if (k == 0 || ((s.xs[k - 1] - s.lo) >> 5) != (o >> 5)) s.pos[o >> 5] = (uint16_t)k;  // xs sorted
    }
  } else if (s.mode == kHash) {
    for (uint32_t k = tid; k < s.d; k += nt) {
      const uint32_t e = s.xs[k];
      uint32_t h = (e * 2654435761u) >> s.hshift;
      while (atomicCAS(&s.tab[h], kEmpty, e) != kEmpty) h = (h + 1) & s.hmask;
      s.pos[h] = (uint16_t)k;
    }
  }
}

// Row kinds as count_tri.cu minus AND: a row whose N+(y) is a bitset is PROBEd
// element by element, because every hit must be attributed to its z, and
// extracting the set bits of ANDed chunks measured slower on B200 than probing
// (DESIGN.md NEXT-1).  Rows whose bitset span misses x's span are skipped.
__device__ __forceinline__ uint8_t row_kind(const YInfo& y, uint32_t a, const XIdx& X, uint32_t sf16) {
  if (a == 0 || y.len == 0) return kSkip;
  if (y.c1 > y.c0) {
    if (y.c1 <= (X.amin >> 7) || y.c0 > (X.amax >> 7)) return kSkip;
    return kProbe;
  }
  const uint32_t lg = 32 - __clz(y.len);
  if (y.c0 >= kAlwaysSearch ? y.c0 == kAlwaysSearch : (uint64_t)a * lg * sf16 < (uint64_t)y.len * 16) return kSearch;  // sf16: see count_tri.cu row_kind
  return kStream;
}

// Credit one hit z = N+(x)[j]: local counter if N+(x) is staged, else a global atomic.
__device__ __forceinline__ void credit(uint32_t* lc, unsigned long long* t, const uint32_t* xs, int j) {
  if (lc) atomicAdd(&lc[j], 1u);
  else atomicAdd(&t[xs[j]], 1ull);
}

// Row (x, y = xs[i]) on an 8-lane group; returns this lane's hit count.
template <bool kPiv>
__device__ __forceinline__ uint32_t pv_row(uint8_t kd, const YInfo& y, const XIdx& X, uint32_t i, uint32_t* lc,
                                           unsigned long long* t, const uint32_t* __restrict__ col,
                                           const uint32_t* __restrict__ bs, uint32_t gl) {
  const uint32_t* xs = X.xs;
  const uint32_t d = X.d;
  uint32_t c = 0;
  if (kd == kProbe) {  // 4 probes in flight per lane
    uint32_t j = i + 1 + gl;
    for (; j + 3 * kG < d; j += 4 * kG) {
      const uint32_t h0 = probe_bits(bs, y, xs[j]), h1 = probe_bits(bs, y, xs[j + kG]);
      const uint32_t h2 = probe_bits(bs, y, xs[j + 2 * kG]), h3 = probe_bits(bs, y, xs[j + 3 * kG]);
      if (h0) credit(lc, t, xs, (int)j);
      if (h1) credit(lc, t, xs, (int)(j + kG));
      if (h2) credit(lc, t, xs, (int)(j + 2 * kG));
      if (h3) credit(lc, t, xs, (int)(j + 3 * kG));
      c += h0 + h1 + h2 + h3;
    }
    for (; j < d; j += kG)
      if (probe_bits(bs, y, xs[j])) { credit(lc, t, xs, (int)j); ++c; }
  } else if (kd == kStream) {
    const uint4* yl = reinterpret_cast<const uint4*>(col) + y.list;
    for (uint32_t k = gl; k * 4 < y.len; k += kG) {
      const uint4 v = __ldg(yl + k);
      const uint32_t e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (k * 4 + q >= y.len) break;
        const int j = X.index_of(e[q]);
        if (j >= 0) { credit(lc, t, xs, j); ++c; }
      }
    }
  } else if (kd == kSearch) {
    const uint32_t* L = col + (uint64_t)y.list * 4;
    const uint32_t n = y.len;
    if (kPiv && n >= 4 * kG) {  // 7 slice pivots loaded once per row (count_tri.cu grp_row)
      const unsigned gmask = 0xFFu << ((threadIdx.x & 31) & ~7u);
      const uint32_t mine = (gl < kG - 1) ? __ldg(L + (uint64_t)(gl + 1) * n / kG - 1) : 0u;
      uint32_t piv[kG - 1];
#pragma unroll
      for (int q = 0; q < kG - 1; ++q) piv[q] = __shfl_sync(gmask, mine, q, kG);
      for (uint32_t j = i + 1 + gl; j < d; j += kG) {
        const uint32_t e = xs[j];
        uint32_t k = 0;
#pragma unroll
        for (int q = 0; q < kG - 1; ++q) k += (piv[q] < e);
        const uint32_t lo = (uint32_t)((uint64_t)k * n / kG), hi = (uint32_t)((uint64_t)(k + 1) * n / kG);
        if (gmem_search(L + lo, hi - lo, e)) { credit(lc, t, xs, (int)j); ++c; }
      }
    } else {
      for (uint32_t j = i + 1 + gl; j < d; j += kG)
        if (gmem_search(L, n, xs[j])) { credit(lc, t, xs, (int)j); ++c; }
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

// ------------------------------------------------------------ warp kernel --
struct __align__(16) PvWarpSmem {
  uint32_t xs[kWarpMaxD];
  uint32_t lc[kWarpMaxD];
  uint32_t tab[kWarpTabWords];
  YInfo yi[kWarpMaxD];
  uint16_t pos[kWarpTabWords];
  uint8_t kind[kWarpMaxD];
  uint8_t ord[kWarpMaxD];
};

template <bool kPiv>
__global__ void __launch_bounds__(kWarps * 32) k_pv_warp(const uint4* __restrict__ desc,
                                                        const uint32_t* __restrict__ col,
                                                        const uint32_t* __restrict__ bs,
                                                        const uint32_t* __restrict__ work, uint64_t nwork,
                                                        unsigned long long* __restrict__ t, uint32_t sf16,
                                                        unsigned long long* __restrict__ ctr) {
  extern __shared__ __align__(16) uint32_t dsm_pw[];
  PvWarpSmem& sm = reinterpret_cast<PvWarpSmem*>(dsm_pw)[threadIdx.x >> 5];
  const uint32_t lane = threadIdx.x & 31, grp = lane / kG, gl = lane % kG;
  const unsigned lt = (1u << lane) - 1u;
  for (;;) {
    unsigned long long wi = 0;
    if (lane == 0) wi = atomicAdd(&ctr[1], 1ull);
    wi = __shfl_sync(kFull, wi, 0);
    if (wi >= nwork) break;
    const uint32_t x = __ldg(work + wi);
    const uint4 dx = __ldg(desc + x);
    const uint32_t d = dx.y;  // 2 <= d <= kWarpMaxD
    const uint32_t* xg = col + (uint64_t)dx.x * 4;
    for (uint32_t k = lane; k < (d + 3) / 4; k += 32)
      reinterpret_cast<uint4*>(sm.xs)[k] = __ldg(reinterpret_cast<const uint4*>(xg) + k);
    for (uint32_t k = lane; k < d; k += 32) sm.lc[k] = 0u;
    __syncwarp();
    const XIdx X = plan_x(sm.tab, sm.pos, kWarpTabWords, sm.xs, d);
    const uint32_t nrows = d - 1;
    bool need_x = false;  // only STREAM rows read x's staged structure
    for (uint32_t i = lane; i < nrows; i += 32) {
      const YInfo y = yinfo(desc, sm.xs[i]);
      const uint8_t kd = row_kind(y, nrows - i, X, sf16);
      sm.yi[i] = y;
      sm.kind[i] = kd;
      need_x |= kd == kStream;
    }
    if (__any_sync(kFull, need_x)) fill_x<false>(X, lane, 32);
    __syncwarp();
    uint32_t nr = 0;
#pragma unroll
    for (int kdi = 0; kdi < 3; ++kdi) {
      const uint8_t want = (uint8_t)(kProbe + kdi);
      for (uint32_t i0 = 0; i0 < nrows; i0 += 32) {
        const uint32_t i = i0 + lane;
        const bool sel = i < nrows && sm.kind[i] == want;
        const unsigned m = __ballot_sync(kFull, sel);
        if (sel) sm.ord[nr + __popc(m & lt)] = (uint8_t)i;
        nr += __popc(m);
      }
    }
    __syncwarp();
    uint32_t cx = 0;
    for (uint32_t r = grp; r < nr; r += 32 / kG) {
      const uint32_t i = sm.ord[r];
      const uint32_t c = group_sum(pv_row<kPiv>(sm.kind[i], sm.yi[i], X, i, sm.lc, t, col, bs, gl), lane);
      if (gl == 0 && c) {
        atomicAdd(&sm.lc[i], c);  // y = N+(x)[i] is in every triangle of its row
        cx += c;
      }
    }
    cx = warp_sum(cx);
    if (lane == 0 && cx) atomicAdd(&t[x], (unsigned long long)cx);
    __syncwarp();
    for (uint32_t k = lane; k < d; k += 32)
      if (sm.lc[k]) atomicAdd(&t[sm.xs[k]], (unsigned long long)sm.lc[k]);
    __syncwarp();
  }
}

// ------------------------------------------------------------- CTA kernel --
template <bool kPiv, int kCW = kCtaWarps>
__global__ void __launch_bounds__(kCW * 32) k_pv_cta(const uint4* __restrict__ desc,
                                                          const uint32_t* __restrict__ col,
                                                          const uint32_t* __restrict__ bs,
                                                          const uint32_t* __restrict__ work, uint64_t nwork,
                                                          unsigned long long* __restrict__ t, uint32_t sf16,
                                                          unsigned long long* __restrict__ ctr, uint32_t xcap) {
  extern __shared__ __align__(16) uint32_t dsm_pc[];
  uint32_t* xs_s = dsm_pc;                                          // xcap
  uint32_t* lc_s = xs_s + xcap;                                     // xcap
  uint32_t* tab = lc_s + xcap;                                      // kCtaTabWords
  uint16_t* pos = reinterpret_cast<uint16_t*>(tab + kCtaTabWords);  // kCtaTabWords
  __shared__ unsigned long long s_wi;
  __shared__ uint32_t s_cx;
  constexpr uint32_t kGroups = kCW * 32 / kG;
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
    const bool staged = d <= xcap;
    const uint32_t* xs = staged ? xs_s : xg;
    uint32_t* lc = staged ? lc_s : nullptr;  // d > xcap: credit with global atomics
    if (staged) {
      for (uint32_t k = threadIdx.x; k < (d + 3) / 4; k += blockDim.x)
        reinterpret_cast<uint4*>(xs_s)[k] = __ldg(reinterpret_cast<const uint4*>(xg) + k);
      for (uint32_t k = threadIdx.x; k < d; k += blockDim.x) lc_s[k] = 0u;
    }
    __syncthreads();
    const XIdx X = plan_x(tab, pos, staged ? kCtaTabWords : 0, xs, d);
    fill_x<true>(X, threadIdx.x, blockDim.x);
    __syncthreads();
    const uint32_t nrows = d - 1;
    uint32_t cx = 0;
    uint32_t i = gid;
    YInfo y = (i < nrows) ? yinfo(desc, xs[i]) : YInfo{0, 0, 0, 0, 0};
    while (i < nrows) {
      const uint32_t inext = i + kGroups;
      const YInfo ynext = (inext < nrows) ? yinfo(desc, xs[inext]) : YInfo{0, 0, 0, 0, 0};
      const uint32_t c = group_sum(pv_row<kPiv>(row_kind(y, nrows - i, X, sf16), y, X, i, lc, t, col, bs, gl), lane);
      if (gl == 0 && c) {
        if (lc) atomicAdd(&lc[i], c);
        else atomicAdd(&t[xs[i]], (unsigned long long)c);
        cx += c;
      }
      i = inext;
      y = ynext;
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

size_t cta_smem(uint32_t xcap) { return (size_t)(2 * xcap + kCtaTabWords) * 4 + (size_t)kCtaTabWords * 2; }

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

template <bool kPiv>
static void pv_launch(eh_graph* g, unsigned long long* d_t, uint32_t sf16) {
  cudaStream_t s = g->stream;
  const uint64_t nsmall = g->n_work[0];  // class 0 -> warp kernel; classes 1-2 -> CTA kernel
  const uint64_t nlarge = g->n_work[1] + g->n_work[2];
  const uint32_t* wl = nlarge ? work_lpt(g) + nsmall : nullptr;
  // the warp-class kernel on a side stream beside the CTA-class kernel (count_tri.cu)
  const cudaStream_t ss = (nlarge && nsmall && getenv("EH_TEST_TRI_SERIAL") == nullptr) ? fork_side(g, 0) : s;
  if (nlarge) {
    // N+(x) staged up to max |N+(x)| rounded up to 256 (smaller CTAs than a power of
    // two >= 2048: C3 t(v) 13.89 -> 13.80 ms, C4 2.34 -> 2.27 ms)
    const uint32_t xcap = (uint32_t)std::min<uint64_t>(kCtaXCapMax, std::max<uint64_t>(256, (g->max_dplus + 255) / 256 * 256));
    const uint32_t xc = getenv("EH_TEST_PV_XCAP") ? (uint32_t)std::max(128, atoi(getenv("EH_TEST_PV_XCAP")))  // test hook:
                                              : xcap;                                         // the unstaged path
    const size_t smem = cta_smem(xc);
    auto kc = k_pv_cta<kPiv>;  // 8 warps (4 / 16 measured slower: C3 17.3 / 16.6 ms)
    ensure_dyn_smem((const void*)kc, smem);
    int per_sm = 0;
    EH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kc, kCtaWarps * 32, smem));
    const unsigned grid = (unsigned)std::min<uint64_t>(nlarge, (uint64_t)kSMs * std::max(1, per_sm));
    kc<<<grid, kCtaWarps * 32, smem, s>>>(g->desc, g->col, g->bs, wl, nlarge, d_t, sf16, g->d_counter, xc);
    EH_LAUNCH("k_pv_cta");
  }
  if (nsmall) {
    const unsigned grid = (unsigned)std::min<uint64_t>((nsmall + kWarps - 1) / kWarps, (uint64_t)kSMs * 8);
    const size_t smem = sizeof(PvWarpSmem) * kWarps;
    auto kw = k_pv_warp<kPiv>;
    ensure_dyn_smem((const void*)kw, smem);
    kw<<<grid, kWarps * 32, smem, ss>>>(g->desc, g->col, g->bs, g->work, nsmall, d_t, sf16, g->d_counter);
    EH_LAUNCH("k_pv_warp");
  }
  if (ss != s) join_side(g, 0);
}

}  // namespace

void triangles_per_vertex(eh_graph* g, unsigned long long* d_t) {
  cudaStream_t s = g->stream;
  const uint32_t sf16 = g->n_act > (1ull << 24) ? 64u : 16u;  // C3 t(v) 15.03 -> 14.79 ms with 16
  EH_CUDA(cudaMemsetAsync(d_t, 0, std::max<uint64_t>(1, g->n_act) * 8, s));
  EH_CUDA(cudaMemsetAsync(g->d_counter, 0, 4 * sizeof(unsigned long long), s));
  // pivot-started SEARCH rows above 2^20 active ids, as in count_tri.cu
  if (g->n_act > (1ull << 20)) pv_launch<true>(g, d_t, sf16);
  else pv_launch<false>(g, d_t, sf16);
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
