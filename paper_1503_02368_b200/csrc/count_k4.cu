// count_k4.cu -- SURVEY.md §8(a) row a9: the 4-clique Generic-Join.
//
// 4Clique(x,y,z,w) :- R(x,y),S(y,z),T(x,z),U(x,w),V(y,w),Q(z,w),
// attribute order x, y, z, w on the pruned relation:
//     for x:  for y in N+(x):  for z in N+(x) cap N+(y):
//        K += | N+(x) cap N+(y) cap N+(z) |
// Every 4-clique x<y<z<w (rank order) is counted once, at its lowest vertex x.
//
// B200 formulation (same count): for one x, index N+(x) locally
// (x_0 < x_1 < ... < x_{d-1}) and build in shared memory the bit-matrix L of the
// subgraph G[N+(x)]:  bit j of row i  <=>  x_j in N+(x_i)  (so j > i).  Row i is
// the intersection N+(x) after x_i  cap  N+(x_i) -- exactly the triangle row of
// edge (x, x_i) -- computed with the same layout dispatch:
//   PROBE  N+(x_i) bitset: each x_j (j > i) tests its bit;
//   STREAM N+(x_i) uint: stream its list, look each element up in a shared-memory
//          hash of N+(x) that returns the local index j;
//   SEARCH |A| log|B| << |B|: each x_j binary-searches N+(x_i).
// Then the innermost loop is a bit-parallel AND:
//     K(x) = sum over set bits (i, j) of popcount(L_i & L_j restricted to > j),
// i.e. |P cap N+(z)| with P = N+(x) cap N+(y), y = x_i, z = x_j, counted 32 w
// at a time.  |N+(x)| <= 128: one warp per x (rows on 8-lane groups, then 2- or
// 4-lane groups over the <= 2 / 4 words of a row; a half-size instance for
// |N+(x)| <= 64); 128 < |N+(x)| <= 1024: one CTA per x (three shapes of 8 / 32 / 32
// warps, L up to 135 KB of shared memory); larger x (rare when pruned; the hubs of
// the symmetric data): one CTA per row (k_k4_big).  COUNT(*) accumulates per lane in u64 (K4 > 2^32 on C4).
#include "eh_internal.cuh"
#include "primitives.cuh"
#include "rows.cuh"
#include "sets.cuh"

namespace eh {

namespace {

constexpr int kG = 8;                 // lanes per row group (row fill)
constexpr int kWMaxD = 128;           // warp kernel: d <= 128 -> rows of <= 4 words
constexpr int kWWarps = 8;
constexpr int kCMaxD = 1024;          // CTA kernels: d <= 1024 -> rows of <= 32 words; three shapes
                                      // (d <= 256: 8 warps, ~25 KB; <= 512: 32 warps, ~82 KB; larger: 32 warps, 224 KB)
constexpr uint32_t kEmptyK = 0xFFFFFFFFu;

enum K4Kind : uint8_t { kKSkip = 0, kKProbe = 1, kKStream = 2, kKSearch = 3 };

// N+(x) -> local index, open addressing (load <= 1/4)
struct LocalHash {
  const uint32_t* keys;
  const uint16_t* idx;
  uint32_t shift, mask, amin, amax;
  __device__ __forceinline__ int lookup(uint32_t e) const {
    if (e < amin || e > amax) return -1;
    uint32_t s = (e * 2654435761u) >> shift;
    for (;;) {
      const uint32_t v = keys[s];
      if (v == e) return idx[s];
      if (v == kEmptyK) return -1;
      s = (s + 1) & mask;
    }
  }
};

template <bool kCta>
__device__ __forceinline__ LocalHash build_local_hash(uint32_t* keys, uint16_t* idx, const uint32_t* xs, uint32_t d,
                                                      int tid, int nt) {
  uint32_t hbits = 5;
  while ((1u << hbits) < 4 * d) ++hbits;
  LocalHash H{keys, idx, 32 - hbits, (1u << hbits) - 1u, xs[0], xs[d - 1]};
  for (uint32_t k = tid; k < (1u << hbits); k += nt) keys[k] = kEmptyK;
  if (kCta) __syncthreads(); else __syncwarp();
  for (uint32_t k = tid; k < d; k += nt) {
    const uint32_t e = xs[k];
    uint32_t h = (e * 2654435761u) >> H.shift;
    while (atomicCAS(&keys[h], kEmptyK, e) != kEmptyK) h = (h + 1) & H.mask;
    idx[h] = (uint16_t)k;
  }
  return H;
}

__device__ __forceinline__ uint8_t k4_kind(const YInfo& y, uint32_t a, uint32_t sf16) {
  if (a == 0 || y.len == 0) return kKSkip;
  if (y.c1 > y.c0) return kKProbe;
  const uint32_t lg = 32 - __clz(y.len);
  if (y.c0 >= kAlwaysSearch ? y.c0 == kAlwaysSearch : (uint64_t)a * lg * sf16 < (uint64_t)y.len * 16) return kKSearch;  // sf16: see count_tri.cu row_kind
  return kKStream;
}

// Fill row i of L (stride W words) with the 8-lane group's lane gl.  kU
// (NEXT-2, unpruned nest on the symmetric trie): the row is all of
// N(x) cap N(x_i), not only the part after x_i.
template <bool kU>
__device__ __forceinline__ void fill_row(uint8_t kd, const uint32_t* __restrict__ col, const uint32_t* __restrict__ bs,
                                         const YInfo& y, const uint32_t* xs, uint32_t d, uint32_t i, const LocalHash& H,
                                         uint32_t* Lrow, uint32_t gl) {
  if (kd == kKProbe) {
    for (uint32_t j = (kU ? 0 : i + 1) + gl; j < d; j += kG)
      if (probe_bits(bs, y, xs[j])) atomicOr(&Lrow[j >> 5], 1u << (j & 31));
  } else if (kd == kKStream) {
    const uint4* yl = reinterpret_cast<const uint4*>(col) + y.list;
    const uint32_t nfull = y.len >> 2;
    for (uint32_t k = gl; k < nfull; k += kG) {
      const uint4 v = __ldg(yl + k);
      const uint32_t e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = H.lookup(e[q]);
        if (j >= 0) atomicOr(&Lrow[j >> 5], 1u << (j & 31));
      }
    }
    if (gl < (y.len & 3)) {
      const int j = H.lookup(__ldg(col + (uint64_t)y.list * 4 + nfull * 4 + gl));
      if (j >= 0) atomicOr(&Lrow[j >> 5], 1u << (j & 31));
    }
  } else if (kd == kKSearch) {
    for (uint32_t j = (kU ? 0 : i + 1) + gl; j < d; j += kG)
      if (gmem_search(col + (uint64_t)y.list * 4, y.len, xs[j])) atomicOr(&Lrow[j >> 5], 1u << (j & 31));
  }
}

// ------------------------------------------------------------ warp kernel --
// per-warp shared memory of the warp kernel for |N+(x)| <= kMD: rows of kMD / 32
// words, a local hash of 4 kMD slots
template <int kMD>
struct __align__(16) K4WarpSmem {
  static constexpr int kW = kMD / 32;
  uint32_t xs[kMD];
  uint32_t hkeys[4 * kMD];
  uint32_t L[kMD * kW];
  YInfo yi[kMD];
  uint16_t hidx[4 * kMD];
  uint8_t kind[kMD];
  uint8_t ord[kMD];
};

// kMD = 64 (class 0) or kWMaxD = 128; the smaller instance has half the shared
// memory per warp, so about twice as many warps per SM
template <bool kU, int kMD = kWMaxD>
__global__ void __launch_bounds__(kWWarps * 32) k_k4_warp(const uint4* __restrict__ desc,
                                                          const uint32_t* __restrict__ col,
                                                          const uint32_t* __restrict__ bs,
                                                          const uint32_t* __restrict__ work, uint64_t nwork,
                                                          unsigned long long* __restrict__ ctr, uint32_t sf16,
                                                          uint32_t cslot) {
  constexpr uint32_t kWWd = K4WarpSmem<kMD>::kW;
  extern __shared__ __align__(16) uint32_t dsm_k4w[];
  K4WarpSmem<kMD>& sm = reinterpret_cast<K4WarpSmem<kMD>*>(dsm_k4w)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  unsigned long long cnt = 0;
  for (;;) {
    unsigned long long wi = 0;
    if (lane == 0) wi = atomicAdd(&ctr[cslot], 1ull);
    wi = __shfl_sync(kFull, wi, 0);
    if (wi >= nwork) break;
    const uint32_t x = __ldg(work + wi);
    const uint4 dx = __ldg(desc + x);
    const uint32_t d = dx.y;  // 2 <= d <= kMD
    EH_DASSERT(d >= 2 && d <= (uint32_t)kMD);
    if (d < 3) continue;
    const uint32_t* xg = col + (uint64_t)dx.x * 4;
    for (uint32_t k = lane; k < (d + 3) / 4; k += 32)
      reinterpret_cast<uint4*>(sm.xs)[k] = __ldg(reinterpret_cast<const uint4*>(xg) + k);
    for (uint32_t k = lane; k < d * kWWd; k += 32) sm.L[k] = 0u;
    __syncwarp();
    const LocalHash H = build_local_hash<false>(sm.hkeys, sm.hidx, sm.xs, d, lane, 32);
    const uint32_t nrows = kU ? d : d - 1;
    for (uint32_t i = lane; i < nrows; i += 32) {
      const YInfo y = yinfo(desc, sm.xs[i]);
      sm.yi[i] = y;
      sm.kind[i] = k4_kind(y, kU ? d : nrows - i, sf16);
    }
    __syncwarp();
    uint32_t nr = 0;
#pragma unroll
    for (int kdi = 0; kdi < 3; ++kdi) {
      const uint8_t want = (uint8_t)(kKProbe + kdi);
      for (uint32_t i0 = 0; i0 < nrows; i0 += 32) {
        const uint32_t i = i0 + lane;
        const bool sel = i < nrows && sm.kind[i] == want;
        const unsigned m = __ballot_sync(kFull, sel);
        if (sel) sm.ord[nr + __popc(m & lt)] = (uint8_t)i;
        nr += __popc(m);
      }
    }
    __syncwarp();
    for (uint32_t r = lane / kG; r < nr; r += 32 / kG) {
      const uint32_t i = sm.ord[r];
      fill_row<kU>(sm.kind[i], col, bs, sm.yi[i], sm.xs, d, i, H, sm.L + i * kWWd, lane % kG);
    }
    __syncwarp();
    // bit-parallel innermost loop: kWWd-lane groups, lane q holds word q of row i
    const uint32_t W = (d + 31) >> 5, q = lane & (kWWd - 1);
    for (uint32_t i0 = 0; i0 < d; i0 += 32 / kWWd) {
      const uint32_t i = i0 + lane / kWWd;
      const uint32_t li = (i < d && q < W) ? sm.L[i * kWWd + q] : 0u;
      for (uint32_t kk = 0; kk < W; ++kk) {
        uint32_t wb = __shfl_sync(kFull, li, (lane & ~(kWWd - 1)) + kk);
        while (wb) {
          const uint32_t b = __ffs(wb) - 1;
          wb &= wb - 1;
          const uint32_t j = kk * 32 + b;
          if (kU ? q < W : (q >= kk && q < W)) {  // unpruned: all w, else w after z
            cnt += __popc(li & sm.L[j * kWWd + q]);  // row j's bits all lie above j
          }
        }
      }
    }
    __syncwarp();
  }
  cnt = warp_sum(cnt);
  if (lane == 0 && cnt) atomicAdd(&ctr[0], cnt);
}

// ------------------------------------------------------------- CTA kernel --
template <int kMaxD, int kCWarps>
constexpr size_t k4_cta_smem() {
  return (size_t)(kMaxD + 4 * kMaxD + 2 * kMaxD + kMaxD * (kMaxD / 32 + 1)) * 4 + (size_t)kCWarps * kMaxD * 2;
}

// One CTA per x with dlo < d <= dhi (<= kMaxD); ctr slot `cslot` is its work cursor.
template <bool kU, int kMaxD, int kCWarps>
__global__ void __launch_bounds__(kCWarps * 32) k_k4_cta(const uint4* __restrict__ desc,
                                                          const uint32_t* __restrict__ col,
                                                          const uint32_t* __restrict__ bs,
                                                          const uint32_t* __restrict__ work, uint64_t nwork,
                                                          unsigned long long* __restrict__ ctr, uint32_t dlo,
                                                          uint32_t cslot, uint32_t sf16) {
  constexpr int kCHash = 4 * kMaxD;
  extern __shared__ __align__(16) uint32_t dsm_k4c[];
  uint32_t* xs = dsm_k4c;                                   // kMaxD
  uint32_t* hkeys = xs + kMaxD;                             // kCHash
  uint16_t* hidx = reinterpret_cast<uint16_t*>(hkeys + kCHash);  // kCHash u16
  uint32_t* L = hkeys + kCHash + kCHash / 2;                // d rows of S = W|1 words
  uint16_t* jl_all = reinterpret_cast<uint16_t*>(L + kMaxD * (kMaxD / 32 + 1));  // per-warp edge lists
  __shared__ unsigned long long s_wi;
  constexpr uint32_t kGroups = kCWarps * 32 / kG;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t gid = threadIdx.x / kG, gl = threadIdx.x % kG;
  unsigned long long cnt = 0;
  for (;;) {
    if (threadIdx.x == 0) s_wi = atomicAdd(&ctr[cslot], 1ull);
    __syncthreads();
    const unsigned long long wi = s_wi;
    if (wi >= nwork) break;
    const uint32_t x = __ldg(work + wi);
    const uint4 dx = __ldg(desc + x);
    const uint32_t d = dx.y;
    if (d > (uint32_t)kMaxD || d <= dlo || d < 3) {  // the other shape / fallback handles these
      __syncthreads();
      continue;
    }
    const uint32_t W = (d + 31) >> 5;
    const uint32_t S = W | 1u;  // odd row stride: 32 lanes reading 32 different rows hit 32 banks
    const uint32_t* xg = col + (uint64_t)dx.x * 4;
    for (uint32_t k = threadIdx.x; k < (d + 3) / 4; k += blockDim.x)
      reinterpret_cast<uint4*>(xs)[k] = __ldg(reinterpret_cast<const uint4*>(xg) + k);
    for (uint32_t k = threadIdx.x; k < d * S; k += blockDim.x) L[k] = 0u;
    __syncthreads();
    const LocalHash H = build_local_hash<true>(hkeys, hidx, xs, d, threadIdx.x, blockDim.x);
    __syncthreads();
    const uint32_t nrows = kU ? d : d - 1;
    uint32_t i = gid;
    YInfo y = (i < nrows) ? yinfo(desc, xs[i]) : YInfo{0, 0, 0, 0, 0};
    while (i < nrows) {
      const uint32_t inext = i + kGroups;
      const YInfo ynext = (inext < nrows) ? yinfo(desc, xs[inext]) : YInfo{0, 0, 0, 0, 0};
      fill_row<kU>(k4_kind(y, kU ? d : nrows - i, sf16), col, bs, y, xs, d, i, H, L + i * S, gl);
      i = inext;
      y = ynext;
    }
    __syncthreads();
    // bit-parallel innermost loop: one warp per row i; the set bits j of L_i (the
    // local edges) are listed, then each LANE takes one edge and ANDs the words
    // of L_i and L_j above j (broadcast read of L_i, conflict-free reads of L_j).
    uint16_t* jl = jl_all + w * kMaxD;
    for (uint32_t r = w; r < d; r += kCWarps) {
      const uint32_t* Li = L + r * S;
      const uint32_t wv = ((uint32_t)lane < W) ? Li[lane] : 0u;
      const uint32_t c = __popc(wv);
      const uint32_t incl = warp_inclusive_scan(c);
      const uint32_t ne = __shfl_sync(kFull, incl, 31);
      uint32_t p = incl - c, t = wv;
      EH_DASSERT(incl <= d);
      while (t) {
        const uint32_t b = __ffs(t) - 1;
        t &= t - 1;
        jl[p++] = (uint16_t)(lane * 32 + b);
      }
      __syncwarp();
      for (uint32_t e = lane; e < ne; e += 32) {
        const uint32_t j = jl[e];
        const uint32_t kk = j >> 5;
        const uint32_t* Lj = L + j * S;
        uint32_t acc = 0;
        if (kU) {  // all w
          for (uint32_t k = 0; k < W; ++k) acc += __popc(Li[k] & Lj[k]);
        } else {   // w after z
          // every bit of row j lies above j (row j = N+(x) after x_j cap N+(x_j)), so the
          // words of L_i AND L_j need no mask
          acc = __popc(Li[kk] & Lj[kk]);
          for (uint32_t k = kk + 1; k < W; ++k) acc += __popc(Li[k] & Lj[k]);
        }
        cnt += acc;
      }
      __syncwarp();
    }
    __syncthreads();
  }
  cnt = warp_sum(cnt);
  if (lane == 0 && cnt) atomicAdd(&ctr[0], cnt);
}


// ------------------------------------------- hub rows: |N+(x)| > kCMaxD --
// Rows (x, y = x_i) of the big x are flattened into one index space (prefix
// sums of their row counts) and taken one per CTA.  The row's
//   P = N+(x) after y  cap  N+(y)        (kU: all of N(x) cap N(y))
// is built in order (stream the smaller side, O(1) bitset probe or binary search
// into the other; block-ordered compaction) in shared memory (global scratch
// when it could exceed the staging capacity), then every z in P is a warp task
// (taken from a shared cursor):  |P after z cap N+(z)|  (kU: all of P) by the
// cheaper of  (a) probing each p into N+(z) (bit test, or binary search of
// N+(z)) and (b) streaming N+(z) with coalesced loads, each element binary-
// searched in P on chip -- the min property applied per (x, y, z) (PAPER.md:
// 164-170, 628-642).  Before this kernel the hub rows probed all of P for every
// z with global binary searches (|P|^2 log d work): C4 unpruned 14.4 s.
constexpr int kBigThreads = 512;
constexpr uint32_t kBigPCap = 8192;   // P staged on chip up to this many elements (32 KB)
constexpr uint32_t kBigBmMaxWords = 40960;  // P's bitmap on chip for id spaces up to 1.31 M (160 KB)

struct BigPred {
  const uint4* desc;
  const uint32_t* work;
  __device__ bool operator()(uint64_t k) const { return desc[work[k]].y > (uint32_t)kCMaxD; }
};
struct BigEmit {
  const uint4* desc;
  const uint32_t* work;
  uint32_t* bx;
  uint32_t* brows;
  __device__ void operator()(uint64_t pos, uint64_t k) const {
    bx[pos] = work[k];
    brows[pos] = desc[work[k]].y;
  }
};

__device__ __forceinline__ uint32_t lower_bound_gen(const uint32_t* a, uint32_t n, uint32_t e) {
  uint32_t lo = 0, len = n;  // generic pointer: shared or global
  while (len > 0) {
    const uint32_t h = len >> 1;
    if (a[lo + h] < e) { lo += h + 1; len -= h + 1; } else { len = h; }
  }
  return lo;
}

template <bool kU>
__global__ void __launch_bounds__(kBigThreads) k_k4_big(const uint4* __restrict__ desc, const uint32_t* __restrict__ col,
                                                        const uint32_t* __restrict__ bs, const uint32_t* __restrict__ bx,
                                                        const uint64_t* __restrict__ boff, uint64_t nbig, uint64_t nrows,
                                                        uint32_t* __restrict__ pscratch, uint32_t pstride,
                                                        unsigned long long* __restrict__ ctr, uint32_t bm_words) {
  extern __shared__ __align__(16) uint32_t Psm[];  // kBigPCap, then (bm_words > 0) P as a bitmap over all ids
  uint32_t* bm = Psm + kBigPCap;
  constexpr int kW = kBigThreads / 32;
  for (uint32_t t = threadIdx.x; t < bm_words; t += kBigThreads) bm[t] = 0u;
  __shared__ unsigned long long s_r;
  __shared__ uint32_t s_wc[kW], s_z;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t* Pglob = pscratch + (uint64_t)blockIdx.x * pstride;
  unsigned long long cnt = 0;
  for (;;) {
    if (threadIdx.x == 0) { s_r = atomicAdd(&ctr[3], 1ull); s_z = 0; }
    __syncthreads();
    const unsigned long long r = s_r;
    if (r >= nrows) break;
    uint64_t lo = 0, hi = nbig;  // the big x whose rows contain r: last boff[k] <= r
    while (hi - lo > 1) {
      const uint64_t mid = (lo + hi) >> 1;
      if (boff[mid] <= r) lo = mid; else hi = mid;
    }
    const uint32_t x = bx[lo], i = (uint32_t)(r - boff[lo]);
    const uint4 dx = __ldg(desc + x);
    const uint32_t d = dx.y;
    const uint32_t* xs = col + (uint64_t)dx.x * 4;
    const uint32_t y = __ldg(xs + i);
    const SetRef sy = set_of(desc, col, bs, y);
    const uint32_t a0 = kU ? 0u : i + 1;  // A = xs[a0, d)
    if (a0 + 1 >= d || sy.len < 2) {      // |P| < 2 for every z
      __syncthreads();
      continue;
    }
    // P = A cap N(y), in order: stream the smaller side, probe the other
    const bool stream_a = (d - a0) <= sy.len;
    const SetRef sx = set_of(desc, col, bs, x);
    const uint32_t nsrc = stream_a ? d - a0 : sy.len;
    const uint32_t* src = stream_a ? xs + a0 : sy.list;
    uint32_t* P = (min(d - a0, sy.len) <= kBigPCap) ? Psm : Pglob;
    EH_DASSERT(min(d - a0, sy.len) <= pstride);
    uint32_t np = 0;
    for (uint32_t j0 = 0; j0 < nsrc; j0 += kBigThreads) {
      const uint32_t j = j0 + threadIdx.x;
      const uint32_t e = (j < nsrc) ? __ldg(src + j) : 0u;
      // streaming N(y) against all of N(x): keep only the elements of A (after y)
      const uint32_t hit = (j < nsrc) && (stream_a ? member(sy, e) : ((kU || e > y) && member(sx, e)));
      const unsigned m = __ballot_sync(kFull, hit);
      if (lane == 0) s_wc[w] = __popc(m);
      __syncthreads();
      uint32_t base = np, tot = 0;
#pragma unroll
      for (int q = 0; q < kW; ++q) {
        const uint32_t c = s_wc[q];
        if (q < w) base += c;
        tot += c;
      }
      if (hit) P[base + __popc(m & lt)] = e;
      np += tot;
      __syncthreads();
    }
    if (bm_words) {  // P's bitmap (cleared again after the row)
      for (uint32_t t = threadIdx.x; t < np; t += kBigThreads) atomicOr(&bm[P[t] >> 5], 1u << (P[t] & 31));
      __syncthreads();
    }
    // z tasks: warp per z from a shared cursor
    for (;;) {
      uint32_t k = 0;
      if (lane == 0) k = atomicAdd(&s_z, 1u);
      k = __shfl_sync(kFull, k, 0);
      if (k >= np) break;
      const uint32_t z = P[k];
      const SetRef sz = set_of(desc, col, bs, z);
      if (sz.len == 0) continue;
      const uint32_t* T = kU ? P : P + k + 1;  // the part of P that can meet N+(z)
      const uint32_t nt = kU ? np : np - k - 1;
      if (nt == 0) continue;
      const uint32_t lgt = 32 - __clz(nt), lgz = 32 - __clz(sz.len);
      // costs in element steps: probe each p of T into N(z); stream N(z) against P
      // (bit test in P's bitmap, else binary search of T); AND N(z)'s bitset chunks
      // with P's bitmap (every element of P below z misses N+(z), so the whole
      // bitmap is exact for the pruned nest too)
      const uint64_t probe_cost = (uint64_t)nt * (sz.bits ? 2u : 2u * lgz);
      const uint64_t stream_cost = (uint64_t)sz.len * (bm_words ? 1u : lgt);
      const uint64_t and_cost = (bm_words && sz.bits) ? (uint64_t)(sz.c1 - sz.c0) * 2u : ~0ull;
      uint32_t c = 0;
      if (and_cost <= probe_cost && and_cost <= stream_cost) {
        const uint4* zb = reinterpret_cast<const uint4*>(sz.bits);
        for (uint32_t ch = sz.c0 + lane; ch < sz.c1; ch += 32) {
          const uint4 zw = __ldg(zb + (ch - sz.c0));
          if (4 * ch + 3 < bm_words) {
            const uint4 pw = reinterpret_cast<const uint4*>(bm)[ch];
            c += __popc(zw.x & pw.x) + __popc(zw.y & pw.y) + __popc(zw.z & pw.z) + __popc(zw.w & pw.w);
          } else {
            const uint32_t zz[4] = {zw.x, zw.y, zw.z, zw.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (4 * ch + q < bm_words) c += __popc(zz[q] & bm[4 * ch + q]);
          }
        }
      } else if (probe_cost <= stream_cost) {
        for (uint32_t t = lane; t < nt; t += 32) c += member(sz, T[t]);
      } else if (bm_words) {
        for (uint32_t t = lane; t < sz.len; t += 32) {
          const uint32_t e = __ldg(sz.list + t);
          c += (bm[e >> 5] >> (e & 31)) & 1u;
        }
      } else {
        for (uint32_t t = lane; t < sz.len; t += 32) {
          const uint32_t e = __ldg(sz.list + t);
          const uint32_t p = lower_bound_gen(T, nt, e);
          c += (p < nt && T[p] == e) ? 1u : 0u;
        }
      }
      cnt += c;
    }
    __syncthreads();
    if (bm_words)
      for (uint32_t t = threadIdx.x; t < np; t += kBigThreads) bm[P[t] >> 5] = 0u;
  }
  cnt = warp_sum(cnt);
  if (lane == 0 && cnt) atomicAdd(&ctr[0], cnt);
}

template <bool kU, int kMaxD, int kCWarps>
void launch_k4_cta(eh_graph* g, const uint32_t* wl, uint64_t nlarge, uint32_t dlo, uint32_t cslot, uint32_t sf16,
                   cudaStream_t st) {
  constexpr size_t smem = k4_cta_smem<kMaxD, kCWarps>();
  auto k = k_k4_cta<kU, kMaxD, kCWarps>;
  ensure_dyn_smem((const void*)k, smem);
  int per_sm = 0;
  EH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kCWarps * 32, smem));
  const unsigned grid = (unsigned)std::min<uint64_t>(nlarge, (uint64_t)kSMs * std::max(1, per_sm));
  k<<<grid, kCWarps * 32, smem, st>>>(g->desc, g->col, g->bs, wl, nlarge, g->d_counter, dlo, cslot, sf16);
  EH_LAUNCH("k_k4_cta");
}

template <bool kU>
uint64_t k4_impl(eh_graph* g) {
  cudaStream_t s = g->stream;
  const uint32_t sf16 = g->n_act > (1ull << 24) ? 64u : 16u;  // C4 K4 7.44 -> 7.39 ms with 16
  EH_CUDA(cudaMemsetAsync(g->d_counter, 0, 8 * sizeof(unsigned long long), s));
  const uint64_t nsmall = g->n_work[0] + g->n_work[1];  // d <= tri_warp_max_degree() = kWMaxD
  const uint64_t nlarge = g->n_work[2];
  const uint32_t* wl = work_lpt(g) + nsmall;  // class 2 heaviest first
  // the warp-class kernel runs on a side stream beside the CTA-class kernels (they
  // share only the count, an atomic); test hook EH_TEST_K4_SERIAL keeps one stream
  // and the three CTA shapes run on streams of their own, so their tails overlap too
  // (measured: C2 K4 1.537 -> 1.467 -> 1.405 ms, C4 7.41 -> 7.35 -> 7.26, C3 45.45 -> 45.42 -> 45.33)
  const bool serial = getenv("EH_TEST_K4_SERIAL") != nullptr;
  const bool shapes = !serial;
  const cudaStream_t ss = (!serial && nsmall && nlarge) ? fork_side(g, 0) : s;
  const cudaStream_t s1 = (shapes && nlarge) ? fork_side(g, 1) : s;
  const cudaStream_t s2 = (shapes && nlarge && g->max_dplus > 512) ? fork_side(g, 2) : s;
  if (nsmall) {
    // class 0 (|N+(x)| <= 64) on the half-size instance when it holds all of it, the
    // rest (<= 128) after it on the same stream (its own work cursor, slot 6)
    const uint64_t n64 = (g->class0_max <= 64 && getenv("EH_TEST_K4_W128") == nullptr) ? g->n_work[0] : 0;
    if (n64) {
      auto kw = k_k4_warp<kU, 64>;
      const size_t smem = sizeof(K4WarpSmem<64>) * kWWarps;
      ensure_dyn_smem((const void*)kw, smem);
      int per_sm = 0;
      EH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kw, kWWarps * 32, smem));
      const unsigned grid = (unsigned)std::min<uint64_t>((n64 + kWWarps - 1) / kWWarps, (uint64_t)kSMs * std::max(1, per_sm));
      kw<<<grid, kWWarps * 32, smem, ss>>>(g->desc, g->col, g->bs, g->work, n64, g->d_counter, sf16, 6u);
      EH_LAUNCH("k_k4_warp");
    }
    if (nsmall > n64 && n64 && getenv("EH_TEST_K4_W128") == nullptr) {
      // class 1 (64 < |N+(x)| <= 128) as 4-warp CTAs over its LPT list (cursor slot 7):
      // ~7 KB each, 16 per SM, where the 128-entry warp instance holds 8.4 KB per warp
      // (measured: C3 K4 34.3 -> 32.7 ms, C2 1.24 -> 1.18, C4 5.89 -> 5.80; 2 / 8 warps
      // per CTA close behind)
      launch_k4_cta<kU, 128, 4>(g, work_lpt(g) + g->n_work[0], nsmall - n64, 0u, 7u, sf16, ss);
    } else if (nsmall > n64) {
      auto kw = k_k4_warp<kU, kWMaxD>;
      const size_t smem = sizeof(K4WarpSmem<kWMaxD>) * kWWarps;
      ensure_dyn_smem((const void*)kw, smem);
      const unsigned grid = (unsigned)std::min<uint64_t>((nsmall - n64 + kWWarps - 1) / kWWarps, (uint64_t)kSMs * 8);
      kw<<<grid, kWWarps * 32, smem, ss>>>(g->desc, g->col, g->bs, g->work + n64, nsmall - n64, g->d_counter, sf16,
                                            1u);
      EH_LAUNCH("k_k4_warp");
    }
  }
  if (nlarge) {
    // d <= 256: 8-warp CTAs (~25 KB); d <= 512: 32-warp CTAs (~82 KB); d <= 1024: 32 warps
    // (224 KB, one CTA per SM): more warps per x than round 1's 4 / 8 / 16 -- the fills
    // and the bit-parallel loop of one x are latency-bound, so more of them in flight
    // (measured: C4 K4 6.78 -> 6.20 (256: 8, 512: 16) -> 5.96 ms (512, 1024: 32), C3 43.4
    // -> 39.7 -> 34.9; 256-shape with 16 warps slower).  Test hooks EH_TEST_K4_W256 /
    // _W512 / _W1024 select other warp counts.
    const char* w256 = getenv("EH_TEST_K4_W256");
    const char* w512 = getenv("EH_TEST_K4_W512");
    const int nw256 = w256 ? atoi(w256) : 8, nw512 = w512 ? atoi(w512) : 32;
    if (nw256 == 4) launch_k4_cta<kU, 256, 4>(g, wl, nlarge, 0u, 5u, sf16, s);
    else if (nw256 == 16) launch_k4_cta<kU, 256, 16>(g, wl, nlarge, 0u, 5u, sf16, s);
    else launch_k4_cta<kU, 256, 8>(g, wl, nlarge, 0u, 5u, sf16, s);
    if (nw512 == 8) launch_k4_cta<kU, 512, 8>(g, wl, nlarge, 256u, 2u, sf16, s1);
    else if (nw512 == 16) launch_k4_cta<kU, 512, 16>(g, wl, nlarge, 256u, 2u, sf16, s1);
    else launch_k4_cta<kU, 512, 32>(g, wl, nlarge, 256u, 2u, sf16, s1);
    if (g->max_dplus > 512) {
      const char* w1024 = getenv("EH_TEST_K4_W1024");
      if (w1024 && atoi(w1024) == 16) launch_k4_cta<kU, kCMaxD, 16>(g, wl, nlarge, 512u, 4u, sf16, s2);
      else launch_k4_cta<kU, kCMaxD, 32>(g, wl, nlarge, 512u, 4u, sf16, s2);
    }
    if (g->max_dplus > (uint64_t)kCMaxD) {
      DBuf<uint32_t> bx(g->alloc, nlarge), brows(g->alloc, nlarge);
      const uint64_t nbig = select_if(nlarge, BigPred{g->desc, wl}, BigEmit{g->desc, wl, bx.p, brows.p}, g->alloc, s);
      DBuf<uint64_t> boff(g->alloc, nbig + 1), tot(g->alloc, 1);
      scan_exclusive_u32(brows.p, boff.p, nbig, tot.p, g->alloc, s);
      const uint64_t nrows = nbig ? read_scalar(tot.p, s) : 0;
      // P's bitmap over all ids on chip when it fits next to the P list (C2: 32 KB, C4: 80 KB)
      const uint32_t bm_words = (g->n_act + 127) / 128 * 4 <= kBigBmMaxWords ? (uint32_t)((g->n_act + 127) / 128 * 4) : 0u;
      const size_t smem = ((size_t)kBigPCap + bm_words) * 4;
      ensure_dyn_smem((const void*)k_k4_big<kU>, smem);
      int per_sm = 0;
      EH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_k4_big<kU>, kBigThreads, smem));
      const unsigned gb = (unsigned)std::min<uint64_t>(nrows, (uint64_t)kSMs * std::max(1, per_sm));
      const uint32_t stride = (uint32_t)g->max_dplus;  // |P| <= max |N+(x)|
      DBuf<uint32_t> scratch(g->alloc, (size_t)std::max(1u, gb) * stride);
      if (nrows) {  // a rank range (eh_count_4cliques_range) may hold none of the big x
        k_k4_big<kU><<<gb, kBigThreads, smem, s>>>(g->desc, g->col, g->bs, bx.p, boff.p, nbig, nrows, scratch.p,
                                                    stride, g->d_counter, bm_words);
        EH_LAUNCH("k_k4_big");
      }
      EH_CUDA(cudaStreamSynchronize(s));  // scratch is released on return
    }
  }
  if (ss != s) join_side(g, 0);
  if (s1 != s) join_side(g, 1);
  if (s2 != s) join_side(g, 2);
  EH_CUDA(cudaMemcpyAsync(g->h_counter, g->d_counter, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaStreamSynchronize(s));
  return g->h_counter[0];
}

}  // namespace

uint64_t count_4cliques(eh_graph* g) { return k4_impl<false>(g); }

// NEXT-2: the unpruned 4-clique nest over the symmetric trie = 24 K4.  Hub
// lists (> 1024) take the CTA-per-row kernel k_k4_big (DESIGN.md NEXT-2).
uint64_t count_4cliques_unpruned(eh_graph* g) { return k4_impl<true>(symmetric_trie(g)); }

}  // namespace eh
