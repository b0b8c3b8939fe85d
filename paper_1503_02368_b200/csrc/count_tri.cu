// count_tri.cu -- SURVEY.md §8(a) rows a7 (work classes), a8 (triangle
// Generic-Join) and a10 (warp-shuffle uint64 reduction).
//
// Loop nest with R = S = T = E+ in rank space:
//     for x:  for y in N+(x):  Q += | N+(y) cap N+(x) |
// Every element of N+(y) is larger than y, so |N+(y) cap N+(x)| equals
// |N+(y) cap A| with A = N+(x) after y: a
// membership test against the WHOLE of N+(x) is exact, and a loop over A only
// needs the suffix.
//
// Each edge (x, y) -- a "row" of x -- picks the cheapest intersection for its
// layout pair (min property):
//   PROBE  N+(y) bitset: every a in A tests its bit in y's bitset (uint cap
//          bitset).
//   AND    N+(y) bitset and x staged as a bitmap in shared memory: AND the
//          overlapping 128-bit chunks and popcount (bitset cap bitset,
//          PAPER.md:636) when the overlap is small relative to |A|.
//   STREAM N+(y) uint: stream y's list with coalesced 128-bit loads and test
//          each element against N+(x) staged in shared memory -- an exact
//          bitmap over x's span when it fits, else an open-addressing hash
//          table (O(1) per element; a B200 replacement for the paper's SIMD
//          shuffling merge, same result).
//   SEARCH N+(y) uint and |A| log|B| << |B|: each a in A binary-searches B
//          (the galloping side of the uint hybrid).
// Rows are short (tens of units), so each row runs on an 8-lane sub-warp
// group: 4 rows in flight per warp, and 8 lanes x 16 B still read one full
// 128-B line per load.  Work classes (a7): 2 <= |N+(x)| <= kWarpMaxD run one
// warp per x (rows ordered by kind so the 4 groups of a warp rarely diverge);
// larger x run one CTA per x (its groups take rows round-robin).  COUNT(*) is a per-lane
// u64, reduced with __shfl_xor_sync, one atomicAdd(unsigned long long) per warp
// (PAPER.md:243).
#include "eh_internal.cuh"
#include "primitives.cuh"
#include "rows.cuh"
#include "sets.cuh"

namespace eh {

namespace {

// ------------------------------------------------------------ tunables --
constexpr int kG = 8;                 // lanes per row group
constexpr int kWarpMaxD = 128;        // warp kernel handles 2 <= d <= kWarpMaxD
constexpr int kWarpBmWords = 512;     // warp-kernel x structure: 2 KB (bitmap of 16384 ids or 512-slot hash)
constexpr int kWK_Warps = 8;
// CTA kernel shapes (measured on C2-C5): small CTAs with an 8 KB x
// structure (bitmap of 65536 ids), many per SM, balance the per-x tails best --
// unless the id space is so large that the spans of N+(x) outgrow that bitmap
// (C5: 2^26 ids), where 16-warp CTAs with a 64 KB structure win.
constexpr uint32_t kCtaXCapMax = 16384;  // CTA kernel stages N+(x) in smem up to xcap = max |N+(x)|
constexpr uint32_t kCtaXCapNarrow = 4096; // rounded up to 256, clamped to these (wide / narrow shape)
constexpr uint64_t kWideIds = 1ull << 24;  // n_active above this -> the wide shape
constexpr uint32_t kRowsPerItem = 1024;    // NEXT-2: rows of one CTA work item
constexpr uint64_t kHubBitmapBudget = 4ull << 30;  // NEXT-2: device bytes for the hub bitmaps
constexpr uint32_t kAndFactor = 8;    // AND when overlap chunks <= kAndFactor * |A| + 8
constexpr uint32_t kEmpty = 0xFFFFFFFFu;

enum RowKind : uint8_t { kSkip = 0, kProbe = 1, kAnd = 2, kStream = 3, kSearchGlobal = 4 };
enum XMode : uint32_t { kBitmap = 0, kHash = 1, kSorted = 2, kHashF = 3 };
#ifndef EH_HASH_FILTER
#define EH_HASH_FILTER 1
#endif
#ifndef EH_HASH_FILTER_MUL
#define EH_HASH_FILTER_MUL 4
#endif

// ---------------------------------------------- x's membership structure --
// N+(x) in shared memory as (a) an exact bitmap over [lo, lo + nbits), (b) an
// open-addressing hash table with 2^hbits slots (load <= 1/2), alone (kHash) or
// behind a one-hash filter with 32 bits per home slot (kHashF: a miss -- most
// lookups of a STREAM row -- is one shared-memory load and never walks a probe
// chain; C5 855 -> 728 ms), or (c) the sorted list itself (binary search; CTA
// kernel only when |N+(x)| > xcap).
struct XSet {
  uint32_t* tab;        // bitmap words or hash slots (shared memory)
  const uint32_t* xs;   // sorted N+(x) (shared or global)
  uint32_t mode, lo, nbits, hshift, hmask, d, amin, amax;

  __device__ __forceinline__ uint32_t contains(uint32_t e) const {
    if (mode == kBitmap) {
      const uint32_t o = e - lo;
      return (o < nbits) ? (tab[o >> 5] >> (o & 31)) & 1u : 0u;
    }
    if (e < amin || e > amax) return 0u;
    if (mode == kHashF) {
      // filter word w = the hash slot's home index: one bit per (w, next 5 hash bits)
      const uint32_t h = e * 2654435761u;
      uint32_t s = h >> hshift;
      if (!((tab[s] >> ((h >> (hshift - 5)) & 31)) & 1u)) return 0u;
      const uint32_t* slots = tab + hmask + 1;
      for (;;) {
        const uint32_t v = slots[s];
        if (v == e) return 1u;
        if (v == kEmpty) return 0u;
        s = (s + 1) & hmask;
      }
    }
    if (mode == kHash) {
      uint32_t s = (e * 2654435761u) >> hshift;
      for (;;) {
        const uint32_t v = tab[s];
        if (v == e) return 1u;
        if (v == kEmpty) return 0u;
        s = (s + 1) & hmask;
      }
    }
    uint32_t lo2 = 0, len = d;
    while (len > 0) {
      const uint32_t h = len >> 1;
      if (xs[lo2 + h] < e) { lo2 += h + 1; len -= h + 1; } else { len = h; }
    }
    return (lo2 < d && xs[lo2] == e) ? 1u : 0u;
  }
};

// Choose the structure (no shared-memory writes): exact bitmap if x's span fits
// the budget; else, when 4d words fit, a one-hash filter in front of a hash table
// (kHashF); else a hash with load <= 1/2 (<= 1/8 when the budget allows); else a
// binary search of the staged list.
__device__ __forceinline__ XSet plan_xset(uint32_t* tab, uint32_t tab_words, const uint32_t* xs, uint32_t d) {
  XSet s;
  s.tab = tab;
  s.xs = xs;
  s.d = d;
  s.amin = xs[0];
  s.amax = xs[d - 1];
  const uint32_t lo = (s.amin >> 7) << 7;
  const uint64_t span_bits = (uint64_t)(((s.amax >> 7) + 1) << 7) - lo;
  uint32_t hbits = 5;  // smallest table >= 8d that fits the budget
  while ((1u << hbits) < 8 * d && (2u << hbits) <= tab_words) ++hbits;
  if (span_bits <= 32ull * tab_words) {
    EH_DASSERT(d >= 1 && s.amin <= s.amax);
    s.mode = kBitmap;
    s.lo = lo;
    s.nbits = (uint32_t)span_bits;
    s.hshift = s.hmask = 0;
  } else if (EH_HASH_FILTER && tab_words >= 64 && EH_HASH_FILTER_MUL * d <= tab_words) {
    // half the budget as a one-hash filter (16 * tab_words bits, <= d of them set), half as
    // the hash table (load <= 1/2): a miss -- most lookups -- costs one load and never probes
    const uint32_t half = tab_words / 2;  // a power of two
    s.mode = kHashF;
    s.lo = s.nbits = 0;
    s.hshift = 32 - (31 - __clz(half));
    s.hmask = half - 1u;
  } else if ((1u << hbits) <= tab_words && (1u << hbits) >= 2 * d) {
    s.mode = kHash;
    s.lo = s.nbits = 0;
    s.hshift = 32 - hbits;
    s.hmask = (1u << hbits) - 1u;
  } else {
    s.mode = kSorted;
    s.lo = s.nbits = s.hshift = s.hmask = 0;
  }
  return s;
}

// Fill the planned structure cooperatively (tid in [0, nthreads)); caller syncs afterwards.
__device__ __forceinline__ void fill_xset(const XSet& s, int tid, int nthreads) {
  uint32_t* tab = s.tab;
  const uint32_t* xs = s.xs;
  const uint32_t d = s.d;
  if (s.mode == kBitmap) {
    for (uint32_t k = tid; k < s.nbits / 32; k += nthreads) tab[k] = 0u;
  } else if (s.mode == kHash) {
    for (uint32_t k = tid; k <= s.hmask; k += nthreads) tab[k] = kEmpty;
  } else if (s.mode == kHashF) {
    for (uint32_t k = tid; k <= s.hmask; k += nthreads) { tab[k] = 0u; tab[s.hmask + 1 + k] = kEmpty; }
  }
  if (nthreads == 32) __syncwarp(); else __syncthreads();
  const uint32_t lo = s.lo;
  if (s.mode == kBitmap) {
    for (uint32_t k = tid; k < d; k += nthreads) {
      const uint32_t o = xs[k] - lo;
      EH_DASSERT(o < s.nbits);
      atomicOr(&tab[o >> 5], 1u << (o & 31));
    }
  } else if (s.mode == kHash) {
    for (uint32_t k = tid; k < d; k += nthreads) {
      const uint32_t e = xs[k];
      uint32_t h = (e * 2654435761u) >> s.hshift;
      while (atomicCAS(&tab[h], kEmpty, e) != kEmpty) h = (h + 1) & s.hmask;
    }
  } else if (s.mode == kHashF) {
    uint32_t* slots = tab + s.hmask + 1;
    for (uint32_t k = tid; k < d; k += nthreads) {
      const uint32_t e = xs[k];
      const uint32_t hh = e * 2654435761u;
      uint32_t h = hh >> s.hshift;
      atomicOr(&tab[h], 1u << ((hh >> (s.hshift - 5)) & 31));
      while (atomicCAS(&slots[h], kEmpty, e) != kEmpty) h = (h + 1) & s.hmask;
    }
  }
}

__device__ __forceinline__ XSet build_xset(uint32_t* tab, uint32_t tab_words, const uint32_t* xs, uint32_t d,
                                           int tid, int nthreads) {
  const XSet s = plan_xset(tab, tab_words, xs, d);
  fill_xset(s, tid, nthreads);
  return s;
}

// Decide the intersection for row i of x (y = xs[i], |A| = a).
// sf16: the SEARCH side is taken when |A| log2|B| sf16/16 < |B| (c13).  A binary
// search costs log2|B| dependent loads, cheap when the lists are L2-resident
// (narrow graphs: sf16 = 16) and dear when they stream from HBM (above 2^24 active
// ids, the wide kernels: sf16 = 64; a compile-time constant -- as a runtime value
// it also changed the wide kernel's code generation, C5 900 -> 1050 ms).  Measured: C3 9.46 -> 9.20 ms, C4 1.52 -> 1.47, C2 0.333 -> 0.318
// with 16 instead of 64; C5 903 ms with 64 vs 956 with 16.
template <uint32_t sf16>
__device__ __forceinline__ uint8_t row_kind(const YInfo& y, uint32_t a, const XSet& X) {
  if (a == 0 || y.len == 0) return kSkip;
  if (y.c1 > y.c0) {
    if (X.mode == kBitmap) {
      const uint32_t xc0 = X.lo >> 7, xc1 = xc0 + (X.nbits >> 7);
      const uint32_t lo = max(y.c0, xc0), hi = min(y.c1, xc1);
      if (hi <= lo) return kSkip;
      if (hi - lo <= kAndFactor * a + 8) return kAnd;
    }
    return kProbe;
  }
  const uint32_t lg = 32 - __clz(y.len);
  if (y.c0 >= kAlwaysSearch ? y.c0 == kAlwaysSearch : (uint64_t)a * lg * sf16 < (uint64_t)y.len * 16) return kSearchGlobal;
  return kStream;
}

// Unpruned rows (NEXT-2) meet every combination of |A| = d(x) and |N(y)|
// (hubs on both sides), so the choice uses explicit costs: PROBE a bit tests,
// STREAM |N(y)| lookups in x's structure (log2 d when it is the sorted list),
// SEARCH a binary searches of N(y), AND as above.
template <uint32_t sf16>
__device__ __forceinline__ uint8_t row_kind_unpruned(const YInfo& y, uint32_t a, const XSet& X) {
  if (a == 0 || y.len == 0) return kSkip;
  const uint32_t lgx = (X.mode == kSorted) ? (32 - __clz(X.d)) : 1u;
  const uint64_t stream = (uint64_t)y.len * lgx;
  if (y.c1 > y.c0) {
    if (X.mode == kBitmap) {
      const uint32_t xc0 = X.lo >> 7, xc1 = xc0 + (X.nbits >> 7);
      const uint32_t lo = max(y.c0, xc0), hi = min(y.c1, xc1);
      if (hi <= lo) return kSkip;
      if (hi - lo <= kAndFactor * a + 8) return kAnd;
    }
    return (stream < a) ? kStream : kProbe;
  }
  const uint64_t search = (uint64_t)a * (32 - __clz(y.len)) * sf16;
  return (y.c0 >= kAlwaysSearch ? y.c0 == kAlwaysSearch : search < stream * 16) ? kSearchGlobal : kStream;
}

// ---- group-level row bodies: kG lanes, gl = lane within the group --------
__device__ __forceinline__ uint32_t and4(const uint4 u, const uint4 v) {
  return __popc(u.x & v.x) + __popc(u.y & v.y) + __popc(u.z & v.z) + __popc(u.w & v.w);
}

template <int G = kG, bool kPiv = false, int kSl = 8, int kAndU = 2>  // kSl: pivot slices (16 measured: C3 +2 %, C5 -0.5 %)
__device__ __forceinline__ uint32_t grp_row(uint8_t kd, const uint32_t* __restrict__ col,
                                            const uint32_t* __restrict__ bs, const YInfo& y, const XSet& X,
                                            const uint32_t* A, uint32_t na, uint32_t gl) {
  uint32_t c = 0;
  if (kd == kProbe) {  // (4 probes in flight per lane measured slower: C3 8.63 -> 8.75 ms)
    for (uint32_t j = gl; j < na; j += G) c += probe_bits(bs, y, A[j]);
  } else if (kd == kAnd) {
    const uint32_t xc0 = X.lo >> 7, xc1 = xc0 + (X.nbits >> 7);
    const uint32_t lo = max(y.c0, xc0), hi = min(y.c1, xc1);
    const uint4* yb = reinterpret_cast<const uint4*>(bs) + y.pool;  // chunk y.c0
    const uint4* xb = reinterpret_cast<const uint4*>(X.tab);        // chunk xc0
    EH_DASSERT(X.mode == kBitmap && lo >= y.c0 && hi <= y.c1 && lo >= xc0 && hi <= xc1);
    uint32_t k = lo + gl;                                            // absolute chunk index
    if (kAndU == 4) {  // 4 chunk loads in flight per lane (narrow shape on large graphs: C3 8.90 -> 8.63 ms)
      for (; k + 3 * G < hi; k += 4 * G) {
        const uint4 u0 = __ldg(yb + (k - y.c0)), u1 = __ldg(yb + (k + G - y.c0));
        const uint4 u2 = __ldg(yb + (k + 2 * G - y.c0)), u3 = __ldg(yb + (k + 3 * G - y.c0));
        c += and4(u0, xb[k - xc0]) + and4(u1, xb[k + G - xc0]) + and4(u2, xb[k + 2 * G - xc0]) +
             and4(u3, xb[k + 3 * G - xc0]);
      }
      for (; k < hi; k += G) c += and4(__ldg(yb + (k - y.c0)), xb[k - xc0]);
    } else {  // 2 in flight (C2, C4, and the wide shape: C5 879 vs 907 ms with 4)
      for (; k + G < hi; k += 2 * G) {
        const uint4 u0 = __ldg(yb + (k - y.c0)), u1 = __ldg(yb + (k + G - y.c0));
        c += and4(u0, xb[k - xc0]) + and4(u1, xb[k + G - xc0]);
      }
      if (k < hi) c += and4(__ldg(yb + (k - y.c0)), xb[k - xc0]);
    }
  } else if (kd == kStream) {
    const uint4* yl = reinterpret_cast<const uint4*>(col) + y.list;
    const uint32_t nfull = y.len >> 2;
    uint32_t k = gl;
    for (; k + G < nfull; k += 2 * G) {
      const uint4 v0 = __ldg(yl + k), v1 = __ldg(yl + k + G);
      c += X.contains(v0.x) + X.contains(v0.y) + X.contains(v0.z) + X.contains(v0.w);
      c += X.contains(v1.x) + X.contains(v1.y) + X.contains(v1.z) + X.contains(v1.w);
    }
    if (k < nfull) {
      const uint4 v = __ldg(yl + k);
      c += X.contains(v.x) + X.contains(v.y) + X.contains(v.z) + X.contains(v.w);
    }
    if (gl < (y.len & 3)) c += X.contains(__ldg(col + (uint64_t)y.list * 4 + nfull * 4 + gl));
  } else if (kd == kSearchGlobal) {
    const uint32_t* L = col + (uint64_t)y.list * 4;
    const uint32_t n = y.len;
    if (kPiv && n >= 4 * kSl) {
      // the group's lanes load kSl-1 pivots (the last element of each of kSl equal
      // slices of N+(y)) in one round; every search then starts inside one slice,
      // log2(kSl) fewer dependent loads per element of A
      constexpr int kPer = kSl / G;  // pivots per lane
      const uint32_t gbase = (threadIdx.x & 31) & ~(uint32_t)(G - 1);
      const unsigned gmask = (G == 32) ? 0xFFFFFFFFu : (((1u << G) - 1u) << gbase);
      uint32_t mine[kPer];
#pragma unroll
      for (int r = 0; r < kPer; ++r) {
        const uint32_t q = gl * kPer + r;
        mine[r] = (q < kSl - 1) ? __ldg(L + (uint64_t)(q + 1) * n / kSl - 1) : 0u;
      }
      uint32_t piv[kSl - 1];
#pragma unroll
      for (int q = 0; q < kSl - 1; ++q) piv[q] = __shfl_sync(gmask, mine[q % kPer], q / kPer, G);
      for (uint32_t j = gl; j < na; j += G) {
        const uint32_t e = A[j];
        uint32_t k = 0;
#pragma unroll
        for (int q = 0; q < kSl - 1; ++q) k += (piv[q] < e);
        const uint32_t lo = (uint32_t)((uint64_t)k * n / kSl), hi = (uint32_t)((uint64_t)(k + 1) * n / kSl);
        c += gmem_search(L + lo, hi - lo, e);
      }
    } else {
      for (uint32_t j = gl; j < na; j += G) c += gmem_search(L, n, A[j]);
    }
  }
  return c;
}

// ---- NEXT-3 block-level (composite) layout (EH_BLOCK_LAYOUT, trie.cu) -------
struct BlockView {
  const uint4* bdesc;
  const uint32_t* bcol;
  const uint32_t* bcid;
  const uint4* bmask;
};

// y's composite set as a YInfo: list/len = its uint (sparse) part, pool = first
// dense block, c0 = number of dense blocks, c1 = 0 (no set-level bitset).
__device__ __forceinline__ YInfo yinfo_block(const BlockView& bv, uint32_t y) {
  const uint4 b = __ldg(bv.bdesc + y);
  const uint32_t z1 = __ldg(&bv.bdesc[y + 1].z);
  return YInfo{b.x, b.y, b.z, z1 - b.z, 0u};
}

// Min property on composite sets: when |A| is small against y, every a in A is
// looked up (binary search of its block among y's dense blocks, then a bit test
// or a binary search of the sparse part) -- kProbe; otherwise the sparse part
// follows the uint rules (kSearchGlobal / kStream) and the dense blocks are
// ANDed (rows with only dense blocks: kAnd).
__device__ __forceinline__ uint8_t row_kind_block(const YInfo& y, uint32_t a) {
  if (a == 0 || (y.len == 0 && y.c0 == 0)) return kSkip;
  const uint32_t lgs = 32 - __clz(y.len), lgd = 32 - __clz(y.c0);
  if ((uint64_t)a * (lgs + lgd) * 4 < (uint64_t)y.len + 4ull * y.c0) return kProbe;
  if (y.len == 0) return kAnd;
  if ((uint64_t)a * lgs * 4 < y.len) return kSearchGlobal;
  return kStream;
}

__device__ __forceinline__ uint32_t block_member(const BlockView& bv, const YInfo& y, uint32_t e) {
  const uint32_t c = e >> 7;
  uint32_t lo = 0, len = y.c0;  // lower_bound of c among the dense block numbers
  const uint32_t* ids = bv.bcid + y.pool;
  while (len > 0) {
    const uint32_t h = len >> 1;
    if (__ldg(ids + lo + h) < c) { lo += h + 1; len -= h + 1; } else { len = h; }
  }
  if (lo < y.c0 && __ldg(ids + lo) == c) {
    const uint4 m = __ldg(bv.bmask + y.pool + lo);
    const uint32_t q = (e >> 5) & 3, w = q == 0 ? m.x : q == 1 ? m.y : q == 2 ? m.z : m.w;
    return (w >> (e & 31)) & 1u;
  }
  return gmem_search(bv.bcol + (uint64_t)y.list * 4, y.len, e);
}

// |A cap N+(y)| = |A cap sparse(y)| + |A cap dense(y)|: the sparse part as a uint
// row, each dense block ANDed with x's staged bitmap chunk (bitset cap bitset,
// PAPER.md:636) or, when x is hashed, its bits looked up one by one.
template <int G = kG>
__device__ __forceinline__ uint32_t grp_row_block(uint8_t kd, const BlockView& bv, const uint32_t* __restrict__ bs,
                                                  const YInfo& y, const XSet& X, const uint32_t* A, uint32_t na,
                                                  uint32_t gl) {
  if (kd == kProbe) {
    uint32_t c = 0;
    for (uint32_t j = gl; j < na; j += G) c += block_member(bv, y, A[j]);
    return c;
  }
  uint32_t c = (kd == kStream || kd == kSearchGlobal) ? grp_row<G>(kd, bv.bcol, bs, y, X, A, na, gl) : 0u;
  const uint32_t nd = y.c0;
  const uint32_t xc0 = X.lo >> 7, xc1 = xc0 + (X.nbits >> 7);
  const uint4* xb = reinterpret_cast<const uint4*>(X.tab);
  for (uint32_t k = gl; k < nd; k += G) {
    const uint32_t cc = __ldg(bv.bcid + y.pool + k);
    const uint4 m = __ldg(bv.bmask + y.pool + k);
    if (X.mode == kBitmap) {
      if (cc >= xc0 && cc < xc1) c += and4(m, xb[cc - xc0]);
    } else {
      const uint32_t w[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t t = w[q];
        while (t) {
          const uint32_t b = __ffs(t) - 1;
          t &= t - 1;
          c += X.contains(cc * 128 + q * 32 + b);
        }
      }
    }
  }
  return c;
}

// ------------------------------------------------------------ warp kernel --
// One warp per x with 2 <= |N+(x)| <= kWarpMaxD.  Lanes classify the rows in
// parallel, rows are ordered by kind, then the 4 groups take rows round-robin.
template <int kMaxD>
struct __align__(16) WarpSmem {
  uint32_t xs[kMaxD];
  uint32_t tab[kWarpBmWords];
  YInfo yi[kMaxD];
  uint8_t kind[kMaxD];
  uint8_t ord[kMaxD];  // non-skip rows grouped by kind
};

// kUnpruned (NEXT-2, unpruned nest on the symmetric trie): row i intersects all of
// N(x) with N(y) (no suffix restriction) and every element of N(x) is a row.
template <bool kUnpruned, bool kBlock, int kMaxD, int kMinB, int kWG = kG, uint32_t kSF = 64, bool kPiv = false,
          int kAU = (kPiv && kSF == 16) ? 4 : 2>
__global__ void __launch_bounds__(kWK_Warps * 32, kMinB) k_tri_warp(const uint4* __restrict__ desc,
                                                             const uint32_t* __restrict__ col,
                                                             const uint32_t* __restrict__ bs,
                                                             const uint32_t* __restrict__ work, uint64_t nwork,
                                                             unsigned long long* __restrict__ ctr, BlockView bv,
                                                             uint32_t cslot) {
  extern __shared__ __align__(16) uint32_t dsm_w[];
  WarpSmem<kMaxD>* sm_all = reinterpret_cast<WarpSmem<kMaxD>*>(dsm_w);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t grp = lane / kWG, gl = lane % kWG;
  WarpSmem<kMaxD>& sm = sm_all[w];
  const unsigned lt = (1u << lane) - 1u;
  unsigned long long cnt = 0;
  for (;;) {
    unsigned long long wi = 0;
    if (lane == 0) wi = atomicAdd(&ctr[cslot], 1ull);  // (grabbing 2-8 x per atomic measured no faster)
    wi = __shfl_sync(kFull, wi, 0);
    if (wi >= nwork) break;
    const uint32_t x = __ldg(work + wi);
    const uint4 dx = __ldg(desc + x);
    const uint32_t d = dx.y;  // 2 <= d <= kWarpMaxD
    EH_DASSERT(d >= 2 && d <= (uint32_t)kMaxD);
    const uint32_t* xg = col + (uint64_t)dx.x * 4;
    for (uint32_t k = lane; k < (d + 3) / 4; k += 32)
      reinterpret_cast<uint4*>(sm.xs)[k] = __ldg(reinterpret_cast<const uint4*>(xg) + k);
    __syncwarp();
    const XSet X = plan_xset(sm.tab, kWarpBmWords, sm.xs, d);
    const uint32_t nrows = kUnpruned ? d : d - 1;
    bool need_x = false;  // only AND and STREAM rows read x's staged structure
    for (uint32_t i = lane; i < nrows; i += 32) {
      const YInfo y = kBlock ? yinfo_block(bv, sm.xs[i]) : yinfo(desc, sm.xs[i]);
      const uint8_t kd = kBlock ? row_kind_block(y, nrows - i)
                       : kUnpruned ? row_kind_unpruned<kSF>(y, d, X) : row_kind<kSF>(y, nrows - i, X);
      sm.yi[i] = y;
      sm.kind[i] = kd;
      need_x |= kBlock || (kd == kAnd || kd == kStream);
    }
    if (__any_sync(kFull, need_x)) fill_xset(X, lane, 32);
    __syncwarp();
    uint32_t nr = 0;
#pragma unroll
    for (int kdi = 0; kdi < 4; ++kdi) {
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
    for (uint32_t r = grp; r < nr; r += 32 / kWG) {
      const uint32_t i = sm.ord[r];
      cnt += kBlock ? grp_row_block<kWG>(sm.kind[i], bv, bs, sm.yi[i], X, sm.xs + i + 1, nrows - i, gl)
           : kUnpruned ? grp_row<kWG>(sm.kind[i], col, bs, sm.yi[i], X, sm.xs, d, gl)
                       : grp_row<kWG, kPiv, 8, kAU>(sm.kind[i], col, bs, sm.yi[i], X, sm.xs + i + 1, nrows - i, gl);
    }
    __syncwarp();
  }
  cnt = warp_sum(cnt);
  if (lane == 0 && cnt) atomicAdd(&ctr[0], cnt);
}

// ----------------------------------------------------------- thread kernel --
// a7 thread class: one THREAD per x with 2 <= |N+(x)| <= bin_thread_max (C3:
// 923 k of the 1.56 M warp-class x, but only 2.7 M of their 15 M rows and 7 M
// of their 161 M wedges).  A warp per such x spends its time on the per-x
// staging / classification / ordering with most lanes idle; here 32 x run side
// by side.  Row (x, y = x_i): every a in A = N+(x) after y is a bit probe of
// y's bitset (uint cap bitset) or, y uint, a binary search of N+(y) that
// resumes where the previous a stopped (A is increasing; the galloping side
// of the uint hybrid) -- |A| <= 15, so the min property always
// favours probing A over streaming N+(y).  N+(x) is staged per thread in
// shared memory with an odd stride (a warp's 32 threads hit 32 banks).
constexpr int kTMax = 16;
constexpr int kTBlock = 256;
constexpr int kTStride = kTMax + 1;

__global__ void __launch_bounds__(kTBlock) k_tri_thread(const uint4* __restrict__ desc,
                                                        const uint32_t* __restrict__ col,
                                                        const uint32_t* __restrict__ bs,
                                                        const uint32_t* __restrict__ work, uint64_t nwork,
                                                        unsigned long long* __restrict__ ctr) {
  __shared__ uint32_t sxs[kTBlock * kTStride];
  uint32_t* xs = sxs + threadIdx.x * kTStride;
  unsigned long long cnt = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nwork; k += stride) {
    const uint32_t x = __ldg(work + k);
    const uint4 dx = __ldg(desc + x);
    const uint32_t d = dx.y;  // 2 <= d <= kTMax
    EH_DASSERT(d >= 2 && d <= (uint32_t)kTMax);
    const uint4* xg = reinterpret_cast<const uint4*>(col) + dx.x;
    for (uint32_t q = 0; q < (d + 3) / 4; ++q) {
      const uint4 v = __ldg(xg + q);
      xs[4 * q] = v.x;
      xs[4 * q + 1] = v.y;
      xs[4 * q + 2] = v.z;
      xs[4 * q + 3] = v.w;
    }
    for (uint32_t i = 0; i + 1 < d; ++i) {
      const YInfo y = yinfo(desc, xs[i]);
      if (y.len == 0) continue;
      if (y.c1 > y.c0) {
        for (uint32_t j = i + 1; j < d; ++j) cnt += probe_bits(bs, y, xs[j]);
      } else {
        const uint32_t* L = col + (uint64_t)y.list * 4;
        uint32_t lo = 0;
        for (uint32_t j = i + 1; j < d; ++j) {
          const uint32_t e = xs[j];
          uint32_t len = y.len - lo;
          while (len > 0) {
            const uint32_t h = len >> 1;
            if (__ldg(L + lo + h) < e) { lo += h + 1; len -= h + 1; } else { len = h; }
          }
          if (lo == y.len) break;
          cnt += (__ldg(L + lo) == e);
        }
      }
    }
  }
  cnt = warp_sum(cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&ctr[0], cnt);
}

void launch_thread(eh_graph* g, uint64_t nt, cudaStream_t st) {
  if (nt == 0) return;
  int per_sm = 0;
  EH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tri_thread, kTBlock, 0));
  const unsigned grid = (unsigned)std::min<uint64_t>((nt + kTBlock - 1) / kTBlock, (uint64_t)kSMs * std::max(1, per_sm));
  k_tri_thread<<<grid, kTBlock, 0, st>>>(g->desc, g->col, g->bs, g->work, nt, g->d_counter);
  EH_LAUNCH("k_tri_thread");
}

// ---------------------------------------------- bulk async copy (TMA) --
// 1-D cp.async.bulk global -> shared, completion tracked by an mbarrier
// (transaction bytes); one thread arms and issues, every thread waits.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}

// ------------------------------------------------------------- CTA kernel --
// One CTA per x (classes 1-2); its 8-lane groups take rows round-robin
// (row i has |A| = d-1-i, so the loads even out), prefetching the next row's
// descriptor before working on the current one.
template <int kCtaWarps, int kTabW, int kXCap, bool kUnpruned, bool kBlock, int kMinB, int kCG = kG, uint32_t kSF = 64,
          bool kPiv = false, bool kTma = !kUnpruned && !kBlock && kCtaWarps == 16,
          int kAU = (kPiv && kCtaWarps == 4) ? 4 : 2>  // kXCap > 0: compile-time staging capacity
__global__ void __launch_bounds__(kCtaWarps * 32, kMinB) k_tri_cta(const uint4* __restrict__ desc,
                                                            const uint32_t* __restrict__ col,
                                                            const uint32_t* __restrict__ bs,
                                                            const uint32_t* __restrict__ work, uint64_t nwork,
                                                            unsigned long long* __restrict__ ctr, uint32_t xcap_rt,
                                                            const unsigned long long* __restrict__ items,
                                                            const uint32_t* __restrict__ hslot,
                                                            uint32_t* __restrict__ hub_bm, uint32_t hub_words,
                                                            BlockView bv, uint32_t cslot) {
  // kUnpruned: work items are (x << 32 | first row) over row ranges of kRowsPerItem
  // (hub lists of the symmetric trie would otherwise leave one CTA with 10^5 rows)
  const uint32_t xcap = kXCap > 0 ? (uint32_t)kXCap : xcap_rt;
  extern __shared__ __align__(16) uint32_t dsm[];
  uint32_t* xs_s = dsm;                         // xcap (kTma: two buffers)
  uint32_t* tab = dsm + (kTma ? 2 : 1) * xcap;  // kTabW
  __shared__ unsigned long long s_wi;
  constexpr uint32_t kGroups = kCtaWarps * 32 / kCG;
  const int lane = threadIdx.x & 31;
  const uint32_t gid = threadIdx.x / kCG, gl = threadIdx.x % kCG;
  unsigned long long cnt = 0;
  if constexpr (kTma) {
    // the rows of x (as in the loop below)
    auto rows = [&](const uint32_t* xs, const XSet& X, uint32_t d, uint32_t nrows, uint32_t r0) {
      uint32_t i = r0 + gid;
      YInfo y = (i < nrows) ? (kBlock ? yinfo_block(bv, xs[i]) : yinfo(desc, xs[i])) : YInfo{0, 0, 0, 0, 0};
      while (i < nrows) {
        const uint32_t inext = i + kGroups;
        const YInfo ynext = (inext < nrows) ? (kBlock ? yinfo_block(bv, xs[inext]) : yinfo(desc, xs[inext]))
                                            : YInfo{0, 0, 0, 0, 0};
        const uint32_t na = kUnpruned ? d : nrows - i;
        if (kBlock) {
          cnt += grp_row_block<kCG>(row_kind_block(y, na), bv, bs, y, X, xs + i + 1, na, gl);
        } else {
          const uint8_t kd = kUnpruned ? row_kind_unpruned<kSF>(y, na, X) : row_kind<kSF>(y, na, X);
          cnt += grp_row<kCG, kPiv && !kUnpruned, 8, kAU>(kd, col, bs, y, X, kUnpruned ? xs : xs + i + 1, na, gl);
        }
        i = inext;
        y = ynext;
      }
    };
    // Pruned set-level nest, wide shape (> 2^24 active ids): N+(x) arrives by TMA
    // (1-D cp.async.bulk, mbarrier transaction count) into one of two buffers while
    // the previous x's rows run; thread 0 takes the next work item and issues its
    // copy at the start of each x.  Measured: C5 887 -> 878 ms; on the narrow
    // 4-warp shape it is slower (C3 8.90 -> 9.52 ms: thread 0's dependent loads
    // delay the CTA's next barrier), so that shape keeps plain staged loads.
    __shared__ __align__(8) unsigned long long s_bar[2];
    __shared__ uint4 s_dx[2];
    __shared__ unsigned long long s_wi2[2];
    auto prefetch = [&](int b) {  // thread 0
      const unsigned long long w = atomicAdd(&ctr[cslot], 1ull);
      s_wi2[b] = w;
      if (w < nwork) {
        const uint4 q = __ldg(desc + __ldg(work + w));
        s_dx[b] = q;
        if (q.y <= xcap) {
          const uint32_t bytes = (q.y + 3) / 4 * 16;  // lists are padded to 16 B
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of the buffer
          mbar_arrive_tx(&s_bar[b], bytes);
          bulk_g2s(xs_s + (uint32_t)b * xcap, col + (uint64_t)q.x * 4, bytes, &s_bar[b]);
        } else {
          mbar_arrive(&s_bar[b]);  // unstaged x: complete the phase without a copy
        }
      }
    };
    if (threadIdx.x == 0) {
      mbar_init(&s_bar[0], 1);
      mbar_init(&s_bar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      prefetch(0);
    }
    __syncthreads();
    for (uint32_t it = 0;; ++it) {
      const int cur = it & 1;
      if (s_wi2[cur] >= nwork) break;
      const uint4 dx = s_dx[cur];
      if (threadIdx.x == 0) prefetch(cur ^ 1);
      const uint32_t d = dx.y;
      const uint32_t* xs = col + (uint64_t)dx.x * 4;
      if (d <= xcap) {
        mbar_wait(&s_bar[cur], (it >> 1) & 1u);  // k-th use of a buffer waits on phase parity k & 1
        xs = xs_s + (uint32_t)cur * xcap;
      }
      const XSet X = build_xset(tab, (d <= xcap) ? (uint32_t)kTabW : 0u, xs, d, threadIdx.x, blockDim.x);
      __syncthreads();
      rows(xs, X, d, d - 1, 0u);
      __syncthreads();
    }
    cnt = warp_sum(cnt);
    if (lane == 0 && cnt) atomicAdd(&ctr[0], cnt);
    return;
  }
  for (;;) {
    if (threadIdx.x == 0) s_wi = atomicAdd(&ctr[cslot], 1ull);
    __syncthreads();
    const unsigned long long wi = s_wi;
    if (wi >= nwork) break;
    uint32_t x, r0 = 0, slot = 0xFFFFFFFFu;
    if (kUnpruned) {  // item = (index in the work list << 32) | first row
      const unsigned long long it = __ldg(items + wi);
      const uint32_t k = (uint32_t)(it >> 32);
      x = __ldg(work + k);
      r0 = (uint32_t)it;
      if (hslot) slot = __ldg(hslot + k);
    } else {
      x = __ldg(work + wi);
    }
    const uint4 dx = __ldg(desc + x);
    const uint32_t d = dx.y;
    const uint32_t* xg = col + (uint64_t)dx.x * 4;
    const uint32_t* xs = xg;
    if (d <= xcap) {
      for (uint32_t k = threadIdx.x; k < (d + 3) / 4; k += blockDim.x)
        reinterpret_cast<uint4*>(xs_s)[k] = __ldg(reinterpret_cast<const uint4*>(xg) + k);
      xs = xs_s;
    }
    __syncthreads();
    XSet X;
    if (kUnpruned && slot != 0xFFFFFFFFu) {  // hub: its bitmap over the whole id space, built once, L2-resident
      X.tab = hub_bm + (uint64_t)slot * hub_words;
      X.xs = xs;
      X.mode = kBitmap;
      X.lo = 0;
      X.nbits = hub_words * 32;
      X.hshift = X.hmask = 0;
      X.d = d;
      X.amin = xs[0];
      X.amax = xs[d - 1];
    } else {
      X = build_xset(tab, (d <= xcap) ? (uint32_t)kTabW : 0u, xs, d, threadIdx.x, blockDim.x);
    }
    __syncthreads();
    const uint32_t nrows = kUnpruned ? min(d, r0 + kRowsPerItem) : d - 1;
    uint32_t i = r0 + gid;
    YInfo y = (i < nrows) ? (kBlock ? yinfo_block(bv, xs[i]) : yinfo(desc, xs[i])) : YInfo{0, 0, 0, 0, 0};
    while (i < nrows) {
      const uint32_t inext = i + kGroups;
      const YInfo ynext = (inext < nrows) ? (kBlock ? yinfo_block(bv, xs[inext]) : yinfo(desc, xs[inext]))
                                          : YInfo{0, 0, 0, 0, 0};
      const uint32_t na = kUnpruned ? d : nrows - i;
      if (kBlock) {
        cnt += grp_row_block<kCG>(row_kind_block(y, na), bv, bs, y, X, xs + i + 1, na, gl);
      } else {
        const uint8_t kd = kUnpruned ? row_kind_unpruned<kSF>(y, na, X) : row_kind<kSF>(y, na, X);
        cnt += grp_row<kCG, kPiv && !kUnpruned, 8, kAU>(kd, col, bs, y, X, kUnpruned ? xs : xs + i + 1, na, gl);
      }
      i = inext;
      y = ynext;
    }
    __syncthreads();
  }
  cnt = warp_sum(cnt);
  if (lane == 0 && cnt) atomicAdd(&ctr[0], cnt);
}


// NEXT-2 row-range items: x with d rows becomes ceil(d / kRowsPerItem) items.
__global__ void k_item_count(const uint4* __restrict__ desc, const uint32_t* __restrict__ work, uint64_t n,
                             uint32_t* __restrict__ cnt) {
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x)
    cnt[k] = (desc[work[k]].y + kRowsPerItem - 1) / kRowsPerItem;
}
__global__ void k_item_emit(const uint32_t* __restrict__ work, uint64_t n, const uint32_t* __restrict__ cnt,
                            const uint64_t* __restrict__ off, unsigned long long* __restrict__ items) {
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x)
    for (uint32_t c = 0; c < cnt[k]; ++c) items[off[k] + c] = ((unsigned long long)k << 32) | (c * kRowsPerItem);
}

// NEXT-2 hubs (|N(x)| > xcap): one bitmap of N(x) over the whole id space per hub.
struct HubPred {
  const uint4* desc;
  const uint32_t* work;
  uint32_t xcap;
  __device__ bool operator()(uint64_t k) const { return desc[work[k]].y > xcap; }
};
struct HubEmit {
  uint32_t* hslot;
  uint32_t* hubk;
  __device__ void operator()(uint64_t pos, uint64_t k) const {
    hslot[k] = (uint32_t)pos;
    hubk[pos] = (uint32_t)k;
  }
};
__global__ void k_hub_fill(const uint4* __restrict__ desc, const uint32_t* __restrict__ col,
                           const uint32_t* __restrict__ work, const uint32_t* __restrict__ hubk, uint32_t words,
                           uint32_t* __restrict__ bm) {
  const uint32_t h = blockIdx.x;
  const uint4 d = desc[work[hubk[h]]];
  uint32_t* b = bm + (uint64_t)h * words;
  for (uint32_t k = threadIdx.x; k < d.y; k += blockDim.x) {
    const uint32_t e = col[(uint64_t)d.x * 4 + k];
    atomicOr(&b[e >> 5], 1u << (e & 31));
  }
}

template <int NW, int TABW, int XCAP, bool kUnpruned, bool kBlock, int kMinB = 0, int kCG = kG, uint32_t kSF = 64,
          bool kPiv = false>
void launch_cta(eh_graph* g, uint64_t nsmall, uint64_t nlarge, uint32_t xcap, const uint32_t* work = nullptr,
                cudaStream_t st = nullptr, uint32_t cslot = 2) {
  // work / st / cslot: another work list (default: classes 1-2 of g->work after nsmall
  // entries), stream and work-cursor slot of the count buffer (pruned nests only)
  if (nlarge == 0) return;
  if (!work) work = g->work + nsmall;
  if (XCAP > 0) xcap = XCAP;
  auto k = k_tri_cta<NW, TABW, XCAP, kUnpruned, kBlock, kMinB, kCG, kSF, kPiv>;
  const size_t smem = (size_t)((!kUnpruned && !kBlock && NW == 16 ? 2 : 1) * xcap + TABW) * 4;  // TMA: two buffers
  cudaStream_t s = st ? st : g->stream;
  DBuf<unsigned long long> items;
  DBuf<uint32_t> hslot, hubk, hub_bm;
  uint32_t hub_words = 0;
  uint64_t nitems = nlarge;
  if (kUnpruned) {
    hslot = DBuf<uint32_t>(g->alloc, nlarge);
    hubk = DBuf<uint32_t>(g->alloc, nlarge);
    hub_words = (uint32_t)((g->n_act + 127) / 128 * 4);
    // hubs = lists above the staging capacity, raised until their bitmaps fit the
    // budget; lists above xcap that are not hubs use the global sorted list
    uint64_t hub_min = xcap, nh = 0;
    for (;;) {
      EH_CUDA(cudaMemsetAsync(hslot.p, 0xFF, nlarge * 4, s));
      nh = select_if(nlarge, HubPred{g->desc, work, (uint32_t)std::min<uint64_t>(hub_min, UINT32_MAX)},
                     HubEmit{hslot.p, hubk.p}, g->alloc, s);
      if (nh * hub_words * 4ull <= kHubBitmapBudget || hub_min > g->max_dplus) break;
      hub_min *= 2;
    }
    if (nh * hub_words * 4ull > kHubBitmapBudget) {  // not even the largest lists fit: no hub bitmaps
      EH_CUDA(cudaMemsetAsync(hslot.p, 0xFF, nlarge * 4, s));
      nh = 0;
    }
    if (nh) {
      hub_bm = DBuf<uint32_t>(g->alloc, nh * hub_words);
      EH_CUDA(cudaMemsetAsync(hub_bm.p, 0, hub_bm.bytes(), s));
      k_hub_fill<<<(unsigned)nh, 1024, 0, s>>>(g->desc, g->col, work, hubk.p, hub_words, hub_bm.p);
      EH_LAUNCH("k_hub_fill");
    }
    DBuf<uint32_t> cnt(g->alloc, nlarge);
    DBuf<uint64_t> off(g->alloc, nlarge + 1), tot(g->alloc, 1);
    k_item_count<<<grid_for(nlarge, 1024), 256, 0, s>>>(g->desc, work, nlarge, cnt.p);
    EH_LAUNCH("k_item_count");
    scan_exclusive_u32(cnt.p, off.p, nlarge, tot.p, g->alloc, s);
    nitems = read_scalar(tot.p, s);
    items = DBuf<unsigned long long>(g->alloc, nitems);
    k_item_emit<<<grid_for(nlarge, 1024), 256, 0, s>>>(work, nlarge, cnt.p, off.p, items.p);
    EH_LAUNCH("k_item_emit");
  }
  ensure_dyn_smem((const void*)k, smem);
  int per_sm = 0;
  EH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, NW * 32, smem));
  const unsigned grid = (unsigned)std::min<uint64_t>(nitems, (uint64_t)kSMs * std::max(1, per_sm));
  k<<<grid, NW * 32, smem, s>>>(g->desc, g->col, g->bs, work, nitems, g->d_counter, xcap, items.p,
                                kUnpruned ? hslot.p : nullptr, hub_bm.p, hub_words,
                                BlockView{g->bdesc, g->bcol, g->bcid, g->bmask}, cslot);
  EH_LAUNCH("k_tri_cta");
  if (kUnpruned) EH_CUDA(cudaStreamSynchronize(s));  // items is released on return
}


template <bool kUnpruned, bool kBlock, int kMaxD, int kMinB, int kWG = kG, uint32_t kSF = 64, bool kPiv = false>
void launch_warp(eh_graph* g, uint64_t nsmall, const uint32_t* work = nullptr, uint32_t cslot = 1,
                 cudaStream_t st = nullptr) {
  if (!st) st = g->stream;
  if (nsmall == 0) return;
  if (!work) work = g->work;
  auto k = k_tri_warp<kUnpruned, kBlock, kMaxD, kMinB, kWG, kSF, kPiv>;
  const size_t smem = sizeof(WarpSmem<kMaxD>) * kWK_Warps;
  ensure_dyn_smem((const void*)k, smem);
  int per_sm = 0;
  EH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kWK_Warps * 32, smem));
  const unsigned grid = (unsigned)std::min<uint64_t>((nsmall + kWK_Warps - 1) / kWK_Warps,
                                                     (uint64_t)kSMs * std::max(1, per_sm));
  k<<<grid, kWK_Warps * 32, smem, st>>>(g->desc, g->col, g->bs, work, nsmall, g->d_counter,
                                               BlockView{g->bdesc, g->bcol, g->bcid, g->bmask}, cslot);
  EH_LAUNCH("k_tri_warp");
}

#ifndef EH_MID_NW
#define EH_MID_NW 4
#endif
#ifndef EH_MID_CG
#define EH_MID_CG kG
#endif
#ifndef EH_MID_TABW
#define EH_MID_TABW 2048
#endif
// wide shape: class-2 x with |N+(x)| <= kMidMax (0 / 1 of the 2-way split)
constexpr uint32_t kMidMax = 512;  // the 4-warp CTA's 2048-word table holds filter + hash up to 512 elements
struct MidClass {
  const uint4* desc;
  const uint32_t* w;
  uint32_t mid;
  __device__ int operator()(uint64_t i) const { return desc[w[i]].y <= mid ? 0 : 1; }
};
struct MidEmit {
  const uint32_t* w;
  uint32_t* out;
  __device__ void operator()(int, uint64_t pos, uint64_t i) const { out[pos] = w[i]; }
};

template <bool kUnpruned, bool kBlock>
uint64_t count_impl(eh_graph* g) {
  cudaStream_t s = g->stream;
  EH_CUDA(cudaMemsetAsync(g->d_counter, 0, 8 * sizeof(unsigned long long), s));
  // narrow shape: class 0 -> warp kernel, classes 1-2 -> CTA kernel; wide: classes 0-1 -> warp
  // the symmetric trie's hub lists always take the wide shape (measured: C3 2.70 -> 1.27 s)
  // test hook EH_TEST_TRI_WIDE: the wide (> 2^24 ids) kernels on any graph, so the tests
  // reach their TMA staging (and, with EH_TEST_TRI_XCAP, its unstaged branch)
  const bool wide = g->n_act > kWideIds || kUnpruned || getenv("EH_TEST_TRI_WIDE") != nullptr;
  const uint64_t nsmall = g->n_work[0] + (wide ? g->n_work[1] : 0);
  const uint64_t nlarge = g->n_work[2] + (wide ? 0 : g->n_work[1]);
  // The thread- and warp-class kernels run on a side stream beside the CTA-class
  // kernel (they share only the count, an atomic), so the tail of one overlaps the
  // other; test hook EH_TEST_TRI_SERIAL keeps one stream.
  const cudaStream_t ss = (nlarge && nsmall && getenv("EH_TEST_TRI_SERIAL") == nullptr) ? fork_side(g, 0) : s;
  // a7 thread class (the head of class 0; pruned set-level nest only)
  const uint64_t nt = (!kUnpruned && !kBlock) ? g->n_thread : 0;
  launch_thread(g, nt, ss);
  if (nsmall > nt) {
    // staging sized for class 0 (|N+(x)| <= 64 by default): 30 KB instead of 43 KB
    // per 8-warp CTA, one more CTA per SM (measured: C3 9.48 -> 9.41 ms)
    // SEARCH rows start inside one of 8 pivot slices on the larger graphs (> 2^20 active
    // ids; measured C3 9.15 -> 8.92 ms, C5 900 -> 887; slower on C2 / C4)
    const bool big = g->n_act > (1ull << 20);
    // min 6 CTAs per SM: 40 registers (a few spilled bytes) for one more resident CTA
    // (measured C3 8.59 -> 8.38 ms, C4 1.458 -> 1.419, C2 0.316 -> 0.313)
    const uint32_t* w0 = g->work + nt;
    const uint64_t n0 = nsmall - nt;
    // rows on 4-lane groups below 2^20 active ids (8 rows in flight per warp; measured
    // C4 1.264 -> 1.251, C2 0.270 -> 0.268 ms; above, with the pivot searches, C3 7.87 -> 8.07)
    if (!wide && g->class0_max <= 64 && big) launch_warp<kUnpruned, kBlock, 64, 6, kG, 16, true>(g, n0, w0, 1u, ss);
    else if (!wide && g->class0_max <= 64) launch_warp<kUnpruned, kBlock, 64, 6, 4, 16>(g, n0, w0, 1u, ss);
    else if (!wide) launch_warp<kUnpruned, kBlock, kWarpMaxD, 0, kG, 16>(g, n0, w0, 1u, ss);
    else if (kUnpruned && g->n_act <= kWideIds) launch_warp<kUnpruned, kBlock, kWarpMaxD, 0, kG, 16, true>(g, n0, w0, 1u, ss);
    else if (!kUnpruned && !kBlock && g->class0_max <= 64) {  // wide: class 0 with 64-entry staging, min 6 CTAs/SM
      launch_warp<kUnpruned, kBlock, 64, 6, kG, 64, true>(g, g->n_work[0] - nt, w0, 1u, ss);
      launch_warp<kUnpruned, kBlock, kWarpMaxD, 0, kG, 64, true>(g, nsmall - g->n_work[0], g->work + g->n_work[0], 6u, ss);
    } else launch_warp<kUnpruned, kBlock, kWarpMaxD, 0, kG, 64, true>(g, n0, w0, 1u, ss);
  }
  DBuf<uint32_t> split;  // wide shape: class 2 as (mid x, big x)
  // test hook EH_TEST_TRI_MID: the mid / big boundary (0 = no mid class)
  uint32_t mid_max = kMidMax;
  if (const char* e = getenv("EH_TEST_TRI_MID")) mid_max = (uint32_t)atoi(e);
  if (nlarge) {
    // unpruned: lists above 4096 use the global hub bitmaps (measured: C3 0.93 -> 0.42 s)
    const uint64_t cap = kUnpruned ? 4096 : wide ? kCtaXCapMax : kCtaXCapNarrow;
    uint32_t xcap = (uint32_t)std::min<uint64_t>(cap, std::max<uint64_t>(256, (g->max_dplus + 255) / 256 * 256));
    if (const char* e = getenv("EH_TEST_TRI_XCAP")) xcap = (uint32_t)std::max(128, atoi(e));  // test hook: unstaged path
    // the unpruned nest takes the wide shapes on every graph; its SEARCH factor still
    // follows the graph size (L2-resident lists: C3 unpruned 415.6 -> 386.9 ms)
    if (kUnpruned && g->n_act <= kWideIds && xcap <= 4096) {
      // the same mid / big split as the pruned wide shape below (the launches run one after
      // the other: an unpruned launch ends with a stream synchronisation)
      uint64_t nmid = 0;
      // (measured: C3 unpruned 6T 438.6 -> 424.3 ms, -R 624.8 -> 579.7; C4 / C2 unchanged)
      if (!kBlock && mid_max >= tri_warp_max_degree() + 1) {
        split = DBuf<uint32_t>(g->alloc, nlarge);
        uint64_t st2[3];
        partition_k<2>(nlarge, MidClass{g->desc, g->work + nsmall, mid_max}, MidEmit{g->work + nsmall, split.p}, st2,
                       g->alloc, s);
        nmid = st2[1] - st2[0];
      }
      launch_cta<16, 16384, 4096, kUnpruned, kBlock, 0, kG, 16, true>(g, nsmall, nlarge - nmid, 0,
                                                                    nmid ? split.p + nmid : nullptr);
      if (nmid)
        launch_cta<4, 2048, 0, kUnpruned, kBlock, 0, kG, 16, true>(g, nsmall, nmid, (mid_max + 255) / 256 * 256, split.p,
                                                                  nullptr, 3u);
    } else if (wide && xcap <= 4096 && !getenv("EH_TEST_TRI_XCAP")) {
      // Wide shape, pruned set-level nest: the x with |N+(x)| <= kMidMax take the 4-warp
      // CTAs (8 KB table: one-hash filter + hash table, many CTAs per SM, so the per-x
      // barrier tails overlap), the rest the 16-warp CTAs with the 64 KB table.  The class
      // list is split per call (one stable 2-way partition of its entries).
      uint64_t nmid = 0;
      if (!kUnpruned && !kBlock && mid_max >= tri_warp_max_degree() + 1) {
        split = DBuf<uint32_t>(g->alloc, nlarge);
        uint64_t st2[3];
        partition_k<2>(nlarge, MidClass{g->desc, g->work + nsmall, mid_max}, MidEmit{g->work + nsmall, split.p}, st2,
                       g->alloc, s);
        nmid = st2[1] - st2[0];
      }
      const uint32_t* wbig = nmid ? split.p + nmid : nullptr;
      launch_cta<16, 16384, 4096, kUnpruned, kBlock, 0, kG, 64, true>(g, nsmall, nlarge - nmid, 0, wbig);
      if (nmid) {
        const cudaStream_t sm = (nlarge > nmid && getenv("EH_TEST_TRI_SERIAL") == nullptr) ? fork_side(g, 1) : s;
        launch_cta<EH_MID_NW, EH_MID_TABW, 0, kUnpruned, kBlock, 0, EH_MID_CG, 64, true>(g, nsmall, nmid, (mid_max + 255) / 256 * 256, split.p, sm,
                                                                   3u);
        if (sm != s) join_side(g, 1);
      }
    }
    else if (wide) launch_cta<16, 16384, 0, kUnpruned, kBlock, 0, kG, 64, true>(g, nsmall, nlarge, xcap);
    // rows on 4-lane groups (32 rows in flight per CTA) below 2^20 active ids, 8-lane
    // groups above (measured: C2 0.348 -> 0.325, C4 1.556 -> 1.508, C3 9.42 -> 9.46 ms)
    else if (g->n_act <= (1ull << 20)) launch_cta<4, 2048, 0, kUnpruned, kBlock, 0, 4, 16>(g, nsmall, nlarge, xcap);
    else launch_cta<4, 2048, 0, kUnpruned, kBlock, 0, kG, 16, true>(g, nsmall, nlarge, xcap);
  }
  if (ss != s) join_side(g, 0);
  EH_CUDA(cudaMemcpyAsync(g->h_counter, g->d_counter, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaStreamSynchronize(s));
  return g->h_counter[0];
}

}  // namespace

uint64_t count_triangles(eh_graph* g) {
  return g->bdesc ? count_impl<false, true>(g) : count_impl<false, false>(g);  // NEXT-3 block layout if built
}

// NEXT-2: the unpruned nest over the symmetric trie (built on first use) = 6T.
uint64_t count_triangles_unpruned(eh_graph* g) { return count_impl<true, false>(symmetric_trie(g)); }

uint32_t tri_warp_max_degree() { return kWarpMaxD; }
uint32_t tri_thread_max_degree() { return kTMax; }

}  // namespace eh
