// dedup.cu -- SURVEY.md §8(a) rows a1-a4 as one bucketed pass: canonical keys,
// distinct undirected edges and the degree of every id, without a full key sort.
//
//  PAPER.md:284      values "grouped into sets of distinct values based on their
//                    parent attribute" -- the trie needs each distinct edge once,
//                    grouped by its low end; a total order of the edge keys is not
//                    needed (the CSR's lists are ordered later, per list, by the
//                    segmented sort of segsort.cu).
//  PAPER.md:799-800  symmetric pruning needs the degree of every id first.
//  Readings: c4 degree = distinct neighbours, c5 self-loops dropped,
//  c6 dedup, c7 (u,v) == (v,u).
//
// Design (DESIGN.md §6 "ingest"): the canonical key of a pair is (lo, hi) =
// (min, max) over b-bit ids.  Its bucket is lo's top bb bits (an MSD radix digit),
// its residual r = (lo's low b - bb bits) << b | hi fits 31 bits, so a bucket holds
// all pairs of 2^(b - bb) consecutive lo values.
//   (1) k_bkt_hist: bucket histogram in shared memory (one read of src / dst), kept
//       per (chunk of the input, CTA);
//   (2) k_bkt_colscan + exclusive scan -> bucket offsets and every (chunk, CTA)'s own
//       range inside each bucket;
//   (3) k_bkt_part_smem: every non-loop pair's residual scattered into its bucket with
//       shared-memory cursors -- no global atomics (one read of src / dst, one 4-B
//       write; order within a bucket arbitrary).  Above 2^15 buckets (id spaces beyond
//       ~2^23 ids) the histogram and the cursors are global atomics (k_bkt_part_direct);
//   (4) k_bkt_dedup: one CTA per bucket inserts the residuals into an on-chip
//       open-addressing hash set (shared memory; buckets too large for it use a
//       table in global memory), counts each id's distinct neighbours (lo side in
//       shared memory, hi side with global atomics), and writes the bucket's
//       distinct keys (lo << b) | hi contiguously, grouped by lo.
// The output is the compact array of the m distinct keys; k_scatter_col and the
// orderings consume it like the sorted keys of the radix path (ingest.cu).
#include "eh_internal.cuh"
#include "primitives.cuh"

#include <algorithm>

namespace eh {

namespace {

constexpr uint32_t kEmptyR = 0xFFFFFFFFu;  // residuals have <= 31 bits
constexpr int kMaxLoBits = 12;             // <= 4096 lo values per bucket (shared-memory counters)
constexpr int kHistSmemBits = 15;          // shared-memory histogram up to 2^15 buckets (128 KB, one CTA per SM)
constexpr int kSmallThreads = 512;
constexpr uint32_t kSmallSlots = 16384;    // 64 KB table: buckets of <= kSmallMax pairs
constexpr uint32_t kSmallMax = 8192;
constexpr int kBigThreads = 1024;
constexpr uint32_t kBigSlots = 52224;      // 204 KB table (1 CTA / SM): buckets of <= kBigMax pairs
constexpr uint32_t kBigMax = 36000;
constexpr int kGiantThreads = 1024;

struct BktParams {
  uint32_t b;       // id bits
  uint32_t lobits;  // b - bb: lo bits inside a bucket
};

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7FEB352Du;
  x ^= x >> 15; x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}

// row pitch of the per-(chunk, CTA) histograms: one 128-B line past the power of two (rows at
// exactly 64 KB apart made k_bkt_colscan's strided reads 4.6x slower: 437 vs 95 us at C3)
__host__ __device__ __forceinline__ uint64_t pitch(uint32_t nb) { return (uint64_t)nb + 32; }

// pair -> (bucket, residual); false for a self-loop (dropped, reading c5)
__device__ __forceinline__ bool pair_bucket(uint32_t u, uint32_t v, const BktParams& p, uint32_t& bk, uint32_t& r) {
  if (u == v) return false;
  const uint32_t lo = min(u, v), hi = max(u, v);
  bk = lo >> p.lobits;
  r = ((lo & ((1u << p.lobits) - 1u)) << p.b) | hi;
  return true;
}

// f(u, v, ok) over the pairs [p0, p1) (p0 a multiple of 4), grid-stride, 128-bit loads when
// the inputs are 16-B aligned; every lane of a warp runs the same number of rounds (f may use
// warp collectives)
template <class F>
__device__ __forceinline__ void for_pairs_range(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                                                uint64_t p0, uint64_t p1, F f) {
  const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  uint64_t done = p0;
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {  // 128-bit loads
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    const uint4* d4 = reinterpret_cast<const uint4*>(dst);
    const uint64_t v1 = p1 / 4;
    // the next round's loads are issued before this round's pairs are processed
    uint64_t i = p0 / 4 + t0;
    bool ok = i < v1;
    uint4 a = ok ? __ldcs(s4 + i) : make_uint4(0, 0, 0, 0), c = ok ? __ldcs(d4 + i) : make_uint4(0, 0, 0, 0);
    for (uint64_t i0 = p0 / 4 + t0 - (threadIdx.x & 31); i0 < v1; i0 += nt) {
      const uint64_t in = i + nt;
      const bool okn = in < v1;
      const uint4 an = okn ? __ldcs(s4 + in) : make_uint4(0, 0, 0, 0), cn = okn ? __ldcs(d4 + in) : make_uint4(0, 0, 0, 0);
      f(a.x, c.x, ok); f(a.y, c.y, ok); f(a.z, c.z, ok); f(a.w, c.w, ok);
      i = in; ok = okn; a = an; c = cn;
    }
    done = v1 * 4;
  }
  for (uint64_t i0 = done + t0 - (threadIdx.x & 31); i0 < p1; i0 += nt) {
    const uint64_t i = i0 + (threadIdx.x & 31);
    const bool ok = i < p1;
    f(ok ? src[i] : 0u, ok ? dst[i] : 0u, ok);
  }
}
template <class F>
__device__ __forceinline__ void for_pairs(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                                          uint64_t n, F f) {
  for_pairs_range(src, dst, 0, n, f);
}

// (1) bucket histogram; kSmem: per-CTA shared-memory counters, else warp-aggregated global atomics.
// percta (kSmem only): the input is taken in chunks of `per` pairs and this CTA's own
// histogram of chunk c goes to percta[(c * gridDim.x + blockIdx.x) * nb + .] instead of cnt
// (k_bkt_colscan sums them and turns the entries into the cursors of k_bkt_part_smem).
template <bool kSmem>
__global__ void __launch_bounds__(1024) k_bkt_hist(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                                                  uint64_t n, BktParams p, uint32_t nb, uint32_t* __restrict__ cnt,
                                                  uint32_t* __restrict__ percta, uint64_t per) {
  extern __shared__ uint32_t sh_hist[];
  const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
  if (!percta) per = n;
  uint32_t chunk = 0;
  for (uint64_t p0 = 0; p0 < n || p0 == 0; p0 += per, ++chunk) {
    if (kSmem) {
      for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) sh_hist[i] = 0;
      __syncthreads();
    }
    for_pairs_range(src, dst, p0, min(n, p0 + per), [&](uint32_t u, uint32_t v, bool ok) {
      uint32_t bk = 0xFFFFFFFFu, r;
      if (!(ok && pair_bucket(u, v, p, bk, r))) bk = 0xFFFFFFFFu;
      if (kSmem) {
        if (bk != 0xFFFFFFFFu) atomicAdd(&sh_hist[bk], 1u);
      } else {
        const unsigned peers = __match_any_sync(kFull, bk);
        if (bk != 0xFFFFFFFFu && (peers & lt) == 0) atomicAdd(&cnt[bk], (uint32_t)__popc(peers));
      }
    });
    if (kSmem) {
      __syncthreads();
      uint32_t* mine = percta ? percta + ((uint64_t)chunk * gridDim.x + blockIdx.x) * pitch(nb) : nullptr;
      for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) {
        const uint32_t c = sh_hist[i];
        if (mine) mine[i] = c;
        else if (c) atomicAdd(&cnt[i], c);
      }
      __syncthreads();
    }
    if (per == 0) break;
  }
}

// (2') per-(chunk, CTA) histograms -> exclusive offsets inside each bucket (in part order),
// and the bucket totals.  One CTA per kCsB buckets: thread (bx, seg) owns a contiguous segment
// of the parts of bucket blockIdx.x * kCsB + bx (loads coalesced over bx, independent over
// the segment), the kCsS segment sums are scanned in shared memory, a second pass writes the
// offsets.  (64 segments of 16 buckets: with 32 x 32 the 84 dependent rounds per thread of a
// 2664-part scan took 437 us at C3 with 2^14 buckets.)
constexpr uint32_t kCsB = 16, kCsS = 64;
__global__ void __launch_bounds__(kCsB * kCsS) k_bkt_colscan(uint32_t* __restrict__ percta, uint32_t nparts, uint32_t nb,
                                                            uint32_t* __restrict__ cnt) {
  __shared__ uint32_t seg_sum[kCsS][kCsB + 1];
  const uint32_t bx = threadIdx.x % kCsB, seg = threadIdx.x / kCsB;
  const uint32_t b = blockIdx.x * kCsB + bx;
  const uint32_t per = (nparts + kCsS - 1) / kCsS;
  const uint64_t ld = pitch(nb);
  const uint32_t c0 = min(nparts, seg * per), c1 = min(nparts, c0 + per);
  uint32_t sum = 0;
  if (b < nb) {
#pragma unroll 8
    for (uint32_t c = c0; c < c1; ++c) sum += percta[(uint64_t)c * ld + b];
  }
  seg_sum[seg][bx] = sum;
  __syncthreads();
  if (seg == 0) {  // lane bx scans the segment sums of its bucket
    uint32_t run = 0;
    for (uint32_t q = 0; q < kCsS; ++q) {
      const uint32_t v = seg_sum[q][bx];
      seg_sum[q][bx] = run;
      run += v;
    }
    if (b < nb) cnt[b] = run;
  }
  __syncthreads();
  if (b < nb) {
    uint32_t run = seg_sum[seg][bx];
#pragma unroll 8
    for (uint32_t c = c0; c < c1; ++c) {
      const uint32_t v = percta[(uint64_t)c * ld + b];
      percta[(uint64_t)c * ld + b] = run;
      run += v;
    }
  }
}

// (3'') residuals into their buckets without global atomics: the same grid, chunks and pair
// assignment as k_bkt_hist<true>, whose per-(chunk, CTA) counts (k_bkt_colscan) give every
// CTA its own range inside each bucket for each chunk; the cursors live in shared memory.
// (The global cursor atomics of k_bkt_part_direct ran at ~60 G atomics/s, 69 % of its stall
// samples waiting on their results: C3 1.16 ms for 0.8 GB of traffic.)  A bucket's range is
// laid out chunk-major, so the sectors written during one chunk (all CTAs advance through
// the chunks together) add up to the chunk's own output -- sized to stay in L2 until the
// sectors are complete (unchunked, C3's 4.8 M runs of ~14 entries were evicted half-written:
// 1.97 ms).
__global__ void __launch_bounds__(1024) k_bkt_part_smem(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                                                       uint64_t n, BktParams p, uint32_t nb,
                                                       const uint64_t* __restrict__ boff,
                                                       const uint32_t* __restrict__ percta, uint64_t per,
                                                       uint32_t* __restrict__ part) {
  extern __shared__ uint32_t sh_cur[];
  uint32_t chunk = 0;
  for (uint64_t p0 = 0; p0 < n; p0 += per, ++chunk) {
    const uint32_t* mine = percta + ((uint64_t)chunk * gridDim.x + blockIdx.x) * pitch(nb);
#pragma unroll 8
    for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) sh_cur[i] = (uint32_t)boff[i] + mine[i];
    __syncthreads();
    for_pairs_range(src, dst, p0, min(n, p0 + per), [&](uint32_t u, uint32_t v, bool ok) {
      uint32_t bk, r;
      if (ok && pair_bucket(u, v, p, bk, r)) {
        const uint32_t q = atomicAdd(&sh_cur[bk], 1u);
        EH_DASSERT(q >= boff[bk] && q < boff[bk + 1]);
        part[q] = r;
      }
    });
    __syncthreads();
  }
}

// (3) residuals into their buckets (one cursor atomic per group of equal buckets in the warp)
__global__ void __launch_bounds__(256) k_bkt_part(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                                                  uint64_t n, BktParams p, const uint64_t* __restrict__ boff,
                                                  uint32_t* __restrict__ cur, uint32_t* __restrict__ part) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for_pairs(src, dst, n, [&](uint32_t u, uint32_t v, bool ok) {
    uint32_t bk = 0xFFFFFFFFu, r = 0;
    if (!(ok && pair_bucket(u, v, p, bk, r))) bk = 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(kFull, bk);
    const int leader = __ffs(peers) - 1;
    uint32_t p0 = 0;
    if (bk != 0xFFFFFFFFu && lane == leader) p0 = atomicAdd(&cur[bk], (uint32_t)__popc(peers));
    p0 = __shfl_sync(kFull, p0, leader);
    if (bk != 0xFFFFFFFFu) {
      EH_DASSERT(boff[bk] + p0 + __popc(peers & lt) < boff[bk + 1]);
      part[boff[bk] + p0 + __popc(peers & lt)] = r;
    }
  });
}

// (3') the same without warp aggregation: with >= 2^13 buckets a warp's 32 pairs
// rarely share one, so the match costs more than the atomics it saves; the four
// pairs of a 128-bit load issue their cursor atomics back to back; cur[] starts at the
// buckets' absolute offsets (k_bkt_cursors)
__global__ void __launch_bounds__(256) k_bkt_part_direct(const uint32_t* __restrict__ src,
                                                         const uint32_t* __restrict__ dst, uint64_t n, BktParams p,
                                                         const uint64_t* __restrict__ boff, uint32_t* __restrict__ cur,
                                                         uint32_t* __restrict__ part) {
  const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  uint64_t done = 0;
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    const uint4* d4 = reinterpret_cast<const uint4*>(dst);
    const uint64_t n4 = n / 4;
    for (uint64_t i = t0; i < n4; i += nt) {
      const uint4 a = __ldcs(s4 + i), c = __ldcs(d4 + i);
      const uint32_t u[4] = {a.x, a.y, a.z, a.w}, v[4] = {c.x, c.y, c.z, c.w};
      uint32_t bk[4], r[4], q[4];
      bool ok[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) ok[k] = pair_bucket(u[k], v[k], p, bk[k], r[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k) q[k] = ok[k] ? atomicAdd(&cur[bk[k]], 1u) : 0u;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (ok[k]) {
          EH_DASSERT(q[k] >= boff[bk[k]] && q[k] < boff[bk[k] + 1]);
          part[q[k]] = r[k];
        }
    }
    done = n4 * 4;
  }
  for (uint64_t i = done + t0; i < n; i += nt) {
    uint32_t bk, r;
    if (pair_bucket(src[i], dst[i], p, bk, r)) part[atomicAdd(&cur[bk], 1u)] = r;
  }
}

// cursors of k_bkt_part_direct: absolute positions (n < 2^32), so the scatter needs no offset load
__global__ void k_bkt_cursors(const uint64_t* __restrict__ boff, uint32_t nb, uint32_t* __restrict__ cur) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nb; k += gridDim.x * blockDim.x) cur[k] = (uint32_t)boff[k];
}

// (4a) bucket classes by size: 0 shared-memory table (small CTA), 1 shared-memory
// table (big CTA), 2 global table (slots = 2 * pairs, carved from one scratch buffer)
__global__ void k_bkt_classify(const uint64_t* __restrict__ boff, uint32_t nb, uint32_t* __restrict__ lists,
                               unsigned long long* __restrict__ info, uint64_t* __restrict__ gtab) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (uint32_t k0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); k0 < nb; k0 += gridDim.x * blockDim.x) {
    const uint32_t k = k0 + lane;
    const uint64_t c = k < nb ? boff[k + 1] - boff[k] : 0;
    const int cls = c == 0 ? -1 : (c <= kSmallMax ? 0 : (c <= kBigMax ? 1 : 2));
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const unsigned bal = __ballot_sync(kFull, cls == q);
      if (!bal) continue;
      uint32_t base = 0;
      if (lane == __ffs(bal) - 1) base = (uint32_t)atomicAdd(&info[q], (unsigned long long)__popc(bal));
      base = __shfl_sync(kFull, base, __ffs(bal) - 1);
      if (cls == q) lists[(uint64_t)q * nb + base + __popc(bal & lt)] = k;
    }
    if (cls == 2) gtab[k] = atomicAdd(&info[3], (unsigned long long)(2 * c));
  }
}

// (4b) per bucket: insert, count, emit.  kMode 0 / 1: table in shared memory
// (kSlots entries), 2: table in global memory at gscr + gtab[bucket].
template <int kThreads, int kMode, uint32_t kSlots>
__global__ void __launch_bounds__(kThreads) k_bkt_dedup(const uint32_t* __restrict__ part,
                                                        const uint64_t* __restrict__ boff,
                                                        const uint32_t* __restrict__ list,
                                                        const unsigned long long* __restrict__ info, int cls,
                                                        BktParams p, uint32_t* __restrict__ deg,
                                                        unsigned long long* __restrict__ m_ctr,
                                                        uint64_t* __restrict__ out, uint32_t* __restrict__ gscr,
                                                        const uint64_t* __restrict__ gtab) {
  // dynamic shared memory: [table: kSlots (modes 0 / 1)] [lcnt: 2^lobits]; lcnt[l] = the
  // distinct neighbours above lo0 + l in this bucket, then its emit cursor
  extern __shared__ __align__(16) uint32_t dsm_dedup[];
  __shared__ uint32_t sw[kThreads / 32 + 1];
  __shared__ unsigned long long s_base;
  const uint32_t nlo = 1u << p.lobits;
  uint32_t* lcnt = dsm_dedup + (kMode == 2 ? 0u : kSlots);
  const uint32_t hmask = (p.b >= 32) ? 0xFFFFFFFFu : ((1u << p.b) - 1u);
  const uint64_t nl = info[cls];
  for (uint64_t w = blockIdx.x; w < nl; w += gridDim.x) {
    const uint32_t bk = list[w];
    const uint64_t beg = boff[bk];
    const uint32_t c = (uint32_t)(boff[bk + 1] - beg);
    uint32_t* tab;
    uint32_t ts;
    if (kMode == 2) {
      tab = gscr + gtab[bk];
      ts = 2 * c;
    } else {
      tab = dsm_dedup;
      ts = (kMode == 0) ? min(kSlots, max(64u, 2u * c)) : kSlots;
    }
    for (uint32_t i = threadIdx.x; i < ts; i += kThreads) tab[i] = kEmptyR;
    for (uint32_t i = threadIdx.x; i < nlo; i += kThreads) lcnt[i] = 0;
    __syncthreads();
    // insert: read before CAS, so duplicates of a key already present cost no atomic
    for (uint32_t i = threadIdx.x; i < c; i += kThreads) {
      const uint32_t r = __ldcs(part + beg + i);
      uint32_t h = (uint32_t)(((uint64_t)mix32(r) * ts) >> 32);
      for (;;) {
        uint32_t cur = kMode == 2 ? __ldcg(tab + h) : tab[h];
        if (cur == r) break;
        if (cur == kEmptyR) {
          cur = atomicCAS(tab + h, kEmptyR, r);
          if (cur == kEmptyR) { atomicAdd(&lcnt[r >> p.b], 1u); break; }
          if (cur == r) break;
        }
        h = (h + 1 == ts) ? 0 : h + 1;
      }
    }
    __syncthreads();
    // lo side of the degrees; exclusive scan of the per-lo counts -> emit cursors
    const uint32_t lo0 = bk << p.lobits;
    const uint32_t per = (nlo + kThreads - 1) / kThreads;  // consecutive lo values per thread
    const uint32_t a0 = min(nlo, threadIdx.x * per), a1 = min(nlo, a0 + per);
    uint32_t s = 0;
    for (uint32_t l = a0; l < a1; ++l) {
      const uint32_t v = lcnt[l];
      if (v) atomicAdd(&deg[lo0 + l], v);
      s += v;
    }
    uint32_t tot;
    uint32_t ex = block_exclusive_scan<kThreads>(s, sw, &tot);
    for (uint32_t l = a0; l < a1; ++l) {
      const uint32_t v = lcnt[l];
      lcnt[l] = ex;
      ex += v;
    }
    if (threadIdx.x == 0) s_base = atomicAdd(m_ctr, (unsigned long long)tot);
    __syncthreads();
    const uint64_t obase = s_base;
    for (uint32_t i = threadIdx.x; i < ts; i += kThreads) {
      const uint32_t r = kMode == 2 ? __ldcg(tab + i) : tab[i];
      if (r == kEmptyR) continue;
      const uint32_t l = r >> p.b, hi = r & hmask;
      const uint32_t q = atomicAdd(&lcnt[l], 1u);
      out[obase + q] = ((uint64_t)(lo0 + l) << p.b) | hi;
      atomicAdd(&deg[hi], 1u);
    }
    __syncthreads();  // the table and lcnt are reused by the next bucket
  }
}

template <int kThreads, int kMode, uint32_t kSlots>
void launch_dedup(uint64_t nlist, size_t smem, const uint32_t* part, const uint64_t* boff, const uint32_t* list,
                  const unsigned long long* info, int cls, BktParams p, uint32_t* deg, unsigned long long* m_ctr,
                  uint64_t* out, uint32_t* gscr, const uint64_t* gtab, cudaStream_t s) {
  if (nlist == 0) return;
  auto k = k_bkt_dedup<kThreads, kMode, kSlots>;
  ensure_dyn_smem((const void*)k, smem);
  int per_sm = 1;
  EH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, smem));
  const uint64_t grid = std::min<uint64_t>(nlist, (uint64_t)kSMs * std::max(1, per_sm));
  k<<<(unsigned)grid, kThreads, smem, s>>>(part, boff, list, info, cls, p, deg, m_ctr, out, gscr, gtab);
  EH_LAUNCH("k_bkt_dedup");
}

}  // namespace

// Bucket geometry for b-bit ids and n pairs; false when the residual cannot fit
// 31 bits with a bucket of <= 2^kMaxLoBits lo values (b >= 32: radix path).
bool bucket_dedup_ok(uint32_t b, uint64_t n) {
  return b < 32 && n > 0 && n < (1ull << 32);
}

// a1-a4: distinct canonical keys into `out` (compact, m entries, grouped by bucket
// and lo), deg[id] += distinct neighbours (deg zeroed by the caller), *m_ctr += m.
void bucket_dedup(const uint32_t* src, const uint32_t* dst, uint64_t n, uint32_t b, uint32_t* deg,
                  unsigned long long* m_ctr, uint64_t* out, eh_graph* g, PhaseTimer* tm) {
  Allocator& al = g->alloc;
  cudaStream_t s = g->stream;
  // bb bucket bits: residual <= 31 bits, <= 2^12 lo values per bucket, 4096 - 8192 pairs per bucket
  // on average (measured with the shared-memory partition, EH_TEST_BKT_SHIFT -2 / -1 / 0 / 1 around
  // n >> 12: C3 4.89 / 5.00 / 5.10 / -, C4 1.54 / 1.45 / 1.47 / 1.58, C2 0.670 / 0.676 / 0.688 / 0.710 ms)
  int bb = std::max<int>(2 * (int)b - 31, (int)b - kMaxLoBits);
  bb = std::max<int>(bb, (int)bitlen(n >> 13));
  // chunks of `per` pairs (a multiple of 4) whose residuals (4 B each) fit 32 MB of L2 (test hook
  // EH_TEST_BKT_CHUNK_MB; measured at C3, 8 / 16 / 32 / 64 MB / one chunk: load 8.61 / 5.81 / 5.08 /
  // 5.07 / 5.94 ms)
  uint64_t chunk_mb = 32;
  if (const char* e = getenv("EH_TEST_BKT_CHUNK_MB")) chunk_mb = std::max(1, atoi(e));
  const uint64_t nchunks = std::max<uint64_t>(1, (n * 4 + (chunk_mb << 20) - 1) / (chunk_mb << 20));
  const uint64_t per = ((n + nchunks - 1) / nchunks + 3) / 4 * 4;
  // the per-(chunk, CTA) histograms are read twice by the column scan: keep them L2-sized
  // (C3: 2^14 buckets 175 MB, scan 0.40 ms; 2^13 buckets 87 MB, 0.10 ms)
  // -- first one CTA per SM instead of two (the partition is no faster with two), then fewer buckets
  unsigned cta_per_sm = 2;
  auto hist_bytes = [&](int bits, unsigned k) { return ((n + per - 1) / per) * ((uint64_t)k * kSMs) * (4ull << bits); };
  if (bb <= kHistSmemBits && hist_bytes(bb, 2) > (96ull << 20)) cta_per_sm = 1;
  while (bb > std::max<int>(2 * (int)b - 31, (int)b - kMaxLoBits) && bb <= kHistSmemBits &&
         hist_bytes(bb, cta_per_sm) > (96ull << 20))
    --bb;
  if (const char* e = getenv("EH_TEST_BKT_SHIFT")) bb = std::max<int>(2 * (int)b - 31, bb + atoi(e));  // test hook
  bb = std::max(0, std::min<int>(bb, (int)b));
  const BktParams p{b, b - (uint32_t)bb};
  const uint32_t nb = 1u << bb;
  DBuf<uint32_t> cnt(al, nb), cur(al, nb);
  EH_CUDA(cudaMemsetAsync(cnt.p, 0, nb * 4ull, s));
  EH_CUDA(cudaMemsetAsync(cur.p, 0, nb * 4ull, s));
  const unsigned TB = 256;
  const unsigned grid_stream = grid_for((n + 3) / 4, TB, kSMs * 8);
  // shared-memory histogram / cursors (<= 2^15 buckets): 1024-thread CTAs, as many per SM as the
  // counters allow (one at 2^15 buckets); test hooks: EH_TEST_BKT_GHIST global-atomic histogram,
  // EH_TEST_BKT_PART_ATOMIC global cursor atomics (both for > 2^15 buckets anyway),
  // EH_TEST_BKT_PART_MATCH the warp-matched variant of the latter
  const bool smem_hist = bb <= kHistSmemBits && getenv("EH_TEST_BKT_GHIST") == nullptr;
  const bool smem_part = smem_hist && n < (1ull << 32) && getenv("EH_TEST_BKT_PART_ATOMIC") == nullptr &&
                         getenv("EH_TEST_BKT_PART_MATCH") == nullptr;
  const size_t sm = nb * 4ull;
  const unsigned per_sm = (unsigned)std::max<size_t>(1, std::min<size_t>(cta_per_sm, (200 * 1024) / std::max<size_t>(sm, 1)));
  const unsigned grid_sm = std::min(grid_for((n + 3) / 4, 1024), kSMs * per_sm);
  const uint64_t nparts = (n + per - 1) / per * grid_sm;  // (chunk, CTA) histograms
  DBuf<uint32_t> percta;
  if (smem_part) percta = DBuf<uint32_t>(al, nparts * pitch(nb));
  if (smem_hist) {
    ensure_dyn_smem((const void*)k_bkt_hist<true>, sm);
    prefer_max_smem_carveout((const void*)k_bkt_hist<true>);
    k_bkt_hist<true><<<grid_sm, 1024, sm, s>>>(src, dst, n, p, nb, cnt.p, smem_part ? percta.p : nullptr, per);
  } else {
    k_bkt_hist<false><<<grid_stream, TB, 0, s>>>(src, dst, n, p, nb, cnt.p, nullptr, n);
  }
  EH_LAUNCH("k_bkt_hist");
  if (smem_part) {
    k_bkt_colscan<<<(nb + kCsB - 1) / kCsB, kCsB * kCsS, 0, s>>>(percta.p, (uint32_t)nparts, nb, cnt.p);
    EH_LAUNCH("k_bkt_colscan");
  }
  DBuf<uint64_t> boff(al, nb + 1ull), tot(al, 1);
  scan_exclusive_u32(cnt.p, boff.p, nb, tot.p, al, s);
  EH_CUDA(cudaMemcpyAsync(boff.p + nb, tot.p, 8, cudaMemcpyDeviceToDevice, s));
  DBuf<uint32_t> part(al, n);
  if (tm) tm->mark("bkt_hist");
  if (smem_part) {
    ensure_dyn_smem((const void*)k_bkt_part_smem, sm);
    prefer_max_smem_carveout((const void*)k_bkt_part_smem);
    k_bkt_part_smem<<<grid_sm, 1024, sm, s>>>(src, dst, n, p, nb, boff.p, percta.p, per, part.p);
  } else if (getenv("EH_TEST_BKT_PART_MATCH") == nullptr) {
    k_bkt_cursors<<<grid_for(nb, TB), TB, 0, s>>>(boff.p, nb, cur.p);
    EH_LAUNCH("k_bkt_cursors");
    k_bkt_part_direct<<<grid_stream, TB, 0, s>>>(src, dst, n, p, boff.p, cur.p, part.p);
  } else {
    k_bkt_part<<<grid_stream, TB, 0, s>>>(src, dst, n, p, boff.p, cur.p, part.p);
  }
  EH_LAUNCH("k_bkt_part");
  percta.reset();
  if (tm) tm->mark("bkt_part");
  cur.reset();
  DBuf<uint32_t> lists(al, 3ull * nb);
  DBuf<uint64_t> gtab(al, nb);
  DBuf<unsigned long long> info(al, 4);
  EH_CUDA(cudaMemsetAsync(info.p, 0, 32, s));
  k_bkt_classify<<<grid_for(nb, TB), TB, 0, s>>>(boff.p, nb, lists.p, info.p, gtab.p);
  EH_LAUNCH("k_bkt_classify");
  unsigned long long hinfo[4];
  EH_CUDA(cudaMemcpyAsync(hinfo, info.p, 32, cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaStreamSynchronize(s));
  DBuf<uint32_t> gscr(al, std::max<unsigned long long>(1, hinfo[3]));
  // large buckets first, beside the small ones (side stream); shared only: deg / m atomics
  const bool side = hinfo[0] && (hinfo[1] || hinfo[2]);
  const cudaStream_t ss = side ? fork_side(g, 0) : s;
  const size_t lsm = (size_t)4 << p.lobits;
  launch_dedup<kGiantThreads, 2, 0>(hinfo[2], lsm, part.p, boff.p, lists.p + 2ull * nb, info.p, 2, p, deg, m_ctr, out,
                                    gscr.p, gtab.p, ss);
  launch_dedup<kBigThreads, 1, kBigSlots>(hinfo[1], kBigSlots * 4ull + lsm, part.p, boff.p, lists.p + nb, info.p, 1, p,
                                          deg, m_ctr, out, gscr.p, gtab.p, ss);
  launch_dedup<kSmallThreads, 0, kSmallSlots>(hinfo[0], kSmallSlots * 4ull + lsm, part.p, boff.p, lists.p, info.p, 0, p,
                                              deg, m_ctr, out, gscr.p, gtab.p, s);
  if (side) join_side(g, 0);
}

}  // namespace eh
