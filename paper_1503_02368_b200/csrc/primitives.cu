// primitives.cu -- device-wide scan and one-sweep LSD radix sort (hand-written, sm_100a).
//
// Used by ingest ("hand-written radix sort, dedup",
// the (degree, id) rank sort, dictionary encoding) and by the layout / work-list
// builders.
//
// Radix sort = one-sweep LSD with 8-bit digits (9-bit when that saves a pass):
//   (1) one read of the keys builds the digit histograms of EVERY pass;
//       an exclusive scan per pass gives each digit's global base;
//   (2) per pass, tiles of 4096 keys are taken in launch order from an atomic
//       tile counter; each tile ranks its keys stably (warp sub-tiles in order,
//       __match_any_sync within a round of 32), publishes its per-digit counts,
//       and finds its per-digit exclusive prefix by decoupled look-back over the
//       preceding tiles (status = {flag:2, value:62} in one 64-bit word, so flag
//       and value are published atomically).  Keys are reordered by digit in
//       shared memory and written out in digit runs (coalesced).
// One read + one write of the keys per pass; forward progress holds because a
// tile only waits on tiles that obtained a smaller index, i.e. started earlier.
// Passes whose digit is constant over all keys are skipped.
#include "eh_internal.cuh"
#include "primitives.cuh"

namespace eh {

// ------------------------------------------------------------------- scan --
constexpr int kScanBlock = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanBlock * kScanItems;

template <typename Tin>
__global__ void __launch_bounds__(kScanBlock) k_scan_reduce(const Tin* __restrict__ in, uint64_t n,
                                                            uint64_t* __restrict__ block_sums) {
  __shared__ uint64_t sw[kScanBlock / 32];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t idx = base + (uint64_t)i * kScanBlock + threadIdx.x;
    if (idx < n) s += (uint64_t)in[idx];
  }
  const uint64_t tot = block_reduce_sum<kScanBlock>(s, sw);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

template <typename Tin>
__global__ void __launch_bounds__(kScanBlock) k_scan_down(const Tin* __restrict__ in, uint64_t* __restrict__ out,
                                                          uint64_t n, const uint64_t* __restrict__ block_offs,
                                                          uint64_t* __restrict__ d_total) {
  __shared__ uint64_t sw[kScanBlock / 32 + 1];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  uint64_t v[kScanItems];
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < n) ? (uint64_t)in[base + i] : 0;
    s += v[i];
  }
  uint64_t tot;
  uint64_t run = block_exclusive_scan<kScanBlock>(s, sw, &tot) + (block_offs ? block_offs[blockIdx.x] : 0);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (d_total && blockIdx.x == gridDim.x - 1 && threadIdx.x == kScanBlock - 1) *d_total = run;
}

template <typename Tin>
static void scan_impl(const Tin* in, uint64_t* out, uint64_t n, uint64_t* d_total, Allocator& al, cudaStream_t s) {
  if (n == 0) {
    if (d_total) EH_CUDA(cudaMemsetAsync(d_total, 0, sizeof(uint64_t), s));
    return;
  }
  const uint64_t nt = (n + kScanTile - 1) / kScanTile;
  if (nt == 1) {
    k_scan_down<Tin><<<1, kScanBlock, 0, s>>>(in, out, n, nullptr, d_total);
    EH_LAUNCH("k_scan_down");
    return;
  }
  DBuf<uint64_t> sums(al, nt);
  k_scan_reduce<Tin><<<(unsigned)nt, kScanBlock, 0, s>>>(in, n, sums.p);
  EH_LAUNCH("k_scan_reduce");
  scan_impl<uint64_t>(sums.p, sums.p, nt, nullptr, al, s);  // in-place is safe: block-local reads precede writes
  k_scan_down<Tin><<<(unsigned)nt, kScanBlock, 0, s>>>(in, out, n, sums.p, d_total);
  EH_LAUNCH("k_scan_down");
}

void scan_exclusive_u32(const uint32_t* in, uint64_t* out, uint64_t n, uint64_t* d_total, Allocator& al,
                        cudaStream_t s) {
  scan_impl<uint32_t>(in, out, n, d_total, al, s);
}
void scan_exclusive_u64(const uint64_t* in, uint64_t* out, uint64_t n, uint64_t* d_total, Allocator& al,
                        cudaStream_t s) {
  scan_impl<uint64_t>(in, out, n, d_total, al, s);
}

// ------------------------------------------------------------- radix sort --
constexpr int kRBlock = 256;                  // histogram kernel
constexpr int kRadixDefaultCfg = 2;           // pass kernel tile: 256 threads x 16 keys (measured best, see radix_impl)
constexpr int kRMaxDigits = 512;              // digits of 8 or 9 bits
constexpr int kRMaxPasses = 8;
constexpr uint64_t kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;

// Key source of the first pass: the keys themselves, or (kCanon, SURVEY.md §8(a)
// row a1 fused into the sort) the canonical undirected key (min << b) | max of
// the pair (src[i], dst[i]), self-loops mapped to the all-ones sentinel.
struct CanonSrc {
  const uint32_t* src;
  const uint32_t* dst;
  uint32_t b;
  uint64_t sentinel;
};
template <typename K, bool kCanon>
__device__ __forceinline__ K load_key(const K* __restrict__ keys, const CanonSrc& cs, uint64_t i) {
  if (kCanon) {
    const uint32_t u = __ldg(cs.src + i), v = __ldg(cs.dst + i);
    return (u == v) ? (K)cs.sentinel : (K)((((uint64_t)min(u, v)) << cs.b) | (uint64_t)max(u, v));
  }
  return keys[i];
}

template <typename K>
__global__ void k_canon_fill(CanonSrc cs, uint64_t n, K* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = load_key<K, true>(out, cs, i);
}

// (1) all-pass digit histograms in one read (pass p: bits [begin + p*bits, +bits))
template <typename K, bool kCanon>
__global__ void __launch_bounds__(kRBlock) k_radix_hist(const K* __restrict__ keys, CanonSrc cs, uint64_t n,
                                                        uint32_t passes, uint32_t begin, uint32_t bits,
                                                        unsigned long long* __restrict__ hist) {
  __shared__ uint32_t h[kRMaxPasses * kRMaxDigits];
  const uint32_t nd = 1u << bits, dm = nd - 1u;
  for (int i = threadIdx.x; i < kRMaxPasses * kRMaxDigits; i += kRBlock) h[i] = 0;
  __syncthreads();
  for (uint64_t i = (uint64_t)blockIdx.x * kRBlock + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kRBlock) {
    const K k = load_key<K, kCanon>(keys, cs, i) >> begin;
    for (uint32_t p = 0; p < passes; ++p) atomicAdd(&h[p * nd + ((uint32_t)(k >> (bits * p)) & dm)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (int)(passes * nd); i += kRBlock) {
    const uint32_t c = h[i];
    if (c) atomicAdd(&hist[i], (unsigned long long)c);
  }
}

// per-pass exclusive scan of the digit counts (one CTA per pass, one thread per digit)
__global__ void __launch_bounds__(kRMaxDigits) k_radix_base(const unsigned long long* __restrict__ hist,
                                                            unsigned long long* __restrict__ base,
                                                            uint32_t* __restrict__ trivial, uint64_t n, uint32_t nd) {
  __shared__ unsigned long long sw[kRMaxDigits / 32 + 1];
  const uint32_t p = blockIdx.x;
  const unsigned long long c = (threadIdx.x < nd) ? hist[p * nd + threadIdx.x] : 0ull;
  unsigned long long tot;
  const unsigned long long ex = block_exclusive_scan<kRMaxDigits>(c, sw, &tot);
  if (threadIdx.x < nd) base[p * nd + threadIdx.x] = ex;
  if (c == n) trivial[p] = 1u;  // every key has this digit: the pass is the identity
}

// (2) one pass over digits of kBits bits.  Launch bounds at the occupancy the tile's
// shared memory allows (e.g. the 8192-key u64 tile: 2 CTAs per SM, so 64 registers
// instead of 40 with 184-B spills: C3 load 7.38 -> 7.23 ms).
template <int kPBlock, int kRItems, int kKeyBytes>
constexpr int radix_min_blocks() {  // resident CTAs the shared memory allows (keys + ~8 KB static), <= 1536 threads
  constexpr int by_smem = (200 * 1024) / (kPBlock * kRItems * kKeyBytes + 8 * 1024);
  constexpr int by_thr = 3 * 512 / kPBlock;
  return by_smem < 1 ? 1 : (by_smem < by_thr ? by_smem : by_thr);
}
template <typename K, int kBits, int kPBlock, int kRItems, bool kCanon>
__global__ void __launch_bounds__(kPBlock, radix_min_blocks<kPBlock, kRItems, (int)sizeof(K)>()) k_radix_pass(const K* __restrict__ in, CanonSrc cs,
                                                                           K* __restrict__ out, uint64_t n,
                                                                           uint32_t shift,
                                                                           const unsigned long long* __restrict__ base,
                                                                           unsigned long long* __restrict__ status,
                                                                           uint32_t* __restrict__ tile_ctr) {
  constexpr int kD = 1 << kBits;
  constexpr uint32_t kDM = kD - 1, kInv = kD;    // digit mask, invalid-key marker
  constexpr int kDPT = kD > kPBlock ? kD / kPBlock : 1;  // consecutive digits per thread
  static_assert(kD <= kPBlock * kDPT, "digits per thread");
  constexpr int kRWarps = kPBlock / 32;
  constexpr int kRTile = kPBlock * kRItems;
  extern __shared__ __align__(16) unsigned char dsm_radix[];
  K* skeys = reinterpret_cast<K*>(dsm_radix);    // kRTile keys (dynamic shared memory)
  __shared__ uint16_t wcnt[kRWarps][kD];         // per-warp digit counts (<= 32 * items), then prefixes
  __shared__ uint32_t tdp[kD];                   // tile-local exclusive digit prefix
  __shared__ unsigned long long goff[kD];        // global position of the tile's first key with digit d
  __shared__ uint32_t s_tile;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (int i = threadIdx.x; i < kRWarps * kD; i += kPBlock) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t t0 = tile * kRTile;
  const uint64_t tn = min((uint64_t)kRTile, n - t0);
  const unsigned lt = (1u << lane) - 1u;
  K key[kRItems];
  uint32_t rd[kRItems];  // rank within the warp sub-tile (low 16 bits) | digit << 16 (kInv: invalid)
#pragma unroll
  for (int r = 0; r < kRItems; ++r) {
    const uint32_t li = (uint32_t)w * 32 * kRItems + (uint32_t)r * 32 + lane;
    const bool valid = li < tn;
    key[r] = valid ? load_key<K, kCanon>(in, cs, t0 + li) : K(0);
    const uint32_t d = valid ? ((uint32_t)(key[r] >> shift) & kDM) : kInv;
    const unsigned peers = __match_any_sync(kFull, d);
    const uint32_t before = (d < kInv) ? wcnt[w][d] : 0u;
    __syncwarp();
    if (d < kInv && (peers & lt) == 0) wcnt[w][d] = (uint16_t)(before + __popc(peers));
    __syncwarp();
    rd[r] = (before + __popc(peers & lt)) | (d << 16);
  }
  __syncthreads();
  // thread t owns digits [t*kDPT, t*kDPT + kDPT): per-warp exclusive prefix, tile totals
  const uint32_t d0 = threadIdx.x * kDPT;
  const bool owner = d0 < (uint32_t)kD;
  uint32_t total[kDPT];
  uint32_t tsum = 0;
#pragma unroll
  for (int q = 0; q < kDPT; ++q) {
    total[q] = 0;
    if (owner) {
      uint32_t run = 0;
#pragma unroll
      for (int ww = 0; ww < kRWarps; ++ww) {
        const uint32_t c = wcnt[ww][d0 + q];
        wcnt[ww][d0 + q] = (uint16_t)run;  // prefix <= tile size fits u16
        run += c;
      }
      total[q] = run;
      // publish this tile's aggregate (tile 0: its inclusive prefix)
      __stcg(status + tile * kD + d0 + q, (tile == 0 ? kFlagInc : kFlagAgg) | run);
      if (tile == 0) goff[d0 + q] = base[d0 + q];
    }
    tsum += total[q];
  }
  // the barrier also keeps the compiler from merging the aggregate store above
  // with the inclusive store below (same address): without the early aggregate
  // the look-back degenerates into a serial chain
  __syncthreads();
  // decoupled look-back, one thread per digit, reading a window of 8 preceding
  // tiles per step (independent loads in flight); a tile that has not published
  // yet stops the window and is re-read from there.
  if (tile > 0 && owner) {
#pragma unroll
    for (int q = 0; q < kDPT; ++q) {
      const uint32_t d = d0 + q;
      constexpr int kW = 8;
      unsigned long long excl = 0;
      int64_t t = (int64_t)tile - 1;
      for (;;) {
        unsigned long long sv[kW];
#pragma unroll
        for (int j = 0; j < kW; ++j)
          sv[j] = (t - j >= 0) ? *((volatile unsigned long long*)(status + (uint64_t)(t - j) * kD + d)) : kFlagInc;
        int j = 0;
        bool done = false;
#pragma unroll
        for (int q2 = 0; q2 < kW; ++q2) {
          if (done || j != q2) continue;
          const unsigned long long fl = sv[q2] & ~kValMask;
          if (fl == 0) continue;  // not published yet: stop the window here
          excl += sv[q2] & kValMask;
          ++j;
          if (fl == kFlagInc) done = true;
        }
        if (done) break;
        t -= j;
      }
      __stcg(status + tile * kD + d, kFlagInc | (excl + total[q]));
      goff[d] = base[d] + excl;
    }
  }
  // tile-local exclusive prefix over digits (threads without digits contribute 0)
  {
    __shared__ uint32_t sw[kPBlock / 32 + 1];
    uint32_t tt;
    uint32_t ex = block_exclusive_scan<kPBlock>(tsum, sw, &tt);
    if (owner) {
#pragma unroll
      for (int q = 0; q < kDPT; ++q) { tdp[d0 + q] = ex; ex += total[q]; }
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRItems; ++r)
    if ((rd[r] >> 16) < kInv) {
      EH_DASSERT(tdp[rd[r] >> 16] + wcnt[w][rd[r] >> 16] + (rd[r] & 0xFFFFu) < (uint32_t)kRTile);
      skeys[tdp[rd[r] >> 16] + wcnt[w][rd[r] >> 16] + (rd[r] & 0xFFFFu)] = key[r];
    }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < tn; i += kPBlock) {
    const K k = skeys[i];
    const uint32_t dd = (uint32_t)(k >> shift) & kDM;
    EH_DASSERT(goff[dd] + (i - tdp[dd]) < n);
    out[goff[dd] + (i - tdp[dd])] = k;
  }
}

template <typename K, int kBits, int kPBlock, int kRItems, bool kCanon>
static void launch_pass(const K* src, CanonSrc cs, K* dst, uint64_t n, uint32_t shift, const unsigned long long* bp,
                        unsigned long long* status, uint32_t* ctr, uint64_t tiles, size_t smem, cudaStream_t s) {
  auto k = k_radix_pass<K, kBits, kPBlock, kRItems, kCanon>;
  ensure_dyn_smem((const void*)k, smem);
  k<<<(unsigned)tiles, kPBlock, smem, s>>>(src, cs, dst, n, shift, bp, status, ctr);
  EH_LAUNCH("k_radix_pass");
}

template <typename K, int kBits, bool kCanon>
static void launch_pass_cfg(int cfg, const K* src, CanonSrc cs, K* dst, uint64_t n, uint32_t shift,
                            const unsigned long long* bp, unsigned long long* status, uint32_t* ctr, uint64_t tiles,
                            size_t smem, cudaStream_t s) {
  switch (cfg) {
    case 0: launch_pass<K, kBits, 512, 8, kCanon>(src, cs, dst, n, shift, bp, status, ctr, tiles, smem, s); break;
    case 1: launch_pass<K, kBits, 256, 8, kCanon>(src, cs, dst, n, shift, bp, status, ctr, tiles, smem, s); break;
    case 2: launch_pass<K, kBits, 256, 16, kCanon>(src, cs, dst, n, shift, bp, status, ctr, tiles, smem, s); break;
    default: launch_pass<K, kBits, 512, 16, kCanon>(src, cs, dst, n, shift, bp, status, ctr, tiles, smem, s); break;
  }
}

template <typename K, bool kCanon>
static void launch_pass_bits(uint32_t bits, int cfg, const K* src, CanonSrc cs, K* dst, uint64_t n, uint32_t shift,
                             const unsigned long long* bp, unsigned long long* status, uint32_t* ctr, uint64_t tiles,
                             size_t smem, cudaStream_t s) {
  if (bits == 9) launch_pass_cfg<K, 9, kCanon>(cfg, src, cs, dst, n, shift, bp, status, ctr, tiles, smem, s);
  else launch_pass_cfg<K, 8, kCanon>(cfg, src, cs, dst, n, shift, bp, status, ctr, tiles, smem, s);
}

// LSD sort of keys by bits [begin, key_bits).  Stable, so a key array already
// ordered by its low `begin` bits comes out ordered by the whole key.  With
// cs.src != nullptr (u64 only) the keys are produced from (src, dst) by the
// histogram and the first non-trivial pass (the canonicalisation of row a1 fused
// into the sort); `keys` is then only an output buffer.  Digits are 8 bits, or 9
// when that saves a pass (EH_RADIX_BITS=8|9 forces one).
template <typename K>
static K* radix_impl(K* keys, K* alt, uint64_t n, uint32_t key_bits, uint32_t begin, CanonSrc cs, Allocator& al,
                     cudaStream_t s) {
  const bool canon = cs.src != nullptr;
  if (n == 0) return keys;
  if (key_bits <= begin || n == 1) {
    if (canon) {
      k_canon_fill<K><<<grid_for(n, 1024), 256, 0, s>>>(cs, n, keys);
      EH_LAUNCH("k_canon_fill");
    }
    return keys;
  }
  const uint32_t span = key_bits - begin;
  // 9-bit digits when they save a pass, with the 8192-key tile (its longer digit
  // runs pay for the 512 buckets); the 8192-key tile also for very large inputs.
  // Measured (tools/radix_bench.cu, B200): C3 keys (44 bits) 8-bit/4096 4.07 ms,
  // 9-bit/8192 3.95 ms; C5 keys (52 bits) 8-bit 110 / 92 ms (4096 / 8192), 9-bit/8192 88.7 ms.
  uint32_t bits = ((span + 8) / 9 < (span + 7) / 8) ? 9u : 8u;
  static const int bits_env = [] { const char* e = getenv("EH_RADIX_BITS"); return e ? atoi(e) : 0; }();
  if (bits_env == 8 || bits_env == 9) bits = (uint32_t)bits_env;  // tuning override
  const uint32_t nd = 1u << bits;
  const uint32_t passes = (span + bits - 1) / bits;
  if (passes > (uint32_t)kRMaxPasses) fail(EH_EINVAL, "radix sort: %u key bits", span);
  DBuf<unsigned long long> hist(al, (size_t)passes * nd), base(al, (size_t)passes * nd);
  DBuf<uint32_t> trivial(al, kRMaxPasses), ctr(al, kRMaxPasses);
  EH_CUDA(cudaMemsetAsync(hist.p, 0, hist.bytes(), s));
  EH_CUDA(cudaMemsetAsync(trivial.p, 0, trivial.bytes(), s));
  EH_CUDA(cudaMemsetAsync(ctr.p, 0, ctr.bytes(), s));
  if (canon)
    k_radix_hist<K, true><<<grid_for(n, kRBlock * 16, kSMs * 8), kRBlock, 0, s>>>(keys, cs, n, passes, begin, bits, hist.p);
  else
    k_radix_hist<K, false><<<grid_for(n, kRBlock * 16, kSMs * 8), kRBlock, 0, s>>>(keys, cs, n, passes, begin, bits, hist.p);
  EH_LAUNCH("k_radix_hist");
  k_radix_base<<<passes, kRMaxDigits, 0, s>>>(hist.p, base.p, trivial.p, n, nd);
  EH_LAUNCH("k_radix_base");
  // Skipping a pass whose digit is constant needs the flags on the host (one
  // synchronisation); small sorts just run every pass (a constant-digit pass is
  // an exact stable copy).
  uint32_t triv[kRMaxPasses] = {0};
  if (n >= (1ull << 22)) {
    EH_CUDA(cudaMemcpyAsync(triv, trivial.p, sizeof triv, cudaMemcpyDeviceToHost, s));
    EH_CUDA(cudaStreamSynchronize(s));
  }
  // tile shape (threads x keys per thread); EH_RADIX_CFG selects one for tuning
  static const int cfg_env = [] { const char* e = getenv("EH_RADIX_CFG"); return e ? atoi(e) : -1; }();
  const int cfg = (cfg_env >= 0 && cfg_env <= 3) ? cfg_env
                  : (bits == 9 || n >= (1ull << 28)) ? 3 : kRadixDefaultCfg;
  static const int kThreads[4] = {512, 256, 256, 512}, kItems[4] = {8, 8, 16, 16};
  const uint64_t tile = (uint64_t)kThreads[cfg] * kItems[cfg];
  const uint64_t tiles = (n + tile - 1) / tile;
  if (tiles >= (1ull << 31)) fail(EH_EINVAL, "radix sort: too many keys");
  DBuf<unsigned long long> status(al, (size_t)tiles * nd);
  const size_t smem = tile * sizeof(K);
  // the canonical source is read by the first non-trivial pass, which writes `keys`
  bool from_src = canon;
  K* src = keys;
  K* dst = canon ? keys : alt;
  for (uint32_t p = 0; p < passes; ++p) {
    if (triv[p]) continue;
    EH_CUDA(cudaMemsetAsync(status.p, 0, status.bytes(), s));
    const unsigned long long* bp = base.p + (size_t)p * nd;
    const uint32_t shift = begin + bits * p;
    if (from_src) launch_pass_bits<K, true>(bits, cfg, nullptr, cs, dst, n, shift, bp, status.p, ctr.p + p, tiles, smem, s);
    else launch_pass_bits<K, false>(bits, cfg, src, cs, dst, n, shift, bp, status.p, ctr.p + p, tiles, smem, s);
    if (from_src) { from_src = false; src = keys; dst = alt; continue; }
    K* t = src; src = dst; dst = t;
  }
  if (from_src) {  // every pass trivial: materialise the keys (already in order)
    k_canon_fill<K><<<grid_for(n, 1024), 256, 0, s>>>(cs, n, keys);
    EH_LAUNCH("k_canon_fill");
  }
  return src;
}

uint64_t* radix_sort_u64(uint64_t* keys, uint64_t* alt, uint64_t n, uint32_t key_bits, Allocator& al,
                         cudaStream_t s, uint32_t begin_bit) {
  return radix_impl<uint64_t>(keys, alt, n, key_bits, begin_bit, CanonSrc{nullptr, nullptr, 0, 0}, al, s);
}
uint32_t* radix_sort_u32(uint32_t* keys, uint32_t* alt, uint64_t n, uint32_t key_bits, Allocator& al,
                         cudaStream_t s) {
  return radix_impl<uint32_t>(keys, alt, n, key_bits, 0, CanonSrc{nullptr, nullptr, 0, 0}, al, s);
}
uint64_t* radix_sort_canon(const uint32_t* src, const uint32_t* dst, uint64_t n, uint32_t b, uint64_t* keys,
                           uint64_t* alt, Allocator& al, cudaStream_t s) {
  const uint64_t sentinel = (b >= 32) ? ~0ull : ((1ull << (2 * b)) - 1ull);
  return radix_impl<uint64_t>(keys, alt, n, 2 * b, 0, CanonSrc{src, dst, b, sentinel}, al, s);
}

}  // namespace eh
