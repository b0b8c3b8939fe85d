// primitives.cu -- device-wide scan and LSD radix sort (hand-written, sm_100a).
//
// Used by ingest ("hand-written radix sort, dedup",
// CSR offsets) and by the layout/work-list builders.  Radix sort is the classic
// reduce-then-scan LSD scheme: per pass (i) every CTA histograms the digit over
// its contiguous key range, (ii) one exclusive scan of the digit-major
// [256 x CTAs] table gives every (digit, CTA) its global base, (iii) every CTA
// re-reads its range tile by tile, ranks keys stably inside each warp with
// __match_any_sync and scatters them.  Stable, deterministic, no look-back.
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
constexpr int kRadixBlock = 256;
constexpr int kRadixWarps = kRadixBlock / 32;
constexpr int kRadixItems = 8;                       // keys per lane per tile
constexpr int kRadixTile = kRadixBlock * kRadixItems;  // 2048 keys
constexpr int kRadixDigits = 256;

template <typename K>
__global__ void __launch_bounds__(kRadixBlock) k_radix_upsweep(const K* __restrict__ keys, uint64_t n,
                                                               uint64_t per_cta, uint32_t shift,
                                                               uint64_t* __restrict__ hist) {
  __shared__ uint32_t h[kRadixDigits];
  for (int i = threadIdx.x; i < kRadixDigits; i += kRadixBlock) h[i] = 0;
  __syncthreads();
  const uint64_t b = (uint64_t)blockIdx.x * per_cta;
  const uint64_t e = min(n, b + per_cta);
  for (uint64_t i = b + threadIdx.x; i < e; i += kRadixBlock) {
    const uint32_t d = (uint32_t)(keys[i] >> shift) & 0xFFu;
    atomicAdd(&h[d], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kRadixDigits; d += kRadixBlock) hist[(uint64_t)d * gridDim.x + blockIdx.x] = h[d];
}

template <typename K>
__global__ void __launch_bounds__(kRadixBlock) k_radix_downsweep(const K* __restrict__ keys, K* __restrict__ out,
                                                                 uint64_t n, uint64_t per_cta, uint32_t shift,
                                                                 const uint64_t* __restrict__ offs) {
  __shared__ uint32_t wcnt[kRadixWarps][kRadixDigits];  // per-warp digit counts, then exclusive prefixes
  __shared__ uint32_t ttot[kRadixDigits];               // per-tile digit totals
  __shared__ uint64_t cbase[kRadixDigits];              // global output base of each digit for this tile
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < kRadixDigits; d += kRadixBlock) cbase[d] = offs[(uint64_t)d * gridDim.x + blockIdx.x];
  for (int i = threadIdx.x; i < kRadixWarps * kRadixDigits; i += kRadixBlock) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const uint64_t b = (uint64_t)blockIdx.x * per_cta;
  const uint64_t e = min(n, b + per_cta);
  const unsigned lt = (1u << lane) - 1u;
  for (uint64_t t0 = b; t0 < e; t0 += kRadixTile) {
    K key[kRadixItems];
    uint32_t rk[kRadixItems], dg[kRadixItems];
    // warp w owns the contiguous sub-tile [t0 + w*32*ITEMS, +32*ITEMS), read in rounds of 32:
    // ranking rounds in order and lanes by position keeps the sort stable.
#pragma unroll
    for (int r = 0; r < kRadixItems; ++r) {
      const uint64_t idx = t0 + (uint64_t)w * 32 * kRadixItems + (uint64_t)r * 32 + lane;
      const bool valid = idx < e;
      key[r] = valid ? keys[idx] : K(0);
      const uint32_t d = valid ? ((uint32_t)(key[r] >> shift) & 0xFFu) : 0x100u;
      const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
      const uint32_t before = (d < 0x100u) ? wcnt[w][d] : 0u;
      __syncwarp();
      if (d < 0x100u && (peers & lt) == 0) wcnt[w][d] = before + __popc(peers);
      __syncwarp();
      rk[r] = before + __popc(peers & lt);
      dg[r] = d;
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadixDigits; d += kRadixBlock) {
      uint32_t run = 0;
#pragma unroll
      for (int ww = 0; ww < kRadixWarps; ++ww) {
        const uint32_t c = wcnt[ww][d];
        wcnt[ww][d] = run;
        run += c;
      }
      ttot[d] = run;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRadixItems; ++r)
      if (dg[r] < 0x100u) out[cbase[dg[r]] + wcnt[w][dg[r]] + rk[r]] = key[r];
    __syncthreads();
    for (int d = threadIdx.x; d < kRadixDigits; d += kRadixBlock) cbase[d] += ttot[d];
    for (int i = threadIdx.x; i < kRadixWarps * kRadixDigits; i += kRadixBlock) (&wcnt[0][0])[i] = 0;
    __syncthreads();
  }
}

template <typename K>
static K* radix_impl(K* keys, K* alt, uint64_t n, uint32_t key_bits, Allocator& al, cudaStream_t s) {
  if (n <= 1 || key_bits == 0) return keys;
  const uint64_t tiles = (n + kRadixTile - 1) / kRadixTile;
  const unsigned G = (unsigned)std::min<uint64_t>(tiles, (uint64_t)kSMs * 8);
  const uint64_t per_cta = ((tiles + G - 1) / G) * kRadixTile;
  const unsigned grid = (unsigned)((n + per_cta - 1) / per_cta);
  DBuf<uint64_t> hist(al, (size_t)kRadixDigits * grid);
  K* src = keys;
  K* dst = alt;
  for (uint32_t shift = 0; shift < key_bits; shift += 8) {
    k_radix_upsweep<K><<<grid, kRadixBlock, 0, s>>>(src, n, per_cta, shift, hist.p);
    EH_LAUNCH("k_radix_upsweep");
    scan_exclusive_u64(hist.p, hist.p, (uint64_t)kRadixDigits * grid, nullptr, al, s);
    k_radix_downsweep<K><<<grid, kRadixBlock, 0, s>>>(src, dst, n, per_cta, shift, hist.p);
    EH_LAUNCH("k_radix_downsweep");
    K* t = src; src = dst; dst = t;
  }
  return src;
}

uint64_t* radix_sort_u64(uint64_t* keys, uint64_t* alt, uint64_t n, uint32_t key_bits, Allocator& al,
                         cudaStream_t s) {
  return radix_impl<uint64_t>(keys, alt, n, key_bits, al, s);
}
uint32_t* radix_sort_u32(uint32_t* keys, uint32_t* alt, uint64_t n, uint32_t key_bits, Allocator& al,
                         cudaStream_t s) {
  return radix_impl<uint32_t>(keys, alt, n, key_bits, al, s);
}

}  // namespace eh
