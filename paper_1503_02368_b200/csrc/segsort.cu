// segsort.cu -- sort many short u32 segments, in place or into another layout
// ("CSR with strictly increasing out-lists").
//
// After orientation the out-lists are filled by a counting-sort scatter (atomic
// cursor per list), which leaves each list in arbitrary order.  Degree
// orientation bounds every list: |N+(x)| <= sqrt(2m) (each out-neighbour has
// degree >= deg(x) >= |N+(x)|), so lists are short and sort in on-chip memory:
//   len <= 32          four segments per warp: 8-, 16- or 32-lane bitonic networks
//   len <= 1024        one warp, bitonic network in registers, E = 2, 4, 8, 16 or 32
//                      keys per lane (__shfl_xor_sync across lanes; measured faster than
//                      the shared-memory network for 257..1024: C3 load 7.98 -> 7.73 ms)
//   1025 .. 8192       one CTA, bitonic network in shared memory
//   longer (rare)      gathered as (segment << 32 | value) keys and sorted by the
//                      device-wide LSD radix sort, then scattered back.
#include "eh_internal.cuh"
#include "primitives.cuh"

#include <algorithm>

namespace eh {

namespace {

constexpr uint32_t kPad = 0xFFFFFFFFu;
constexpr int kMidMax = 1024;  // register tiers up to here (E = 32 keys per lane)
constexpr int kBigMax = 8192, kBigThreads = 1024;

struct Seg {
  const uint64_t* off16;  // output segment v starts at element off16[v] * 4
  const uint32_t* len;
  const uint32_t* in;     // out-of-place: input segment v at in + ioff[v] (else in place)
  const uint64_t* ioff;
  __device__ __forceinline__ const uint32_t* src(uint32_t* data, uint32_t v) const {
    return ioff ? in + ioff[v] : data + off16[v] * 4;
  }
};

// Bitonic network over 32 * E keys held E per lane (key index e * 32 + lane, so
// loads and stores are coalesced).
template <int E>
__device__ __forceinline__ void warp_bitonic_regs(uint32_t (&x)[E], int lane) {
#pragma unroll
  for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {  // partner in this lane: e ^ (j / 32)
        const int je = j >> 5;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if (e & je) continue;
          const bool up = (((e * 32 + lane) & k) == 0);
          const uint32_t a = x[e], b = x[e + je];
          x[e] = up ? min(a, b) : max(a, b);
          x[e + je] = up ? max(a, b) : min(a, b);
        }
      } else {  // partner in lane ^ j
        const bool lower = (lane & j) == 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint32_t o = __shfl_xor_sync(kFull, x[e], j);
          const bool up = (((e * 32 + lane) & k) == 0);
          x[e] = (lower == up) ? min(x[e], o) : max(x[e], o);
        }
      }
    }
  }
}

template <int E>
__global__ void k_seg_regs(uint32_t* __restrict__ data, Seg sg, const uint32_t* __restrict__ all_ids,
                           const uint64_t* __restrict__ rng) {
  const uint32_t* ids = all_ids + rng[0];
  const uint64_t nids = rng[1] - rng[0];
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint64_t t = warp; t < nids; t += nw) {
    const uint32_t v = ids[t];
    const uint32_t n = sg.len[v];
    EH_DASSERT(n <= 32u * E);
    uint32_t* p = data + sg.off16[v] * 4;
    const uint32_t* q = sg.src(data, v);
    uint32_t x[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t i = e * 32 + lane;
      x[e] = (i < n) ? q[i] : kPad;
    }
    warp_bitonic_regs<E>(x, lane);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t i = e * 32 + lane;
      if (i < n) p[i] = x[e];
    }
  }
}

// Segments of <= 32 keys, four per warp: when the four are all <= 8 keys they
// are sorted at once by 8-lane bitonic networks, when <= 16 two at a time by
// 16-lane networks, else one at a time by the whole warp (lists of consecutive
// ranks have similar lengths, so the branch is nearly always uniform).
template <int S>
__device__ __forceinline__ uint32_t subwarp_bitonic(uint32_t x, int lane) {
  const int sl = lane & (S - 1);
#pragma unroll
  for (int k = 2; k <= S; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint32_t o = __shfl_xor_sync(kFull, x, j);
      const bool lower = (sl & j) == 0, up = (sl & k) == 0;
      x = (lower == up) ? min(x, o) : max(x, o);
    }
  }
  return x;
}

template <int S>
__device__ __forceinline__ void sort_group(uint32_t* __restrict__ data, const Seg& sg, const uint32_t* __restrict__ ids,
                                           uint64_t t0, uint64_t nids, int lane) {
  const uint64_t t = t0 + lane / S;  // this lane's segment
  const int sl = lane & (S - 1);
  uint32_t n = 0;
  uint32_t* p = nullptr;
  const uint32_t* q = nullptr;
  if (t < nids) {
    const uint32_t v = ids[t];
    n = sg.len[v];
    p = data + sg.off16[v] * 4;
    q = sg.src(data, v);
  }
  EH_DASSERT(n <= (uint32_t)S);
  uint32_t x = ((uint32_t)sl < n) ? q[sl] : kPad;
  x = subwarp_bitonic<S>(x, lane);
  if ((uint32_t)sl < n) p[sl] = x;
}

__global__ void k_seg_small(uint32_t* __restrict__ data, Seg sg, const uint32_t* __restrict__ all_ids,
                            const uint64_t* __restrict__ rng) {
  const uint32_t* ids = all_ids + rng[0];
  const uint64_t nids = rng[1] - rng[0];
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint64_t t0 = warp * 4; t0 < nids; t0 += nw * 4) {
    const uint32_t mylen = (lane < 4 && t0 + lane < nids) ? sg.len[ids[t0 + lane]] : 0u;
    const uint32_t mx = __reduce_max_sync(kFull, mylen);
    if (mx <= 8) {
      sort_group<8>(data, sg, ids, t0, nids, lane);
    } else if (mx <= 16) {
      sort_group<16>(data, sg, ids, t0, nids, lane);
      sort_group<16>(data, sg, ids, t0 + 2, nids, lane);
    } else {
#pragma unroll 1
      for (int q = 0; q < 4; ++q) sort_group<32>(data, sg, ids, t0 + q, nids, lane);
    }
  }
}

// Bitonic sort of s[0..N) (N power of two) by `nt` cooperating threads.
template <bool kCta>
__device__ __forceinline__ void bitonic_smem(uint32_t* s, uint32_t N, uint32_t tid, uint32_t nt) {
  for (uint32_t k = 2; k <= N; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t t = tid; t < N / 2; t += nt) {
        const uint32_t i = 2 * t - (t & (j - 1));
        const uint32_t l = i + j;
        const bool asc = (i & k) == 0;
        const uint32_t a = s[i], b = s[l];
        if ((a > b) == asc) { s[i] = b; s[l] = a; }
      }
      if (kCta) __syncthreads(); else __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(kBigThreads) k_seg_big(uint32_t* __restrict__ data, Seg sg,
                                                          const uint32_t* __restrict__ all_ids,
                                                          const uint64_t* __restrict__ rng) {
  const uint32_t* ids = all_ids + rng[0];
  const uint64_t nids = rng[1] - rng[0];
  __shared__ uint32_t s[kBigMax];
  for (uint64_t t = blockIdx.x; t < nids; t += gridDim.x) {
    const uint32_t v = ids[t];
    const uint32_t n = sg.len[v];
    uint32_t* p = data + sg.off16[v] * 4;
    const uint32_t* q = sg.src(data, v);
    uint32_t N = 2048;
    while (N < n) N <<= 1;
    EH_DASSERT(N <= (uint32_t)kBigMax);
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) s[i] = (i < n) ? q[i] : kPad;
    __syncthreads();
    bitonic_smem<true>(s, N, threadIdx.x, blockDim.x);
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) p[i] = s[i];
    __syncthreads();
  }
}

// ---- fallback for segments longer than kBigMax ----
__global__ void k_seg_gather(uint32_t* __restrict__ data, Seg sg, const uint32_t* __restrict__ ids,
                             uint64_t nids, const uint64_t* __restrict__ goff, uint64_t* __restrict__ keys) {
  for (uint64_t t = blockIdx.x; t < nids; t += gridDim.x) {
    const uint32_t v = ids[t];
    const uint32_t n = sg.len[v];
    const uint32_t* p = sg.src(data, v);
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) keys[goff[t] + i] = (t << 32) | p[i];
  }
}
__global__ void k_seg_scatter(uint32_t* __restrict__ data, Seg sg, const uint32_t* __restrict__ ids,
                              uint64_t nids, const uint64_t* __restrict__ goff, const uint64_t* __restrict__ keys) {
  for (uint64_t t = blockIdx.x; t < nids; t += gridDim.x) {
    const uint32_t v = ids[t];
    const uint32_t n = sg.len[v];
    uint32_t* p = data + sg.off16[v] * 4;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) p[i] = (uint32_t)keys[goff[t] + i];
  }
}

// tier of a segment by its length (-1: nothing to sort), tiers as in segmented_sort_u32
struct TierOf {
  const uint32_t* len;
  uint32_t min_len;  // 2 in place; 1 out of place (single elements are copied)
  __device__ int operator()(uint64_t v) const {
    const uint32_t n = len[v];
    if (n < min_len) return -1;
    if (n <= 32) return 0;
    if (n <= 64) return 1;
    if (n <= 128) return 2;
    if (n <= 256) return 3;
    if (n <= 512) return 4;
    if (n <= (uint32_t)kMidMax) return 5;
    if (n <= (uint32_t)kBigMax) return 6;
    return 7;
  }
};
struct TierEmit {
  uint32_t* out;
  __device__ void operator()(int, uint64_t pos, uint64_t v) const { out[pos] = (uint32_t)v; }
};
__global__ void k_gather_len(const uint32_t* __restrict__ len, const uint32_t* __restrict__ ids, uint64_t n,
                             uint32_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = len[ids[i]];
}

}  // namespace

static void segsort_impl(uint32_t* data, const Seg& sg, uint64_t nseg, uint32_t max_len, Allocator& al,
                         cudaStream_t s, eh_graph* fork) {
  const uint32_t* len = sg.len;
  DBuf<uint32_t> all_ids(al, nseg);
  DBuf<uint64_t> starts(al, 10);  // one partition of the segments by tier, kept on the device:
  partition_k_async<8>(nseg, TierOf{len, sg.ioff ? 1u : 2u}, TierEmit{all_ids.p}, starts.p, al, s);  // no host sync
  // the tier kernels read their range from `starts`; grids are sized for the worst
  // case the host knows (nseg, max_len) and stride over what is there
  const uint32_t tier_min[8] = {1, 33, 65, 129, 257, 513, (uint32_t)kMidMax + 1, (uint32_t)kBigMax + 1};
  // The tiers are independent (disjoint segments) and each kernel is short and latency-bound
  // (ids -> length / offset -> keys), so with a handle to fork from they alternate over the
  // handle's stream and two of its side streams (C3: 0.59 -> see DESIGN.md §6 "ingest").
  cudaStream_t st[3] = {s, s, s};
  int ntier = 0;
  for (int tier = 0; tier < 7 && max_len >= tier_min[tier]; ++tier) ++ntier;
  const bool forked = fork && ntier >= 2 && getenv("EH_TEST_SEG_SERIAL") == nullptr;
  if (forked) {
    st[1] = fork_side(fork, 1);
    if (ntier >= 3) st[2] = fork_side(fork, 2);
  }
  // heaviest first on each stream: tier 0 (all lists <= 32) alone on the handle's stream's head
  const int lane_of[7] = {0, 1, 2, 1, 2, 1, 2};
  for (int tier = 0; tier < 7; ++tier) {
    if (max_len < tier_min[tier]) break;
    const uint64_t* rng = starts.p + tier;
    const uint64_t kmax = std::min<uint64_t>(nseg, 1ull << 24);
    const unsigned g = grid_for(kmax * 32, 256);
    const cudaStream_t ts = st[lane_of[tier]];
    if (tier == 0) k_seg_small<<<grid_for(kmax * 8, 256), 256, 0, ts>>>(data, sg, all_ids.p, rng);
    else if (tier == 1) k_seg_regs<2><<<g, 256, 0, ts>>>(data, sg, all_ids.p, rng);
    else if (tier == 2) k_seg_regs<4><<<g, 256, 0, ts>>>(data, sg, all_ids.p, rng);
    else if (tier == 3) k_seg_regs<8><<<g, 256, 0, ts>>>(data, sg, all_ids.p, rng);
    else if (tier == 4) k_seg_regs<16><<<g, 256, 0, ts>>>(data, sg, all_ids.p, rng);
    else if (tier == 5) k_seg_regs<32><<<g, 256, 0, ts>>>(data, sg, all_ids.p, rng);
    else k_seg_big<<<(unsigned)kSMs * 2, kBigThreads, 0, ts>>>(data, sg, all_ids.p, rng);
    EH_LAUNCH(tier == 6 ? "k_seg_big" : "k_seg_regs");
  }
  if (forked) {
    join_side(fork, 1);
    if (ntier >= 3) join_side(fork, 2);
  }
  if (max_len > (uint32_t)kBigMax) {  // rare: device-wide radix sort of the longest segments
    uint64_t h[2];
    EH_CUDA(cudaMemcpyAsync(h, starts.p + 7, 16, cudaMemcpyDeviceToHost, s));
    EH_CUDA(cudaStreamSynchronize(s));
    const uint64_t k = h[1] - h[0];
    if (k) {
      const uint32_t* tier_ids = all_ids.p + h[0];
      DBuf<uint32_t> lens(al, k);
      DBuf<uint64_t> goff(al, k), tot(al, 1);
      k_gather_len<<<grid_for(k, 256), 256, 0, s>>>(len, tier_ids, k, lens.p);
      EH_LAUNCH("k_gather_len");
      scan_exclusive_u32(lens.p, goff.p, k, tot.p, al, s);
      const uint64_t total = read_scalar(tot.p, s);
      DBuf<uint64_t> keys(al, total), alt(al, total);
      const unsigned g = (unsigned)std::min<uint64_t>(k, (uint64_t)kSMs * 4);
      k_seg_gather<<<g, 512, 0, s>>>(data, sg, tier_ids, k, goff.p, keys.p);
      EH_LAUNCH("k_seg_gather");
      uint64_t* sorted = radix_sort_u64(keys.p, alt.p, total, 32 + bitlen(k - 1), al, s);
      k_seg_scatter<<<g, 512, 0, s>>>(data, sg, tier_ids, k, goff.p, sorted);
      EH_LAUNCH("k_seg_scatter");
      EH_CUDA(cudaStreamSynchronize(s));  // temporaries are released on return
    }
  }
}

void segmented_sort_u32(uint32_t* data, const uint64_t* off16, const uint32_t* len, uint64_t nseg, uint32_t max_len,
                        Allocator& al, cudaStream_t s, eh_graph* fork) {
  if (nseg == 0 || max_len <= 1) return;
  segsort_impl(data, Seg{off16, len, nullptr, nullptr}, nseg, max_len, al, s, fork);
}

void segmented_sort_u32_into(const uint32_t* in, const uint64_t* ioff, uint32_t* out, const uint64_t* off16,
                             const uint32_t* len, uint64_t nseg, uint32_t max_len, Allocator& al, cudaStream_t s,
                             eh_graph* fork) {
  if (nseg == 0 || max_len == 0) return;
  segsort_impl(out, Seg{off16, len, in, ioff}, nseg, max_len, al, s, fork);
}

}  // namespace eh
