// primitives.cuh -- warp / block building blocks shared by the libeh kernels.
#pragma once
#include <cstdint>

namespace eh {

constexpr unsigned kFull = 0xFFFFFFFFu;

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// Sum over the block; every thread gets the total.  sw: BLOCK/32 entries.
template <int BLOCK, typename T>
__device__ __forceinline__ T block_reduce_sum(T v, T* sw) {
  constexpr int NW = BLOCK / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sw[w] = v;
  __syncthreads();
  T t = (lane < NW) ? sw[lane] : T(0);
  t = warp_sum(t);
  __syncthreads();
  return t;
}

// Exclusive scan over the block (thread order).  sw: BLOCK/32 + 1 entries.
template <int BLOCK, typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* sw, T* total) {
  constexpr int NW = BLOCK / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const T inc = warp_inclusive_scan(v);
  if (lane == 31) sw[w] = inc;
  __syncthreads();
  if (w == 0) {
    T x = (lane < NW) ? sw[lane] : T(0);
    x = warp_inclusive_scan(x);
    if (lane < NW) sw[lane] = x;
  }
  __syncthreads();
  const T wp = (w > 0) ? sw[w - 1] : T(0);
  *total = sw[NW - 1];
  __syncthreads();
  return wp + inc - v;
}

}  // namespace eh

// ------------------------------------------------------------- select_if --
// Stable device-wide selection: for i in [0, n) with pred(i), call
// emit(pos, i) where pos is the rank of i among selected indices.  Two passes
// over the predicate (count per tile, then scan + emit), so no flag or offset
// array is materialised.  Returns the number selected (host-synchronising).
#include "eh_internal.cuh"

namespace eh {

constexpr int kSelBlock = 512;
constexpr int kSelItems = 8;
constexpr int kSelTile = kSelBlock * kSelItems;

template <class Pred>
__global__ void __launch_bounds__(kSelBlock) k_select_count(uint64_t n, Pred pred, uint64_t* __restrict__ tile_cnt) {
  __shared__ uint64_t sw[kSelBlock / 32];
  const uint64_t base = (uint64_t)blockIdx.x * kSelTile + (uint64_t)threadIdx.x * kSelItems;
  uint64_t c = 0;
#pragma unroll
  for (int k = 0; k < kSelItems; ++k)
    if (base + k < n && pred(base + k)) ++c;
  c = block_reduce_sum<kSelBlock>(c, sw);
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = c;
}

template <class Pred, class Emit>
__global__ void __launch_bounds__(kSelBlock) k_select_emit(uint64_t n, Pred pred, Emit emit,
                                                           const uint64_t* __restrict__ tile_off) {
  __shared__ uint64_t sw[kSelBlock / 32 + 1];
  const uint64_t base = (uint64_t)blockIdx.x * kSelTile + (uint64_t)threadIdx.x * kSelItems;
  uint32_t bits = 0;
  uint64_t c = 0;
#pragma unroll
  for (int k = 0; k < kSelItems; ++k)
    if (base + k < n && pred(base + k)) { bits |= 1u << k; ++c; }
  uint64_t tot;
  uint64_t pos = block_exclusive_scan<kSelBlock>(c, sw, &tot) + tile_off[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kSelItems; ++k)
    if (bits & (1u << k)) emit(pos++, base + k);
}

template <class Pred, class Emit>
uint64_t select_if(uint64_t n, Pred pred, Emit emit, Allocator& al, cudaStream_t s) {
  if (n == 0) return 0;
  const uint64_t nt = (n + kSelTile - 1) / kSelTile;
  DBuf<uint64_t> cnt(al, nt), tot(al, 1);
  k_select_count<Pred><<<(unsigned)nt, kSelBlock, 0, s>>>(n, pred, cnt.p);
  EH_LAUNCH("k_select_count");
  scan_exclusive_u64(cnt.p, cnt.p, nt, tot.p, al, s);
  k_select_emit<Pred, Emit><<<(unsigned)nt, kSelBlock, 0, s>>>(n, pred, emit, cnt.p);
  EH_LAUNCH("k_select_emit");
  return read_scalar(tot.p, s);
}

// select_if when the caller already knows the count: no host synchronisation.
template <class Pred, class Emit>
void select_emit(uint64_t n, Pred pred, Emit emit, Allocator& al, cudaStream_t s) {
  if (n == 0) return;
  const uint64_t nt = (n + kSelTile - 1) / kSelTile;
  DBuf<uint64_t> cnt(al, nt), tot(al, 1);
  k_select_count<Pred><<<(unsigned)nt, kSelBlock, 0, s>>>(n, pred, cnt.p);
  EH_LAUNCH("k_select_count");
  scan_exclusive_u64(cnt.p, cnt.p, nt, tot.p, al, s);
  k_select_emit<Pred, Emit><<<(unsigned)nt, kSelBlock, 0, s>>>(n, pred, emit, cnt.p);
  EH_LAUNCH("k_select_emit");
}

// ---------------------------------------------------------- partition_k --
// Stable multi-way partition: klass(i) in [0, C) or -1 (dropped) for i in [0, n);
// emit(c, pos, i) with pos the rank of i among the selected indices of class c.
// One count pass (per-tile class counts, class-major), ONE exclusive scan of the
// C x tiles counts, one emit pass, one host read of the C totals -- instead of C
// select_if calls with a host synchronisation each.
constexpr int kPartMaxC = 8;

template <int C, class Klass>
__global__ void __launch_bounds__(kSelBlock) k_part_count(uint64_t n, Klass klass, uint64_t ntiles,
                                                          uint64_t* __restrict__ cnt) {
  __shared__ uint32_t sc[C];
  if (threadIdx.x < C) sc[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kSelTile + (uint64_t)threadIdx.x * kSelItems;
  uint32_t mine[C];
#pragma unroll
  for (int c = 0; c < C; ++c) mine[c] = 0;
#pragma unroll
  for (int k = 0; k < kSelItems; ++k) {
    if (base + k >= n) break;
    const int c = klass(base + k);
#pragma unroll
    for (int q = 0; q < C; ++q) mine[q] += (c == q);
  }
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const uint32_t v = warp_sum(mine[c]);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&sc[c], v);
  }
  __syncthreads();
  if (threadIdx.x < C) cnt[(uint64_t)threadIdx.x * ntiles + blockIdx.x] = sc[threadIdx.x];
}

template <int C, class Klass, class Emit>
__global__ void __launch_bounds__(kSelBlock) k_part_emit(uint64_t n, Klass klass, Emit emit, uint64_t ntiles,
                                                         const uint64_t* __restrict__ off) {
  __shared__ uint64_t sw[kSelBlock / 32 + 1];
  const uint64_t base = (uint64_t)blockIdx.x * kSelTile + (uint64_t)threadIdx.x * kSelItems;
  int cls[kSelItems];
#pragma unroll
  for (int k = 0; k < kSelItems; ++k) cls[k] = (base + k < n) ? klass(base + k) : -1;
#pragma unroll 1
  for (int c = 0; c < C; ++c) {
    uint64_t m = 0;
#pragma unroll
    for (int k = 0; k < kSelItems; ++k) m += (cls[k] == c);
    uint64_t tot;
    uint64_t pos = block_exclusive_scan<kSelBlock>(m, sw, &tot) + off[(uint64_t)c * ntiles + blockIdx.x];
    if (m) {
#pragma unroll
      for (int k = 0; k < kSelItems; ++k)
        if (cls[k] == c) emit(c, pos++, base + k);
    }
  }
}

template <int C>
__global__ void k_part_starts(const uint64_t* __restrict__ off, const uint64_t* __restrict__ total, uint64_t ntiles,
                              uint64_t* __restrict__ starts) {
  const int c = threadIdx.x;
  if (c < C) starts[c] = off[(uint64_t)c * ntiles];
  if (c == C) starts[C] = *total;
}

// The positions are global: class c's indices land in [starts[c], starts[c+1]) of
// one output (class-major, each class in index order).  Returns starts[0..C].
// Device-side variant: d_starts (C + 2 entries, caller-owned) receives starts[0..C]
// on the stream; no host synchronisation.
template <int C, class Klass, class Emit>
void partition_k_async(uint64_t n, Klass klass, Emit emit, uint64_t* d_starts, Allocator& al, cudaStream_t s) {
  static_assert(C <= kPartMaxC, "classes");
  if (n == 0) {
    EH_CUDA(cudaMemsetAsync(d_starts, 0, (C + 2) * sizeof(uint64_t), s));
    return;
  }
  const uint64_t nt = (n + kSelTile - 1) / kSelTile;
  DBuf<uint64_t> cnt(al, (size_t)C * nt), off(al, (size_t)C * nt);
  k_part_count<C, Klass><<<(unsigned)nt, kSelBlock, 0, s>>>(n, klass, nt, cnt.p);
  EH_LAUNCH("k_part_count");
  scan_exclusive_u64(cnt.p, off.p, (uint64_t)C * nt, d_starts + C + 1, al, s);
  k_part_emit<C, Klass, Emit><<<(unsigned)nt, kSelBlock, 0, s>>>(n, klass, emit, nt, off.p);
  EH_LAUNCH("k_part_emit");
  k_part_starts<C><<<1, 32, 0, s>>>(off.p, d_starts + C + 1, nt, d_starts);
  EH_LAUNCH("k_part_starts");
}

template <int C, class Klass, class Emit>
void partition_k(uint64_t n, Klass klass, Emit emit, uint64_t starts[C + 1], Allocator& al, cudaStream_t s) {
  DBuf<uint64_t> st(al, C + 2);
  partition_k_async<C>(n, klass, emit, st.p, al, s);
  EH_CUDA(cudaMemcpyAsync(starts, st.p, (C + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaStreamSynchronize(s));
}

}  // namespace eh
