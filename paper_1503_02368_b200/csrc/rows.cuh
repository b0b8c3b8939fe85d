// rows.cuh -- per-row (edge (x, y)) helpers shared by the triangle and 4-clique
// kernels: the descriptor of N+(y), the uint cap bitset probe and the global
// binary search (galloping side of the uint hybrid).
#pragma once
#include <cstdint>

#include "check.cuh"

namespace eh {

// desc[v].w of every set of an EH_NO_ALGO graph (all uint): row dispatch never
// chooses the galloping (binary-search) side -- the paper's "-RA" ablation.
constexpr uint32_t kNoAlgo = 0xFFFFFFFFu;
// EH_FORCE_SEARCH (all uint): row dispatch always chooses the galloping side.
constexpr uint32_t kAlwaysSearch = 0xFFFFFFFEu;

struct YInfo {
  uint32_t list;  // col offset of N+(y) in 16-B units
  uint32_t len;   // |N+(y)|
  uint32_t pool;  // bitset pool offset of chunk c0 in 16-B chunks (if bitset)
  uint32_t c0;    // first chunk
  uint32_t c1;    // one past last chunk (c1 == c0: no bitset)
};

__device__ __forceinline__ YInfo yinfo(const uint4* __restrict__ desc, uint32_t y) {
  const uint4 d = __ldg(desc + y);
  const uint32_t z1 = __ldg(&desc[y + 1].z);
  return YInfo{d.x, d.y, d.z, d.w, d.w + (z1 - d.z)};
}

// uint cap bitset: mask the low bits to find the chunk, test the bit.
__device__ __forceinline__ uint32_t probe_bits(const uint32_t* __restrict__ bs, const YInfo& y, uint32_t e) {
  const uint32_t c = e >> 7;
  if (c < y.c0 || c >= y.c1) return 0u;
  return (__ldg(bs + (uint64_t)y.pool * 4 + ((e >> 5) - 4u * y.c0)) >> (e & 31)) & 1u;
}

__device__ __forceinline__ uint32_t gmem_search(const uint32_t* __restrict__ a, uint32_t n, uint32_t e) {
  uint32_t lo = 0, len = n;
  while (len > 0) {
    const uint32_t h = len >> 1;
    if (__ldg(a + lo + h) < e) { lo += h + 1; len -= h + 1; } else { len = h; }
  }
  return (lo < n && __ldg(a + lo) == e) ? 1u : 0u;
}

}  // namespace eh
