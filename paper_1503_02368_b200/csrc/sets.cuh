// sets.cuh -- device-side views of one set of the trie and membership probes.
//
// A set N+(v) is read either in its uint layout (sorted u32 run in `col`,
// PAPER.md:592) or, when the set-level optimizer chose it, its bitset layout
// (single span, 128-bit chunks at absolute positions).
#pragma once
#include <cstdint>

namespace eh {

struct SetRef {
  const uint32_t* list;  // uint layout: len sorted elements
  const uint32_t* bits;  // bitset layout (nullptr if none): word w of the span is bits[w - 4*c0]
  uint32_t len;
  uint32_t c0, c1;       // chunk range [c0, c1) of the bitset span
};

__device__ __forceinline__ SetRef set_of(const uint4* __restrict__ desc, const uint32_t* __restrict__ col,
                                         const uint32_t* __restrict__ bs, uint32_t v) {
  const uint4 d = desc[v];
  const uint32_t z1 = desc[v + 1].z;
  SetRef s;
  s.list = col + (uint64_t)d.x * 4;
  s.len = d.y;
  s.c0 = d.w;
  s.c1 = d.w + (z1 - d.z);
  s.bits = (z1 != d.z) ? (bs + (uint64_t)d.z * 4) : nullptr;
  return s;
}

// uint cap bitset probe: mask the low bits to find the block,
// then test the bit.  Valid only when s.bits != nullptr.
__device__ __forceinline__ uint32_t bit_probe(const SetRef& s, uint32_t e) {
  const uint32_t c = e >> 7;
  if (c < s.c0 || c >= s.c1) return 0u;
  return (__ldg(s.bits + ((e >> 5) - 4u * s.c0)) >> (e & 31)) & 1u;
}

// lower_bound of e in a sorted array (binary search: the galloping side of the
// uint cap uint hybrid).
__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* __restrict__ a, uint32_t n, uint32_t e) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < e) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ uint32_t search_probe(const uint32_t* __restrict__ a, uint32_t n, uint32_t e) {
  const uint32_t p = lower_bound_u32(a, n, e);
  return (p < n && __ldg(a + p) == e) ? 1u : 0u;
}

// Generic (non-__ldg) variants for arrays that may live in shared memory.
__device__ __forceinline__ uint32_t search_probe_any(const uint32_t* a, uint32_t n, uint32_t e) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < e) lo = mid + 1; else hi = mid;
  }
  return (lo < n && a[lo] == e) ? 1u : 0u;
}

__device__ __forceinline__ uint32_t member(const SetRef& s, uint32_t e) {
  return s.bits ? bit_probe(s, e) : search_probe(s.list, s.len, e);
}

}  // namespace eh
