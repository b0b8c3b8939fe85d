// count_tri.cu -- SURVEY.md §8(a) rows a8 (triangle Generic-Join) and a10
// (warp-shuffle uint64 reduction).
//
// Loop nest with R = S = T = E+ in rank space:
//     for x:  for y in N+(x):  Q += | N+(y) cap N+(x) |
// Because N+(y) lies above y, only the suffix A = N+(x) after y can match,
// so the intersection is |A cap N+(y)|.
// Dispatch on the layout pair:
//   N+(y) bitset         -> probe each a in A into the bitset (uint cap bitset)
//   N+(y) uint, |A|<=|B| -> each a in A binary-searches B   (galloping side)
//   N+(y) uint, |A|>|B|  -> each b in B binary-searches A    (staged in smem)
// COUNT(*) is accumulated per lane in u64, reduced with __shfl_xor_sync and
// added once per warp with atomicAdd(unsigned long long*).
#include "eh_internal.cuh"
#include "primitives.cuh"
#include "sets.cuh"

namespace eh {

namespace {

constexpr int kTriWarps = 8;
constexpr int kTriBlock = kTriWarps * 32;
constexpr int kXCap = 1024;  // N+(x) staged in shared memory when |N+(x)| <= kXCap

__global__ void __launch_bounds__(kTriBlock) k_tri_warp(const uint4* __restrict__ desc, const uint32_t* __restrict__ col,
                                                        const uint32_t* __restrict__ bs,
                                                        const uint32_t* __restrict__ work, uint64_t nwork,
                                                        unsigned long long* __restrict__ ctr) {
  __shared__ __align__(16) uint32_t xs_s[kTriWarps][kXCap];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long cnt = 0;
  for (;;) {
    unsigned long long wi = 0;
    if (lane == 0) wi = atomicAdd(&ctr[1], 1ull);
    wi = __shfl_sync(kFull, wi, 0);
    if (wi >= nwork) break;
    const uint32_t x = work[wi];
    const uint4 dx = desc[x];
    const uint32_t d = dx.y;
    const uint32_t* xg = col + (uint64_t)dx.x * 4;
    const uint32_t* xs = xg;
    if (d <= kXCap) {
      const uint4* src4 = reinterpret_cast<const uint4*>(xg);
      uint4* dst4 = reinterpret_cast<uint4*>(xs_s[w]);
      for (uint32_t k = lane; k < (d + 3) / 4; k += 32) dst4[k] = __ldg(src4 + k);
      __syncwarp();
      xs = xs_s[w];
    }
    for (uint32_t i = 0; i + 1 < d; ++i) {
      const uint32_t y = xs[i];
      const SetRef sy = set_of(desc, col, bs, y);
      if (sy.len == 0) continue;
      const uint32_t a0 = i + 1, na = d - a0;
      if (sy.bits) {
        for (uint32_t j = a0 + lane; j < d; j += 32) cnt += bit_probe(sy, xs[j]);
      } else if (na <= sy.len) {
        for (uint32_t j = a0 + lane; j < d; j += 32) cnt += search_probe(sy.list, sy.len, xs[j]);
      } else {
        for (uint32_t k = lane; k < sy.len; k += 32) cnt += search_probe_any(xs + a0, na, __ldg(sy.list + k));
      }
    }
    __syncwarp();
  }
  cnt = warp_sum(cnt);
  if (lane == 0 && cnt) atomicAdd(&ctr[0], cnt);
}

}  // namespace

uint64_t count_triangles(eh_graph* g) {
  cudaStream_t s = g->stream;
  EH_CUDA(cudaMemsetAsync(g->d_counter, 0, 2 * sizeof(unsigned long long), s));
  const uint64_t nwork = g->n_work[0] + g->n_work[1] + g->n_work[2];
  if (nwork) {
    const unsigned grid = (unsigned)std::min<uint64_t>((nwork + kTriWarps - 1) / kTriWarps, (uint64_t)kSMs * 8);
    k_tri_warp<<<grid, kTriBlock, 0, s>>>(g->desc, g->col, g->bs, g->work, nwork, g->d_counter);
    EH_LAUNCH("k_tri_warp");
  }
  EH_CUDA(cudaMemcpyAsync(g->h_counter, g->d_counter, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaStreamSynchronize(s));
  return g->h_counter[0];
}

}  // namespace eh
