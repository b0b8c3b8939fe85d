// count_k4.cu -- SURVEY.md §8(a) row a9: the 4-clique Generic-Join.
//
// 4Clique(x,y,z,w) :- R(x,y),S(y,z),T(x,z),U(x,w),V(y,w),Q(z,w),
// attribute order x, y, z, w on the pruned relation:
//     for x:  for y in N+(x):
//        P = N+(x) cap N+(y)                       (materialised per warp, sorted)
//        for z in P:  K += | P cap N+(z) |        (only P after z can match)
// Each intersection uses the same layout dispatch as the triangle kernel.
#include "eh_internal.cuh"
#include "primitives.cuh"
#include "sets.cuh"

namespace eh {

namespace {

constexpr int kK4Warps = 4;
constexpr int kK4Block = kK4Warps * 32;
constexpr int kK4Cap = 1024;  // N+(x) and P staged in shared memory when |N+(x)| <= kK4Cap

__global__ void __launch_bounds__(kK4Block) k_k4_warp(const uint4* __restrict__ desc, const uint32_t* __restrict__ col,
                                                      const uint32_t* __restrict__ bs,
                                                      const uint32_t* __restrict__ work, uint64_t nwork,
                                                      uint32_t* __restrict__ pscratch, uint32_t pstride,
                                                      unsigned long long* __restrict__ ctr) {
  __shared__ __align__(16) uint32_t xs_s[kK4Warps][kK4Cap];
  __shared__ __align__(16) uint32_t ps_s[kK4Warps][kK4Cap];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const uint64_t gw = (uint64_t)blockIdx.x * kK4Warps + w;
  unsigned long long cnt = 0;
  for (;;) {
    unsigned long long wi = 0;
    if (lane == 0) wi = atomicAdd(&ctr[1], 1ull);
    wi = __shfl_sync(kFull, wi, 0);
    if (wi >= nwork) break;
    const uint32_t x = work[wi];
    const uint4 dx = desc[x];
    const uint32_t d = dx.y;
    if (d < 3) continue;
    const uint32_t* xg = col + (uint64_t)dx.x * 4;
    const uint32_t* xs = xg;
    uint32_t* P = pscratch ? pscratch + gw * pstride : nullptr;
    if (d <= kK4Cap) {
      const uint4* src4 = reinterpret_cast<const uint4*>(xg);
      uint4* dst4 = reinterpret_cast<uint4*>(xs_s[w]);
      for (uint32_t k = lane; k < (d + 3) / 4; k += 32) dst4[k] = __ldg(src4 + k);
      __syncwarp();
      xs = xs_s[w];
      P = ps_s[w];
    }
    for (uint32_t i = 0; i + 2 < d; ++i) {
      const uint32_t y = xs[i];
      const SetRef sy = set_of(desc, col, bs, y);
      if (sy.len < 2) continue;
      // P = (N+(x) after y) cap N+(y), kept in increasing order via ballot compaction
      uint32_t np = 0;
      for (uint32_t j0 = i + 1; j0 < d; j0 += 32) {
        const uint32_t j = j0 + lane;
        const uint32_t e = (j < d) ? xs[j] : 0u;
        const uint32_t hit = (j < d) ? member(sy, e) : 0u;
        const unsigned mask = __ballot_sync(kFull, hit);
        if (hit) P[np + __popc(mask & lt)] = e;
        np += __popc(mask);
      }
      __syncwarp();
      // for z in P: K += |P after z cap N+(z)|
      for (uint32_t t = 0; t + 1 < np; ++t) {
        const SetRef sz = set_of(desc, col, bs, P[t]);
        if (sz.len == 0) continue;
        for (uint32_t k = t + 1 + lane; k < np; k += 32) cnt += member(sz, P[k]);
      }
      __syncwarp();
    }
  }
  cnt = warp_sum(cnt);
  if (lane == 0 && cnt) atomicAdd(&ctr[0], cnt);
}

}  // namespace

uint64_t count_4cliques(eh_graph* g) {
  cudaStream_t s = g->stream;
  EH_CUDA(cudaMemsetAsync(g->d_counter, 0, 2 * sizeof(unsigned long long), s));
  const uint64_t nwork = g->n_work[0] + g->n_work[1] + g->n_work[2];
  if (nwork) {
    const unsigned grid = (unsigned)std::min<uint64_t>((nwork + kK4Warps - 1) / kK4Warps, (uint64_t)kSMs * 4);
    DBuf<uint32_t> scratch;
    uint32_t stride = 0;
    if (g->max_dplus > (uint64_t)kK4Cap) {
      stride = (uint32_t)g->max_dplus;
      scratch = DBuf<uint32_t>(g->alloc, (size_t)grid * kK4Warps * stride);
    }
    k_k4_warp<<<grid, kK4Block, 0, s>>>(g->desc, g->col, g->bs, g->work, nwork, scratch.p, stride, g->d_counter);
    EH_LAUNCH("k_k4_warp");
    EH_CUDA(cudaMemcpyAsync(g->h_counter, g->d_counter, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    EH_CUDA(cudaStreamSynchronize(s));
    return g->h_counter[0];
  }
  return 0;
}

}  // namespace eh
