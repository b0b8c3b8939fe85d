// intersect.cu -- the set operation "xs cap ys" (Table `lst:eh_operators`,
// PAPER.md:515-516) behind eh_intersect, with the paper's layout-dependent
// algorithms (set-level layouts PAPER.md:730):
//   * each input gets the set-level layout: bitset iff span < 32 |S| (|S| >= 2);
//   * uint  cap uint  : merge (merge-path partitioned over threads) when the
//                       cardinality ratio is <= 32, else every element of the
//                       smaller set binary-searches the larger ("galloping",
//                       PAPER.md:634; strict > 32, reading c13);
//   * uint  cap bitset: mask the low bits and probe the block;
//   * bitset cap bitset: AND of the overlapping 128-bit chunks.
// The result is always a sorted uint32 array (reading c14).
#include "eh_internal.cuh"
#include "primitives.cuh"

#include <algorithm>

namespace eh {

namespace {

constexpr uint32_t kTauIntersect = 32;

__global__ void k_check_sorted(const uint32_t* __restrict__ a, uint64_t n, uint32_t* __restrict__ bad) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (a[i] >= a[i + 1]) *bad = 1u;
}

__global__ void k_build_bits(const uint32_t* __restrict__ a, uint64_t n, uint32_t c0, uint32_t* __restrict__ bits) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t e = a[i];
    atomicOr(&bits[(e >> 5) - 4ull * c0], 1u << (e & 31));
  }
}

// uint cap bitset: flag[i] = a[i] in bits.
__global__ void k_probe_bits(const uint32_t* __restrict__ a, uint64_t n, const uint32_t* __restrict__ bits,
                             uint32_t c0, uint32_t c1, uint32_t* __restrict__ flag) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t e = a[i], c = e >> 7;
    flag[i] = (c >= c0 && c < c1) ? ((bits[(e >> 5) - 4ull * c0] >> (e & 31)) & 1u) : 0u;
  }
}

// galloping side: flag[i] = a[i] in b (binary search over b).
__global__ void k_probe_search(const uint32_t* __restrict__ a, uint64_t na, const uint32_t* __restrict__ b,
                               uint64_t nb, uint32_t* __restrict__ flag) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t e = a[i];
    uint64_t lo = 0, hi = nb;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (b[mid] < e) lo = mid + 1; else hi = mid;
    }
    flag[i] = (lo < nb && b[lo] == e) ? 1u : 0u;
  }
}

// merge side: the merge of a and b (a[i] before b[j] iff a[i] <= b[j]) is cut
// into windows of kMergeSteps steps along the merge path; each thread finds its
// start by binary search on its diagonal and merges its window, flagging a[i]
// when it meets an equal b[j].
constexpr int kMergeSteps = 16;
__global__ void k_merge_path(const uint32_t* __restrict__ a, uint64_t na, const uint32_t* __restrict__ b,
                             uint64_t nb, uint32_t* __restrict__ flag) {
  const uint64_t total = na + nb;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t * kMergeSteps < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = t * kMergeSteps;
    uint64_t lo = (k > nb) ? k - nb : 0, hi = std::min<uint64_t>(k, na);
    while (lo < hi) {
      const uint64_t mid = (lo + hi + 1) >> 1;
      if (a[mid - 1] <= b[k - mid]) lo = mid; else hi = mid - 1;
    }
    uint64_t i = lo, j = k - lo;
    const uint64_t kend = std::min<uint64_t>(total, k + kMergeSteps);
    for (uint64_t step = k; step < kend; ++step) {
      if (i < na && (j >= nb || a[i] <= b[j])) {
        flag[i] = (j < nb && a[i] == b[j]) ? 1u : 0u;
        ++i;
      } else {
        ++j;
      }
    }
  }
}

struct FlagPred {
  const uint32_t* f;
  __device__ bool operator()(uint64_t i) const { return f[i] != 0; }
};
struct CopyEmit {
  const uint32_t* a;
  uint32_t* out;
  __device__ void operator()(uint64_t pos, uint64_t i) const { if (out) out[pos] = a[i]; }
};

// bitset cap bitset: AND the overlapping chunks, then decode in order.
__global__ void k_and_words(const uint32_t* __restrict__ ba, uint32_t ca0, const uint32_t* __restrict__ bb,
                            uint32_t cb0, uint64_t w0, uint64_t nw, uint32_t* __restrict__ wout,
                            uint32_t* __restrict__ wcnt) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t w = w0 + i;  // absolute word
    const uint32_t v = ba[w - 4ull * ca0] & bb[w - 4ull * cb0];
    wout[i] = v;
    wcnt[i] = __popc(v);
  }
}
__global__ void k_decode_words(const uint32_t* __restrict__ wv, const uint64_t* __restrict__ pos, uint64_t w0,
                               uint64_t nw, uint32_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v = wv[i];
    uint64_t p = pos[i];
    while (v) {
      const int bit = __ffs(v) - 1;
      out[p++] = (uint32_t)((w0 + i) * 32 + bit);
      v &= v - 1;
    }
  }
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) { cudaGetLastError(); return false; }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

struct Layout {
  bool bitset = false;
  uint32_t c0 = 0, c1 = 0;
  DBuf<uint32_t> bits;
};

}  // namespace

int64_t intersect(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb, uint32_t* out) {
  if ((na && !a) || (nb && !b)) fail(EH_EINVAL, "eh_intersect: NULL input with non-zero length");
  int dev = 0;
  EH_CUDA(cudaGetDevice(&dev));
  cudaStream_t s = cudaStreamPerThread;
  Allocator al;
  al.stream = s;
  const unsigned TB = 256;
  // inputs on the device
  DBuf<uint32_t> ha, hb;
  const uint32_t* da = a;
  const uint32_t* db = b;
  if (na && !is_device_ptr(a)) {
    ha = DBuf<uint32_t>(al, na);
    EH_CUDA(cudaMemcpyAsync(ha.p, a, na * 4, cudaMemcpyHostToDevice, s));
    da = ha.p;
  }
  if (nb && !is_device_ptr(b)) {
    hb = DBuf<uint32_t>(al, nb);
    EH_CUDA(cudaMemcpyAsync(hb.p, b, nb * 4, cudaMemcpyHostToDevice, s));
    db = hb.p;
  }
  // validate strict increase, O(na + nb)
  DBuf<uint32_t> bad(al, 1);
  EH_CUDA(cudaMemsetAsync(bad.p, 0, 4, s));
  if (na > 1) {
    k_check_sorted<<<grid_for(na, TB * 4), TB, 0, s>>>(da, na, bad.p);
    EH_LAUNCH("k_check_sorted");
  }
  if (nb > 1) {
    k_check_sorted<<<grid_for(nb, TB * 4), TB, 0, s>>>(db, nb, bad.p);
    EH_LAUNCH("k_check_sorted");
  }
  if (read_scalar(bad.p, s)) fail(EH_EUNSORTED, "eh_intersect: input not strictly increasing");
  if (na == 0 || nb == 0) return 0;
  // smaller set plays `a`
  if (na > nb) { std::swap(da, db); std::swap(na, nb); }
  // set-level layouts
  uint32_t ends[4];
  EH_CUDA(cudaMemcpyAsync(&ends[0], da, 4, cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaMemcpyAsync(&ends[1], da + na - 1, 4, cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaMemcpyAsync(&ends[2], db, 4, cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaMemcpyAsync(&ends[3], db + nb - 1, 4, cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaStreamSynchronize(s));
  Layout la, lb;
  auto choose = [&](Layout& L, const uint32_t* d, uint64_t n, uint32_t first, uint32_t last) {
    const uint64_t span = (uint64_t)last - first + 1;
    if (n >= 2 && span < (uint64_t)kTauIntersect * n) {
      L.bitset = true;
      L.c0 = first >> 7;
      L.c1 = (last >> 7) + 1;
      const uint64_t words = 4ull * (L.c1 - L.c0);
      L.bits = DBuf<uint32_t>(al, words);
      EH_CUDA(cudaMemsetAsync(L.bits.p, 0, words * 4, s));
      k_build_bits<<<grid_for(n, TB * 4), TB, 0, s>>>(d, n, L.c0, L.bits.p);
      EH_LAUNCH("k_build_bits");
    }
  };
  choose(la, da, na, ends[0], ends[1]);
  choose(lb, db, nb, ends[2], ends[3]);
  const bool out_dev = out && is_device_ptr(out);
  DBuf<uint32_t> dout;
  uint32_t* o = nullptr;
  if (out) {
    if (out_dev) o = out;
    else { dout = DBuf<uint32_t>(al, na); o = dout.p; }
  }
  uint64_t count = 0;
  if (la.bitset && lb.bitset) {
    const uint32_t c0 = std::max(la.c0, lb.c0), c1 = std::min(la.c1, lb.c1);
    if (c0 < c1) {
      const uint64_t nw = 4ull * (c1 - c0), w0 = 4ull * c0;
      DBuf<uint32_t> wv(al, nw), wc(al, nw);
      DBuf<uint64_t> pos(al, nw), tot(al, 1);
      k_and_words<<<grid_for(nw, TB * 4), TB, 0, s>>>(la.bits.p, la.c0, lb.bits.p, lb.c0, w0, nw, wv.p, wc.p);
      EH_LAUNCH("k_and_words");
      scan_exclusive_u32(wc.p, pos.p, nw, tot.p, al, s);
      count = read_scalar(tot.p, s);
      if (o && count) {
        k_decode_words<<<grid_for(nw, TB * 4), TB, 0, s>>>(wv.p, pos.p, w0, nw, o);
        EH_LAUNCH("k_decode_words");
      }
    }
  } else {
    DBuf<uint32_t> flag(al, na);
    const uint32_t* probe = da;  // uint side whose elements are flagged
    uint64_t nprobe = na;
    if (lb.bitset) {
      k_probe_bits<<<grid_for(na, TB * 4), TB, 0, s>>>(da, na, lb.bits.p, lb.c0, lb.c1, flag.p);
    } else if (la.bitset) {
      flag = DBuf<uint32_t>(al, nb);
      probe = db;
      nprobe = nb;
      k_probe_bits<<<grid_for(nb, TB * 4), TB, 0, s>>>(db, nb, la.bits.p, la.c0, la.c1, flag.p);
    } else if (nb > 32 * na) {
      k_probe_search<<<grid_for(na, TB * 4), TB, 0, s>>>(da, na, db, nb, flag.p);
    } else {
      EH_CUDA(cudaMemsetAsync(flag.p, 0, na * 4, s));
      k_merge_path<<<grid_for((na + nb + kMergeSteps - 1) / kMergeSteps, TB), TB, 0, s>>>(da, na, db, nb, flag.p);
    }
    EH_LAUNCH("intersect probe");
    count = select_if(nprobe, FlagPred{flag.p}, CopyEmit{probe, o}, al, s);
  }
  if (out && !out_dev && count) EH_CUDA(cudaMemcpyAsync(out, o, count * 4, cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaStreamSynchronize(s));
  return (int64_t)count;
}

}  // namespace eh
