// alloc.cu -- the default device allocation path: cudaMallocAsync plus a
// process-wide exact-size cache of large blocks (see eh_internal.cuh).
#include "eh_internal.cuh"

#include <map>
#include <mutex>
#include <unordered_map>

namespace eh {

namespace {

constexpr size_t kCacheMin = 4ull << 20;   // blocks from 4 MB up are cached
constexpr size_t kCacheGran = 2ull << 20;  // their sizes rounded to 2 MB

struct Cached {
  void* p;
  cudaEvent_t ev;  // recorded on the releasing stream at release
};

struct BlockCache {
  std::mutex mu;
  std::map<std::pair<int, size_t>, std::vector<Cached>> free;  // (device, size) -> idle blocks
  std::unordered_map<void*, std::pair<int, size_t>> big;       // live + idle cached blocks
  size_t idle_bytes = 0, cap = 0;
};

BlockCache& cache() {
  static BlockCache* c = new BlockCache;  // never destroyed: blocks outlive static destructors
  return *c;
}

size_t cache_cap() {  // half of the (current) device's memory
  size_t freeb = 0, total = 0;
  if (cudaMemGetInfo(&freeb, &total) != cudaSuccess) { cudaGetLastError(); return 16ull << 30; }
  return total / 2;
}

// free every idle block (caller holds the lock); the stream waits on each block's event
void flush_locked(BlockCache& c, cudaStream_t s) {
  for (auto& kv : c.free)
    for (Cached& b : kv.second) {
      cudaStreamWaitEvent(s, b.ev, 0);
      cudaFreeAsync(b.p, s);
      cudaEventDestroy(b.ev);
      c.big.erase(b.p);
    }
  c.free.clear();
  c.idle_bytes = 0;
}

void* raw_alloc(size_t bytes, cudaStream_t stream) {
  static const bool trace = getenv("EH_ALLOC_TRACE") != nullptr;
  timespec t0, t1;
  if (trace) clock_gettime(CLOCK_MONOTONIC, &t0);
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, bytes, stream);
  if (trace) {
    clock_gettime(CLOCK_MONOTONIC, &t1);
    const double ms = (t1.tv_sec - t0.tv_sec) * 1e3 + (t1.tv_nsec - t0.tv_nsec) * 1e-6;
    if (ms > 2.0) fprintf(stderr, "[eh alloc] cudaMallocAsync(%zu) took %.1f ms\n", bytes, ms);
  }
  if (e == cudaErrorMemoryAllocation) {  // give the cached blocks back and retry once
    cudaGetLastError();
    BlockCache& c = cache();
    {
      std::lock_guard<std::mutex> lk(c.mu);
      flush_locked(c, stream);
    }
    cudaStreamSynchronize(stream);
    e = cudaMallocAsync(&p, bytes, stream);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(e == cudaErrorMemoryAllocation ? EH_ENOMEM : EH_ECUDA, "cudaMallocAsync(%zu): %s", bytes,
         cudaGetErrorString(e));
  }
  return p;
}

}  // namespace

void* block_cache_alloc(size_t bytes, cudaStream_t stream) {
  static const bool off = getenv("EH_NO_BLOCK_CACHE") != nullptr;  // ablation switch
  if (bytes < kCacheMin || off) return raw_alloc(bytes, stream);
  bytes = (bytes + kCacheGran - 1) / kCacheGran * kCacheGran;
  int dev = 0;
  EH_CUDA(cudaGetDevice(&dev));
  BlockCache& c = cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.free.find({dev, bytes});
    if (it != c.free.end() && !it->second.empty()) {
      Cached b = it->second.back();
      it->second.pop_back();
      c.idle_bytes -= bytes;
      EH_CUDA(cudaStreamWaitEvent(stream, b.ev, 0));  // the previous user's work is done first
      cudaEventDestroy(b.ev);
      return b.p;
    }
  }
  void* p = raw_alloc(bytes, stream);
  std::lock_guard<std::mutex> lk(c.mu);
  c.big[p] = {dev, bytes};
  return p;
}

void block_cache_free(void* p, cudaStream_t stream) {
  BlockCache& c = cache();
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.big.find(p);
  if (it == c.big.end()) {  // a small block: straight back to the stream-ordered pool
    cudaFreeAsync(p, stream);
    return;
  }
  const int dev = it->second.first;
  const size_t bytes = it->second.second;
  if (c.cap == 0) c.cap = cache_cap();
  cudaEvent_t ev;
  if (c.idle_bytes + bytes > c.cap || cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    c.big.erase(it);
    cudaFreeAsync(p, stream);
    return;
  }
  cudaEventRecord(ev, stream);
  c.free[{dev, bytes}].push_back(Cached{p, ev});
  c.idle_bytes += bytes;
}

}  // namespace eh
