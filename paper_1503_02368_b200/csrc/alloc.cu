// alloc.cu -- the default device allocation path: a library-private
// stream-ordered memory pool per device (cudaMemPoolCreate; the device's default
// pool, shared with torch / CuPy / ..., is never touched) plus a process-wide
// exact-size cache of large blocks (see eh_internal.cuh).  Both hold memory
// until eh_release_cached_memory() (or an allocation failure) gives it back.
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

constexpr int kMaxDev = 64;

struct BlockCache {
  std::mutex mu;
  std::map<std::pair<int, size_t>, std::vector<Cached>> free;  // (device, size) -> idle blocks
  std::unordered_map<void*, std::pair<int, size_t>> big;       // live + idle cached blocks
  size_t idle_bytes = 0, cap = 0;
  cudaMemPool_t pool[kMaxDev] = {};  // private pools, created on first use
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

// The library's pool on device dev (caller holds the lock).  Its release threshold
// is unbounded: freed memory stays mapped for the next load (re-mapping costs
// ~100 ms per load at C3 size and up to seconds at C5) until trimmed.
cudaMemPool_t pool_locked(BlockCache& c, int dev) {
  if (dev < 0 || dev >= kMaxDev) fail(EH_EINVAL, "device ordinal %d out of range", dev);
  if (!c.pool[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p;
    EH_CUDA(cudaMemPoolCreate(&p, &props));
    uint64_t thr = UINT64_MAX;
    EH_CUDA(cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr));
    c.pool[dev] = p;
  }
  return c.pool[dev];
}

cudaMemPool_t pool_for(int dev) {
  BlockCache& c = cache();
  std::lock_guard<std::mutex> lk(c.mu);
  return pool_locked(c, dev);
}

void* raw_alloc(size_t bytes, cudaStream_t stream) {
  static const bool trace = getenv("EH_ALLOC_TRACE") != nullptr;
  timespec t0, t1;
  if (trace) clock_gettime(CLOCK_MONOTONIC, &t0);
  int dev = 0;
  EH_CUDA(cudaGetDevice(&dev));
  const cudaMemPool_t pool = pool_for(dev);
  void* p = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, pool, stream);
  if (trace) {
    clock_gettime(CLOCK_MONOTONIC, &t1);
    const double ms = (t1.tv_sec - t0.tv_sec) * 1e3 + (t1.tv_nsec - t0.tv_nsec) * 1e-6;
    if (ms > 2.0) fprintf(stderr, "[eh alloc] cudaMallocAsync(%zu) took %.1f ms\n", bytes, ms);
  }
  if (e == cudaErrorMemoryAllocation) {  // give the cached blocks back (to the driver) and retry once
    cudaGetLastError();
    BlockCache& c = cache();
    {
      std::lock_guard<std::mutex> lk(c.mu);
      flush_locked(c, stream);
    }
    cudaStreamSynchronize(stream);
    cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocFromPoolAsync(&p, bytes, pool, stream);
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

void release_cached_memory() {
  BlockCache& c = cache();
  std::lock_guard<std::mutex> lk(c.mu);
  int prev = -1;
  cudaGetDevice(&prev);
  for (auto& kv : c.free)
    for (Cached& b : kv.second) {
      cudaSetDevice(kv.first.first);
      cudaEventSynchronize(b.ev);  // the last user's work on the block is done
      cudaFreeAsync(b.p, 0);
      cudaEventDestroy(b.ev);
      c.big.erase(b.p);
    }
  c.free.clear();
  c.idle_bytes = 0;
  for (int d = 0; d < kMaxDev; ++d)
    if (c.pool[d]) {
      cudaSetDevice(d);
      cudaDeviceSynchronize();  // frees still pending in some stream complete first
      cudaMemPoolTrimTo(c.pool[d], 0);
    }
  if (prev >= 0) cudaSetDevice(prev);
  cudaGetLastError();
}

}  // namespace eh
