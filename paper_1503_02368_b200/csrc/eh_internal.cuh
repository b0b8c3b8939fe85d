// eh_internal.cuh -- internal types, error plumbing and allocation for libeh.
// Product code (sm_100a).  Shares nothing with oracle/.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "check.cuh"
#include "eh.h"

namespace eh {

constexpr uint32_t kNone = 0xFFFFFFFFu;  // pad value of `col` (masked by length, never by value)
constexpr int kSMs = 148;

// Internal failures are C++ exceptions caught at the ABI boundary (eh_api.cu).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  throw Error(code, buf);
}

inline void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    const int code = (e == cudaErrorMemoryAllocation) ? EH_ENOMEM : EH_ECUDA;
    cudaGetLastError();  // clear sticky-free errors
    fail(code, "%s: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
  }
}
#define EH_CUDA(call) ::eh::check_cuda((call), #call, __FILE__, __LINE__)
// Every kernel launch is followed by exactly one EH_LAUNCH, which also counts it
// (eh_launch_count(), used by bench.py's "gpu_launches").
extern std::atomic<unsigned long long> g_launches;
#define EH_LAUNCH(what) \
  (::eh::g_launches.fetch_add(1, std::memory_order_relaxed), \
   ::eh::check_cuda(cudaGetLastError(), what, __FILE__, __LINE__))

// Raises a kernel's dynamic shared-memory limit to at least `bytes` on the current device.
// The limit only ever grows (per device and kernel): two host threads launching the same
// kernel with different sizes (eh_count_batch's lanes) cannot lower it under each other.
void ensure_dyn_smem(const void* kernel, size_t bytes);
// Asks for the largest shared-memory carveout for a kernel whose residency is bounded by
// shared memory (the default heuristic sized the carveout for ONE 32 KB CTA of the bucket
// histogram / partition kernels: `launch__occupancy_limit_shared_mem` 1 instead of 2).
void prefer_max_smem_carveout(const void* kernel);

// Device allocator: the caller's hooks (e.g. torch's caching allocator) or cudaMallocAsync.
// Default device allocation path (no allocator hook): cudaMallocAsync on the
// handle's stream, with a process-wide cache of large blocks (>= 4 MB, sizes
// rounded to 2 MB) reused by exact size across loads -- at C5 scale (10.7 GB key
// buffers) the stream-ordered pool alone re-maps memory on later loads, with single
// cudaMallocAsync calls blocking for up to 1.8 s.  A cached block carries an event
// recorded at its release; a new user waits on it (stream order is preserved
// across streams).  Cache size is bounded; on allocation failure it is flushed and
// the allocation retried once.  (alloc.cu)
void* block_cache_alloc(size_t bytes, cudaStream_t stream);
void block_cache_free(void* p, cudaStream_t stream);
// Give every idle cached block and the unused memory of the private pools back
// to the driver (eh_release_cached_memory).
void release_cached_memory();

struct Allocator {
  void* (*hook_alloc)(size_t, void*, void*) = nullptr;
  void (*hook_free)(void*, void*, void*) = nullptr;
  void* ctx = nullptr;
  cudaStream_t stream = nullptr;

  void* alloc(size_t bytes) {
    if (bytes == 0) bytes = 16;
    bytes = (bytes + 255) & ~size_t(255);
    void* p = nullptr;
    if (hook_alloc) {
      p = hook_alloc(bytes, (void*)stream, ctx);
      if (!p) fail(EH_ENOMEM, "allocator hook returned NULL for %zu bytes", bytes);
    } else {
      p = block_cache_alloc(bytes, stream);
    }
    return p;
  }
  void release(void* p) {
    if (!p) return;
    if (hook_free) hook_free(p, (void*)stream, ctx);
    else block_cache_free(p, stream);
  }
};

// RAII device buffer bound to an Allocator.
template <typename T>
struct DBuf {
  Allocator* a = nullptr;
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(Allocator& al, size_t count) : a(&al), p((T*)al.alloc(count * sizeof(T))), n(count) {}
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : a(o.a), p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { reset(); a = o.a; p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { reset(); }
  void reset() { if (p && a) a->release(p); p = nullptr; n = 0; }
  T* release_ptr() { T* q = p; p = nullptr; n = 0; return q; }
  size_t bytes() const { return n * sizeof(T); }
};

inline uint32_t bitlen(uint64_t v) {  // number of bits needed to represent v (0 -> 0)
  uint32_t b = 0;
  while (v) { ++b; v >>= 1; }
  return b;
}

inline unsigned grid_for(uint64_t work, unsigned per_block, unsigned cap = kSMs * 16) {
  uint64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

// ---------------------------------------------------------------- primitives
// (primitives.cu)  device-wide exclusive scan of u32 or u64 counts into u64
// offsets; the total is written to *d_total (device) when non-null.
void scan_exclusive_u32(const uint32_t* in, uint64_t* out, uint64_t n, uint64_t* d_total, Allocator& al,
                        cudaStream_t s);
void scan_exclusive_u64(const uint64_t* in, uint64_t* out, uint64_t n, uint64_t* d_total, Allocator& al,
                        cudaStream_t s);

// LSD radix sort of u64 keys over bits [0, key_bits), 8-bit digits, stable.
// Returns the buffer holding the result (keys or alt).
uint64_t* radix_sort_u64(uint64_t* keys, uint64_t* alt, uint64_t n, uint32_t key_bits, Allocator& al,
                         cudaStream_t s, uint32_t begin_bit = 0);
// a1 + a2 fused: sort the canonical keys (min << b) | max of (src[i], dst[i]) (self-loops -> the
// all-ones sentinel of 2b bits) without materialising them first; keys / alt: n-element buffers
uint64_t* radix_sort_canon(const uint32_t* src, const uint32_t* dst, uint64_t n, uint32_t b, uint64_t* keys,
                           uint64_t* alt, Allocator& al, cudaStream_t s);
// Sort segment v = data[off16[v]*4 .. + len[v]) in place for v < nseg (segsort.cu).
// fork: a handle whose side streams the independent tier kernels may use (nullptr: one stream).
void segmented_sort_u32(uint32_t* data, const uint64_t* off16, const uint32_t* len, uint64_t nseg, uint32_t max_len,
                        Allocator& al, cudaStream_t s, eh_graph* fork = nullptr);
// Out of place: segment v = in[ioff[v] .. + len[v]) sorted into out[off16[v]*4 ..) (segments of one
// element are copied; pads between output segments are left untouched).
void segmented_sort_u32_into(const uint32_t* in, const uint64_t* ioff, uint32_t* out, const uint64_t* off16,
                             const uint32_t* len, uint64_t nseg, uint32_t max_len, Allocator& al, cudaStream_t s,
                             eh_graph* fork = nullptr);
// Same for u32 keys.
uint32_t* radix_sort_u32(uint32_t* keys, uint32_t* alt, uint64_t n, uint32_t key_bits, Allocator& al,
                         cudaStream_t s);

// Optional phase timing (EH_TIMING=1 in the environment): CUDA events between
// phases, reported on stderr.  Development aid; off by default.
struct PhaseTimer {
  cudaStream_t s;
  bool on;
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  std::vector<double> host_ms;
  static double now_ms() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
  }
  explicit PhaseTimer(cudaStream_t st) : s(st) {
    const char* e = getenv("EH_TIMING");
    on = e && e[0] == '1';
    mark("start");
  }
  void mark(const char* name) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.emplace_back(name, e);
    host_ms.push_back(now_ms());
  }
  void report(const char* what) {
    if (!on || ev.size() < 2) return;
    cudaEventSynchronize(ev.back().second);
    fprintf(stderr, "[eh timing] %s (gpu ms / host ms at mark):", what);
    for (size_t i = 1; i < ev.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
      fprintf(stderr, " %s=%.3f/%.3f", ev[i].first, ms, host_ms[i] - host_ms[i - 1]);
    }
    fprintf(stderr, "\n");
  }
  ~PhaseTimer() {
    for (auto& p : ev) cudaEventDestroy(p.second);
  }
};

template <typename T>
inline T read_scalar(const T* d, cudaStream_t s) {
  T h;
  EH_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  EH_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace eh

// ------------------------------------------------------------- the handle --
struct eh_graph {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  eh::Allocator alloc;
  uint32_t flags = 0, tau = 32, min_bitset_card = 2;
  uint32_t bin_small_max = 0, bin_large_min = 0, bin_thread_max = 0;
  uint32_t order = 0;  // NEXT-4: EH_ORDER_*

  uint64_t n_input = 0, m = 0, n_act = 0, max_dplus = 0;
  uint64_t n_bitsets = 0, bs_words = 0, col_elems = 0;
  uint64_t alg_bytes_tri = 0, wedge_work = 0;
  uint64_t alg_bytes_k4 = 0;  // B_K4(tau = 32), computed on first request (eh_alg_bytes_k4)

  // Device trie (rank space).  desc[v] = {col offset in 16-B units, |N+(v)|,
  // bitset pool offset in 16-B chunks (prefix; n_chunks = desc[v+1].z - desc[v].z),
  // first 128-bit chunk index of the bitset span}; desc has n_act+1 entries.
  uint4* desc = nullptr;
  uint32_t* col = nullptr;      // padded per list to 4 elements with kNone
  uint32_t* bs = nullptr;       // bitset pool (128-bit aligned chunks at absolute id/128)
  uint32_t* orig_id = nullptr;  // original id of each rank
  uint32_t* deg_rank = nullptr; // degree (distinct neighbours) of each rank
  uint32_t* bytes32 = nullptr;  // bytes(N+(v)) at tau = 32 (B_tri accounting)
  // NEXT-3 block-level (composite) layout, built with EH_BLOCK_LAYOUT (trie.cu):
  // bdesc[v] = {sparse list offset (16-B units in bcol), #sparse elements, first dense
  // block (prefix into bcid / bmask), 0}; #dense blocks = bdesc[v+1].z - bdesc[v].z.
  uint4* bdesc = nullptr;
  uint32_t* bcol = nullptr;     // sparse elements, padded per list to 16 B
  uint32_t* bcid = nullptr;     // dense 128-id block numbers (absolute), ascending per set
  uint4* bmask = nullptr;       // their 128-bit masks
  uint64_t n_dense_blocks = 0, n_sparse_elems = 0;
  bool stats_ready = false;
  // Count-kernel work lists (vertices with |N+| >= 2 by class), see count_tri.cu.
  uint32_t* work = nullptr;
  uint32_t* work_lpt = nullptr;  // same lists, classes 1-2 heaviest first (work_lpt(), on demand)
  uint64_t n_work[3] = {0, 0, 0};
  uint64_t n_thread = 0;    // the first n_thread entries of class 0: the thread class (d <= bin_thread_max)
  uint32_t class0_max = 0;  // largest |N+(x)| of class 0 (the warp kernels' staging bound)
  unsigned long long* d_counter = nullptr;  // 8 x u64: count, work cursors, y-major queue size
  unsigned long long h_counter[2] = {0, 0};  // host mirror (8-byte D2H per count)
  eh_graph* sym = nullptr;  // NEXT-2: symmetric (unpruned) trie, built on first use (sym.cu)


  std::vector<void*> owned;  // every device allocation above
  uint64_t device_bytes = 0;

  void* own(size_t bytes) {
    void* p = alloc.alloc(bytes);
    owned.push_back(p);
    device_bytes += (bytes + 255) & ~size_t(255);
    return p;
  }
};

namespace eh {
// ingest.cu: canonicalise, sort, dedup, degree rank, orient, CSR; fills g->desc/col/orig_id.
void build_trie(eh_graph* g, const uint32_t* d_src, const uint32_t* d_dst, uint64_t n, PhaseTimer* t = nullptr);
// dedup.cu: the bucketed a1-a4 pass (distinct keys, compact; degrees; *m_ctr += m)
bool bucket_dedup_ok(uint32_t b, uint64_t n);
void bucket_dedup(const uint32_t* src, const uint32_t* dst, uint64_t n, uint32_t b, uint32_t* deg,
                  unsigned long long* m_ctr, uint64_t* out, eh_graph* g, PhaseTimer* tm = nullptr);
// trie.cu: set-level layout (uint / bitset) and the bitset pool; work lists.
void build_layouts(eh_graph* g);
const uint32_t* work_lpt(eh_graph* g);  // lazy: LPT-ordered work lists (trie.cu)
void compute_stats(eh_graph* g);  // lazy: B_tri, wedge work, #bitset sets
void build_block_layout(eh_graph* g);  // NEXT-3 composite layout (EH_BLOCK_LAYOUT)
void build_worklists(eh_graph* g);
uint64_t alg_bytes_k4(eh_graph* g);  // lazy: B_K4 = B_tri + sum over triangles of bytes(N+(z)) (tau = 32)
// eh_count_*_range: while alive, the handle's work lists hold only the x with rank in
// [r0, r1) (class-major, each class and the LPT order preserved); restored on exit.
class WorkRange {
 public:
  WorkRange(eh_graph* g, uint64_t r0, uint64_t r1);
  ~WorkRange();
  WorkRange(const WorkRange&) = delete;
  WorkRange& operator=(const WorkRange&) = delete;

 private:
  eh_graph* g_;
  uint32_t* saved_work_;
  uint32_t* saved_lpt_;
  uint64_t saved_n_[3], saved_nt_;
  DBuf<uint32_t> work_, lpt_;
};
// Side streams of the count kernels: per host thread and device, created once
// (non-blocking) with their fork / join events, so a count on a fresh handle pays
// no stream creation.  Fork: side stream k waits for the work queued so far on the
// handle's stream.  Join: the handle's stream waits for everything queued on side
// stream k.  (Every count call joins before it returns.)
struct SideStreams {
  static constexpr int kSides = 3;
  cudaStream_t s[kSides] = {};
  cudaEvent_t fork = nullptr, join[kSides] = {};
  SideStreams() = default;
  SideStreams(const SideStreams&) = delete;
  SideStreams& operator=(const SideStreams&) = delete;
  ~SideStreams() {  // at thread exit (e.g. an eh_count_batch lane); errors after CUDA teardown are ignored
    for (int k = 0; k < kSides; ++k) {
      if (s[k]) cudaStreamDestroy(s[k]);
      if (join[k]) cudaEventDestroy(join[k]);
    }
    if (fork) cudaEventDestroy(fork);
  }
};
SideStreams& side_streams(int device);  // eh_api.cu
inline cudaStream_t fork_side(eh_graph* g, int k) {
  SideStreams& ss = side_streams(g->device);
  if (!ss.fork) EH_CUDA(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
  if (!ss.s[k]) {
    EH_CUDA(cudaStreamCreateWithFlags(&ss.s[k], cudaStreamNonBlocking));
    EH_CUDA(cudaEventCreateWithFlags(&ss.join[k], cudaEventDisableTiming));
  }
  EH_CUDA(cudaEventRecord(ss.fork, g->stream));
  EH_CUDA(cudaStreamWaitEvent(ss.s[k], ss.fork, 0));
  return ss.s[k];
}
inline void join_side(eh_graph* g, int k) {
  SideStreams& ss = side_streams(g->device);
  EH_CUDA(cudaEventRecord(ss.join[k], ss.s[k]));
  EH_CUDA(cudaStreamWaitEvent(g->stream, ss.join[k], 0));
}
// count_tri.cu / count_k4.cu
uint64_t count_triangles(eh_graph* g);
uint32_t tri_warp_max_degree();  // largest |N+(x)| the warp-per-x kernels accept
uint32_t tri_thread_max_degree();  // largest |N+(x)| the thread-per-x kernel accepts
constexpr uint32_t kThreadMaxDefault = 12;  // default bin_thread_max (a7 thread class) up to 2^19 active ids; 16 above, 4 above 2^24
uint64_t count_4cliques(eh_graph* g);
// count_pv.cu (NEXT-1): t(v) per rank into a device array; Lollipop / Barbell 128-bit counts
void triangles_per_vertex(eh_graph* g, unsigned long long* d_t);
void count_lollipop_barbell(eh_graph* g, bool barbell, uint64_t out2[2]);
// sym.cu / count_tri.cu (NEXT-2): the symmetric trie (lazy) and the unpruned triangle nest (= 6T)
eh_graph* symmetric_trie(eh_graph* g);
uint64_t count_triangles_unpruned(eh_graph* g);
uint64_t count_4cliques_unpruned(eh_graph* g);  // count_k4.cu: = 24 K4
// intersect.cu
int64_t intersect(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb, uint32_t* out);
}  // namespace eh
