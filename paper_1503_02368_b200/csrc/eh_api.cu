// eh_api.cu -- the extern "C" boundary declared in include/eh.h.
//
// Every entry point: validate arguments, select the device, run the CUDA path,
// translate internal exceptions into the documented return codes and the
// thread-local status / message.  There is no CPU fallback anywhere.
#include "eh_internal.cuh"

#include <cstring>
#include <exception>
#include <map>
#include <mutex>
#include <thread>

namespace eh {
std::atomic<unsigned long long> g_launches{0};

void prefer_max_smem_carveout(const void* kernel) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, bool> done;
  int dev = 0;
  EH_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  bool& d = done[{dev, kernel}];
  if (d) return;
  EH_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
  d = true;
}

void ensure_dyn_smem(const void* kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return;  // within the default limit
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> limit;
  int dev = 0;
  EH_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = limit[{dev, kernel}];
  if (bytes <= cur) return;
  EH_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  cur = bytes;
}

SideStreams& side_streams(int device) {
  constexpr int kMaxDev = 64;
  if (device < 0 || device >= kMaxDev) fail(EH_EINVAL, "device ordinal %d out of range", device);
  thread_local SideStreams per_dev[kMaxDev];  // process lifetime of the thread; never destroyed
  return per_dev[device];
}
}

namespace {

thread_local int t_status = EH_OK;
thread_local char t_msg[512] = "";

void set_status(int code, const char* msg) {
  t_status = code;
  std::snprintf(t_msg, sizeof t_msg, "%s", msg ? msg : "");
}
void ok() { set_status(EH_OK, ""); }

// int-returning entry points: the EH_E* status of the failure itself (EH_EINVAL,
// EH_ENOMEM, EH_ECUDA), not a fixed code
template <class F>
int guarded_status(F&& f);

template <class R, class F>
R guarded(R on_error, F&& f) {
  try {
    R r = f();
    ok();
    return r;
  } catch (const eh::Error& e) {
    set_status(e.code, e.what());
  } catch (const std::bad_alloc&) {
    set_status(EH_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    set_status(EH_ECUDA, e.what());
  }
  return on_error;
}

template <class F>
int guarded_status(F&& f) {
  const int r = guarded<int>(INT32_MIN, std::forward<F>(f));
  return r == INT32_MIN ? t_status : r;
}

void destroy(eh_graph* g) {
  if (!g) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(g->device);
  if (g->stream) cudaStreamSynchronize(g->stream);
  if (g->sym) {
    eh_graph* h = g->sym;
    for (void* p : h->owned) h->alloc.release(p);
    delete h;
  }
  for (void* p : g->owned) g->alloc.release(p);
  if (g->stream) cudaStreamSynchronize(g->stream);
  if (g->own_stream && g->stream) cudaStreamDestroy(g->stream);
  if (prev >= 0) cudaSetDevice(prev);
  delete g;
}

struct DeviceGuard {  // restores the caller's current device
  int prev = -1;
  explicit DeviceGuard(int dev) {
    EH_CUDA(cudaGetDevice(&prev));
    if (dev != prev) EH_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

// The whole of eh_load_edges_ex below the ABI guard (also used by eh_count_batch).
eh_graph* load_impl(const uint32_t* src, const uint32_t* dst, uint64_t n, const eh_config* cfg) {
  {
    eh_config c;
    std::memset(&c, 0, sizeof c);
    if (cfg) c = *cfg;
    if (n && (!src || !dst)) eh::fail(EH_EINVAL, "eh_load_edges: NULL src/dst with n = %llu", (unsigned long long)n);
    if ((c.dev_alloc == nullptr) != (c.dev_free == nullptr))
      eh::fail(EH_EINVAL, "eh_load_edges: dev_alloc and dev_free must be set together");
    if (c.flags & ~(uint32_t)(EH_INPUT_ON_DEVICE | EH_SET_DEVICE | EH_ALL_UINT | EH_NO_ALGO | EH_BLOCK_LAYOUT | EH_FORCE_SEARCH))
      eh::fail(EH_EINVAL, "eh_load_edges: unknown flags 0x%x", c.flags);
    int ndev = 0;
    EH_CUDA(cudaGetDeviceCount(&ndev));
    if (ndev <= 0) eh::fail(EH_ECUDA, "no CUDA device");
    int dev = 0;
    EH_CUDA(cudaGetDevice(&dev));
    if (c.flags & EH_SET_DEVICE) {
      if (c.device < 0 || c.device >= ndev) eh::fail(EH_EINVAL, "eh_load_edges: bad device %d", c.device);
      dev = c.device;
    }
    DeviceGuard guard(dev);
    eh_graph* g = new eh_graph();
    try {
      g->device = dev;
      g->flags = c.flags | ((c.flags & (EH_NO_ALGO | EH_FORCE_SEARCH)) ? EH_ALL_UINT : 0u);  // -RA implies -R
      g->tau = c.bitset_tau ? c.bitset_tau : 128;
      g->min_bitset_card = c.min_bitset_card ? c.min_bitset_card : 2;
      g->bin_small_max = c.bin_small_max;
      g->bin_large_min = c.bin_large_min;
      g->bin_thread_max = c.bin_thread_max;
      if (c.order > EH_ORDER_ID) eh::fail(EH_EINVAL, "eh_load_edges: unknown order %u", c.order);
      g->order = c.order;
      if (c.stream) {
        g->stream = (cudaStream_t)c.stream;
      } else {
        // a BLOCKING stream: it is ordered after the work pending on the legacy default
        // stream (e.g. torch's default stream writing device-resident inputs)
        EH_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamDefault));
        g->own_stream = true;
      }
      g->alloc.hook_alloc = c.dev_alloc;
      g->alloc.hook_free = c.dev_free;
      g->alloc.ctx = c.alloc_ctx;
      g->alloc.stream = g->stream;
      eh::PhaseTimer timer(g->stream);
      g->d_counter = (unsigned long long*)g->own(8 * sizeof(unsigned long long));
      timer.mark("alloc");
      // a1: upload (borrowed inputs are copied)
      eh::DBuf<uint32_t> in;
      const uint32_t* d_src = src;
      const uint32_t* d_dst = dst;
      if (n && !(c.flags & EH_INPUT_ON_DEVICE)) {
        in = eh::DBuf<uint32_t>(g->alloc, 2 * n);
        EH_CUDA(cudaMemcpyAsync(in.p, src, n * 4, cudaMemcpyHostToDevice, g->stream));
        EH_CUDA(cudaMemcpyAsync(in.p + n, dst, n * 4, cudaMemcpyHostToDevice, g->stream));
        d_src = in.p;
        d_dst = in.p + n;
      }
      timer.mark("upload");
      eh::build_trie(g, d_src, d_dst, n, &timer);
      in.reset();
      eh::build_layouts(g);
      if (g->flags & EH_BLOCK_LAYOUT) eh::build_block_layout(g);
      timer.mark("layouts");
      eh::build_worklists(g);
      timer.mark("worklists");
      EH_CUDA(cudaStreamSynchronize(g->stream));
      timer.report("eh_load_edges");
    } catch (...) {
      destroy(g);
      throw;
    }
    return g;
  }
}



// One lane of eh_count_batch: lists first, first + step, ... in order on one compute
// stream (the caller's, else a blocking library stream), uploads on a non-blocking
// copy stream into two device input buffers (ping-pong): the upload of the lane's
// next list overlaps the load + count of the current one.
void batch_lane(const uint32_t* const* src, const uint32_t* const* dst, const uint64_t* n, uint64_t k,
                uint64_t first, uint64_t step, uint32_t query, const eh_config& c, uint64_t* counts) {
  uint64_t nmax = 0;
  for (uint64_t i = first; i < k; i += step) nmax = std::max(nmax, n[i]);
  cudaStream_t cs = (cudaStream_t)c.stream, up = nullptr;
  bool own_cs = false;
  cudaEvent_t landed[2] = {nullptr, nullptr}, read[2] = {nullptr, nullptr};
  eh::Allocator al;
  al.hook_alloc = c.dev_alloc;
  al.hook_free = c.dev_free;
  al.ctx = c.alloc_ctx;
  void* buf[2] = {nullptr, nullptr};
  auto cleanup = [&]() {
    if (cs) cudaStreamSynchronize(cs);
    if (up) cudaStreamSynchronize(up);
    for (int b = 0; b < 2; ++b) {
      if (buf[b]) al.release(buf[b]);
      if (landed[b]) cudaEventDestroy(landed[b]);
      if (read[b]) cudaEventDestroy(read[b]);
    }
    if (cs) cudaStreamSynchronize(cs);
    if (up) cudaStreamDestroy(up);
    if (own_cs && cs) cudaStreamDestroy(cs);
  };
  try {
    if (!cs) {
      EH_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamDefault));
      own_cs = true;
    }
    EH_CUDA(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
    al.stream = cs;
    for (int b = 0; b < 2; ++b) {
      EH_CUDA(cudaEventCreateWithFlags(&landed[b], cudaEventDisableTiming));
      EH_CUDA(cudaEventCreateWithFlags(&read[b], cudaEventDisableTiming));
      buf[b] = al.alloc(std::max<uint64_t>(1, 2 * nmax) * 4);
    }
    EH_CUDA(cudaStreamSynchronize(cs));  // the buffers exist before the copy stream writes them
    auto upload = [&](uint64_t j) {  // j-th list of this lane
      const uint64_t i = first + j * step;
      const int b = (int)(j & 1);
      uint32_t* d = (uint32_t*)buf[b];
      if (j >= 2) EH_CUDA(cudaStreamWaitEvent(up, read[b], 0));  // the lane's list j-2 has been read
      if (n[i]) {
        EH_CUDA(cudaMemcpyAsync(d, src[i], n[i] * 4, cudaMemcpyHostToDevice, up));
        EH_CUDA(cudaMemcpyAsync(d + n[i], dst[i], n[i] * 4, cudaMemcpyHostToDevice, up));
      }
      EH_CUDA(cudaEventRecord(landed[b], up));
    };
    eh_config gc = c;
    gc.flags |= EH_INPUT_ON_DEVICE;
    gc.flags &= ~(uint32_t)EH_SET_DEVICE;
    gc.stream = cs;
    const uint64_t nl = (k - first + step - 1) / step;
    upload(0);
    for (uint64_t j = 0; j < nl; ++j) {
      if (j + 1 < nl) upload(j + 1);  // overlaps the load and count of list j
      const uint64_t i = first + j * step;
      const int b = (int)(j & 1);
      EH_CUDA(cudaStreamWaitEvent(cs, landed[b], 0));
      const uint32_t* d = (const uint32_t*)buf[b];
      eh_graph* g = load_impl(d, d + n[i], n[i], &gc);  // synchronous on cs: inputs read on return
      EH_CUDA(cudaEventRecord(read[b], cs));
      try {
        counts[i] = query == EH_QUERY_4CLIQUES ? eh::count_4cliques(g) : eh::count_triangles(g);
      } catch (...) {
        destroy(g);
        throw;
      }
      destroy(g);
    }
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}

}  // namespace

extern "C" {

eh_graph* eh_load_edges_ex(const uint32_t* src, const uint32_t* dst, uint64_t n, const eh_config* cfg) {
  return guarded<eh_graph*>(nullptr, [&]() -> eh_graph* { return load_impl(src, dst, n, cfg); });
}

eh_graph* eh_load_edges(const uint32_t* src, const uint32_t* dst, uint64_t n) {
  return eh_load_edges_ex(src, dst, n, nullptr);
}

int eh_count_batch(const uint32_t* const* src, const uint32_t* const* dst, const uint64_t* n, uint64_t k,
                   uint32_t query, const eh_config* cfg, uint64_t* counts) {
  return guarded_status([&]() -> int {
    if (k && (!src || !dst || !n || !counts)) eh::fail(EH_EINVAL, "eh_count_batch: NULL argument");
    if (query != EH_QUERY_TRIANGLES && query != EH_QUERY_4CLIQUES)
      eh::fail(EH_EINVAL, "eh_count_batch: unknown query %u", query);
    eh_config c;
    std::memset(&c, 0, sizeof c);
    if (cfg) c = *cfg;
    if (c.flags & EH_INPUT_ON_DEVICE) eh::fail(EH_EINVAL, "eh_count_batch: inputs are host memory");
    if (k == 0) return EH_OK;
    for (uint64_t i = 0; i < k; ++i)
      if (n[i] && (!src[i] || !dst[i])) eh::fail(EH_EINVAL, "eh_count_batch: NULL list %llu", (unsigned long long)i);
    int dev = 0, ndev = 0;
    EH_CUDA(cudaGetDeviceCount(&ndev));
    if (ndev <= 0) eh::fail(EH_ECUDA, "no CUDA device");
    EH_CUDA(cudaGetDevice(&dev));
    if (c.flags & EH_SET_DEVICE) {
      if (c.device < 0 || c.device >= ndev) eh::fail(EH_EINVAL, "eh_count_batch: bad device %d", c.device);
      dev = c.device;
    }
    DeviceGuard guard(dev);
    // lanes: with the caller's stream one lane runs every list on it; otherwise small
    // lists (<= 2^23 input edges) take two lanes (host threads with streams of their
    // own, alternate lists), so one list's ingest and count kernels fill the gaps of
    // the other's; large lists keep one lane -- two graphs in flight evict each other's
    // L2-resident hub lists (measured, ms per list: C2 1.48 -> 1.37 with two lanes,
    // C4 K4 10.69 -> 10.76, C3 16.8 -> 18.2).  Test hook EH_TEST_BATCH_LANES=1|2.
    uint64_t nmax = 0;
    for (uint64_t i = 0; i < k; ++i) nmax = std::max(nmax, n[i]);
    int lanes = (c.stream || nmax > (1ull << 23)) ? 1 : 2;
    if (const char* e = getenv("EH_TEST_BATCH_LANES")) lanes = std::max(1, std::min(2, atoi(e)));
    if ((uint64_t)lanes > k) lanes = (int)k;
    std::exception_ptr err[2];
    auto run = [&](int lane) {
      try {
        EH_CUDA(cudaSetDevice(dev));
        batch_lane(src, dst, n, k, (uint64_t)lane, (uint64_t)lanes, query, c, counts);
      } catch (...) {
        err[lane] = std::current_exception();
      }
    };
    std::thread other;
    if (lanes == 2) other = std::thread(run, 1);
    run(0);
    if (other.joinable()) other.join();
    for (int l = 0; l < lanes; ++l)
      if (err[l]) std::rethrow_exception(err[l]);
    return EH_OK;
  });
}

uint64_t eh_count_triangles(eh_graph* g) {
  return guarded<uint64_t>(EH_COUNT_ERROR, [&]() -> uint64_t {
    if (!g) eh::fail(EH_EINVAL, "eh_count_triangles: NULL graph");
    DeviceGuard guard(g->device);
    return eh::count_triangles(g);
  });
}

uint64_t eh_count_4cliques(eh_graph* g) {
  return guarded<uint64_t>(EH_COUNT_ERROR, [&]() -> uint64_t {
    if (!g) eh::fail(EH_EINVAL, "eh_count_4cliques: NULL graph");
    DeviceGuard guard(g->device);
    return eh::count_4cliques(g);
  });
}

uint64_t eh_count_triangles_range(eh_graph* g, uint64_t r0, uint64_t r1) {
  return guarded<uint64_t>(EH_COUNT_ERROR, [&]() -> uint64_t {
    if (!g) eh::fail(EH_EINVAL, "eh_count_triangles_range: NULL graph");
    DeviceGuard guard(g->device);
    eh::WorkRange range(g, r0, r1);
    return eh::count_triangles(g);
  });
}

uint64_t eh_count_4cliques_range(eh_graph* g, uint64_t r0, uint64_t r1) {
  return guarded<uint64_t>(EH_COUNT_ERROR, [&]() -> uint64_t {
    if (!g) eh::fail(EH_EINVAL, "eh_count_4cliques_range: NULL graph");
    DeviceGuard guard(g->device);
    eh::work_lpt(g);  // the full LPT order first: the range keeps its sub-order
    eh::WorkRange range(g, r0, r1);
    return eh::count_4cliques(g);
  });
}

uint64_t eh_alg_bytes_k4(eh_graph* g) {
  return guarded<uint64_t>(EH_COUNT_ERROR, [&]() -> uint64_t {
    if (!g) eh::fail(EH_EINVAL, "eh_alg_bytes_k4: NULL graph");
    DeviceGuard guard(g->device);
    return eh::alg_bytes_k4(g);
  });
}

uint64_t eh_count_triangles_unpruned(eh_graph* g) {
  return guarded<uint64_t>(EH_COUNT_ERROR, [&]() -> uint64_t {
    if (!g) eh::fail(EH_EINVAL, "eh_count_triangles_unpruned: NULL graph");
    DeviceGuard guard(g->device);
    return eh::count_triangles_unpruned(g);
  });
}

uint64_t eh_count_4cliques_unpruned(eh_graph* g) {
  return guarded<uint64_t>(EH_COUNT_ERROR, [&]() -> uint64_t {
    if (!g) eh::fail(EH_EINVAL, "eh_count_4cliques_unpruned: NULL graph");
    DeviceGuard guard(g->device);
    return eh::count_4cliques_unpruned(g);
  });
}

int eh_symmetric_stats(eh_graph* g, eh_stats* out) {
  return guarded_status([&]() -> int {
    if (!g || !out) eh::fail(EH_EINVAL, "eh_symmetric_stats: NULL argument");
    DeviceGuard guard(g->device);
    eh_graph* h = eh::symmetric_trie(g);
    eh::compute_stats(h);
    out->n_input = h->n_input;
    out->m_undirected = h->m;
    out->n_active = h->n_act;
    out->max_out_degree = h->max_dplus;
    out->n_bitset_sets = h->n_bitsets;
    out->bitset_words = h->bs_words;
    out->device_bytes = h->device_bytes;
    out->alg_bytes_tri = h->alg_bytes_tri;
    out->wedge_work = h->wedge_work;
    return EH_OK;
  });
}

int eh_triangles_per_vertex(eh_graph* g, uint64_t* t) {
  return guarded_status([&]() -> int {
    if (!g || (!t && g->n_act)) eh::fail(EH_EINVAL, "eh_triangles_per_vertex: NULL argument");
    DeviceGuard guard(g->device);
    if (g->n_act == 0) return EH_OK;
    cudaPointerAttributes pa{};
    EH_CUDA(cudaPointerGetAttributes(&pa, t));
    const bool on_device = pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged;
    if (on_device && pa.device != g->device)
      eh::fail(EH_EINVAL, "eh_triangles_per_vertex: output on device %d, graph on device %d", pa.device, g->device);
    if (on_device) {
      eh::triangles_per_vertex(g, reinterpret_cast<unsigned long long*>(t));
      EH_CUDA(cudaStreamSynchronize(g->stream));
    } else {
      eh::DBuf<unsigned long long> d(g->alloc, g->n_act);
      eh::triangles_per_vertex(g, d.p);
      EH_CUDA(cudaMemcpyAsync(t, d.p, g->n_act * 8, cudaMemcpyDeviceToHost, g->stream));
      EH_CUDA(cudaStreamSynchronize(g->stream));
    }
    return EH_OK;
  });
}

static int count128(eh_graph* g, uint64_t* out, bool barbell, const char* what) {
  return guarded_status([&]() -> int {
    if (!g || !out) eh::fail(EH_EINVAL, "%s: NULL argument", what);
    DeviceGuard guard(g->device);
    eh::count_lollipop_barbell(g, barbell, out);
    return EH_OK;
  });
}

int eh_count_lollipop(eh_graph* g, uint64_t out[2]) { return count128(g, out, false, "eh_count_lollipop"); }
int eh_count_barbell(eh_graph* g, uint64_t out[2]) { return count128(g, out, true, "eh_count_barbell"); }

int64_t eh_intersect(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb, uint32_t* out) {
  int64_t r = guarded<int64_t>(INT64_MIN, [&]() -> int64_t { return eh::intersect(a, na, b, nb, out); });
  return r == INT64_MIN ? (int64_t)t_status : r;
}

int eh_graph_stats(const eh_graph* g, eh_stats* out) {
  if (!g || !out) {
    set_status(EH_EINVAL, "eh_graph_stats: NULL argument");
    return EH_EINVAL;
  }
  const int rc = guarded_status([&]() -> int {
    DeviceGuard guard(g->device);
    eh::compute_stats(const_cast<eh_graph*>(g));  // cached, logically const
    return EH_OK;
  });
  if (rc != EH_OK) return t_status;
  out->n_input = g->n_input;
  out->m_undirected = g->m;
  out->n_active = g->n_act;
  out->max_out_degree = g->max_dplus;
  out->n_bitset_sets = g->n_bitsets;
  out->bitset_words = g->bs_words;
  out->device_bytes = g->device_bytes;
  out->alg_bytes_tri = g->alg_bytes_tri;
  out->wedge_work = g->wedge_work;
  ok();
  return EH_OK;
}

int eh_graph_export(const eh_graph* g, uint64_t* row_ptr, uint32_t* col, uint32_t* orig_id, uint8_t* is_bitset) {
  return guarded_status([&]() -> int {
    if (!g) eh::fail(EH_EINVAL, "eh_graph_export: NULL graph");
    DeviceGuard guard(g->device);
    const uint64_t n = g->n_act;
    std::vector<uint4> desc(n + 1);
    EH_CUDA(cudaMemcpyAsync(desc.data(), g->desc, (n + 1) * sizeof(uint4), cudaMemcpyDeviceToHost, g->stream));
    std::vector<uint32_t> padded(g->col_elems);
    if (g->col_elems)
      EH_CUDA(cudaMemcpyAsync(padded.data(), g->col, g->col_elems * 4, cudaMemcpyDeviceToHost, g->stream));
    if (orig_id && n) EH_CUDA(cudaMemcpyAsync(orig_id, g->orig_id, n * 4, cudaMemcpyDeviceToHost, g->stream));
    EH_CUDA(cudaStreamSynchronize(g->stream));
    uint64_t pos = 0;
    for (uint64_t v = 0; v < n; ++v) {
      if (row_ptr) row_ptr[v] = pos;
      if (col) std::memcpy(col + pos, padded.data() + (uint64_t)desc[v].x * 4, (size_t)desc[v].y * 4);
      if (is_bitset) is_bitset[v] = desc[v + 1].z != desc[v].z;
      pos += desc[v].y;
    }
    if (row_ptr) row_ptr[n] = pos;
    return EH_OK;
  });
}

void eh_free(eh_graph* g) { destroy(g); }

void eh_release_cached_memory(void) {
  eh::release_cached_memory();
  ok();
}

uint64_t eh_launch_count(void) { return eh::g_launches.load(); }

int eh_last_status(void) { return t_status; }
const char* eh_last_error(void) { return t_msg; }

}  // extern "C"
