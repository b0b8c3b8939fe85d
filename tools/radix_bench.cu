// radix_bench.cu -- dev microbenchmark (not product code): the library's
// one-sweep radix sort vs cub::DeviceRadixSort on the same u64 keys.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//        -Ipaper_1503_02368_b200/csrc tools/radix_bench.cu -o /tmp/radix_bench
//   radix_bench KEYS.bin BITS [REPS]      (KEYS.bin: raw little-endian u64)
#include <algorithm>
#include <cub/device/device_radix_sort.cuh>

#include "../paper_1503_02368_b200/csrc/primitives.cu"

namespace eh { std::atomic<unsigned long long> g_launches{0}; }

int main(int argc, char** argv) {
  if (argc < 3) { fprintf(stderr, "usage: %s KEYS.bin BITS [REPS]\n", argv[0]); return 2; }
  FILE* f = fopen(argv[1], "rb");
  if (!f) { perror("open"); return 2; }
  fseek(f, 0, SEEK_END);
  const size_t n = ftell(f) / 8;
  fseek(f, 0, SEEK_SET);
  std::vector<uint64_t> h(n);
  if (fread(h.data(), 8, n, f) != n) return 2;
  fclose(f);
  const uint32_t bits = atoi(argv[2]);
  const int reps = argc > 3 ? atoi(argv[3]) : 5;
  cudaStream_t s;
  cudaStreamCreate(&s);
  eh::Allocator al;
  al.stream = s;
  uint64_t *src, *a, *b, *c;
  cudaMalloc(&src, n * 8); cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8); cudaMalloc(&c, n * 8);
  cudaMemcpy(src, h.data(), n * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  std::vector<float> ours, cubt;
  uint64_t* res = nullptr;
  for (int r = 0; r < reps; ++r) {
    cudaMemcpyAsync(a, src, n * 8, cudaMemcpyDeviceToDevice, s);
    cudaEventRecord(e0, s);
    res = eh::radix_sort_u64(a, b, n, bits, al, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ours.push_back(ms);
  }
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, a, c, (int64_t)n, 0, (int)bits, s);
  void* tmp; cudaMalloc(&tmp, tmp_bytes);
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0, s);
    cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, src, c, (int64_t)n, 0, (int)bits, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); cubt.push_back(ms);
  }
  std::vector<uint64_t> x(n), y(n);
  cudaMemcpy(x.data(), res, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(y.data(), c, n * 8, cudaMemcpyDeviceToHost);
  const bool same = x == y;
  auto best = [](std::vector<float> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
  printf("{\"n\": %zu, \"bits\": %u, \"ours_ms\": %.4f, \"cub_ms\": %.4f, \"identical\": %s, \"err\": \"%s\"}\n", n, bits,
         best(ours), best(cubt), same ? "true" : "false", cudaGetErrorString(cudaGetLastError()));
  return same ? 0 : 1;
}
