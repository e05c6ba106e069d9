// Host issue cost and transfer time of the ways to DMA per-chunk pinned
// caches ([L][rows][row_bytes] each) into a layer-major device store
// ([L][cap][row_bytes]): 1-D copies per (chunk, layer), one 2-D copy per chunk,
// one cudaMemcpyBatchAsync for everything.
// nvcc -O2 -o scripts/micro_h2d.bin scripts/micro_h2d.cu
#include <chrono>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

int main() {
  const int C = 64, L = 28, rows = 544, body = 512;
  const size_t rb = 1024;  // 4 kv heads x 128 x bf16
  const size_t cap = 32832;
  std::vector<void*> host(C);
  for (int c = 0; c < C; ++c) cudaHostAlloc(&host[c], (size_t)L * rows * rb, cudaHostAllocDefault);
  void* dst;
  cudaMalloc(&dst, (size_t)L * cap * rb);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto d) { return std::chrono::duration<double, std::milli>(d).count(); };
  const double gb = (double)C * L * body * rb / 1e9;

  for (int rep = 0; rep < 3; ++rep) {
    // (a) 1-D per (chunk, layer)
    cudaEventRecord(a, st);
    auto t0 = now();
    for (int l = 0; l < L; ++l)
      for (int c = 0; c < C; ++c)
        cudaMemcpyAsync((char*)dst + ((size_t)l * cap + 32 + (size_t)c * body) * rb,
                        (char*)host[c] + ((size_t)l * rows + 32) * rb, body * rb, cudaMemcpyHostToDevice, st);
    auto t1 = now();
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float g;
    cudaEventElapsedTime(&g, a, b);
    printf("1-D x%d: issue %.2f ms, gpu %.2f ms (%.1f GB/s)\n", C * L, ms(t1 - t0), g, gb / g * 1e3);

    // (b) 2-D per chunk
    cudaEventRecord(a, st);
    t0 = now();
    for (int c = 0; c < C; ++c)
      cudaMemcpy2DAsync((char*)dst + (32 + (size_t)c * body) * rb, cap * rb, (char*)host[c] + 32 * rb, rows * rb,
                        body * rb, L, cudaMemcpyHostToDevice, st);
    t1 = now();
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&g, a, b);
    printf("2-D x%d: issue %.2f ms, gpu %.2f ms (%.1f GB/s)\n", C, ms(t1 - t0), g, gb / g * 1e3);

    // (c) one batch
    std::vector<void*> ds, ss;
    std::vector<size_t> sz;
    for (int l = 0; l < L; ++l)
      for (int c = 0; c < C; ++c) {
        ds.push_back((char*)dst + ((size_t)l * cap + 32 + (size_t)c * body) * rb);
        ss.push_back((char*)host[c] + ((size_t)l * rows + 32) * rb);
        sz.push_back(body * rb);
      }
    cudaMemcpyAttributes at = {};
    at.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
    at.flags = cudaMemcpyFlagPreferOverlapWithCompute;
    size_t idx = 0, fail = 0;
    cudaEventRecord(a, st);
    t0 = now();
    cudaError_t e = cudaMemcpyBatchAsync(ds.data(), ss.data(), sz.data(), ds.size(), &at, &idx, 1, &fail, st);
    t1 = now();
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&g, a, b);
    printf("batch x%zu (%s): issue %.2f ms, gpu %.2f ms (%.1f GB/s)\n", ds.size(), cudaGetErrorString(e), ms(t1 - t0),
           g, gb / g * 1e3);
  }
  return 0;
}
