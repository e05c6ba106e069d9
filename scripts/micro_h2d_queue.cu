// When does cudaMemcpy(2D)Async from pinned memory start blocking the host?
// Host issue time vs number / size / shape of queued H2D copies.
// nvcc -O2 -o scripts/micro_h2d_queue.bin scripts/micro_h2d_queue.cu
#include <chrono>
#include <cstdio>

#include <cuda_runtime.h>

int main() {
  const size_t host_bytes = 1ull << 30, dev_bytes = 1ull << 30;
  void *h, *d;
  cudaHostAlloc(&h, host_bytes, cudaHostAllocDefault);
  cudaMalloc(&d, dev_bytes);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const size_t sizes[] = {64 << 10, 256 << 10, 1 << 20};
  const int counts[] = {128, 256, 512, 1024, 2048, 4096};
  for (size_t sz : sizes)
    for (int n : counts) {
      if ((size_t)n * sz > 8ull * host_bytes) continue;
      cudaDeviceSynchronize();
      auto t0 = now();
      double first_block = -1;
      for (int i = 0; i < n; ++i) {
        auto a = now();
        const size_t off = ((size_t)i * sz) % (host_bytes - sz);
        cudaMemcpyAsync((char*)d + off % (dev_bytes - sz), (char*)h + off, sz, cudaMemcpyHostToDevice, st);
        if (first_block < 0 && ms(a, now()) > 0.2) first_block = i;
      }
      auto t1 = now();
      cudaDeviceSynchronize();
      auto t2 = now();
      printf("1-D %5zu KB x %5d: issue %7.2f ms (first blocking call #%5.0f), drain %7.2f ms, %5.1f GB/s\n", sz >> 10,
             n, ms(t0, t1), first_block, ms(t0, t2), n * sz / ms(t0, t2) / 1e6);
    }
  // 2-D: 128 rows of width w, height h per call
  const int heights[] = {1, 4, 8};
  for (int hgt : heights)
    for (int n : {128, 512, 1024}) {
      const size_t w = 256 << 10;
      cudaDeviceSynchronize();
      auto t0 = now();
      double first_block = -1;
      for (int i = 0; i < n; ++i) {
        auto a = now();
        cudaMemcpy2DAsync(d, 2 * w, (char*)h + (i % 64) * w, 64 * w, w, hgt, cudaMemcpyHostToDevice, st);
        if (first_block < 0 && ms(a, now()) > 0.2) first_block = i;
      }
      auto t1 = now();
      cudaDeviceSynchronize();
      auto t2 = now();
      printf("2-D 256 KB x h%d x %5d: issue %7.2f ms (first blocking call #%5.0f), drain %7.2f ms, %5.1f GB/s\n", hgt,
             n, ms(t0, t1), first_block, ms(t0, t2), (double)n * hgt * w / ms(t0, t2) / 1e6);
    }
  return 0;
}
