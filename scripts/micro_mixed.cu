// Does tcgen05.mma kind::f16 accept A in fp16 and B in bf16 (separate a/b
// format fields of the instruction descriptor)? One CTA: A = 1.5 (f16) or
// per-row values, B = 2.0 (bf16), K = 16, M = 128, N = 64; D read back.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2510_10129_b200/csrc \
//        -o scripts/micro_mixed.bin scripts/micro_mixed.cu -lcuda && scripts/micro_mixed.bin
#include <cstdio>

#include <cuda_fp16.h>

#include "cc_common.cuh"

using namespace cc;

// idesc with explicit a/b formats: 0 = f16, 1 = bf16 (bits 7-9 a, 10-12 b), c = f32 (bit 4)
__host__ __device__ constexpr uint32_t idesc_ab(int m, int n, uint32_t afmt, uint32_t bfmt) {
  return (1u << 4) | (afmt << 7) | (bfmt << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__global__ void mixed_kernel(float* out, uint32_t afmt, uint32_t bfmt) {
  __shared__ __align__(1024) uint8_t smem[32 * 1024];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&slot, 64);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  // A: 128 rows x 16 K (32 B per row) in a K-major SW128 layout; only the
  // first 32 bytes of each 128-byte row matter for K = 16. Row r holds value (r % 4 + 1) * 0.5.
  // B: 64 rows x 16 K, value 2.0 (bf16 0x4000) or f16 2.0 (0x4000 as well).
  uint16_t* a = reinterpret_cast<uint16_t*>(smem);
  uint16_t* b = reinterpret_cast<uint16_t*>(smem + 16 * 1024);
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64;
    const float v = (r % 4 + 1) * 0.5f;
    __half h = __float2half(v);
    __nv_bfloat16 bh = __float2bfloat16(v);
    a[i] = afmt == 0 ? *reinterpret_cast<uint16_t*>(&h) : *reinterpret_cast<uint16_t*>(&bh);
  }
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) b[i] = 0x4000;  // 2.0 in both formats
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_ab(128, 64, afmt, bfmt);
    tc_mma<false>(tmem, umma_desc_sw128(smem_u32(a)), umma_desc_sw128(smem_u32(b)), id, 0u);
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[16];
  tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), v);
  out[warp * 32 + lane] = v[0];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * sizeof(float));
  const char* names[2] = {"f16", "bf16"};
  for (uint32_t af = 0; af < 2; ++af)
    for (uint32_t bf = 0; bf < 2; ++bf) {
      cudaMemset(d, 0, 128 * sizeof(float));
      mixed_kernel<<<1, 128>>>(d, af, bf);
      cudaError_t e = cudaDeviceSynchronize();
      float h[128];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      // expected D[r][0] = 16 * (r%4+1)*0.5 * 2 = 16 * (r%4+1)
      int bad = 0;
      for (int r = 0; r < 128; ++r) bad += h[r] != 16.0f * (r % 4 + 1);
      printf("A %-4s B %-4s: D[0..3] = %g %g %g %g  mismatches %d  (%s)\n", names[af], names[bf], h[0], h[1], h[2],
             h[3], bad, cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
    }
  return 0;
}
