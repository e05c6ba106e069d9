// tcgen05.mma issue-rate micro-benchmark (sm_100a): SM clocks per MMA for the
// attention / GEMM shapes, one CTA per SM, back-to-back MMAs into TMEM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2510_10129_b200/csrc \
//        -o /tmp/micro_umma scripts/micro_umma.cu -lcuda && /tmp/micro_umma
#include "cc_common.cuh"

using namespace cc;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

// MODE 0: SS (A, B from smem), 1: TS (A from TMEM), 2: SS with B MN-major
// LDW background warps (warps 4..) stream tcgen05.ld x32 over TMEM columns
// [0, 256) of their lane quarter while warp 0 issues MMAs (softmax-like load)
template <int MODE, int N, int LDW>
__global__ void __launch_bounds__(128 + 32 * LDW, 1) umma_kernel(long long* cyc, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ uint32_t stop;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    stop = 1u;
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = umma_idesc(128, N, false) | (MODE == 2 ? (1u << 16) : 0u);
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 32 * 1024);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (MODE == 1)
          mma_ts(tmem + 256, tmem + k * 8, umma_desc_sw128(b0 + (k & 3) * 32), idesc, 1u);
        else
          tc_mma<false>(tmem + 256, umma_desc_sw128(a0 + (k & 3) * 32), umma_desc_sw128(b0 + (k & 3) * 32), idesc,
                        1u);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
    asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(smem_u32(&stop)), "r"(0u));
  }
  if (LDW > 0 && warp >= 4) {
    float v[32], acc = 0.f;
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    for (int it = 0; it < iters * 4; ++it) {
      tmem_ld32(base + (it & 7) * 32, v);
      acc += v[it & 31];
      if (*(volatile uint32_t*)&stop == 0u) break;
    }
    if (acc == 12345.f) cyc[1000] = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// attention pattern: S = Q K^T (Q 128x128, K 128 keys x 128, K-major SW128, two
// 64-element K-blocks) into cols [0,128); O += P V with P from TMEM cols [0,64)
// and V MN-major (LBO 16 KB, SBO 1 KB) into cols [128, 256). Random smem data.
__device__ __forceinline__ uint64_t desc_mn(uint32_t a, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
template <int PATTERN>
__global__ void __launch_bounds__(128, 1) attn_mma_kernel(long long* cyc, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  uint32_t x = 12345u + threadIdx.x * 7919u + blockIdx.x;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) {
    x = x * 1664525u + 1013904223u;
    reinterpret_cast<uint32_t*>(smem)[i] = (x & 0x3FFF3FFFu) | 0x3C003C00u;  // bf16 pairs in [1, 2)
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t idS = umma_idesc(128, 128, false);
  constexpr uint32_t idPV = umma_idesc(128, 128, false) | (1u << 16);
  if (threadIdx.x == 0) {
    const uint32_t q0 = smem_u32(smem), k0 = smem_u32(smem + 32 * 1024), v0 = smem_u32(smem + 64 * 1024);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (PATTERN & 1) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t off = (k >> 2) * (128 * 128) + (k & 3) * 32;
          tc_mma<false>(tmem + 256, umma_desc_sw128(q0 + off), umma_desc_sw128(k0 + off), idS, k > 0 ? 1u : 0u);
        }
      }
      if (PATTERN & 2) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          mma_ts(tmem + 384, tmem + k * 8, desc_mn(v0 + k * 16 * 128, 128 * 128, 1024), idPV, 1u);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int PATTERN>
void run_attn(const char* name) {
  long long* d;
  const int ctas = 148, iters = 2000;
  cudaMalloc(&d, sizeof(long long) * ctas);
  cudaFuncSetAttribute(attn_mma_kernel<PATTERN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 97 * 1024);
  attn_mma_kernel<PATTERN><<<ctas, 128, 97 * 1024>>>(d, iters);
  attn_mma_kernel<PATTERN><<<ctas, 128, 97 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(long long) * ctas, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < ctas; ++i) mx = h[i] > mx ? h[i] : mx;
  const int groups = (PATTERN == 3 ? 2 : 1);
  printf("%-34s %7.1f clk per 8-MMA group (ideal 512)  %s\n", name, mx / (iters * groups),
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

template <int MODE, int N, int LDW = 0>
void run(const char* name, int ctas) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * ctas);
  const int iters = 2000;
  cudaFuncSetAttribute(umma_kernel<MODE, N, LDW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  umma_kernel<MODE, N, LDW><<<ctas, 128 + 32 * LDW, 96 * 1024>>>(d, iters);
  umma_kernel<MODE, N, LDW><<<ctas, 128 + 32 * LDW, 96 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(long long) * ctas, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < ctas; ++i) mx = h[i] > mx ? h[i] : mx;
  const double per = mx / (iters * 8.0);
  const double ideal = 128.0 * N * 16 * 2 / 8192.0;
  printf("%-28s ctas %3d: %7.1f clk per MMA (ideal %5.1f at 8192 flop/clk/SM) -> %.2f  %s\n", name, ctas, per,
         ideal, ideal / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run_attn<1>("attn S only (random data)");
  run_attn<2>("attn PV only (random data)");
  run_attn<3>("attn S + PV alternating");
  run<0, 128, 4>("SS N128 + 4 ld warps", 148);
  run<0, 128, 8>("SS N128 + 8 ld warps", 148);
  run<1, 128, 8>("TS N128 + 8 ld warps", 148);
  for (int ctas : {148}) {
    run<0, 128>("SS M128 N128 K16", ctas);
    run<0, 256>("SS M128 N256 K16", ctas);
    run<1, 128>("TS M128 N128 K16 (A tmem)", ctas);
    run<1, 256>("TS M128 N256 K16 (A tmem)", ctas);
    run<2, 128>("SS M128 N128 B MN-major", ctas);
  }
  return 0;
}
