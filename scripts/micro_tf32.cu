// tcgen05.mma kind::tf32 vs kind::f16 issue rate (sm_100a): SM clocks per MMA
// for the 3xTF32 GEMM's shapes, one CTA per SM, back-to-back SS MMAs into TMEM
// with random operands (no loads, no epilogue): is the scoring GEMM MMA-bound?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2510_10129_b200/csrc \
//        -o /tmp/micro_tf32 scripts/micro_tf32.cu -lcuda && /tmp/micro_tf32
#include <cstdio>
#include <vector>

#include "cc_common.cuh"

using namespace cc;

// KIND 0: bf16 (K=16 per MMA), 1: tf32 (K=8 per MMA). N columns, M=128.
template <int KIND, int N>
__global__ void __launch_bounds__(128, 1) mma_rate_kernel(long long* cyc, int iters, uint32_t fill) {
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
    reinterpret_cast<uint32_t*>(smem)[i] = (x & 0x007FFFFFu) | fill;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = umma_idesc(128, N, KIND == 1);
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 32 * 1024);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        tc_mma<KIND == 1>(tmem, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc, 1u);
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

// the 3xTF32 GEMM's k-step: tf32 N=256 MMA into [0, 256) then N=128 into
// DOFF + [0, 128) (DOFF 128: overlaps the first MMA's columns, as in the kernel;
// 256: a separate accumulator)
// EXTRA bit 0: tcgen05.commit to a ring barrier per K-block (4 k-steps);
// bit 1: tcgen05.fence::after_thread_sync per K-block; bit 2: wait on the ring
// barrier committed 3 K-blocks earlier (the GEMM's stage release + refill)
// bit 4: nine more warps wait (mbarrier.try_wait loop) on a barrier the MMA
// thread completes only at the end, as the GEMM's epilogue and producer warps do
template <int DOFF, int EXTRA = 0>
__global__ void __launch_bounds__(320, 1) pair_kernel(long long* cyc, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ uint64_t ring[3];
  __shared__ uint64_t gate;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int r = 0; r < 3; ++r) mbar_init(&ring[r], 1);
    mbar_init(&gate, 1);
    fence_barrier_init();
  }
  uint32_t x = 12345u + threadIdx.x * 7919u + blockIdx.x;
  for (int i = threadIdx.x; i < 192 * 1024 / 4; i += blockDim.x) {
    x = x * 1664525u + 1013904223u;
    uint32_t v = (x & 0x007FFFFFu) | 0x3F800000u;
    if (EXTRA & 32) {  // random sign and exponent in [2^-24, 2^3], like split activations/weights
      const uint32_t y = x * 2654435761u;
      v = (x & 0x007FFFFFu) | ((y >> 31) << 31) | ((103u + (y >> 8) % 27u) << 23);
    }
    if ((EXTRA & 64) && (i & 1)) v = 0u;  // half the elements zero
    reinterpret_cast<uint32_t*>(smem)[i] = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id256 = umma_idesc(128, 256, true), id128 = umma_idesc(128, 128, true);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      // bit 3: the GEMM's smem layout, 3 stages x [A_hi | A_lo] (32 KB) then 3 x [B_hi | B_lo] (32 KB)
      const int st = (EXTRA & 8) ? it % 3 : 0;
      const uint32_t a0 = smem_u32(smem) + st * 32768, a1 = a0 + 16384;
      const uint32_t b0 = smem_u32(smem) + ((EXTRA & 8) ? 3 * 32768 + st * 32768 : 32768);
      if ((EXTRA & 4) && it >= 3) mbar_wait(&ring[it % 3], (uint32_t)((it / 3 - 1) & 1));
      if (EXTRA & 2) tc_fence_after();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        // bit 7: alternate the accumulator buffer (columns [0,256) / [256,512)) every 4 K-blocks
        const uint32_t dbase = (EXTRA & 128) ? (uint32_t)((it >> 2) & 1) * 256u : 0u;
        // bit 8: accumulate = 0 on the first k-step of every 4th K-block (a phase start)
        const uint32_t accf = ((EXTRA & 256) && (it & 3) == 0 && k == 0) ? 0u : 1u;
        tc_mma<true>(tmem + dbase, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), id256, accf);
        tc_mma<true>(tmem + dbase + DOFF, umma_desc_sw128(a1 + k * 32), umma_desc_sw128(b0 + k * 32), id128, 1u);
      }
      if (EXTRA & 1) tc_commit(&ring[it % 3]);
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
    mbar_arrive(&gate);
  } else if ((EXTRA & 16) && warp >= 1) {
    mbar_wait(&gate, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int DOFF, int EXTRA = 0>
static void run_pair(const char* label) {
  const int iters = 2048, blocks = 148;
  long long* d;
  cudaMalloc(&d, blocks * sizeof(long long));
  auto k = pair_kernel<DOFF, EXTRA>;
  const int sm = (EXTRA & 512) ? 232448 - 2048 : 200 * 1024;  // bit 9: the GEMM's full shared-memory carve-out
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  const int threads = (EXTRA & 16) ? 320 : 128;
  k<<<blocks, threads, sm>>>(d, 16);
  k<<<blocks, threads, sm>>>(d, iters);
  cudaDeviceSynchronize();
  std::vector<long long> h(blocks);
  cudaMemcpy(h.data(), d, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (auto v : h) avg += (double)v;
  avg /= blocks;
  printf("%-40s %7.1f clk per k-step (ideal 192)  (%s)\n", label, avg / (iters * 4.0),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

template <int KIND, int N>
static void run(const char* label) {
  const int iters = 4096, blocks = 148;
  long long* d;
  cudaMalloc(&d, blocks * sizeof(long long));
  auto k = mma_rate_kernel<KIND, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const uint32_t fill = KIND == 1 ? 0x3F800000u : 0x3C003C00u;
  k<<<blocks, 128, 100 * 1024>>>(d, 16, fill);
  k<<<blocks, 128, 100 * 1024>>>(d, iters, fill);
  cudaDeviceSynchronize();
  std::vector<long long> h(blocks);
  cudaMemcpy(h.data(), d, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (auto v : h) avg += (double)v;
  avg /= blocks;
  const double per = avg / (iters * 4.0);
  const double flops = 2.0 * 128 * N * (KIND == 1 ? 8 : 16);
  printf("%-28s %7.1f clk/MMA  %7.0f flop/clk/SM  (%s)\n", label, per, flops / per,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<0, 256>("bf16 M128 N256 K16");
  run<0, 128>("bf16 M128 N128 K16");
  run<1, 256>("tf32 M128 N256 K8");
  run<1, 128>("tf32 M128 N128 K8");
  run<1, 64>("tf32 M128 N64 K8");
  run_pair<128>("tf32 N256 [0,256) + N128 [128,256)");
  run_pair<256>("tf32 N256 [0,256) + N128 [256,384)");
  run_pair<0>("tf32 N256 [0,256) + N128 [0,128)");
  run_pair<128, 1>("  + commit per K-block");
  run_pair<128, 2>("  + fence::after_thread_sync per K-block");
  run_pair<128, 3>("  + commit + fence");
  run_pair<128, 5>("  + commit + ring wait (3 deep)");
  run_pair<128, 7>("  + commit + ring wait + fence");
  run_pair<128, 8>("  3 rotating 64 KB stages");
  run_pair<128, 15>("  3 stages + commit + ring + fence");
  run_pair<128, 31>("  ... + 9 warps in mbarrier try_wait");
  run_pair<128, 8 + 32>("  3 stages, random sign/exponent data");
  run_pair<128, 8 + 64>("  3 stages, half zeros");
  run_pair<128, 8 + 32 + 64>("  3 stages, random exp + half zeros");
  run_pair<128, 8 + 128>("  3 stages, alternating accumulators");
  run_pair<128, 8 + 256>("  3 stages, accumulate=0 per phase");
  run_pair<128, 8 + 128 + 256 + 7>("  3 stages, alt acc + acc0 + commit/ring/fence");
  run_pair<128, 8 + 512>("  3 stages, 227 KB smem carve-out");
  run_pair<128, 8 + 16 + 512 + 7>("  3 stages, 227 KB, 320 thr, commit/ring/fence");
  return 0;
}
