// TMEM read bandwidth (tcgen05.ld.32x32b) per SM on sm_100a, alone and while
// one thread keeps the tensor core busy with back-to-back SS MMAs into other
// TMEM columns: does reading accumulators out of TMEM (the 3xTF32 phase folds,
// the attention's S rows) contend with the MMA?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2510_10129_b200/csrc \
//        -o scripts/micro_tmem.bin scripts/micro_tmem.cu -lcuda && scripts/micro_tmem.bin
#include <cstdio>
#include <vector>

#include "cc_common.cuh"

using namespace cc;

__device__ __forceinline__ void ld32_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// LDW loader warps (warps 1..LDW, lane quarter = warp % 4) each read BATCH x 32
// columns then wait, `iters` times; warp 0 lane 0 optionally issues MMAs
// (bf16 M128 N256 K16 into columns [256, 512)) for the whole loader run.
template <int LDW, int BATCH, bool MMA, bool NOLD = false>
__global__ void __launch_bounds__(32 * (LDW + 1), 1) tmem_bw_kernel(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ volatile uint32_t done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&slot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    done = 0;
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3C003C00u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    if (MMA && lane == 0) {
      const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 16 * 1024);
      constexpr uint32_t idesc = umma_idesc(128, 256, false);
      long long n = 0;
      const long long t0 = clock64();
      while (done < LDW) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma<false>(tmem + 256, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc, 1u);
        n += 4;
        if ((n & 63) == 0) {  // keep the issue queue bounded
          tc_commit(&bar);
          mbar_wait(&bar, (uint32_t)((n >> 6) - 1) & 1u);
        }
      }
      const long long t1 = clock64();
      out[gridDim.x * 2 + blockIdx.x] = (long long)((double)n * 128.0 / (double)(t1 - t0) * 1000.0);  // MMA duty x1000
    }
  } else {
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t r[BATCH][32];
    uint32_t acc = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (NOLD) {
        __nanosleep(200);
        continue;
      }
#pragma unroll
      for (int b = 0; b < BATCH; ++b) ld32_nowait(base + ((it * BATCH + b) & 7) * 32, r[b]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int b = 0; b < BATCH; ++b)
#pragma unroll
        for (int c = 0; c < 32; ++c) acc ^= r[b][c];
    }
    const long long t1 = clock64();
    if (lane == 0) {
      atomicAdd((unsigned int*)&done, 1u);
      if (warp == 1) out[blockIdx.x] = t1 - t0;
    }
    if (acc == 0xdeadbeef) out[gridDim.x * 3] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int LDW, int BATCH, bool MMA, bool NOLD = false>
static void run() {
  const int blocks = 148, iters = 2000;
  long long* d;
  cudaMalloc(&d, (blocks * 3 + 1) * sizeof(long long));
  cudaMemset(d, 0, (blocks * 3 + 1) * sizeof(long long));
  auto k = tmem_bw_kernel<LDW, BATCH, MMA, NOLD>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  k<<<blocks, 32 * (LDW + 1), 80 * 1024>>>(d, 50);
  k<<<blocks, 32 * (LDW + 1), 80 * 1024>>>(d, iters);
  cudaDeviceSynchronize();
  std::vector<long long> h(blocks * 3 + 1);
  cudaMemcpy(h.data(), d, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
  double cyc = 0, duty = 0;
  for (int b = 0; b < blocks; ++b) {
    cyc += (double)h[b];
    duty += (double)h[blocks * 2 + b] / 1000.0;
  }
  cyc /= blocks;
  duty /= blocks;
  const double bytes = (double)LDW * iters * BATCH * 32 * 32 * 4;  // per SM
  printf(NOLD ? "(no loads)  " : "");
  printf("loaders=%2d batch=%d mma=%d : %6.1f B/clk/SM TMEM read  %s%5.2f  (%s)\n", LDW, BATCH, (int)MMA,
         bytes / cyc, MMA ? "MMA duty " : "", MMA ? duty : 0.0, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<1, 1, false>();
  run<4, 1, false>();
  run<4, 4, false>();
  run<8, 1, false>();
  run<8, 4, false>();
  run<4, 4, true, true>();
  run<4, 4, true>();
  run<8, 4, true>();
  return 0;
}
