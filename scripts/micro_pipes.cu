// Pipe micro-benchmarks for the attention softmax budget (sm_100a):
// cycles per warp-instruction of MUFU.EX2, FFMA2, FADD2, F2FP with W warps
// per SM issuing independent chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/micro_pipes scripts/micro_pipes.cu && /tmp/micro_pipes
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>

constexpr int CH = 8;      // independent chains per thread
constexpr int ITERS = 4096;

template <int OP>
__global__ void pipe_kernel(float* out, long long* cyc, float seed) {
  float v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = seed * (c + 1) * 1e-3f - 0.5f;
  float2 w[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) w[c] = make_float2(v[c], v[c] + 0.25f);
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[c]));
      } else if (OP == 1) {
        w[c] = __ffma2_rn(w[c], make_float2(0.999f, 0.999f), make_float2(1e-4f, 1e-4f));
      } else if (OP == 2) {
        w[c] = __fadd2_rn(w[c], make_float2(1e-4f, -1e-4f));
      } else if (OP == 3) {
        __nv_bfloat162 b = __floats2bfloat162_rn(w[c].x, w[c].y);
        acc += *reinterpret_cast<uint32_t*>(&b);
        w[c].x += 1e-3f;
      } else if (OP == 4) {
        v[c] = fmaf(v[c], 0.999f, 1e-4f);
      } else if (OP == 5) {  // EX2 + F2FP
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[c]));
        __nv_bfloat162 b = __floats2bfloat162_rn(w[c].x, w[c].y);
        acc += *reinterpret_cast<uint32_t*>(&b);
        w[c].x += 1e-3f;
      } else if (OP == 6) {  // EX2 + FFMA2
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[c]));
        w[c] = __ffma2_rn(w[c], make_float2(0.999f, 0.999f), make_float2(1e-4f, 1e-4f));
      } else if (OP == 7) {  // F2FP + FFMA2
        __nv_bfloat162 b = __floats2bfloat162_rn(w[c].x, w[c].y);
        acc += *reinterpret_cast<uint32_t*>(&b);
        w[c] = __ffma2_rn(w[c], make_float2(0.999f, 0.999f), make_float2(1e-4f, 1e-4f));
      } else if (OP == 9) {  // EX2 on packed bf16x2 (two exps per instruction)
        uint32_t u = __float_as_uint(w[c].x);
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u));
        w[c].x = __uint_as_float(u);
      } else if (OP == 10) {  // EX2 on packed f16x2
        uint32_t u = __float_as_uint(w[c].y);
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u));
        w[c].y = __uint_as_float(u);
      } else if (OP == 8) {  // FMNMX3
        v[c] = fmaxf(v[c], fmaxf(w[c].x, w[c].y));
        w[c].x = -w[c].x;
      }
    }
  }
  const long long t1 = clock64();
  __syncthreads();
  float s = acc;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c] + w[c].x + w[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  for (int rep = 0; rep < 2; ++rep) pipe_kernel<OP><<<148, warps * 32>>>(out, cyc, 1.0f);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const double per = (double)h[0] / (ITERS * CH);  // cycles per warp-instruction per warp
  printf("%-11s warps/SM %2d: %6.2f cyc per instr per warp -> %5.2f warp-instr/clk/SM\n", name, warps, per,
         warps / per);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("EX2", w);
    run<1>("FFMA2", w);
    run<2>("FADD2", w);
    run<3>("F2FP", w);
    run<4>("FFMA", w);
    run<5>("EX2+F2FP", w);
    run<6>("EX2+FFMA2", w);
    run<7>("F2FP+FFMA2", w);
    run<8>("FMNMX3", w);
    run<9>("EX2.BF16X2", w);
    run<10>("EX2.F16X2", w);
  }
  return 0;
}
