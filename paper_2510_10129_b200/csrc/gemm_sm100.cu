// Persistent warp-specialised tcgen05 GEMM for sm_100a with fused epilogues.
//
//   C[M,N] = A[M,K] · B[N,K]^T      (A activations, B weights [out, in], both K-major)
//
// Roles per CTA (192 threads, one CTA per SM):
//   warp 0      TMA producer: A/B tiles -> 128B-swizzled smem ring (mbarrier full/empty)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, fp32 in TMEM)
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> registers -> fused op -> global
// Two TMEM accumulators (2 x BN columns) let the epilogue of tile i overlap the
// MMAs of tile i+1. kind::f16 (bf16) for the primary model; kind::tf32 for the
// scoring model as 3xTF32 (fp32-faithful): operands are stored split, A' =
// [hi|hi|lo] and B' = [hi|lo|hi]; a pipeline stage holds the hi and lo
// sub-tiles of both (each loaded once) and feeds three MMAs: hi*hi into one
// accumulator, hi*lo + lo*hi into a second; the epilogue adds the two in fp32.
//
// Replaces the numpy `x @ W` of attention_qkv / _attn_project_out / _mlp
// (model.py:340-432) and fuses bias, RoPE + K/V scatter (model.py:709-714),
// residual add and the gated activation (model.py:418-426) into the epilogue.
#include "cc_common.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

namespace cc {

constexpr int kBM = 128;
constexpr int kEpiWarps = 8;  // two per TMEM lane quarter (column halves)
constexpr int kGemmThreads = 64 + 32 * kEpiWarps;
constexpr int kEpiStageBytes = 32 * 32 * 4;
// 3xTF32: K-blocks (32 K each) accumulated in TMEM before the epilogue folds
// the partial into fp32 registers (see the MMA loop). 8 (256 K): the CTA-pair
// kernel's per-phase handshake (commit, fold, remote arrive) stalls the MMA
// warp at 4 (C3 scoring GEMMs 6.95 ms per pass at 4, 6.54 at 8, 6.46 with no
// phases); scoring error vs fp64 median 6.4e-7 -> 6.9e-7, p99 2.79e-6 ->
// 2.84e-6, selections still exact at C2/C3 (profiles/r2_tf32_phases.md)
#ifndef CC_TF32_KB_PER_PHASE
#define CC_TF32_KB_PER_PHASE 8
#endif
constexpr int kTf32KbPerPhase = CC_TF32_KB_PER_PHASE;

#ifdef CC_GEMM_TRACE  // debug builds only: MMA-warp wait timeline of block 0 (clock64)
__device__ long long g_gemm_trace[5 * 4096];
#define GT(slot, i)                                                            \
  do {                                                                         \
    if (blockIdx.x == 0 && lane == 0 && (i) < 4096) g_gemm_trace[(slot) * 4096 + (i)] = clock64(); \
  } while (0)
#else
#define GT(slot, i) \
  do {              \
  } while (0)
#endif

template <int BN, bool kTF32>
struct GemmCfg {
  static constexpr int ELEM = kTF32 ? 4 : 2;
  static constexpr int BK = 128 / ELEM;  // one 128-byte swizzle row per tile row
  static constexpr int UK = kTF32 ? 8 : 16;
  static constexpr int KSTEPS = BK / UK;
  // 3xTF32: a stage holds the hi and lo sub-tiles of both operands (loaded
  // once, consumed by the three MMAs hi*hi, hi*lo, lo*hi)
  static constexpr int NSUB = kTF32 ? 2 : 1;
  static constexpr int A_SUB = kBM * 128;
  static constexpr int B_SUB = BN * 128;
  static constexpr int A_BYTES = NSUB * A_SUB;
  static constexpr int B_BYTES = NSUB * B_SUB;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int FIXED = kEpiWarps * kEpiStageBytes + 1024 + 256;
  static constexpr int FIT = (232448 - FIXED) / STAGE_BYTES;
  static constexpr int STAGES = FIT > 6 ? 6 : FIT;
  // two accumulator buffers; 3xTF32 keeps hi*hi and the hi*lo + lo*hi
  // corrections in separate accumulators (summed in fp32 by the epilogue)
  static constexpr int ACC_STRIDE = kTF32 ? 2 * BN : BN;
  static constexpr int TMEM_COLS = 2 * ACC_STRIDE;
  static_assert(TMEM_COLS <= 512, "TMEM holds 512 columns");
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + FIXED;
  static constexpr uint32_t IDESC = umma_idesc(kBM, BN, kTF32);
  static constexpr uint32_t IDESC2 = umma_idesc(kBM, 2 * BN, kTF32);  // 3xTF32: [B_hi; B_lo] in one MMA
  static_assert(!kTF32 || 2 * BN <= 256, "3xTF32 fused hi*[hi;lo] MMA needs N = 2*BN <= 256");
  static_assert(STAGES >= 2, "GEMM pipeline needs two stages");
  static_assert(SMEM_BYTES <= 232448, "GEMM shared memory over the sm_100 per-CTA limit");
};

struct EpiParams {
  int epilogue;
  int64_t M, N;
  const float* bias;
  void* C;
  int64_t ldc;
  int c_mode;
  int act;
  int glu_block;
  int64_t n_out;
  int n_q_heads, n_kv_heads, head_dim;
  const float* rope_cos;
  const float* rope_sin;
  void* q_out;
  int64_t ldq;
  int q_mode;
  void* k_cache;
  void* v_cache;
  int cache_dtype;
  const int64_t* dst_rows;
  void* k_raw;
  const int64_t* raw_rows;
  // fused RMSNorm (see cc_gemm_args)
  void* xn_out;
  int64_t ldxn;
  const float* norm_gain;
  float* ssq_out;
  const float* ssq_in;  // inv_rms [M]
  int64_t ld_ssq;
  // or the producer's partial sums (1/rms formed in the epilogue)
  const float* ssq_parts;
  int n_parts;
  int64_t ld_parts;
  float eps;
  float inv_d;
};

// The epilogue mode: a compile-time constant when the kernel is specialised
// on it (kEpi >= 0; fewer live registers, no spills to L2-backed local memory
// under the full shared-memory carve-out), else the runtime field.
__device__ __forceinline__ int epi_of(const EpiParams& ep, int kEpi) { return kEpi >= 0 ? kEpi : ep.epilogue; }

// 1 / rms of GEMM row m: given (cc_norm_finalize reduced the producer's
// partial sums), or formed here from the partials with the same arithmetic
// and summation order (32 loads in flight)
__device__ __forceinline__ bool row_scaled(const EpiParams& ep) { return ep.ssq_in || ep.ssq_parts; }
__device__ __forceinline__ float row_inv_rms(const EpiParams& ep, int64_t m) {
  if (m >= ep.M) return 0.f;
  if (ep.ssq_in) return __ldg(ep.ssq_in + m);
  const float* p = ep.ssq_parts + m;
  float s = 0.f;
  int i = 0;
  for (; i + 32 <= ep.n_parts; i += 32) {
    float t[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) t[j] = __ldg(p + (int64_t)(i + j) * ep.ld_parts);
#pragma unroll
    for (int j = 0; j < 32; ++j) s = __fadd_rn(s, t[j]);
  }
  for (; i + 8 <= ep.n_parts; i += 8) {
    float t[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) t[j] = __ldg(p + (int64_t)(i + j) * ep.ld_parts);
#pragma unroll
    for (int j = 0; j < 8; ++j) s = __fadd_rn(s, t[j]);
  }
  for (; i < ep.n_parts; ++i) s = __fadd_rn(s, __ldg(p + (int64_t)i * ep.ld_parts));
  return __frcp_rn(__fsqrt_rn(__fadd_rn(__fmul_rn(s, ep.inv_d), ep.eps)));
}

__device__ __forceinline__ float act_apply(int act, float x) {
  return act == CC_ACT_SILU ? silu_f(x) : gelu_tanh_f(x);
}

// Store 4 consecutive values of one row (cols [col, col+4)) in `mode`; the
// split layout keeps a 3*ld row pitch with [hi | hi | lo] segments `width` apart
// (activations: only the hi and lo segments are written; the 3xTF32 GEMM reads
// A_hi at column k and A_lo at 2K + k).
__device__ __forceinline__ void store4(void* base, int mode, int64_t row, int64_t ld, int64_t col, int64_t width,
                                       float4 v) {
  if (mode == CC_BF16) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(base) + row * ld + col) = u;
  } else if (mode == CC_F32) {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(base) + row * ld + col) = v;
  } else {  // CC_F32_SPLIT3 : [hi | hi | lo]
    float* p = reinterpret_cast<float*>(base) + row * ld * 3 + col;
    const float e[4] = {v.x, v.y, v.z, v.w};
    float hi[4], lh[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float lo, ll;
      split_tf32(e[i], hi[i], lo);
      split_tf32(lo, lh[i], ll);
    }
    const float4 h4 = make_float4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<float4*>(p) = h4;  // the middle hi copy is never read (the GEMM loads hi and lo only)
    *reinterpret_cast<float4*>(p + 2 * width) = make_float4(lh[0], lh[1], lh[2], lh[3]);
  }
}

__device__ __forceinline__ float4 ld_bias4(const float* b, int64_t col) {
  return b ? *reinterpret_cast<const float4*>(b + col) : make_float4(0.f, 0.f, 0.f, 0.f);
}

// Epilogue staging: each epilogue warp owns a 32 x 32 fp32 tile in smem.
// Element (r, c) lives at r*32 + ((c/4) ^ (r%8))*4 + c%4 — a 16-byte-granule
// XOR swizzle, so both the row-per-lane writes (TMEM layout) and the
// 8-lanes-per-row reads (coalesced global layout) are bank-conflict free.
__device__ __forceinline__ void stage_row32(float* stg, int r, const float* v) {
#pragma unroll
  for (int g = 0; g < 8; ++g)
    *reinterpret_cast<float4*>(stg + r * 32 + ((g ^ (r & 7)) << 2)) =
        make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
}
__device__ __forceinline__ float4 unstage4(const float* stg, int r, int g) {
  return *reinterpret_cast<const float4*>(stg + r * 32 + ((g ^ (r & 7)) << 2));
}

// One 32-row x 32-column chunk of the accumulator: TMEM -> registers (lane =
// row) -> swizzled smem -> 8 passes of 4 rows x 8 lanes x 4 columns, so every
// global access is a contiguous 128-byte (fp32) / 64-byte (bf16) row segment.
// Row-local math (GLU) runs in the lane-per-row layout; column-indexed math
// (bias, RoPE pairs, residual) runs in the coalesced layout.
// First weight row of half `h` (0: columns [0, BN/2), 1: [BN/2, BN)) of tile
// column block nb. GLU weights interleave gate/up in blocks of glu_block rows;
// a GLU tile holds BN/2 gate rows and the matching BN/2 up rows, so the
// epilogue finds gate at accumulator column c and up at c + BN/2.
template <int BN, int kEpi = -1>
__device__ __forceinline__ int b_row(const EpiParams& ep, int nb, int h) {
  if (epi_of(ep, kEpi) != CC_EPI_GLU) return nb * BN + h * (BN / 2);
  const int per_blk = 2 * ep.glu_block / BN;  // tiles per gate/up block pair
  return (nb / per_blk) * 2 * ep.glu_block + (nb % per_blk) * (BN / 2) + h * ep.glu_block;
}

// accumulator columns [c, c+n) (+ the 3xTF32 correction accumulator)
template <int BN, bool kTF32>
__device__ __forceinline__ void acc_ld16(uint32_t taddr, float* v) {
  tmem_ld16(taddr, v);
  if constexpr (kTF32) {
    float w[16];
    tmem_ld16(taddr + BN, w);
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __fadd_rn(v[j], w[j]);
  }
}

// gate/up -> act(gate + b_gate) * (up + b_up) for 16 accumulator columns
// [c, c + 16) of a GLU tile (lane-per-row layout)
template <int BN, int kEpi = -1>
__device__ __forceinline__ void glu16(const EpiParams& ep, int nb, int c, float* g16, const float* u16) {
  const int64_t gcol = b_row<BN, kEpi>(ep, nb, 0) + c;  // interleaved gate row of column c
  float up[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    up[j] = u16[j];
    if (ep.bias) {
      g16[j] += ep.bias[gcol + j];
      up[j] += ep.bias[gcol + ep.glu_block + j];
    }
  }
  if (ep.act == CC_ACT_SILU) {
    silu_n<16>(g16);
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) g16[j] = gelu_tanh_f(g16[j]);
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) g16[j] = __fmul_rn(g16[j], up[j]);
}

template <int BN, int kEpi = -1>
__device__ __forceinline__ void epilogue_tail(const EpiParams& ep, float* v, int c0, int64_t row0, int nb,
                                              float* stg, int lane);

// split-K: the other K-slices' fp32 partial accumulators of this lane's row,
// [n_parts][128 rows][BN], added onto the owner's own in slice order (fixed,
// so the result is deterministic)
struct SplitParts {
  const float* p;  // this tile's first partial, row 0 of the CTA (nullptr: no split)
  int n;           // partials to add
  int lrow;        // this lane's row within the 128-row tile
};
template <int BN>
__device__ __forceinline__ void add_parts16(const SplitParts& sp, int col, float* v) {
  for (int s = 0; s < sp.n; ++s) {
    const float4* src = reinterpret_cast<const float4*>(sp.p + ((size_t)s * kBM + sp.lrow) * BN + col);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 x = __ldcg(src + i);
      v[4 * i] += x.x;
      v[4 * i + 1] += x.y;
      v[4 * i + 2] += x.z;
      v[4 * i + 3] += x.w;
    }
  }
}

// rs: this lane's row 1/rms (row_inv_rms, formed once per tile by the caller)
template <int BN, bool kTF32, int kEpi = -1>
__device__ __forceinline__ void epilogue_chunk(const EpiParams& ep, uint32_t tbase, int c0, int64_t row0, int nb,
                                               float* stg, int lane, float rs,
                                               const SplitParts& sp = SplitParts{nullptr, 0, 0}) {
  float v[32];
  const bool scaled = row_scaled(ep);
  if (epi_of(ep, kEpi) == CC_EPI_GLU) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {  // 16 columns at a time (register budget)
      float u[16];
      acc_ld16<BN, kTF32>(tbase + c0 + 16 * hh, v + 16 * hh);
      acc_ld16<BN, kTF32>(tbase + c0 + 16 * hh + BN / 2, u);
      if (sp.p) {
        add_parts16<BN>(sp, c0 + 16 * hh, v + 16 * hh);
        add_parts16<BN>(sp, c0 + 16 * hh + BN / 2, u);
      }
      if (scaled) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          v[16 * hh + j] = __fmul_rn(v[16 * hh + j], rs);
          u[j] = __fmul_rn(u[j], rs);
        }
      }
      glu16<BN, kEpi>(ep, nb, c0 + 16 * hh, v + 16 * hh, u);
    }
  } else {
    acc_ld16<BN, kTF32>(tbase + c0, v);
    acc_ld16<BN, kTF32>(tbase + c0 + 16, v + 16);
    if (sp.p) {
      add_parts16<BN>(sp, c0, v);
      add_parts16<BN>(sp, c0 + 16, v + 16);
    }
    if (scaled) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = __fmul_rn(v[j], rs);
    }
  }
  epilogue_tail<BN, kEpi>(ep, v, c0, row0, nb, stg, lane);
}

// v: the 32 output values of accumulator columns [c0, c0 + 32) of this lane's
// row (GLU: already combined); staged through smem and stored coalesced
template <int BN, int kEpi>
__device__ __forceinline__ void epilogue_tail(const EpiParams& ep, float* v, int c0, int64_t row0, int nb,
                                              float* stg, int lane) {
  const int epi = epi_of(ep, kEpi);
  int64_t colbase;  // global output column of the chunk's column 0
  int64_t width;    // logical output width (column bound)
  if (epi == CC_EPI_GLU) {
    colbase = (int64_t)nb * (BN / 2) + c0;
    width = ep.n_out;
  } else {
    colbase = (int64_t)nb * BN + c0;
    width = ep.N;
  }
  stage_row32(stg, lane, v);
  __syncwarp();
  const int g = lane & 7;
  const int64_t col = colbase + 4 * g;
  if (col >= width) {
    __syncwarp();
    return;
  }
  // pass p covers rows 4p + lane/8; every global load of the chunk is issued
  // before the first dependent store (eight independent requests in flight)
  const int rl = lane >> 3;
  const int64_t m_left = ep.M - row0;
  switch (epi) {
    case CC_EPI_GLU:
#pragma unroll
      for (int ps = 0; ps < 8; ++ps)
        if (ps * 4 + rl < m_left) store4(ep.C, ep.c_mode, row0 + ps * 4 + rl, ep.ldc, col, width,
                                         unstage4(stg, ps * 4 + rl, g));
      break;
    case CC_EPI_STORE:
    case CC_EPI_ACT: {
      const float4 b = ld_bias4(ep.bias, col);
#pragma unroll
      for (int ps = 0; ps < 8; ++ps) {
        const int r = ps * 4 + rl;
        if (r >= m_left) continue;
        float4 x = unstage4(stg, r, g);
        x.x += b.x;
        x.y += b.y;
        x.z += b.z;
        x.w += b.w;
        if (epi == CC_EPI_ACT) {
          x.x = act_apply(ep.act, x.x);
          x.y = act_apply(ep.act, x.y);
          x.z = act_apply(ep.act, x.z);
          x.w = act_apply(ep.act, x.w);
        }
        store4(ep.C, ep.c_mode, row0 + r, ep.ldc, col, width, x);
      }
      break;
    }
    case CC_EPI_RESIDUAL: {
      const float4 b = ld_bias4(ep.bias, col);
      float* hb = reinterpret_cast<float*>(ep.C) + row0 * ep.ldc + col;
      float4 o[8];
#pragma unroll
      for (int ps = 0; ps < 8; ++ps)
        if (ps * 4 + rl < m_left) o[ps] = *reinterpret_cast<const float4*>(hb + (ps * 4 + rl) * ep.ldc);
      const bool fuse = ep.ssq_out != nullptr;  // next RMSNorm's operand + partial sums
      const float4 gn = fuse ? *reinterpret_cast<const float4*>(ep.norm_gain + col) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int ps = 0; ps < 8; ++ps) {
        const int r = ps * 4 + rl;
        float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < m_left) {
          const float4 x = unstage4(stg, r, g);
          y = o[ps];
          y.x = __fadd_rn(y.x, x.x + b.x);
          y.y = __fadd_rn(y.y, x.y + b.y);
          y.z = __fadd_rn(y.z, x.z + b.z);
          y.w = __fadd_rn(y.w, x.w + b.w);
          *reinterpret_cast<float4*>(hb + r * ep.ldc) = y;
          if (fuse)
            store4(ep.xn_out, CC_BF16, row0 + r, ep.ldxn, col, width,
                   make_float4(__fmul_rn(y.x, gn.x), __fmul_rn(y.y, gn.y), __fmul_rn(y.z, gn.z), __fmul_rn(y.w, gn.w)));
        }
        if (fuse) {  // warp-uniform: the 8 lanes of a row reduce their 4 columns in a fixed order
          float ss = __fmaf_rn(y.w, y.w, __fmaf_rn(y.z, y.z, __fmaf_rn(y.y, y.y, __fmul_rn(y.x, y.x))));
          ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, 1));
          ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, 2));
          ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, 4));
          if (g == 0 && r < m_left) ep.ssq_out[(colbase >> 5) * ep.ld_ssq + row0 + r] = ss;
        }
      }
      break;
    }
    case CC_EPI_QKV_ROPE: {
      const float4 b = ld_bias4(ep.bias, col);
      const int dh = ep.head_dim;
      const int64_t qw = (int64_t)ep.n_q_heads * dh, kw = (int64_t)ep.n_kv_heads * dh;
      const bool rot = col < qw + kw;
      const int half = dh >> 1;
      const int pr = (int)(col % dh) >> 1;
#pragma unroll
      for (int half_p = 0; half_p < 2; ++half_p) {  // two batches of 4 passes (register budget)
        float2 cs[4], sn[4];
        int64_t drow[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = (half_p * 4 + q) * 4 + rl;
          const int64_t grow = row0 + r;
          if (r >= m_left) continue;
          if (rot) {
            cs[q] = *reinterpret_cast<const float2*>(ep.rope_cos + grow * half + pr);
            sn[q] = *reinterpret_cast<const float2*>(ep.rope_sin + grow * half + pr);
          }
          if (col >= qw) drow[q] = ep.dst_rows ? ep.dst_rows[grow] : grow;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = (half_p * 4 + q) * 4 + rl;
          if (r >= m_left) continue;
          const int64_t grow = row0 + r;
          float4 x = unstage4(stg, r, g);
          x.x += b.x;
          x.y += b.y;
          x.z += b.z;
          x.w += b.w;
          if (rot) {
            float4 r4;
            rope_pair(x.x, x.y, cs[q].x, sn[q].x, r4.x, r4.y);
            rope_pair(x.z, x.w, cs[q].y, sn[q].y, r4.z, r4.w);
            if (col < qw) {
              store4(ep.q_out, ep.q_mode, grow, ep.ldq, col, qw, r4);
            } else {
              store4(ep.k_cache, ep.cache_dtype, drow[q], kw, col - qw, kw, r4);
              if (ep.k_raw) {
                const int64_t rrow = ep.raw_rows ? ep.raw_rows[grow] : grow;
                store4(ep.k_raw, ep.cache_dtype, rrow, kw, col - qw, kw, x);
              }
            }
          } else {
            store4(ep.v_cache, ep.cache_dtype, drow[q], kw, col - qw - kw, kw, x);
          }
        }
      }
      break;
    }
    default:
      break;
  }
  __syncwarp();  // the staging tile is reused by the next chunk
}

// Tile t of a persistent schedule -> (m tile, n tile). group_m = 0: m fastest
// over all m (a wave shares the B panels of a few n tiles and re-reads all of
// A per wave: right when A stays in L2 and B does not). group_m = g: m fastest
// inside bands of g m tiles, so a wave covers ~g x (wave / g) tiles and reads
// each A and B panel about once per band.
__device__ __forceinline__ void tile_mn(int t, int num_m, int num_n, int group_m, int& mb, int& nb) {
  if (group_m <= 0 || group_m >= num_m) {
    mb = t % num_m;
    nb = t / num_m;
    return;
  }
  const int per = group_m * num_n;  // tiles per full band (every band but the last is full)
  const int g = t / per, local = t - g * per;
  const int m0 = g * group_m, gm = min(group_m, num_m - m0);
  mb = m0 + local % gm;
  nb = local / gm;
}


// Band size for a persistent GEMM schedule (tile_mn): a wave of the grid over
// an a x b block of tiles reads ~(a + b) operand panels from DRAM. m fastest
// over all m is right only when A is small enough to stay in L2 and B is not
// (the recompute's gate/up: A 47 MB, B 271 MB, B read once); otherwise band
// (measured on the CTA-pair kernel, ncu DRAM read: down 1.79 -> 1.20 GB, qkv
// 189 -> 143 MB, o 292 -> 213 MB; at M = 34,816 rows (chunk precompute, full
// prefill) m fastest re-reads all of A for every n tile). CC_GEMM_GROUP=g in
// the environment forces a band of g (0: m fastest).
static int schedule_band(const cc_gemm_args* a, double elem, int band) {
  static const int group_env = [] {
    const char* e = getenv("CC_GEMM_GROUP");
    return e ? atoi(e) : -1;
  }();
  if (group_env >= 0) return group_env;
  const double l2_half = 60e6;
  const bool a_small = (double)a->M * a->K * elem <= l2_half, b_small = (double)a->N * a->K * elem <= l2_half;
  return (a_small && !b_small) ? 0 : band;
}

template <int BN, bool kTF32, int kEpi = -1>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, EpiParams ep,
                int num_m, int num_n, int num_kb, int k_orig, int kb_per_phase, int group_m) {
  using Cfg = GemmCfg<BN, kTF32>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + Cfg::STAGES * Cfg::A_BYTES;
  uint8_t* smem_epi = smem + Cfg::STAGES * Cfg::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_epi + kEpiWarps * kEpiStageBytes);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles = num_m * num_n;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // the prologue above touched no global memory
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
#ifdef CC_DBG_GEMM_NO_LOADS  // perf experiments only: after the first ring, stages are released without data
      int issued = 0;
#endif
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int mb, nb;
        tile_mn(t, num_m, num_n, group_m, mb, nb);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
#ifdef CC_DBG_GEMM_NO_LOADS
          if (issued++ >= Cfg::STAGES) {
            mbar_arrive(&full[stage]);
            if (++stage == Cfg::STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
#endif
          mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          uint8_t* sa = smem_a + stage * Cfg::A_BYTES;
          uint8_t* sb = smem_b + stage * Cfg::B_BYTES;
          tma_load_2d(sa, &tmA, &full[stage], kb * Cfg::BK, mb * kBM);
          const int br0 = b_row<BN, kEpi>(ep, nb, 0), br1 = b_row<BN, kEpi>(ep, nb, 1);
          tma_load_2d(sb, &tmB, &full[stage], kb * Cfg::BK, br0);
          tma_load_2d(sb + Cfg::B_SUB / 2, &tmB, &full[stage], kb * Cfg::BK, br1);
          if constexpr (kTF32) {  // A' = [hi | hi | lo], B' = [hi | lo | hi]
            tma_load_2d(sa + Cfg::A_SUB, &tmA, &full[stage], 2 * k_orig + kb * Cfg::BK, mb * kBM);
            tma_load_2d(sb + Cfg::B_SUB, &tmB, &full[stage], k_orig + kb * Cfg::BK, br0);
            tma_load_2d(sb + Cfg::B_SUB + Cfg::B_SUB / 2, &tmB, &full[stage], k_orig + kb * Cfg::BK, br1);
          }
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    // 3xTF32: the accumulator buffer rotates every kb_per_phase K-blocks (a
    // "phase"); the epilogue folds each finished phase into fp32 registers with
    // round-to-nearest adds. The tensor core's accumulation truncates once per
    // MMA, a bias that grows linearly with the K steps it accumulates; phases
    // bound that to kb_per_phase * KSTEPS steps (parity at depth).
    // bf16: one phase per tile (the whole K in one accumulator).
    const int per_phase = kTF32 ? kb_per_phase : num_kb;
    int gi = 0;  // trace index (CC_GEMM_TRACE builds)
#ifdef CC_DBG_GEMM_FILL  // perf experiments only (with CC_DBG_GEMM_NO_LOADS): synthetic operand data
    for (int st = 0; st < Cfg::STAGES; ++st) mbar_wait(&full[st], 0);
    for (int i = lane; i < Cfg::STAGES * Cfg::STAGE_BYTES / 4; i += 32) {
      uint32_t x = 12345u + (uint32_t)i * 7919u;
      x = x * 1664525u + 1013904223u;
      reinterpret_cast<uint32_t*>(smem)[i] = (x & 0x007FFFFFu) | 0x3F800000u;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
#endif
    // The whole warp runs the issue loop with warp-uniform operands; one lane
    // elected inside each tcgen05 asm issues (tc_mma_warp). Descriptors are
    // formed once: stage s, k-step k is the base descriptor plus the byte
    // offset >> 4 in its start-address field (< 256 KB: no carry out).
    const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint64_t adesc0 = umma_desc_sw128(smem_u32(smem_a));
    const uint64_t bdesc0 = umma_desc_sw128(smem_u32(smem_b));
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      uint32_t d_tmem = 0;
      for (int kb = 0; kb < num_kb; ++kb, ++gi) {
        const int kp = kb % per_phase;
        GT(0, gi);
        if (kp == 0) {
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          d_tmem = tmem_u + acc * Cfg::ACC_STRIDE;
        }
        GT(1, gi);
        mbar_wait(&full[stage], phase);
        GT(2, gi);
        tc_fence_after();
        const uint64_t ad = adesc0 + (uint64_t)((stage * Cfg::A_BYTES) >> 4);
        const uint64_t bd = bdesc0 + (uint64_t)((stage * Cfg::B_BYTES) >> 4);
#pragma unroll
        for (int k = 0; k < Cfg::KSTEPS; ++k) {
          if constexpr (kTF32) {
            // hi*hi and hi*lo as ONE N = 2*BN MMA: B_hi and B_lo are adjacent
            // 128-byte-row sub-tiles (one 2*BN-row operand) and the two
            // accumulators adjacent TMEM columns, so A_hi is read once; then
            // lo*hi into the correction accumulator
            tc_mma_warp<kTF32>(d_tmem, ad + 2 * k, bd + 2 * k, Cfg::IDESC2, (kp | k) != 0 ? 1u : 0u);
#ifndef CC_DBG_TF32_NO_LOHI  // perf experiments only: drop the lo*hi MMA
            tc_mma_warp<kTF32>(d_tmem + BN, ad + (Cfg::A_SUB >> 4) + 2 * k, bd + 2 * k, Cfg::IDESC, 1u);
#endif
          } else {
            tc_mma_warp<kTF32>(d_tmem, ad + 2 * k, bd + 2 * k, Cfg::IDESC, (kp | k) != 0 ? 1u : 0u);
          }
        }
        tc_commit_warp(&empty[stage]);
        if (kp == per_phase - 1 || kb == num_kb - 1) tc_commit_warp(&tfull[acc]);
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
        if (kp == per_phase - 1 || kb == num_kb - 1) {
          if (++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else {
    // epilogue warps 2..9: TMEM lane quarter = warp % 4, column half = (warp - 2) / 4
    const int ew = warp - 2;
    const int quarter = warp & 3;
    const int chalf = ew >> 2;
    float* stg = reinterpret_cast<float*>(smem_epi + ew * kEpiStageBytes);
    int acc = 0;
    uint32_t acc_phase = 0;
    // GLU tiles produce BN/2 output columns (gate/up pairs), others BN
    const bool glu = epi_of(ep, kEpi) == CC_EPI_GLU;
    const int cols = glu ? BN / 2 : BN;
    const int c_begin = chalf * (cols / 2), c_end = c_begin + cols / 2;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    int epi_i = 0, tile_i = 0;  // trace indices (CC_GEMM_TRACE builds)
    (void)epi_i;
    (void)tile_i;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      int mb, nb;
      tile_mn(t, num_m, num_n, group_m, mb, nb);
      const int64_t row0 = (int64_t)mb * kBM + quarter * 32;
      if constexpr (kTF32) {
        // this warp's accumulator columns, BN/2 per row (GLU: its gate columns
        // then the matching up columns), summed over the phases in registers
        constexpr int NV = BN / 2;
        float run[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) run[j] = 0.f;
        const int n_phases = (num_kb + kb_per_phase - 1) / kb_per_phase;
        for (int ph = 0; ph < n_phases; ++ph) {
          if (ew == 0) GT(3, 2 * epi_i);
          mbar_wait(&tfull[acc], acc_phase);
          if (ew == 0) GT(3, 2 * epi_i + 1);
          ++epi_i;
          tc_fence_after();
          const uint32_t tb = tmem_base + acc * Cfg::ACC_STRIDE + lane_off;
#ifdef CC_DBG_GEMM_NO_EPI  // perf experiments only: no folds, no output
          if (false)
#endif
#pragma unroll
          for (int j = 0; j < NV; j += 16) {
            const int col = (glu && j >= NV / 2) ? c_begin + BN / 2 + (j - NV / 2) : c_begin + j;
            float m16[16], c16[16];
            tmem_ld16(tb + col, m16);
            tmem_ld16(tb + BN + col, c16);
#pragma unroll
            for (int i = 0; i < 16; ++i) run[j + i] = __fadd_rn(run[j + i], __fadd_rn(m16[i], c16[i]));
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
          if (++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
        if (ew == 0) GT(4, 3 * tile_i);
#if defined(CC_DBG_GEMM_NO_EPI) || defined(CC_DBG_GEMM_NO_FINAL)
        if (false)
#endif
        if (glu) {
          // NV/2 = BN/4 output columns: one 32-column chunk (BN = 128)
#pragma unroll
          for (int cc = 0; cc < NV / 2; cc += 32) {
            glu16<BN, kEpi>(ep, nb, c_begin + cc, run + cc, run + NV / 2 + cc);
            glu16<BN, kEpi>(ep, nb, c_begin + cc + 16, run + cc + 16, run + NV / 2 + cc + 16);
            if (ew == 0) GT(4, 3 * tile_i + 1);
            epilogue_tail<BN, kEpi>(ep, run + cc, c_begin + cc, row0, nb, stg, lane);
          }
        } else {
#pragma unroll
          for (int cc = 0; cc < NV; cc += 32) epilogue_tail<BN, kEpi>(ep, run + cc, c_begin + cc, row0, nb, stg, lane);
        }
        if (ew == 0) GT(4, 3 * tile_i + 2);
        ++tile_i;
      } else {
        // 1/rms of this lane's row, formed while the tile's MMAs run
        const float rs = row_scaled(ep) ? row_inv_rms(ep, row0 + lane) : 1.f;
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const uint32_t tbase = tmem_base + acc * Cfg::ACC_STRIDE + lane_off;
        for (int c0 = c_begin; c0 < c_end; c0 += 32)
          epilogue_chunk<BN, kTF32, kEpi>(ep, tbase, c0, row0, nb, stg, lane, rs);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// Split-K variant for bf16 GEMMs whose output tiles cannot fill the SMs (few
// rows: decode steps, the default 8/5 window rule's tens of recomputed rows).
// Such GEMMs stream the weights once and are HBM-bound, but tiles << SMs
// leave most of the machine idle. Work unit u = (tile u / S, K-slice u % S),
// one unit per CTA (grid <= SMs, so every CTA is resident). Slices 0..S-2
// write their raw fp32 accumulator to a per-stream workspace and bump the
// tile's counter (release); slice S-1, the owner, waits for the count
// (acquire), adds the partials in slice order and runs the normal fused
// epilogue, then re-arms the counter. Owners are at most tiles < SMs / 2, so
// the slices they wait for always find an SM.
// ---------------------------------------------------------------------------
template <int BN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_splitk_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       EpiParams ep, int num_m, int num_kb, int S, float* __restrict__ parts,
                       int* __restrict__ counters) {
  using Cfg = GemmCfg<BN, false>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + Cfg::STAGES * Cfg::A_BYTES;
  uint8_t* smem_epi = smem + Cfg::STAGES * Cfg::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_epi + kEpiWarps * kEpiStageBytes);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x / S, ks = blockIdx.x % S;
  const int mb = tile % num_m, nb = tile / num_m;
  const int per = (num_kb + S - 1) / S;
  const int kb0 = min(num_kb, ks * per), kb1 = min(num_kb, kb0 + per);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int st = 0; st < Cfg::STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // the prologue above touched no global memory
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
        uint8_t* sa = smem_a + stage * Cfg::A_BYTES;
        uint8_t* sb = smem_b + stage * Cfg::B_BYTES;
        tma_load_2d(sa, &tmA, &full[stage], kb * Cfg::BK, mb * kBM);
        tma_load_2d(sb, &tmB, &full[stage], kb * Cfg::BK, b_row<BN>(ep, nb, 0));
        tma_load_2d(sb + Cfg::B_SUB / 2, &tmB, &full[stage], kb * Cfg::BK, b_row<BN>(ep, nb, 1));
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {  // warp-wide issue from uniform descriptors (tc_mma_warp)
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint64_t adesc0 = umma_desc_sw128(smem_u32(smem_a));
    const uint64_t bdesc0 = umma_desc_sw128(smem_u32(smem_b));
    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      const uint64_t ad = adesc0 + (uint64_t)((stage * Cfg::A_BYTES) >> 4);
      const uint64_t bd = bdesc0 + (uint64_t)((stage * Cfg::B_BYTES) >> 4);
#pragma unroll
      for (int k = 0; k < Cfg::KSTEPS; ++k)
        tc_mma_warp<false>(tmem_u, ad + 2 * k, bd + 2 * k, Cfg::IDESC, (kb > kb0 || k > 0) ? 1u : 0u);
      tc_commit_warp(&empty[stage]);
      if (kb == kb1 - 1) tc_commit_warp(tfull);
      if (++stage == Cfg::STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else {
    const int ew = warp - 2, quarter = warp & 3, chalf = ew >> 2;
    const int lrow = quarter * 32 + lane;
    float* stg = reinterpret_cast<float*>(smem_epi + ew * kEpiStageBytes);
    const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16);
    const int64_t row0 = (int64_t)mb * kBM + quarter * 32;
    const bool rows_live = row0 < ep.M;  // warp-uniform: this lane quarter holds output rows
    float* tile_parts = parts + (size_t)tile * (S - 1) * kBM * BN;
    mbar_wait(tfull, 0);
    tc_fence_after();
    if (ks < S - 1) {
      // a K-slice: raw accumulator columns [chalf * BN/2, +BN/2) of this lane's row
      if (rows_live) {
        float* dst = tile_parts + ((size_t)ks * kBM + lrow) * BN;
        for (int c = chalf * (BN / 2); c < (chalf + 1) * (BN / 2); c += 16) {
          float v[16];
          tmem_ld16(tbase + c, v);
          if (row0 + lane < ep.M) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              __stcg(reinterpret_cast<float4*>(dst + c) + i,
                     make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
          }
        }
      }
      __threadfence();
      asm volatile("bar.sync 2, %0;" ::"n"(32 * kEpiWarps) : "memory");
      if (ew == 0 && lane == 0)
        asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(counters + tile) : "memory");
    } else {
      // the owner: wait for the S-1 slices, add them in order, fused epilogue
      if (ew == 0 && lane == 0) {
        int seen = 0;
        while (true) {
          asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(counters + tile) : "memory");
          if (seen >= S - 1) break;
          __nanosleep(64);
        }
      }
      asm volatile("bar.sync 2, %0;" ::"n"(32 * kEpiWarps) : "memory");
      if (rows_live) {
        const bool glu = ep.epilogue == CC_EPI_GLU;
        const int cols = glu ? BN / 2 : BN;
        const int c_begin = chalf * (cols / 2), c_end = c_begin + cols / 2;
        const SplitParts sp{tile_parts, S - 1, lrow};
        const float rs = row_scaled(ep) ? row_inv_rms(ep, row0 + lane) : 1.f;
        for (int c0 = c_begin; c0 < c_end; c0 += 32)
          epilogue_chunk<BN, false>(ep, tbase, c0, row0, nb, stg, lane, rs, sp);
      }
      asm volatile("bar.sync 2, %0;" ::"n"(32 * kEpiWarps) : "memory");
      if (ew == 0 && lane == 0) counters[tile] = 0;  // re-armed for the next launch on this stream
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, BN);
  }
}

// ---------------------------------------------------------------------------
// CTA-pair (cta_group::2) variant for large bf16 GEMMs: a cluster of two CTAs
// on one TPC owns a 256 x BN tile. Each CTA TMA-loads its own 128 rows of A
// and one BN/2-row half of B; the leader issues M=256 tcgen05.mma for the
// pair, which reads both CTAs' shared memory, so each SM moves half the B
// bytes (64 instead of 96 bytes of operand per clock at full rate). Each
// CTA's TMEM holds the accumulator of its own 128 rows; both CTAs run the
// same epilogue on their rows.
//   barriers: full[s] (leader; expects both CTAs' bytes), empty[s] and
//   tfull[a] (both CTAs; multicast tcgen05.commit from the leader),
//   tempty[a] (leader; both CTAs' epilogue warps arrive, the peer remotely)
// ---------------------------------------------------------------------------
template <int BN, bool kTF32>
struct Gemm2Cfg {
  static constexpr int ELEM = kTF32 ? 4 : 2;
  static constexpr int BK = 128 / ELEM;            // one 128-byte swizzle row per tile row
  static constexpr int UK = kTF32 ? 8 : 16;
  static constexpr int KSTEPS = BK / UK;
  static constexpr int NSUB = kTF32 ? 2 : 1;       // 3xTF32: hi and lo sub-tiles per stage
  static constexpr int A_SUB = 128 * 128;          // own 128 rows x one 128-byte K row
  static constexpr int B_SUB = (BN / 2) * 128;     // own half of B
  static constexpr int A_BYTES = NSUB * A_SUB;
  static constexpr int B_BYTES = NSUB * B_SUB;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int FIXED = kEpiWarps * kEpiStageBytes + 1024 + 256;
  static constexpr int FIT = (232448 - FIXED) / STAGE_BYTES;
  static constexpr int STAGES = FIT > 6 ? 6 : FIT;
  static constexpr int ACC_STRIDE = kTF32 ? 2 * BN : BN;  // 3xTF32: hi*hi | corrections
  static constexpr int TMEM_COLS = 2 * ACC_STRIDE;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + FIXED;
  static constexpr uint32_t IDESC = umma_idesc(256, BN, kTF32);
  static_assert(TMEM_COLS <= 512 && SMEM_BYTES <= 232448 && STAGES >= 2, "pair GEMM resources");
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_to_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const void* desc, uint32_t leader_bar, int32_t x,
                                                 int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(desc), "r"(leader_bar), "r"(x), "r"(y)
      : "memory");
}
template <bool kTF32>
__device__ __forceinline__ void tc_mma_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
  }
}
// warp-wide forms (see tc_mma_warp): the whole warp calls with uniform operands
template <bool kTF32>
__device__ __forceinline__ void tc_mma_pair_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
  }
}
__device__ __forceinline__ void tc_commit_pair_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {  // arrive on `bar` in both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

template <int BN, bool kTF32, int kEpi = -1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, EpiParams ep,
                 int num_m2, int num_n, int num_kb, int k_orig, int kb_per_phase, int group_m) {
  using Cfg = Gemm2Cfg<BN, kTF32>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + Cfg::STAGES * Cfg::A_BYTES;
  uint8_t* smem_epi = smem + Cfg::STAGES * Cfg::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_epi + kEpiWarps * kEpiStageBytes);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  const int tiles = num_m2 * num_n;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int st = 0; st < Cfg::STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(Cfg::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  __syncthreads();  // also a CTA barrier for tools that do not model barrier.cluster (racecheck)
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // the prologue above touched no global memory
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {  // both CTAs: own A rows and own B half, completion counted on the leader's barrier
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster_id; t < tiles; t += n_clusters) {
        int mb, nb;
        tile_mn(t, num_m2, num_n, group_m, mb, nb);
        const int arow = mb * 256 + (int)rank * 128;
        const int brow = b_row<BN, kEpi>(ep, nb, (int)rank);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * Cfg::STAGE_BYTES);
          const uint32_t lbar = map_to_rank(&full[stage], 0);
          uint8_t* sa = smem_a + stage * Cfg::A_BYTES;
          uint8_t* sb = smem_b + stage * Cfg::B_BYTES;
          tma_load_2d_pair(sa, &tmA, lbar, kb * Cfg::BK, arow);
          tma_load_2d_pair(sb, &tmB, lbar, kb * Cfg::BK, brow);
          if constexpr (kTF32) {  // A' = [hi | hi | lo], B' = [hi | lo | hi]
            tma_load_2d_pair(sa + Cfg::A_SUB, &tmA, lbar, 2 * k_orig + kb * Cfg::BK, arow);
            tma_load_2d_pair(sb + Cfg::B_SUB, &tmB, lbar, k_orig + kb * Cfg::BK, brow);
          }
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // the pair's MMA issuer: the whole warp, one elected lane per tcgen05 op
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem_base, 0);
      const uint64_t adesc0 = umma_desc_sw128(smem_u32(smem_a));
      const uint64_t bdesc0 = umma_desc_sw128(smem_u32(smem_b));
      // 3xTF32: the accumulator buffer rotates every kb_per_phase K-blocks, as
      // in gemm_kernel (the epilogue folds each phase into fp32 registers);
      // bf16: one phase per tile
      const int per_phase = kTF32 ? kb_per_phase : num_kb;
      for (int t = cluster_id; t < tiles; t += n_clusters) {
        uint32_t d_tmem = 0;
        for (int kb = 0; kb < num_kb; ++kb) {
          const int kp = kb % per_phase;
          if (kp == 0) {
            mbar_wait(&tempty[acc], acc_phase ^ 1);
            tc_fence_after();
            d_tmem = tmem_u + acc * Cfg::ACC_STRIDE;
          }
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = adesc0 + (uint64_t)((stage * Cfg::A_BYTES) >> 4);
          const uint64_t bd = bdesc0 + (uint64_t)((stage * Cfg::B_BYTES) >> 4);
#pragma unroll
          for (int k = 0; k < Cfg::KSTEPS; ++k) {
            tc_mma_pair_warp<kTF32>(d_tmem, ad + 2 * k, bd + 2 * k, Cfg::IDESC, (kp | k) != 0 ? 1u : 0u);
            if constexpr (kTF32) {  // corrections hi*lo + lo*hi into the second accumulator (each CTA holds
                                    // half of B_hi and of B_lo, so hi*[hi;lo] cannot be one N=2*BN MMA here)
              tc_mma_pair_warp<kTF32>(d_tmem + BN, ad + 2 * k, bd + (Cfg::B_SUB >> 4) + 2 * k, Cfg::IDESC,
                                      (kp | k) != 0 ? 1u : 0u);
              tc_mma_pair_warp<kTF32>(d_tmem + BN, ad + (Cfg::A_SUB >> 4) + 2 * k, bd + 2 * k, Cfg::IDESC, 1u);
            }
          }
          tc_commit_pair_warp(&empty[stage]);
          const bool phase_end = kp == per_phase - 1 || kb == num_kb - 1;
          if (phase_end) tc_commit_pair_warp(&tfull[acc]);
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
          if (phase_end && ++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
      }
    }
  } else {
    const int ew = warp - 2;
    const int quarter = warp & 3;
    const int chalf = ew >> 2;
    float* stg = reinterpret_cast<float*>(smem_epi + ew * kEpiStageBytes);
    int acc = 0;
    uint32_t acc_phase = 0;
    const int cols = (epi_of(ep, kEpi) == CC_EPI_GLU) ? BN / 2 : BN;
    const int c_begin = chalf * (cols / 2), c_end = c_begin + cols / 2;
    for (int t = cluster_id; t < tiles; t += n_clusters) {
      int mb, nb;
      tile_mn(t, num_m2, num_n, group_m, mb, nb);
      const int64_t row0 = (int64_t)mb * 256 + (int64_t)rank * 128 + quarter * 32;
      if constexpr (kTF32) {
        // phases folded in registers exactly as gemm_kernel does (bitwise the
        // same sums), then the same register epilogue
        const bool glu = epi_of(ep, kEpi) == CC_EPI_GLU;
        constexpr int NV = BN / 2;
        float run[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) run[j] = 0.f;
        const int n_phases = (num_kb + kb_per_phase - 1) / kb_per_phase;
        for (int ph = 0; ph < n_phases; ++ph) {
          mbar_wait(&tfull[acc], acc_phase);
          tc_fence_after();
          const uint32_t tb = tmem_base + acc * Cfg::ACC_STRIDE + ((uint32_t)(quarter * 32) << 16);
#pragma unroll
          for (int j = 0; j < NV; j += 16) {
            const int col = (glu && j >= NV / 2) ? c_begin + BN / 2 + (j - NV / 2) : c_begin + j;
            float m16[16], c16[16];
            tmem_ld16(tb + col, m16);
            tmem_ld16(tb + BN + col, c16);
#pragma unroll
            for (int i = 0; i < 16; ++i) run[j + i] = __fadd_rn(run[j + i], __fadd_rn(m16[i], c16[i]));
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(map_to_rank(&tempty[acc], 0));
          if (++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
        if (glu) {
#pragma unroll
          for (int cc = 0; cc < NV / 2; cc += 32) {
            glu16<BN, kEpi>(ep, nb, c_begin + cc, run + cc, run + NV / 2 + cc);
            glu16<BN, kEpi>(ep, nb, c_begin + cc + 16, run + cc + 16, run + NV / 2 + cc + 16);
            epilogue_tail<BN, kEpi>(ep, run + cc, c_begin + cc, row0, nb, stg, lane);
          }
        } else {
#pragma unroll
          for (int cc = 0; cc < NV; cc += 32) epilogue_tail<BN, kEpi>(ep, run + cc, c_begin + cc, row0, nb, stg, lane);
        }
        continue;
      }
      // 1/rms of this lane's row, formed while the tile's MMAs run
      const float rs = row_scaled(ep) ? row_inv_rms(ep, row0 + lane) : 1.f;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * Cfg::ACC_STRIDE + ((uint32_t)(quarter * 32) << 16);
      for (int c0 = c_begin; c0 < c_end; c0 += 32)
        epilogue_chunk<BN, kTF32, kEpi>(ep, tbase, c0, row0, nb, stg, lane, rs);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(map_to_rank(&tempty[acc], 0));
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();  // no CTA leaves while its peer may still arrive on / read from it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(Cfg::TMEM_COLS)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static int make_map(CUtensorMap* map, const void* ptr, bool f32, int64_t inner, int64_t rows, int64_t ld,
                    int box_inner, int box_rows) {
  auto enc = get_encode();
  if (!enc) return fail(CC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int esz = f32 ? 4 : 2;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * esz)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return CC_OK;
}

template <int BN, bool kTF32, int kEpi = -1>
static int launch(const cc_gemm_args* a, const EpiParams& ep, int64_t kop, cudaStream_t st) {
  using Cfg = GemmCfg<BN, kTF32>;
  CUtensorMap ta, tb;
  int rc = make_map(&ta, a->A, kTF32, kop, a->M, a->lda, Cfg::BK, kBM);
  if (rc) return rc;
  rc = make_map(&tb, a->B, kTF32, kop, a->N, a->ldb, Cfg::BK, BN / 2);
  if (rc) return rc;
  set_smem_once<gemm_kernel<BN, kTF32, kEpi>>(Cfg::SMEM_BYTES);
  const int num_m = (int)((a->M + kBM - 1) / kBM);
  const int num_n = (int)((a->N + BN - 1) / BN);
  // 3xTF32 iterates the original K (hi/lo sub-tiles per stage)
  const int num_kb = (int)(((kTF32 ? a->K : kop) + Cfg::BK - 1) / Cfg::BK);
  const int tiles = num_m * num_n;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  ProfScope ps(st, kTF32 ? OP_GEMM_TF32X3 : OP_GEMM_BF16, 2.0 * (double)a->M * (double)a->N * (double)a->K);
  // 3xTF32 operands are split planes: 3 x 4 bytes per element in A's and B's panels
  const int group_m = schedule_band(a, kTF32 ? 12.0 : 2.0, 16);
  const cudaError_t e = launch_pdl(gemm_kernel<BN, kTF32, kEpi>, dim3(grid), dim3(kGemmThreads), Cfg::SMEM_BYTES, st,
                                   ta, tb, ep, num_m, num_n, num_kb, (int)a->K,
                                   kTF32 ? kTf32KbPerPhase : num_kb, group_m);
  if (e != cudaSuccess) return fail(CC_ERR_CUDA, "gemm launch failed: %s", cudaGetErrorString(e));
  return CC_OK;
}

template <int BN, bool kTF32, int kEpi = -1>
static int launch_pair(const cc_gemm_args* a, const EpiParams& ep, int64_t kop, cudaStream_t st) {
  using Cfg = Gemm2Cfg<BN, kTF32>;
  CUtensorMap ta, tb;
  int rc = make_map(&ta, a->A, kTF32, kop, a->M, a->lda, Cfg::BK, 128);
  if (rc) return rc;
  rc = make_map(&tb, a->B, kTF32, kop, a->N, a->ldb, Cfg::BK, BN / 2);
  if (rc) return rc;
  set_smem_once<gemm2_kernel<BN, kTF32, kEpi>>(Cfg::SMEM_BYTES);
  const int num_m2 = (int)((a->M + 255) / 256);
  const int num_n = (int)((a->N + BN - 1) / BN);
  // 3xTF32 iterates the original K (hi/lo sub-tiles per stage)
  const int num_kb = (int)(((kTF32 ? a->K : kop) + Cfg::BK - 1) / Cfg::BK);
  const int tiles = num_m2 * num_n;
  const int clusters = tiles < num_sms() / 2 ? tiles : num_sms() / 2;
  const int group_m = schedule_band(a, kTF32 ? 12.0 : 2.0, 8);  // bands of 8 m-pairs
  ProfScope ps(st, kTF32 ? OP_GEMM_TF32X3 : OP_GEMM_BF16, 2.0 * (double)a->M * (double)a->N * (double)a->K);
  const cudaError_t e = launch_pdl(gemm2_kernel<BN, kTF32, kEpi>, dim3(2 * clusters), dim3(kGemmThreads),
                                   Cfg::SMEM_BYTES, st, ta, tb, ep, num_m2, num_n, num_kb, (int)a->K,
                                   kTF32 ? kTf32KbPerPhase : num_kb, group_m);
  if (e != cudaSuccess) return fail(CC_ERR_CUDA, "gemm (CTA pair) launch failed: %s", cudaGetErrorString(e));
  return CC_OK;
}

// Split-K workspace per (device, stream): fp32 partials for every unit of a
// grid of <= num_sms units, and one counter per tile (zeroed once; each owner
// re-arms its counter). Per stream, so concurrent streams never share one.
struct SplitKWs {
  float* parts = nullptr;
  int* counters = nullptr;
};
constexpr int kSplitKMaxTiles = 1024;
static int splitk_ws(cudaStream_t st, SplitKWs* out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, SplitKWs> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({dev, st});
  if (it == cache.end()) {
    SplitKWs w;
    if (cudaMalloc(&w.parts, (size_t)num_sms() * kBM * 256 * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&w.counters, kSplitKMaxTiles * sizeof(int)) != cudaSuccess ||
        cudaMemset(w.counters, 0, kSplitKMaxTiles * sizeof(int)) != cudaSuccess)
      return fail(CC_ERR_CUDA, "split-K workspace allocation failed");
    it = cache.emplace(std::make_pair(dev, st), w).first;
  }
  *out = it->second;
  return CC_OK;
}

// ---------------------------------------------------------------------------
// Weight-streaming GEMV for bf16 GEMMs of M <= 4 rows (a decode step, the
// query row of a tiny request). A tcgen05 tile of 128 rows would hold one
// live row; the launch is bound by how fast the weights stream from HBM, so
// the CUDA cores do the dot products and every load is a contiguous 16-byte
// segment of a K-major weight row. One CTA per 32-column output chunk (64
// weight rows for GLU: 32 gate + 32 up), 8 warps x 4 weight rows each (16
// x 4 for GLU: every warp takes 4 rows of the chunk per pass), lanes striding
// K with four 16-byte loads per row in flight; each warp butterfly-reduces
// its (row, weight row) sums into smem; warp 0 then holds the chunk as the
// tensor-core kernels' epilogue expects it (lane = row, 32 columns) and runs
// the same fused epilogue code (bias, RoPE + K/V scatter, residual + RMSNorm
// partials, GLU, 1/rms scaling).
// ---------------------------------------------------------------------------
constexpr int kGemvMaxRows = 4;
constexpr int kGemvWarps = 8;
constexpr int kGemvRowsPerWarp = 4;  // weight rows a warp reduces per pass
constexpr int kGemvUnroll = 4;       // 16-byte K segments per weight row in flight per lane
#ifndef CC_GEMV_PREFETCH
#define CC_GEMV_PREFETCH 4096
#endif
constexpr int64_t kGemvPrefetchBytes = CC_GEMV_PREFETCH;  // L2 prefetch per weight row (bounded: L2 holds it)

template <int MR, int kEpi>
__global__ void __launch_bounds__(32 * kGemvWarps) gemv_kernel(const __nv_bfloat16* __restrict__ A, int64_t lda,
                                                               const __nv_bfloat16* __restrict__ B, int64_t ldb,
                                                               int K, EpiParams ep) {
  constexpr bool kGlu = kEpi == CC_EPI_GLU;
  constexpr int kRows = kGlu ? 64 : 32;  // weight rows of the chunk
  __shared__ float res[MR][kRows];
  __shared__ __align__(16) float stg[32 * 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x;  // output chunk of 32 columns
  int nb, c0;
  int64_t wrow0, wrow1;  // first weight row of the chunk's (gate,) up half
  if constexpr (kGlu) {
    nb = q >> 1;
    c0 = (q & 1) * 32;
    wrow0 = b_row<128, kEpi>(ep, nb, 0) + c0;
    wrow1 = b_row<128, kEpi>(ep, nb, 1) + c0;
  } else {
    nb = q >> 2;
    c0 = (q & 3) * 32;
    wrow0 = (int64_t)q * 32;
    wrow1 = 0;
  }
  // The weights are constant (no predecessor writes them): one thread per
  // weight row starts an L2 bulk prefetch of its head before the dependency
  // wait, so the stream from HBM overlaps the previous kernel's tail and the
  // K loop below mostly hits L2.
  if (kGemvPrefetchBytes > 0 && threadIdx.x < kRows) {
    const int j = threadIdx.x;
    const int64_t row = (kGlu && j >= 32) ? wrow1 + (j - 32) : wrow0 + j;
    const int64_t row_bytes = (int64_t)K * 2;
    const uint32_t bytes = (uint32_t)(row_bytes < kGemvPrefetchBytes ? row_bytes : kGemvPrefetchBytes);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(B + row * ldb), "r"(bytes) : "memory");
  }
  pdl_wait();
  pdl_trigger();
  const int k8 = K >> 3;
  for (int j0 = warp * kGemvRowsPerWarp; j0 < kRows; j0 += kGemvWarps * kGemvRowsPerWarp) {
    const uint4* w[kGemvRowsPerWarp];
#pragma unroll
    for (int r = 0; r < kGemvRowsPerWarp; ++r) {
      const int j = j0 + r;
      const int64_t row = (kGlu && j >= 32) ? wrow1 + (j - 32) : wrow0 + j;
      w[r] = reinterpret_cast<const uint4*>(B + row * ldb);
    }
    float acc[kGemvRowsPerWarp][MR];
#pragma unroll
    for (int r = 0; r < kGemvRowsPerWarp; ++r)
#pragma unroll
      for (int m = 0; m < MR; ++m) acc[r][m] = 0.f;
    for (int base = lane; base < k8; base += 32 * kGemvUnroll) {
      uint4 wv[kGemvUnroll][kGemvRowsPerWarp];
      uint4 av[kGemvUnroll][MR];
#pragma unroll
      for (int u = 0; u < kGemvUnroll; ++u) {
        const int c = base + 32 * u;
        const bool ok = c < k8;
#pragma unroll
        for (int r = 0; r < kGemvRowsPerWarp; ++r) wv[u][r] = ok ? __ldcs(w[r] + c) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int m = 0; m < MR; ++m)
          av[u][m] = ok && m < ep.M ? __ldg(reinterpret_cast<const uint4*>(A + m * lda) + c) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < kGemvUnroll; ++u) {
        float af[MR][8];
#pragma unroll
        for (int m = 0; m < MR; ++m) {
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&av[u][m]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(h[e]);
            af[m][2 * e] = f.x;
            af[m][2 * e + 1] = f.y;
          }
        }
#pragma unroll
        for (int r = 0; r < kGemvRowsPerWarp; ++r) {
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&wv[u][r]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(h[e]);
#pragma unroll
            for (int m = 0; m < MR; ++m)
              acc[r][m] = fmaf(f.y, af[m][2 * e + 1], fmaf(f.x, af[m][2 * e], acc[r][m]));
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kGemvRowsPerWarp; ++r)
#pragma unroll
      for (int m = 0; m < MR; ++m) {
        float x = acc[r][m];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) res[m][j0 + r] = x;
      }
  }
  __syncthreads();
  if (warp != 0) return;
  // lane = output row (rows >= M carry zeros and are never stored)
  const int m = lane < MR ? lane : 0;
  const bool live = lane < MR && lane < ep.M;
  const float rs = row_scaled(ep) ? row_inv_rms(ep, lane) : 1.f;
  float v[32];
  if constexpr (kGlu) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      float u[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        v[16 * hh + j] = live ? res[m][16 * hh + j] : 0.f;
        u[j] = live ? res[m][32 + 16 * hh + j] : 0.f;
        if (row_scaled(ep)) {
          v[16 * hh + j] = __fmul_rn(v[16 * hh + j], rs);
          u[j] = __fmul_rn(u[j], rs);
        }
      }
      glu16<128, kEpi>(ep, nb, c0 + 16 * hh, v + 16 * hh, u);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      v[j] = live ? res[m][j] : 0.f;
      if (row_scaled(ep)) v[j] = __fmul_rn(v[j], rs);
    }
  }
  epilogue_tail<128, kEpi>(ep, v, c0, 0, nb, stg, lane);
}

// CC_GEMM_GEMV=0 in the environment keeps few-row GEMMs on the tensor-core kernels (A/B runs)
static bool gemv_enabled() {
  static const bool on = [] {
    const char* e = getenv("CC_GEMM_GEMV");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int MR>
static int launch_gemv_rows(const cc_gemm_args* a, const EpiParams& ep, cudaStream_t st) {
  const bool glu = a->epilogue == CC_EPI_GLU;
  const int chunks = (int)(glu ? a->N / 64 : a->N / 32);
  const auto* A = static_cast<const __nv_bfloat16*>(a->A);
  const auto* B = static_cast<const __nv_bfloat16*>(a->B);
  const int K = (int)a->K;
  cudaError_t e;
  switch (a->epilogue) {
    case CC_EPI_GLU:
      e = launch_pdl(gemv_kernel<MR, CC_EPI_GLU>, dim3(chunks), dim3(32 * kGemvWarps), 0, st, A, a->lda, B, a->ldb, K, ep);
      break;
    case CC_EPI_RESIDUAL:
      e = launch_pdl(gemv_kernel<MR, CC_EPI_RESIDUAL>, dim3(chunks), dim3(32 * kGemvWarps), 0, st, A, a->lda, B, a->ldb,
                     K, ep);
      break;
    case CC_EPI_QKV_ROPE:
      e = launch_pdl(gemv_kernel<MR, CC_EPI_QKV_ROPE>, dim3(chunks), dim3(32 * kGemvWarps), 0, st, A, a->lda, B, a->ldb,
                     K, ep);
      break;
    default:
      e = launch_pdl(gemv_kernel<MR, -1>, dim3(chunks), dim3(32 * kGemvWarps), 0, st, A, a->lda, B, a->ldb, K, ep);
      break;
  }
  if (e != cudaSuccess) return fail(CC_ERR_CUDA, "gemv launch failed: %s", cudaGetErrorString(e));
  return CC_OK;
}

static int launch_gemv(const cc_gemm_args* a, const EpiParams& ep, cudaStream_t st) {
  ProfScope ps(st, OP_GEMM_BF16, 2.0 * (double)a->M * (double)a->N * (double)a->K);
  if (a->M == 1) return launch_gemv_rows<1>(a, ep, st);
  if (a->M == 2) return launch_gemv_rows<2>(a, ep, st);
  return launch_gemv_rows<4>(a, ep, st);
}

// K-slices for a bf16 GEMM of `tiles` output tiles over num_kb K-blocks: > 1
// only when the tiles fill under half the SMs and each slice keeps >= 8
// K-blocks (CC_GEMM_SPLITK=0 in the environment: never, for A/B runs)
static int splitk_count(int64_t tiles, int num_kb) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("CC_GEMM_SPLITK");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  if (!on || tiles <= 0 || 2 * tiles > num_sms() || tiles > kSplitKMaxTiles) return 1;
  int s = (int)std::min<int64_t>(num_sms() / tiles, num_kb / 8);
  s = std::min(s, 16);
  return s >= 2 ? s : 1;
}

template <int BN>
static int launch_splitk(const cc_gemm_args* a, const EpiParams& ep, int64_t kop, int S, cudaStream_t st) {
  using Cfg = GemmCfg<BN, false>;
  CUtensorMap ta, tb;
  int rc = make_map(&ta, a->A, false, kop, a->M, a->lda, Cfg::BK, kBM);
  if (rc) return rc;
  rc = make_map(&tb, a->B, false, kop, a->N, a->ldb, Cfg::BK, BN / 2);
  if (rc) return rc;
  SplitKWs ws;
  rc = splitk_ws(st, &ws);
  if (rc) return rc;
  set_smem_once<gemm_splitk_kernel<BN>>(Cfg::SMEM_BYTES);
  const int num_m = (int)((a->M + kBM - 1) / kBM);
  const int num_n = (int)((a->N + BN - 1) / BN);
  const int num_kb = (int)((kop + Cfg::BK - 1) / Cfg::BK);
  ProfScope ps(st, OP_GEMM_BF16, 2.0 * (double)a->M * (double)a->N * (double)a->K);
  const cudaError_t e = launch_pdl(gemm_splitk_kernel<BN>, dim3(num_m * num_n * S), dim3(kGemmThreads),
                                   Cfg::SMEM_BYTES, st, ta, tb, ep, num_m, num_kb, S, ws.parts, ws.counters);
  if (e != cudaSuccess) return fail(CC_ERR_CUDA, "gemm (split-K) launch failed: %s", cudaGetErrorString(e));
  return CC_OK;
}

// CC_GEMM_PAIR=0 in the environment keeps every bf16 GEMM on single-CTA tiles (A/B runs)
static bool pair_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("CC_GEMM_PAIR");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// CC_TF32_PAIR=0 keeps every 3xTF32 GEMM on single-CTA tiles (A/B runs)
static bool tf32_pair_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("CC_TF32_PAIR");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

}  // namespace cc

using namespace cc;

#ifdef CC_GEMM_TRACE
extern "C" int cc_debug_gemm_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, g_gemm_trace, sizeof(long long) * 5 * 4096) == cudaSuccess ? 0 : 1;
}
#endif

extern "C" int cc_gemm(const cc_gemm_args* a, void* stream) {
  CC_CHECK_ARG(a, CC_ERR_VALUE, "null gemm args");
  CC_CHECK_ARG(a->M >= 0 && a->N > 0 && a->K > 0, CC_ERR_DIMENSION, "bad GEMM shape M=%lld N=%lld K=%lld",
               (long long)a->M, (long long)a->N, (long long)a->K);
  if (a->M == 0) return CC_OK;
  const bool tf32 = a->kind == CC_GEMM_TF32X3;
  CC_CHECK_ARG(tf32 || a->kind == CC_GEMM_BF16, CC_ERR_UNSUPPORTED, "gemm kind %d", a->kind);
  CC_CHECK_ARG(!tf32 || a->K % 32 == 0, CC_ERR_UNSUPPORTED, "3xTF32 GEMM needs K %% 32 == 0 (K=%lld)",
               (long long)a->K);
  const int64_t kop = tf32 ? 3 * a->K : a->K;
  const int esz = tf32 ? 4 : 2;
  CC_CHECK_ARG(a->lda >= kop && a->ldb >= kop, CC_ERR_DIMENSION, "leading dimension smaller than K");
  CC_CHECK_ARG((a->lda * esz) % 16 == 0 && (a->ldb * esz) % 16 == 0, CC_ERR_UNSUPPORTED,
               "operand rows must be 16-byte aligned");
  CC_CHECK_ARG(((uintptr_t)a->A % 16) == 0 && ((uintptr_t)a->B % 16) == 0, CC_ERR_UNSUPPORTED,
               "operands must be 16-byte aligned");
  CC_CHECK_ARG(a->N % 16 == 0, CC_ERR_UNSUPPORTED, "N=%lld must be a multiple of 16", (long long)a->N);
  // the epilogue writes 4-column vectors (16 B fp32 / 8 B bf16)
  CC_CHECK_ARG(a->ldc % 4 == 0 && a->ldq % 4 == 0 && a->n_out % 4 == 0 && ((uintptr_t)a->C % 16) == 0 &&
                   ((uintptr_t)a->q_out % 16) == 0,
               CC_ERR_UNSUPPORTED, "GEMM outputs must be 16-byte aligned with row pitches a multiple of 4");
  EpiParams ep{};
  ep.epilogue = a->epilogue;
  ep.M = a->M;
  ep.N = a->N;
  ep.bias = a->bias;
  ep.C = a->C;
  ep.ldc = a->ldc;
  ep.c_mode = a->c_mode;
  ep.act = a->act;
  ep.glu_block = a->glu_block;
  ep.n_out = a->n_out;
  ep.n_q_heads = a->n_q_heads;
  ep.n_kv_heads = a->n_kv_heads;
  ep.head_dim = a->head_dim;
  ep.rope_cos = a->rope_cos;
  ep.rope_sin = a->rope_sin;
  ep.q_out = a->q_out;
  ep.ldq = a->ldq;
  ep.q_mode = a->q_mode;
  ep.k_cache = a->k_cache;
  ep.v_cache = a->v_cache;
  ep.cache_dtype = a->cache_dtype;
  ep.dst_rows = a->dst_rows;
  ep.k_raw = a->k_raw;
  ep.raw_rows = a->raw_rows;
  ep.xn_out = a->xn_out;
  ep.ldxn = a->ldxn;
  ep.norm_gain = a->norm_gain;
  ep.ssq_out = a->ssq_out;
  ep.ssq_in = a->inv_rms;
  ep.ld_ssq = a->ld_ssq;
  ep.ssq_parts = a->inv_rms ? nullptr : a->ssq_in;
  ep.n_parts = a->n_ssq;
  ep.ld_parts = a->ld_ssq_in;
  ep.eps = a->norm_eps;
  ep.inv_d = a->n_ssq > 0 ? 1.0f / (float)(32 * a->n_ssq) : 0.f;
  if (a->ssq_out || a->inv_rms || a->ssq_in) CC_CHECK_ARG(!tf32, CC_ERR_UNSUPPORTED, "fused RMSNorm runs on bf16 GEMMs");
  if (a->ssq_in && !a->inv_rms)
    CC_CHECK_ARG(a->n_ssq > 0 && a->ld_ssq_in >= a->M, CC_ERR_DIMENSION, "ssq_in needs n_ssq > 0 and ld_ssq_in >= M");
  if (a->ssq_out)
    CC_CHECK_ARG(a->ld_ssq >= a->M, CC_ERR_DIMENSION, "ld_ssq %lld < M %lld", (long long)a->ld_ssq, (long long)a->M);
  if (a->ssq_out) {
    CC_CHECK_ARG(a->epilogue == CC_EPI_RESIDUAL && a->N % 32 == 0 && a->xn_out && a->norm_gain &&
                     a->ldxn % 4 == 0 && ((uintptr_t)a->xn_out % 16) == 0 && ((uintptr_t)a->norm_gain % 16) == 0,
                 CC_ERR_UNSUPPORTED, "RMSNorm partials come from a RESIDUAL epilogue with N %% 32 == 0, xn and gain");
  }
  if (a->inv_rms || a->ssq_in)
    CC_CHECK_ARG(a->epilogue != CC_EPI_RESIDUAL, CC_ERR_UNSUPPORTED,
                 "row RMS scaling applies to QKV / GLU / STORE / ACT epilogues");
  bool wide;
  if (a->epilogue == CC_EPI_GLU) {
    CC_CHECK_ARG(a->glu_block == 128 && a->N % 256 == 0, CC_ERR_UNSUPPORTED,
                 "GLU needs gate/up interleaved in blocks of 128 (N=%lld)", (long long)a->N);
    wide = true;
  } else if (a->epilogue == CC_EPI_QKV_ROPE) {
    CC_CHECK_ARG(a->head_dim % 32 == 0 && a->rope_cos && a->rope_sin && a->k_cache && a->v_cache && a->q_out,
                 CC_ERR_UNSUPPORTED, "QKV epilogue needs head_dim %% 32 == 0 and all outputs");
    CC_CHECK_ARG(a->N == (int64_t)(a->n_q_heads + 2 * a->n_kv_heads) * a->head_dim ||
                     a->N == (int64_t)(a->n_q_heads + a->n_kv_heads) * a->head_dim,
                 CC_ERR_DIMENSION, "QKV width mismatch");
    wide = a->N >= 2048;
  } else {
    const int64_t t256 = ((a->M + 127) / 128) * ((a->N + 255) / 256);
    wide = t256 >= 2 * num_sms() || a->N % 128 != 0;
  }
  cudaStream_t st = as_stream(stream);
  // 3xTF32 runs 128-wide tiles: two accumulators (hi*hi, corrections) x two buffers fill TMEM
  if (tf32) {
    // small-M scoring GEMMs (few chunks): 64-wide tiles double the CTAs when
    // 128-wide tiles would leave over half the SMs idle (GLU tiles need >= 128)
    const int64_t t128 = ((a->M + kBM - 1) / kBM) * ((a->N + 127) / 128);
    const bool narrow = a->epilogue != CC_EPI_GLU && 2 * t128 <= num_sms();
    // large M (the C3 scoring pass, M = 2048): 256-row CTA-pair tiles, each
    // CTA loading half of B (48 instead of 64 KB of operands per K-block per
    // SM; the split operands make these GEMMs operand-bandwidth bound):
    // 7.10 -> 6.5 ms per 24-layer pass on the C3 shapes (scripts/bench_gemm.py)
    if (tf32_pair_enabled() && a->M >= 1024 && a->N % 128 == 0) {
      switch (a->epilogue) {
        case CC_EPI_GLU:
          return launch_pair<128, true, CC_EPI_GLU>(a, ep, kop, st);
        case CC_EPI_RESIDUAL:
          return launch_pair<128, true, CC_EPI_RESIDUAL>(a, ep, kop, st);
        case CC_EPI_QKV_ROPE:
          return launch_pair<128, true, CC_EPI_QKV_ROPE>(a, ep, kop, st);
        default:
          return launch_pair<128, true>(a, ep, kop, st);
      }
    }
    // specialised on the epilogue (the scoring model's four), generic otherwise
    switch (a->epilogue) {
      case CC_EPI_GLU:
        return launch<128, true, CC_EPI_GLU>(a, ep, kop, st);
      case CC_EPI_RESIDUAL:
        return narrow ? launch<64, true, CC_EPI_RESIDUAL>(a, ep, kop, st)
                      : launch<128, true, CC_EPI_RESIDUAL>(a, ep, kop, st);
      case CC_EPI_QKV_ROPE:
        return narrow ? launch<64, true, CC_EPI_QKV_ROPE>(a, ep, kop, st)
                      : launch<128, true, CC_EPI_QKV_ROPE>(a, ep, kop, st);
      default:
        return narrow ? launch<64, true>(a, ep, kop, st) : launch<128, true>(a, ep, kop, st);
    }
  }
  // at most 4 rows: stream the weights through the CUDA cores (GEMV)
  if (a->M <= kGemvMaxRows && a->N % 32 == 0 && a->K % 8 == 0 && gemv_enabled())
    return launch_gemv(a, ep, st);
  // bf16 GEMMs of few tiles (few rows): 128-wide tiles cut along K
  if (a->N % 128 == 0) {
    const int64_t t128 = ((a->M + kBM - 1) / kBM) * (a->N / 128);
    const int S = splitk_count(t128, (int)((kop + 63) / 64));
    if (S > 1) return launch_splitk<128>(a, ep, kop, S, st);
  }
  // large bf16 GEMMs on CTA pairs: 256-row tiles, half the B traffic per SM
  if (pair_enabled() && a->M >= 512 && a->N % 256 == 0) {
    switch (a->epilogue) {  // specialised on the recompute layer's three epilogues
      case CC_EPI_QKV_ROPE:
        return launch_pair<256, false, CC_EPI_QKV_ROPE>(a, ep, kop, st);
      case CC_EPI_RESIDUAL:
        return launch_pair<256, false, CC_EPI_RESIDUAL>(a, ep, kop, st);
      case CC_EPI_GLU:
        return launch_pair<256, false, CC_EPI_GLU>(a, ep, kop, st);
      default:
        return launch_pair<256, false>(a, ep, kop, st);
    }
  }
  switch (a->epilogue) {  // specialised on the recompute layer's epilogues (few-row GEMMs land here)
    case CC_EPI_QKV_ROPE:
      return wide ? launch<256, false, CC_EPI_QKV_ROPE>(a, ep, kop, st)
                  : launch<128, false, CC_EPI_QKV_ROPE>(a, ep, kop, st);
    case CC_EPI_RESIDUAL:
      return wide ? launch<256, false, CC_EPI_RESIDUAL>(a, ep, kop, st)
                  : launch<128, false, CC_EPI_RESIDUAL>(a, ep, kop, st);
    case CC_EPI_GLU:
      return launch<256, false, CC_EPI_GLU>(a, ep, kop, st);
    default:
      return wide ? launch<256, false>(a, ep, kop, st) : launch<128, false>(a, ep, kop, st);
  }
}
