// Sparse-row flash attention on tcgen05 (sm_100a).
//
// causal_attention(q, bank_k, bank_v, row_limits=idx+1) of selective_forward
// (model.py:715-720) — and the mask_offset rule of layer_forward
// (model.py:467-476) for query rows and dense prefill — without materialising
// the (H, m, n) logits of tensor_core.py:166-170.
//
// One CTA = two 128-row query tiles x one KV head. GQA packing: packed row
// p = i*G + g is selected row i, query head kvh*G + g, so every K/V tile is
// fetched once for all G heads (and both query tiles) that share it. Keys
// stream in 128-key tiles up to the CTA's largest row limit (rows are sorted
// by position, so a tile spans a narrow range and little work is masked).
//
//   warp 0      TMA producer: K and V tiles ([keys][D] bf16, 128B swizzle), 2 stages
//   warp 1      tcgen05.mma issuer, ping-pong over the two query tiles:
//               PV_A(j) | S_A(j+1) | PV_B(j) | S_B(j+1) ...  S = Q K^T lands in
//               TMEM; O += P V reads P straight from TMEM (A operand) and V
//               from smem as an MN-major operand.
//   warps 2..3  idle after the prologue (warpgroup 0 gives up registers)
//   warps 4..7  softmax of tile A, warps 8..11 of tile B: thread t owns row t,
//               reads its S row with tcgen05.ld, does max / exp2 / sum in-thread,
//               writes P (bf16 pairs) back over its S row with tcgen05.st.
//               Lazy rescale: the running max moves (and O is rescaled in TMEM)
//               only when a tile raises it by > 2^8. One FFMA per element
//               folds scale and max; 4 of 16 exp2 pairs (the first of each
//               32-key chunk) run as a degree-3
//               polynomial on the FMA pipe to offload MUFU. P goes back in
//               four 32-key parts, each released to the PV MMA as soon as it
//               is in TMEM.
#include "cc_common.cuh"

#include <algorithm>
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

namespace cc {

#ifdef CC_FA_TRACE  // debug builds only: SM-clock timeline of the heaviest CTA
__device__ long long g_fa_trace[16 * 128];
#define FA_T(slot, j)                                                                        \
  do {                                                                                       \
    if (blockIdx.x == 0 && lane == 0 && (j) < 128)                                              \
      g_fa_trace[(slot) * 128 + (j)] = clock64();                                            \
  } while (0)
#else
#define FA_T(slot, j) \
  do {                \
  } while (0)
#endif

constexpr int kFaTileRows = 128;
constexpr int kFaKeys = 128;
constexpr int kFaThreads = 384;  // 3 warpgroups: producer/MMA, softmax A, softmax B
constexpr int kFaCtlRegs = 56;    // setmaxnreg budgets: 128*56 + 256*224 = 384*168 (the launch allocation)
constexpr int kFaSoftmaxRegs = 224;
constexpr float kFaRescaleThreshold = 8.0f;  // log2 domain
constexpr int kMaxAttnSplits = 32;
constexpr int kFaMinSplitTiles = 8;  // a split part covers at least this many key tiles (1024 keys)

template <int D>
struct FaCfg {
  static constexpr int KB = D / 64;                   // 128-byte K-blocks per row of Q / K
  static constexpr int QT_BYTES = kFaTileRows * D * 2;  // one query tile
  static constexpr int KT_BYTES = kFaKeys * D * 2;      // one K (or V) tile
  static constexpr int STAGES = 2;
  static constexpr int SMEM = 2 * QT_BYTES + 2 * STAGES * KT_BYTES + 1024 + 256;
  static constexpr uint32_t IDESC_S = umma_idesc(128, kFaKeys, false);
  static constexpr uint32_t IDESC_PV = umma_idesc(128, D, false) | (1u << 16);  // B (V) MN-major
  __host__ __device__ static constexpr int s_col(int t) { return t * 256; }
  __host__ __device__ static constexpr int o_col(int t) { return t * 256 + 128; }
};

// MN-major 128B-swizzled operand: 64-element rows of 128 B, MN atoms LBO
// apart, 8-row K groups SBO apart.
__device__ __forceinline__ uint64_t umma_desc_mn_sw128(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void tma_load_3d(void* dst, const void* desc, uint64_t* bar, int32_t x, int32_t y,
                                            int32_t z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(desc), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// warp-wide form (see tc_mma_warp in cc_common.cuh): the whole warp calls
// with uniform operands, one elected lane issues
__device__ __forceinline__ void tc_mma_ts_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}

// 32 columns without the trailing wait (the caller issues tcgen05.wait::ld
// once for several loads before touching the values)
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
#ifdef CC_SYNC_TMEM_LD  // sanitizer builds: no register is pending an async TMEM load across other code
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#endif
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_st16u(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint32_t pack2_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float ex2_mufu(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

#ifndef CC_FA_POLY_DEG
#define CC_FA_POLY_DEG 3
#endif

// 2^x for a pair on the FMA pipe, with the sm_100 paired-FP32 instructions
// (FADD2/FFMA2, half the issue slots): round-to-nearest split x = n + f,
// |f| <= 1/2, a polynomial for 2^f, 2^n via the exponent field.
// t = x + 1.5*2^23 holds n in its low mantissa bits and the magic's own bits
// vanish under << 23, so 2^n scaling is one IMAD.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -126.0f);
  x.y = fmaxf(x.y, -126.0f);
  const float2 magic = make_float2(12582912.0f, 12582912.0f);
  const float2 t = __fadd2_rn(x, magic);
  const float2 n = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
  const float2 f = __ffma2_rn(n, make_float2(-1.0f, -1.0f), x);
#if CC_FA_POLY_DEG == 3
  // degree-3 minimax for 2^f on [-1/2, 1/2]: |rel err| < 1.1e-4, still 20x
  // below the bf16 rounding of P
  float2 p = __ffma2_rn(f, make_float2(5.5008930e-2f, 5.5008930e-2f), make_float2(2.4221098e-1f, 2.4221098e-1f));
  p = __ffma2_rn(p, f, make_float2(6.9328293e-1f, 6.9328293e-1f));
#else
  float2 p = __ffma2_rn(f, make_float2(9.6181291e-3f, 9.6181291e-3f), make_float2(5.5504109e-2f, 5.5504109e-2f));
  p = __ffma2_rn(p, f, make_float2(2.4022651e-1f, 2.4022651e-1f));
  p = __ffma2_rn(p, f, make_float2(6.9314718e-1f, 6.9314718e-1f));
#endif
  p = __ffma2_rn(p, f, make_float2(1.0f, 1.0f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// pairs (of 16 per 32-key chunk) whose exponentials run on the FMA pipe
#ifndef CC_FA_POLY
#define CC_FA_POLY 4
#endif
constexpr int kFaPolyPairs = CC_FA_POLY;
// where in a chunk's 16 pairs the polynomial ones sit: 0 spread evenly, 1 first, 2 last
#ifndef CC_FA_POLY_POS
#define CC_FA_POLY_POS 1
#endif
__host__ __device__ constexpr bool fa_poly_pair(int e) {
  return CC_FA_POLY_POS == 1   ? e < kFaPolyPairs
         : CC_FA_POLY_POS == 2 ? e >= 16 - kFaPolyPairs
                               : (e & 15) * kFaPolyPairs % 16 >= 16 - kFaPolyPairs;
}

// P is handed to the PV MMA in this many key parts: the MMA warp starts
// O += P V on the first part while the softmax warps still exponentiate the
// rest, so part of the softmax leaves the S -> softmax -> PV -> S chain
#ifndef CC_FA_PV_PARTS
#define CC_FA_PV_PARTS 4
#endif
constexpr int kFaPvParts = CC_FA_PV_PARTS;
static_assert(kFaPvParts == 1 || kFaPvParts == 2 || kFaPvParts == 4, "P parts: 1, 2 or 4 (32-key chunks per part)");

template <int D>
__global__ void __launch_bounds__(kFaThreads, 1)
    fa_sparse_row_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                         const __nv_bfloat16* __restrict__ q, int64_t ldq, const int64_t* __restrict__ pos,
                         const int64_t* __restrict__ kstart, int64_t m,
                         int64_t n_keys, int n_q_heads, int n_kv_heads, float factor,
                         const float* __restrict__ row_factor, __nv_bfloat16* __restrict__ out, int64_t ldo,
                         int n_ctas, void* __restrict__ o_part, float* __restrict__ lse_part, int part_bf16) {
  using Cfg = FaCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sQ = smem;                                   // [2 tiles][KB][128 rows][128 B]
  uint8_t* sK = sQ + 2 * Cfg::QT_BYTES;                  // [STAGES][KB][128 keys][128 B]
  uint8_t* sV = sK + Cfg::STAGES * Cfg::KT_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + Cfg::STAGES * Cfg::KT_BYTES);
  uint64_t* k_full = bars;        // [2]
  uint64_t* v_full = bars + 2;    // [2]
  uint64_t* kv_empty = bars + 4;  // [2]
  uint64_t* s_full = bars + 6;    // [2 tiles]
  uint64_t* p_full = bars + 8;    // [2 tiles][kFaPvParts]
  uint64_t* pv_done = bars + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);
  int* s_kmax = reinterpret_cast<int*>(bars + 18);
  int* s_kmin = s_kmax + 1;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = n_q_heads / n_kv_heads;
  // heavy (late-position) tiles first ACROSS all KV heads: block b takes tile
  // n_ctas-1 - b / Hkv of head b % Hkv, so the launch order is the
  // longest-first schedule of the whole grid, not per head
  const int kvh = (int)blockIdx.x % n_kv_heads;
  const int cta = n_ctas - 1 - (int)blockIdx.x / n_kv_heads;
  const int64_t packed_total = m * G;
  const int64_t p0 = (int64_t)cta * 2 * kFaTileRows;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&kv_empty[s], 1);
      mbar_init(&s_full[s], 1);
    }
    for (int b = 0; b < 2 * kFaPvParts; ++b) mbar_init(&p_full[b], 4);
    mbar_init(pv_done, 1);
    *s_kmax = 0;
    *s_kmin = 0x7fffffff;
    fence_barrier_init();
  }
  // the key-range bounds are initialised before the prologue's atomics (found
  // by compute-sanitizer: under its serialisation the init could land after
  // some warps' atomicMax/atomicMin and reset them)
  __syncthreads();
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  pdl_wait();  // nothing above touched global memory
  pdl_trigger();

  // ---- prologue: row ranges -> the CTA's key tiles; then the Q gather ----
  const int tq = warp >= 4 ? (warp - 4) >> 2 : 0;  // query tile of this softmax warp
  const int quarter = warp & 3;                     // TMEM lane quarter
  const int r = quarter * 32 + lane;                // row within the tile
  int lim = 0, ks = 0x7fffffff;  // this row sees keys [ks, lim)
  float scale2 = 0.f;
  int64_t qrow = -1;  // selected row of this thread's packed row (-1: padding)
  int qhead = 0;
  if (warp >= 4) {
    const int64_t p = p0 + tq * kFaTileRows + r;
    if (p < packed_total) {
      const int64_t i = p / G;
      qhead = kvh * G + (int)(p % G);
      qrow = i;
      ks = kstart ? (int)kstart[i] : 0;
      lim = (int)min(ks + pos[i] + 1, n_keys);
      scale2 = (row_factor ? row_factor[i] : factor) * 1.4426950408889634f;
    }
    int mx = lim, mn = ks;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if (lane == 0) {
      atomicMax(s_kmax, mx);
      atomicMin(s_kmin, mn);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // key tiles [j0, j0 + n_tiles) cover every row's range (rows are sorted, so a
  // CTA's ranges are nearly contiguous; tiles outside a row's range are masked)
  int j0 = *s_kmax > 0 ? *s_kmin / kFaKeys : 0;
  int n_tiles = (*s_kmax + kFaKeys - 1) / kFaKeys - j0;
  if (gridDim.z > 1) {
    // split-KV: this CTA takes part blockIdx.z of its tile range. Work-aware:
    // a CTA uses at most one part per kFaMinSplitTiles tiles, so short ranges
    // (early-position rows) stay whole and only the long ones are cut; the
    // unused parts leave LSE = -inf, which the merge skips.
    const int parts = min((int)gridDim.z, max(1, n_tiles / kFaMinSplitTiles));
    const int per = (n_tiles + parts - 1) / parts;
    const int z = (int)blockIdx.z;
    const int a = z < parts ? min(n_tiles, z * per) : n_tiles;
    const int b = z < parts ? min(n_tiles, a + per) : n_tiles;
    j0 += a;
    n_tiles = b - a;
    o_part = static_cast<uint8_t*>(o_part) + (size_t)blockIdx.z * m * n_q_heads * D * (part_bf16 ? 2 : 4);
    lse_part += (int64_t)blockIdx.z * m * n_q_heads;
    if (n_tiles == 0) {  // an unused part: no keys, LSE = -inf for every row (O is never read)
      if (qrow >= 0) lse_part[qrow * n_q_heads + qhead] = -INFINITY;
      tc_fence_before();
      __syncthreads();
      if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
      }
      return;
    }
  }
  if (warp >= 4) {  // softmax warps gather their Q rows into swizzled smem
    const uint4 zero = make_uint4(0, 0, 0, 0);
    const uint4* src = qrow >= 0 ? reinterpret_cast<const uint4*>(q + qrow * ldq + (int64_t)qhead * D) : nullptr;
    uint8_t* qt = sQ + tq * Cfg::QT_BYTES;
#pragma unroll
    for (int c = 0; c < D / 8; ++c) {
      const uint4 v = src ? __ldg(src + c) : zero;
      const int kb = c >> 3, cc = c & 7;
      *reinterpret_cast<uint4*>(qt + kb * (kFaTileRows * 128) + r * 128 + ((cc ^ (r & 7)) << 4)) = v;
    }
    fence_proxy_async_smem();
  }
  // Q is in shared memory before the first S = Q K^T issue: the MMA warp and
  // the softmax warps meet on named barrier 1 (the TMA producer is already
  // streaming the first K/V tiles)
  if (warp == 1 || warp >= 4) asm volatile("bar.sync 1, %0;" ::"n"(kFaThreads - 96) : "memory");

  if (warp < 4) {
#ifndef CC_NO_SETMAXNREG  // sanitizer builds: no register reallocation under instrumentation
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kFaCtlRegs));
#endif
    if (warp == 0) {
      // ---------------- TMA producer ----------------
      if (lane == 0 && n_tiles > 0) {
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
        for (int j = 0; j < n_tiles; ++j) {
          const int s = j & 1;
          const uint32_t ph = (j >> 1) & 1;
          mbar_wait(&kv_empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&k_full[s], Cfg::KT_BYTES);
  #pragma unroll
          for (int kb = 0; kb < Cfg::KB; ++kb)
            tma_load_3d(sK + s * Cfg::KT_BYTES + kb * (kFaKeys * 128), &tmK, &k_full[s], kb * 64, kvh, (j0 + j) * kFaKeys);
          mbar_arrive_expect_tx(&v_full[s], Cfg::KT_BYTES);
  #pragma unroll
          for (int kb = 0; kb < Cfg::KB; ++kb)
            tma_load_3d(sV + s * Cfg::KT_BYTES + kb * (kFaKeys * 128), &tmV, &v_full[s], kb * 64, kvh, (j0 + j) * kFaKeys);
        }
      }
    } else if (warp == 1) {
      // ---------------- MMA issuer (ping-pong over the two query tiles) ----------------
      // the whole warp issues (one elected lane per tcgen05 op) from
      // warp-uniform descriptors formed once
      const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
      const uint64_t qdesc0 = umma_desc_sw128(smem_u32(sQ));
      const uint64_t kdesc0 = umma_desc_sw128(smem_u32(sK));
      const uint64_t vdesc0 = umma_desc_mn_sw128(smem_u32(sV), kFaKeys * 128, 1024);
      auto issue_s = [&](int t, int j) {  // S_t(j) = Q_t K_j^T
        const uint64_t qd = qdesc0 + (uint64_t)((t * Cfg::QT_BYTES) >> 4);
        const uint64_t kd = kdesc0 + (uint64_t)(((j & 1) * Cfg::KT_BYTES) >> 4);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t qo = (k >> 2) * (kFaTileRows * 128) + (k & 3) * 32;
          const uint32_t ko = (k >> 2) * (kFaKeys * 128) + (k & 3) * 32;
          tc_mma_warp<false>(tmem_u + Cfg::s_col(t), qd + (qo >> 4), kd + (ko >> 4), Cfg::IDESC_S, k > 0 ? 1u : 0u);
        }
        tc_commit_warp(&s_full[t]);
      };
      auto issue_pv = [&](int t, int j) {  // O_t += P_t(j) V_j, P read from TMEM (over S_t), part by part
        const uint64_t vd = vdesc0 + (uint64_t)(((j & 1) * Cfg::KT_BYTES) >> 4);
        constexpr int kPer = kFaKeys / 16 / kFaPvParts;  // K=16 MMAs per part
#pragma unroll
        for (int part = 0; part < kFaPvParts; ++part) {
          mbar_wait(&p_full[t * kFaPvParts + part], j & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kPer; ++kk) {
            const int k = part * kPer + kk;
            tc_mma_ts_warp(tmem_u + Cfg::o_col(t), tmem_u + Cfg::s_col(t) + k * 8, vd + ((k * 16 * 128) >> 4),
                           Cfg::IDESC_PV, (j > 0 || k > 0) ? 1u : 0u);
          }
        }
      };
      if (n_tiles > 0) {
        mbar_wait(&k_full[0], 0);
        tc_fence_after();
        issue_s(0, 0);
        issue_s(1, 0);
        for (int j = 0; j < n_tiles; ++j) {
          const bool more = j + 1 < n_tiles;
          mbar_wait(&v_full[j & 1], (j >> 1) & 1);
          issue_pv(0, j);
          FA_T(4, j);
          if (more) {
            mbar_wait(&k_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
            tc_fence_after();
            issue_s(0, j + 1);
            FA_T(5, j);
          }
          issue_pv(1, j);
          FA_T(6, j);
          tc_commit_warp(&kv_empty[j & 1]);
          if (more) issue_s(1, j + 1);
          FA_T(7, j);
        }
        tc_commit_warp(pv_done);
      }
    }
  } else {
#ifndef CC_NO_SETMAXNREG
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kFaSoftmaxRegs));
#endif
    // ---------------- softmax + epilogue (row per thread) ----------------
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t s_addr = tmem + lane_base + Cfg::s_col(tq);
    const uint32_t o_addr = tmem + lane_base + Cfg::o_col(tq);
    int warp_min = qrow >= 0 ? lim : 0x7fffffff, warp_ks = qrow >= 0 ? ks : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      warp_min = min(warp_min, __shfl_xor_sync(0xffffffffu, warp_min, o));
      warp_ks = max(warp_ks, __shfl_xor_sync(0xffffffffu, warp_ks, o));
    }
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      mbar_wait(&s_full[tq], j & 1);
      if (quarter == 0) FA_T(tq * 2, j);
      tc_fence_after();
      float sv[kFaKeys];
#pragma unroll
      for (int c = 0; c < kFaKeys / 32; ++c) tmem_ld32_async(s_addr + c * 32, sv + c * 32);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");  // one wait for the whole row
      const int key0 = (j0 + j) * kFaKeys;
      if (key0 + kFaKeys > warp_min || key0 < warp_ks) {  // boundary tile: apply the per-row key range
#pragma unroll
        for (int c = 0; c < kFaKeys; ++c) sv[c] = (key0 + c < lim && key0 + c >= ks) ? sv[c] : -INFINITY;
      }
      // row max as four independent 3-input chains (FMNMX3), short dependency depth
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < kFaKeys; c += 8) {
#pragma unroll
        for (int u = 0; u < 4; ++u) m4[u] = fmaxf(m4[u], fmaxf(sv[c + 2 * u], sv[c + 2 * u + 1]));
      }
      const float mt = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
      const float m_tile = mt * scale2;  // scale2 > 0: max commutes with the scale
      float alpha = 1.f;
      bool resc = false;
      if (m_tile > m_run + kFaRescaleThreshold) {
        alpha = (m_run == -INFINITY) ? 0.f : ex2_mufu(m_run - m_tile);
        m_run = m_tile;
        resc = true;
      }
      if (j > 0 && __any_sync(0xffffffffu, resc)) {
        // O is stable here: PV_t(j-1) completed before S_t(j) (in-order
        // tcgen05 pipe); rescaled before the first part of P is handed over
        const float a = resc ? alpha : 1.f;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          float ov[32];
          tmem_ld32(o_addr + c * 32, ov);
#pragma unroll
          for (int e = 0; e < 32; ++e) ov[e] *= a;
          tmem_st32(o_addr + c * 32, ov);
        }
      }
      const float nbase = (m_run == -INFINITY) ? 0.f : -m_run;
      const float2 sc2 = make_float2(scale2, scale2), nb2 = make_float2(nbase, nbase);
      float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      constexpr int kChunksPerPart = kFaKeys / 32 / kFaPvParts;
#pragma unroll
      for (int c = 0; c < kFaKeys / 32; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float2 x = __ffma2_rn(make_float2(sv[c * 32 + 2 * e], sv[c * 32 + 2 * e + 1]), sc2, nb2);
          float2 p;
          if (fa_poly_pair(e)) {  // kFaPolyPairs of 16 pairs on the FMA pipe
            p = ex2_poly2(x);
          } else {
            p.x = ex2_mufu(x.x);
            p.y = ex2_mufu(x.y);
          }
          acc[e & 3] = __fadd2_rn(acc[e & 3], p);
          pk[e] = pack2_bf16(p.x, p.y);
        }
        tmem_st16u(s_addr + c * 16, pk);  // P over the S row: column c*16+e holds keys (2e, 2e+1) of chunk c
        if ((c + 1) % kChunksPerPart == 0) {  // a part of P is in TMEM: hand it to the PV MMA
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[tq * kFaPvParts + c / kChunksPerPart]);
        }
      }
      const float2 s01 = __fadd2_rn(acc[0], acc[1]), s23 = __fadd2_rn(acc[2], acc[3]);
      const float lsum = (s01.x + s01.y) + (s23.x + s23.y);
      l_run = l_run * alpha + lsum;
      if (quarter == 0) FA_T(tq * 2 + 1, j);
    }
    if (n_tiles > 0) {
      mbar_wait(pv_done, 0);
      tc_fence_after();
    }
    const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
    const int64_t part_row = qrow >= 0 ? qrow * n_q_heads + qhead : -1;
    const int64_t out_off = qrow >= 0 ? qrow * ldo + (int64_t)qhead * D : -1;
    if (o_part && part_row >= 0)  // split-KV partial: log2-domain LSE of this shard's keys
      lse_part[part_row] = (l_run > 0.f && m_run != -INFINITY) ? m_run + __log2f(l_run) : -INFINITY;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      float ov[32];
      tmem_ld32(o_addr + c * 32, ov);
      if (o_part) {
        if (part_row >= 0 && l_run > 0.f) {  // rows with no visible key here: LSE -inf, O never read
          const bool live = n_tiles > 0;
          const float sc = live ? inv : 0.f;
          if (part_bf16) {  // bf16 partials: half the exchange and merge bytes
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(o_part) + part_row * D + c * 32);
#pragma unroll
            for (int qd = 0; qd < 4; ++qd)
              dst[qd] = make_uint4(pack2_bf16(ov[8 * qd] * sc, ov[8 * qd + 1] * sc),
                                   pack2_bf16(ov[8 * qd + 2] * sc, ov[8 * qd + 3] * sc),
                                   pack2_bf16(ov[8 * qd + 4] * sc, ov[8 * qd + 5] * sc),
                                   pack2_bf16(ov[8 * qd + 6] * sc, ov[8 * qd + 7] * sc));
          } else {
            float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(o_part) + part_row * D + c * 32);
#pragma unroll
            for (int qd = 0; qd < 8; ++qd)
              dst[qd] = make_float4(ov[4 * qd] * sc, ov[4 * qd + 1] * sc, ov[4 * qd + 2] * sc, ov[4 * qd + 3] * sc);
          }
        }
      } else if (out_off >= 0) {
        uint4* dst = reinterpret_cast<uint4*>(out + out_off + c * 32);
#pragma unroll
        for (int qd = 0; qd < 4; ++qd)
          dst[qd] = make_uint4(pack2_bf16(ov[8 * qd] * inv, ov[8 * qd + 1] * inv),
                               pack2_bf16(ov[8 * qd + 2] * inv, ov[8 * qd + 3] * inv),
                               pack2_bf16(ov[8 * qd + 4] * inv, ov[8 * qd + 5] * inv),
                               pack2_bf16(ov[8 * qd + 6] * inv, ov[8 * qd + 7] * inv));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 fa_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// [n_keys][Hkv][D] bf16 bank as a 3-D tensor map, box {64, 1, 128 keys}.
static int make_kv_map(CUtensorMap* map, const void* base, int64_t n_keys, int hkv, int d) {
  auto enc = fa_encode();
  if (!enc) return fail(CC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)hkv, (cuuint64_t)n_keys};
  cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)hkv * d * 2};
  cuuint32_t box[3] = {64, 1, (cuuint32_t)kFaKeys};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CC_ERR_CUDA, "cuTensorMapEncodeTiled (kv) failed (%d)", (int)r);
  return CC_OK;
}

template <int D>
static int fa_launch(const void* q, int64_t ldq, const int64_t* positions, const int64_t* kstart, int64_t m,
                     const void* k_cache,
                     const void* v_cache, int64_t n_keys, int32_t hq, int32_t hkv, float factor,
                     const float* row_factor, void* out, int64_t ldo, cudaStream_t st, double flops,
                     void* o_part = nullptr, float* lse_part = nullptr, int part_bf16 = 0, int n_splits = 1) {
  CUtensorMap tk, tv;
  int rc = make_kv_map(&tk, k_cache, n_keys, hkv, D);
  if (rc) return rc;
  rc = make_kv_map(&tv, v_cache, n_keys, hkv, D);
  if (rc) return rc;
  set_smem_once<fa_sparse_row_kernel<D>>(FaCfg<D>::SMEM);
  const int G = hq / hkv;
  const int n_ctas = (int)((m * G + 2 * kFaTileRows - 1) / (2 * kFaTileRows));
  dim3 grid(n_ctas * hkv, 1, n_splits);
  ProfScope ps(st, OP_ATTENTION, flops);
  const cudaError_t e = launch_pdl(fa_sparse_row_kernel<D>, grid, dim3(kFaThreads), FaCfg<D>::SMEM, st,
      tk, tv, (const __nv_bfloat16*)q, ldq, positions, kstart, m, n_keys, hq, hkv, factor, row_factor,
      (__nv_bfloat16*)out, ldo, n_ctas, o_part, lse_part, part_bf16);
  if (e != cudaSuccess) return fail(CC_ERR_CUDA, "fa_sparse_row launch failed: %s", cudaGetErrorString(e));
  return CC_OK;
}

// Split-KV merge: one warp per (row, head). Lane w reads part w's LSE (parts
// beyond 32 folded in a second pass), the warp reduces the max, and each lane
// keeps its part's weight; then every lane owns 4 (D=128) or 2 (D=64) head-dim
// columns and walks the parts with the weights broadcast by shuffle, four
// parts' loads in flight at a time (the merge is latency-bound otherwise).
template <typename P, int D>
__global__ void lse_merge_kernel(const P* __restrict__ o_parts, const float* __restrict__ lse_parts, int n_parts,
                                 int64_t part_stride, int64_t m, int hq, void* __restrict__ out, int64_t ldo,
                                 int out_dtype) {
  constexpr int C = D / 32;  // columns per lane
  pdl_wait();
  pdl_trigger();
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= m * hq) return;
  const int64_t i = gw / hq;
  const int h = (int)(gw % hq);
  const int64_t pstride = part_stride * hq;  // rows of (row, head) between consecutive parts
  float mx = -INFINITY;
  for (int w = lane; w < n_parts; w += 32) mx = fmaxf(mx, lse_parts[w * pstride + i * hq + h]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float acc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c] = 0.f;
  float wsum = 0.f;
  for (int w0 = 0; w0 < n_parts; w0 += 32) {
    const int w = w0 + lane;
    const float l = w < n_parts ? lse_parts[w * pstride + i * hq + h] : -INFINITY;
    const float a = (l == -INFINITY || mx == -INFINITY) ? 0.f : exp2f(l - mx);
    const int n = min(32, n_parts - w0);
    for (int k = 0; k < n; k += 4) {
      float aw[4];
      float v[4][C];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        aw[u] = __shfl_sync(0xffffffffu, a, (k + u) & 31);
        const bool live = k + u < n && aw[u] != 0.f;  // -inf parts are never read (their O is not written)
        const P* src = o_parts + ((int64_t)(w0 + k + u) * pstride + i * hq + h) * D + lane * C;
#pragma unroll
        for (int c = 0; c < C; ++c) v[u][c] = live ? static_cast<float>(src[c]) : 0.f;
        if (!(k + u < n)) aw[u] = 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        wsum += aw[u];
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] = fmaf(aw[u], v[u][c], acc[c]);
      }
    }
  }
  const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int64_t off = i * ldo + (int64_t)h * D + lane * C + c;
    if (out_dtype == CC_BF16)
      reinterpret_cast<__nv_bfloat16*>(out)[off] = __float2bfloat16_rn(acc[c] * inv);
    else
      reinterpret_cast<float*>(out)[off] = acc[c] * inv;
  }
}

__global__ void fill_neg_inf_kernel(float* __restrict__ p, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = -INFINITY;
}

__global__ void local_limits_kernel(const int64_t* __restrict__ row_pos, int64_t m,
                                    const int64_t* __restrict__ local_pos, int64_t n, int64_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t p = row_pos[i];
  int64_t lo = 0, hi = n;  // first index with local_pos > p
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (local_pos[mid] <= p) lo = mid + 1; else hi = mid;
  }
  out[i] = lo - 1;
}

}  // namespace cc

using namespace cc;

#ifdef CC_FA_TRACE
extern "C" int cc_debug_fa_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, g_fa_trace, sizeof(long long) * 16 * 128) == cudaSuccess ? 0 : 1;
}
#endif

// algorithmic work of the next attention launch, for the launch profiler (set
// by the executor, which knows sum(pos+1) on the host; 0 when unknown).
// Thread-local: each host thread driving the library has its own.
thread_local double g_attn_flops = 0.0;

extern "C" int cc_sparse_row_attention_ranged(const void* q, int64_t ldq, const int64_t* positions,
                                              const int64_t* key_start, int64_t m, const void* k_cache,
                                              const void* v_cache, int64_t n_keys, int32_t n_q_heads,
                                              int32_t n_kv_heads, int32_t head_dim, float factor,
                                              const float* row_factor, void* out, int64_t ldo, void* stream) {
  CC_CHECK_ARG(n_kv_heads > 0 && n_q_heads % n_kv_heads == 0, CC_ERR_DIMENSION,
               "query heads %d not a multiple of kv heads %d", n_q_heads, n_kv_heads);
  CC_CHECK_ARG(head_dim == 64 || head_dim == 128, CC_ERR_UNSUPPORTED, "head_dim %d unsupported", head_dim);
  CC_CHECK_ARG(n_keys > 0, CC_ERR_VALUE, "attention row with no visible keys");
  CC_CHECK_ARG(n_keys < (int64_t)1 << 31, CC_ERR_UNSUPPORTED, "key bank of %lld rows too large",
               (long long)n_keys);
  CC_CHECK_ARG(((uintptr_t)k_cache % 16) == 0 && ((uintptr_t)v_cache % 16) == 0 && ((uintptr_t)q % 16) == 0 &&
                   (ldq % 8) == 0 && (ldo % 8) == 0,
               CC_ERR_UNSUPPORTED, "attention operands must be 16-byte aligned");
  if (m <= 0) return CC_OK;
  cudaStream_t st = as_stream(stream);
  if (head_dim == 128)
    return fa_launch<128>(q, ldq, positions, key_start, m, k_cache, v_cache, n_keys, n_q_heads, n_kv_heads, factor,
                          row_factor, out, ldo, st, g_attn_flops);
  return fa_launch<64>(q, ldq, positions, key_start, m, k_cache, v_cache, n_keys, n_q_heads, n_kv_heads, factor,
                       row_factor, out, ldo, st, g_attn_flops);
}

// Split-KV count for a launch of m rows over n_keys keys. A launch of G*m
// packed rows runs ceil(G*m / 256) x Hkv CTAs; when that is under one wave of
// the SMs (decode steps, the last layer's head row, the default 8/5 window
// rule's few hundred rows) and the keys are long, the grid gets S parts per
// CTA, S bringing it to about two waves. Inside the kernel a CTA uses only as
// many parts as its own key range has 8-tile blocks, so the long
// (late-position) ranges are cut and the short ones stay whole; the parts are
// merged by log-sum-exp. Grids of a wave or more are never split.
extern "C" int32_t cc_attention_splits(int64_t m, int32_t n_q_heads, int32_t n_kv_heads, int64_t n_keys) {
  static int enabled = -1;  // CC_ATTN_SPLIT=0 in the environment: never split (A/B runs)
  if (enabled < 0) {
    const char* e = getenv("CC_ATTN_SPLIT");
    enabled = (e && e[0] == '0') ? 0 : 1;
  }
  if (!enabled || m <= 0 || n_kv_heads <= 0 || n_q_heads % n_kv_heads) return 1;
  if (n_keys < 4096) return 1;
  const int64_t G = n_q_heads / n_kv_heads;
  const int64_t ctas = (m * G + 2 * kFaTileRows - 1) / (2 * kFaTileRows) * n_kv_heads;
  // a grid of one wave or more is left whole: the heavy-first order balances
  // it, and the partial stores + merge would cost more than the fuller grid
  // gains (measured at C2 20 %: 184 CTAs, attention 4.5 + merge 0.9 ms)
  if (ctas >= (int64_t)num_sms()) return 1;
  const int64_t waves2 = 2 * (int64_t)num_sms();
  int64_t s = (waves2 + ctas - 1) / ctas;
  s = std::min<int64_t>(s, kMaxAttnSplits);
  s = std::min<int64_t>(s, n_keys / (kFaMinSplitTiles * kFaKeys));
  return (int32_t)std::max<int64_t>(1, s);
}

extern "C" int cc_sparse_row_attention_split(const void* q, int64_t ldq, const int64_t* positions,
                                             const int64_t* key_start, int64_t m, const void* k_cache,
                                             const void* v_cache, int64_t n_keys, int32_t n_q_heads,
                                             int32_t n_kv_heads, int32_t head_dim, float factor,
                                             const float* row_factor, int32_t n_splits, float* o_parts,
                                             float* lse_parts, void* out, int64_t ldo, void* stream) {
  if (n_splits <= 1)
    return cc_sparse_row_attention_ranged(q, ldq, positions, key_start, m, k_cache, v_cache, n_keys, n_q_heads,
                                          n_kv_heads, head_dim, factor, row_factor, out, ldo, stream);
  CC_CHECK_ARG(n_kv_heads > 0 && n_q_heads % n_kv_heads == 0, CC_ERR_DIMENSION,
               "query heads %d not a multiple of kv heads %d", n_q_heads, n_kv_heads);
  CC_CHECK_ARG(head_dim == 64 || head_dim == 128, CC_ERR_UNSUPPORTED, "head_dim %d unsupported", head_dim);
  CC_CHECK_ARG(n_keys > 0 && n_keys < (int64_t)1 << 31, CC_ERR_VALUE, "bad key bank size");
  CC_CHECK_ARG(n_splits <= kMaxAttnSplits && o_parts && lse_parts, CC_ERR_VALUE,
               "split attention needs partial buffers and at most %d parts", kMaxAttnSplits);
  CC_CHECK_ARG(((uintptr_t)k_cache % 16) == 0 && ((uintptr_t)v_cache % 16) == 0 && ((uintptr_t)q % 16) == 0 &&
                   (ldq % 8) == 0 && (ldo % 8) == 0,
               CC_ERR_UNSUPPORTED, "attention operands must be 16-byte aligned");
  if (m <= 0) return CC_OK;
  cudaStream_t st = as_stream(stream);
  const int rc = head_dim == 128
                     ? fa_launch<128>(q, ldq, positions, key_start, m, k_cache, v_cache, n_keys, n_q_heads,
                                      n_kv_heads, factor, row_factor, nullptr, 0, st, g_attn_flops, o_parts,
                                      lse_parts, 0, n_splits)
                     : fa_launch<64>(q, ldq, positions, key_start, m, k_cache, v_cache, n_keys, n_q_heads,
                                     n_kv_heads, factor, row_factor, nullptr, 0, st, g_attn_flops, o_parts,
                                     lse_parts, 0, n_splits);
  if (rc) return rc;
  return cc_lse_merge(o_parts, CC_F32, lse_parts, n_splits, m, m, n_q_heads, head_dim, out, ldo, CC_BF16, stream);
}

extern "C" int cc_sparse_row_attention(const void* q, int64_t ldq, const int64_t* positions, int64_t m,
                                       const void* k_cache, const void* v_cache, int64_t n_keys, int32_t n_q_heads,
                                       int32_t n_kv_heads, int32_t head_dim, float factor, const float* row_factor,
                                       void* out, int64_t ldo, void* stream) {
  return cc_sparse_row_attention_ranged(q, ldq, positions, nullptr, m, k_cache, v_cache, n_keys, n_q_heads,
                                        n_kv_heads, head_dim, factor, row_factor, out, ldo, stream);
}

extern "C" int cc_sparse_row_attention_partial(const void* q, int64_t ldq, const int64_t* limits, int64_t m,
                                               const void* k_cache, const void* v_cache, int64_t n_keys,
                                               int32_t n_q_heads, int32_t n_kv_heads, int32_t head_dim, float factor,
                                               const float* row_factor, void* o_part, int32_t part_dtype, float* lse,
                                               void* stream) {
  CC_CHECK_ARG(n_kv_heads > 0 && n_q_heads % n_kv_heads == 0, CC_ERR_DIMENSION, "bad head counts");
  CC_CHECK_ARG(head_dim == 64 || head_dim == 128, CC_ERR_UNSUPPORTED, "head_dim %d unsupported", head_dim);
  CC_CHECK_ARG(o_part && lse, CC_ERR_VALUE, "partial attention needs o_part and lse outputs");
  CC_CHECK_ARG(part_dtype == CC_F32 || part_dtype == CC_BF16, CC_ERR_UNSUPPORTED, "partial dtype %d", part_dtype);
  const int part_bf16 = part_dtype == CC_BF16;
  if (m <= 0) return CC_OK;
  cudaStream_t st = as_stream(stream);
  if (n_keys <= 0) {  // an empty shard contributes nothing: O = 0, LSE = -inf
    cudaMemsetAsync(o_part, 0, (size_t)m * n_q_heads * head_dim * (part_bf16 ? 2 : 4), st);
    const int64_t n = m * n_q_heads;
    ProfScope ps(st, OP_OTHER, 0);
    fill_neg_inf_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(lse, n);
    CC_LAUNCH_CHECK("partial attention (empty shard)");
    return CC_OK;
  }
  if (head_dim == 128)
    return fa_launch<128>(q, ldq, limits, nullptr, m, k_cache, v_cache, n_keys, n_q_heads, n_kv_heads, factor, row_factor,
                          nullptr, 0, st, g_attn_flops, o_part, lse, part_bf16);
  return fa_launch<64>(q, ldq, limits, nullptr, m, k_cache, v_cache, n_keys, n_q_heads, n_kv_heads, factor, row_factor,
                       nullptr, 0, st, g_attn_flops, o_part, lse, part_bf16);
}

extern "C" int cc_local_limits(const int64_t* row_pos, int64_t m, const int64_t* local_pos, int64_t n_local,
                               int64_t* limits, void* stream) {
  if (m <= 0) return CC_OK;
  ProfScope ps(as_stream(stream), OP_OTHER, 0);
  local_limits_kernel<<<(unsigned)((m + 255) / 256), 256, 0, as_stream(stream)>>>(row_pos, m, local_pos, n_local,
                                                                                  limits);
  CC_LAUNCH_CHECK("local_limits");
  return CC_OK;
}

extern "C" int cc_lse_merge(const void* o_parts, int32_t part_dtype, const float* lse_parts, int32_t n_parts,
                            int64_t part_stride, int64_t m, int32_t n_q_heads, int32_t head_dim, void* out,
                            int64_t ldo, int32_t out_dtype, void* stream) {
  CC_CHECK_ARG(head_dim == 64 || head_dim == 128, CC_ERR_UNSUPPORTED, "head_dim %d unsupported", head_dim);
  CC_CHECK_ARG(part_dtype == CC_F32 || part_dtype == CC_BF16, CC_ERR_UNSUPPORTED, "partial dtype %d", part_dtype);
  if (m <= 0 || n_parts <= 0) return CC_OK;
  const int64_t warps = m * n_q_heads;
  const unsigned grid = (unsigned)((warps * 32 + 255) / 256);
  cudaStream_t st = as_stream(stream);
  ProfScope ps(st, OP_MERGE, 0.0);
#define CC_MERGE(P, D)                                                                                             \
  launch_pdl(lse_merge_kernel<P, D>, dim3(grid), dim3(256), 0, st, static_cast<const P*>(o_parts), lse_parts, n_parts, \
             part_stride, m, n_q_heads, out, ldo, out_dtype)
  if (part_dtype == CC_BF16) {
    if (head_dim == 128) CC_MERGE(__nv_bfloat16, 128); else CC_MERGE(__nv_bfloat16, 64);
  } else {
    if (head_dim == 128) CC_MERGE(float, 128); else CC_MERGE(float, 64);
  }
#undef CC_MERGE
  CC_LAUNCH_CHECK("lse_merge");
  return CC_OK;
}
