// Scoring-model (fp32) banked attention on tcgen05, 3xTF32.
//
// The same operation as banked_f32.cu — causal_attention of peek_forward
// (model.py:568-607 -> tensor_core.py:109-170) for many sequences at once,
// sequence s = one chunk cache's rotated K/V bank plus the query rows, new row
// i seeing bank rows [0, n_bank) and new rows [0, i] — with both matrix
// products on the 5th-gen tensor core:
//
//   S  = Q K^T  as  Qhi Khi + Qhi Klo + Qlo Khi   (kind::tf32, fp32 in TMEM)
//   O  = P V    as  Phi Vhi + Phi Vlo + Plo Vhi   (P from TMEM, V^T K-major smem)
//
// hi = x rounded to tf32, lo = tf32(x - hi): the dropped lo*lo term and the
// tf32 rounding of lo leave ~2^-22 relative error per product (fp32 level).
// A row's 576 logits do not fit TMEM. The scoring layer sweeps the key tiles
// three times to follow the reference's order exactly; context layers make
// one online pass:
//   - last (scoring) layer: the reference's order exactly (tensor_core.py:
//     88-96, 165-170) — max of S * factor, then the sum of exp(x - max), then
//     p = exp(x - max) / sum written as the weights (selector.py:157-165);
//   - other layers: one sweep, online softmax in the log2 domain (MUFU ex2)
//     with a lazy rescale of O, P = 2^(y - max) fed to O += P V, O / sum at
//     the end.
//
// CTA = one sequence x one KV head x (128 / G) query rows; packed row r =
// query i0 + r / G, head kvh*G + r % G, so the K/V tiles are read once for
// all G heads. 8 warps: warp w owns TMEM lane quarter w % 4 (its packed rows)
// and column half w / 4 of every 32-key tile; the two halves combine their
// row statistics once per sweep through shared memory. K/V tiles are
// register-prefetched from global one tile ahead, split hi/lo and written
// into 128B-swizzled smem (V transposed: an MN-major tf32 B operand read back
// as zeros on this part, K-major V^T is exact); one thread issues the MMAs.
#include "cc_common.cuh"

namespace cc {

constexpr int kBtRows = 128;   // packed rows per CTA = TMEM lanes
constexpr int kBtThreads = 256;  // 4 lane quarters x 2 column halves

template <int HD>
struct BtCfg {
  // keys per tile. 64-key tiles for head_dim 64 (half the serial tile steps)
  // were measured slower (C3 step 2.7 -> 3.4 ms): 128 KB of shared memory and
  // 201 registers leave one CTA per SM where 32-key tiles fit two, and the
  // second CTA hides more of the per-tile barrier chain than halving it saves.
  static constexpr int KEYS = 32;
  static constexpr int HC = KEYS / 2;               // columns of a key tile per thread (two halves)
  static constexpr int Q_BYTES = kBtRows * HD * 4;  // one of Q_hi / Q_lo
  static constexpr int K_BYTES = KEYS * HD * 4;     // one of K_hi / K_lo / V_hi / V_lo
  static constexpr int SMEM = 2 * Q_BYTES + 4 * K_BYTES + 4 * kBtRows * 4 + 1024 + 64;
  static constexpr int T_S = 0, T_PH = KEYS, T_PL = 2 * KEYS, T_O = 3 * KEYS;
  static constexpr int TMEM_COLS = (3 * KEYS + HD) <= 256 ? 256 : 512;
  static constexpr int F4 = KEYS * HD / 4 / kBtThreads;  // float4 per thread per K (or V) tile
  static constexpr uint32_t IDESC_S = umma_idesc(128, KEYS, true);
  static constexpr uint32_t IDESC_PV = umma_idesc(128, HD, true);  // B = V^T, K-major
  static_assert(SMEM <= 232448, "banked tile over the shared-memory limit");
};

// byte offset of fp32 element (row, col) in a [R rows] x [cols] 128B-swizzled
// tile stored as 32-column blocks of R x 128 B (K-major: Q, K rows; V^T dim rows)
__device__ __forceinline__ uint32_t sw128_off(int row, int col, int R) {
  const int kb = col >> 5, chunk = (col & 31) >> 2;
  return (uint32_t)(kb * (R * 128) + row * 128 + ((chunk ^ (row & 7)) << 4) + (col & 3) * 4);
}

__device__ __forceinline__ void split4(const float4 v, float4& hi, float4& lo) {
  float t;
  split_tf32(v.x, hi.x, t);
  lo.x = t;
  split_tf32(v.y, hi.y, t);
  lo.y = t;
  split_tf32(v.z, hi.z, t);
  lo.z = t;
  split_tf32(v.w, hi.w, t);
  lo.w = t;
}

__device__ __forceinline__ void fence_proxy_async_bt() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// D[tmem] (+)= A[tmem] * B[smem], tf32
__device__ __forceinline__ void tc_mma_ts_tf32(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// warp-wide form (see tc_mma_warp in cc_common.cuh)
__device__ __forceinline__ void tc_mma_ts_tf32_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                                    uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st32_f(uint32_t taddr, const float* v) {
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

__device__ __forceinline__ void tmem_st16_f(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// tf32 split without the non-finite guard (inputs are finite probabilities / values)
__device__ __forceinline__ void split_tf32_finite(float x, float& hi, float& lo) {
  const uint32_t u = __float_as_uint(x);
  hi = __uint_as_float((u + 0xFFFu + ((u >> 13) & 1u)) & 0xFFFFE000u);
  lo = __fsub_rn(x, hi);
}

template <int HD>
__global__ void __launch_bounds__(kBtThreads) banked_tc_kernel(
    const cc_bank_seq* __restrict__ seqs, const float* __restrict__ q, const float* __restrict__ k_new,
    const float* __restrict__ v_new, int n_q_heads, int n_kv_heads, float factor, int qpb, void* __restrict__ out,
    int out_mode, float* __restrict__ weights_out, int64_t w_col0, int64_t w_ld) {
  using Cfg = BtCfg<HD>;
  constexpr int HC = Cfg::HC;
  constexpr int kBtKeys = Cfg::KEYS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sQh = smem;
  uint8_t* sQl = sQh + Cfg::Q_BYTES;
  uint8_t* sKh = sQl + Cfg::Q_BYTES;
  uint8_t* sKl = sKh + Cfg::K_BYTES;
  uint8_t* sVh = sKl + Cfg::K_BYTES;
  uint8_t* sVl = sVh + Cfg::K_BYTES;
  float* red = reinterpret_cast<float*>(sVl + Cfg::K_BYTES);  // [2 halves][2][128 rows]
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(red + 4 * kBtRows);
  uint64_t* pv_bar = s_bar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_bar + 2);

  pdl_wait();  // first global access below (the bank table)
  pdl_trigger();
  const cc_bank_seq sq = seqs[blockIdx.z];
  const int kvh = blockIdx.y;
  const int G = n_q_heads / n_kv_heads;
  const int i0 = blockIdx.x * qpb;
  if (i0 >= sq.n_new) return;  // uniform over the CTA
  const int nq = min(qpb, (int)(sq.n_new - i0));
  const int nrows = nq * G;
  const int64_t nb = sq.n_bank;
  const int ncols = (int)(nb + i0 + nq);
  const int n_tiles = (ncols + kBtKeys - 1) / kBtKeys;
  const int64_t qw = (int64_t)n_q_heads * HD, kvw = (int64_t)n_kv_heads * HD;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int half = warp >> 2;                 // column half of every key tile
  const int r = (warp & 3) * 32 + lane;       // packed row = TMEM lane
  const bool scoring = weights_out != nullptr;

  if (tid == 0) {
    mbar_init(s_bar, 1);
    mbar_init(pv_bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);

  // ---- packed row r: Q -> split hi/lo, swizzled K-major (each half stages half the dims) ----
  const bool live = r < nrows;
  const int qi = i0 + (live ? r / G : 0);
  const int head = kvh * G + (live ? r % G : 0);
  const int limit = live ? (int)(nb + qi + 1) : 0;
  {
    const float4* src = reinterpret_cast<const float4*>(q + (sq.row0 + qi) * qw + (int64_t)head * HD);
#pragma unroll
    for (int c = 0; c < HD / 8; ++c) {
      const int c4 = half * (HD / 8) + c;
      const float4 v = live ? __ldg(src + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 hi, lo;
      split4(v, hi, lo);
      const uint32_t off = sw128_off(r, 4 * c4, kBtRows);
      *reinterpret_cast<float4*>(sQh + off) = hi;
      *reinterpret_cast<float4*>(sQl + off) = lo;
    }
  }

  // ---- K / V tile prefetch (registers, one tile ahead) ----
  float4 kreg[Cfg::F4], vreg[Cfg::F4];
  auto fetch = [&](int j, bool with_v) {
#pragma unroll
    for (int e = 0; e < Cfg::F4; ++e) {
      const int idx = tid + e * kBtThreads;
      const int key = idx / (HD / 4), c4 = idx % (HD / 4);
      const int64_t col = (int64_t)j * kBtKeys + key;
      if (col < ncols) {
        const int64_t off = (col < nb ? col : sq.row0 + (col - nb)) * kvw + (int64_t)kvh * HD + 4 * c4;
        kreg[e] = __ldg(reinterpret_cast<const float4*>((col < nb ? sq.k : k_new) + off));
        if (with_v) vreg[e] = __ldg(reinterpret_cast<const float4*>((col < nb ? sq.v : v_new) + off));
      } else {
        kreg[e] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (with_v) vreg[e] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  };
  auto stage = [&](bool with_v) {
#pragma unroll
    for (int e = 0; e < Cfg::F4; ++e) {
      const int idx = tid + e * kBtThreads;
      const int key = idx / (HD / 4), c4 = idx % (HD / 4);
      const uint32_t off = sw128_off(key, 4 * c4, kBtKeys);
      float4 hi, lo;
      split4(kreg[e], hi, lo);
      *reinterpret_cast<float4*>(sKh + off) = hi;
      *reinterpret_cast<float4*>(sKl + off) = lo;
      if (with_v) {
        split4(vreg[e], hi, lo);
        // V^T [HD dims][keys], K-major (128-byte blocks of 32 keys per dim)
        const float hv[4] = {hi.x, hi.y, hi.z, hi.w}, lv[4] = {lo.x, lo.y, lo.z, lo.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t o2 = sw128_off(4 * c4 + i, key, HD);
          *reinterpret_cast<float*>(sVh + o2) = hv[i];
          *reinterpret_cast<float*>(sVl + o2) = lv[i];
        }
      }
    }
  };

  fence_proxy_async_bt();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // warp-uniform MMA operands for warp 0's issue (descriptors formed once)
  const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
  const uint64_t dq_h = umma_desc_sw128(smem_u32(sQh)), dq_l = umma_desc_sw128(smem_u32(sQl));
  const uint64_t dk_h = umma_desc_sw128(smem_u32(sKh)), dk_l = umma_desc_sw128(smem_u32(sKl));
  const uint64_t dv_h = umma_desc_sw128(smem_u32(sVh)), dv_l = umma_desc_sw128(smem_u32(sVl));
  const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);  // this warp's TMEM lane quarter
  const uint32_t t_s = tl + Cfg::T_S + half * HC;

  uint32_t s_phase = 0, pv_phase = 0;
  // one sweep over the key tiles: S = Q K^T for tile j, then body(c0 + half*HC, s[HC])
  auto sweep = [&](bool with_v, auto&& body) {
    fetch(0, with_v);
    for (int j = 0; j < n_tiles; ++j) {
      if (with_v && j > 0) {  // PV(j-1) still reads V smem and P in TMEM
        mbar_wait(pv_bar, pv_phase);
        pv_phase ^= 1;
      }
      stage(with_v);
      fence_proxy_async_bt();
      tc_fence_before();
      __syncthreads();  // also: every thread has read S(j-1) before S(j) overwrites it
      tc_fence_after();
      if (warp == 0) {  // warp-wide issue from uniform descriptors (one elected lane per op)
#pragma unroll
        for (int k = 0; k < HD / 8; ++k) {
          const uint32_t qo = ((k >> 2) * (kBtRows * 128) + (k & 3) * 32) >> 4;
          const uint32_t ko = ((k >> 2) * (kBtKeys * 128) + (k & 3) * 32) >> 4;
          tc_mma_warp<true>(tmem_u + Cfg::T_S, dq_h + qo, dk_h + ko, Cfg::IDESC_S, k > 0 ? 1u : 0u);
          tc_mma_warp<true>(tmem_u + Cfg::T_S, dq_h + qo, dk_l + ko, Cfg::IDESC_S, 1u);
          tc_mma_warp<true>(tmem_u + Cfg::T_S, dq_l + qo, dk_h + ko, Cfg::IDESC_S, 1u);
        }
        tc_commit_warp(s_bar);
      }
      if (j + 1 < n_tiles) fetch(j + 1, with_v);  // in flight during the MMA and the softmax
      mbar_wait(s_bar, s_phase);
      s_phase ^= 1;
      tc_fence_after();
      float s[HC];
#pragma unroll
      for (int c = 0; c < HC; c += 16) tmem_ld16(t_s + c, s + c);
      body(j, j * kBtKeys + half * HC, s);
    }
  };
  // combine a per-half row statistic (half 0 first: deterministic order)
  auto exchange = [&](float a, float b, float& a1, float& b1) {
    red[(half * 2 + 0) * kBtRows + r] = a;
    red[(half * 2 + 1) * kBtRows + r] = b;
    __syncthreads();
    a1 = red[((half ^ 1) * 2 + 0) * kBtRows + r];
    b1 = red[((half ^ 1) * 2 + 1) * kBtRows + r];
    __syncthreads();
  };

  if (scoring) {
    // Exact reference order for the weights that become importance scores:
    // max of (S * factor), then sum of exp(x - max), then exp(x - max) / sum.
    float mx = -INFINITY;
    sweep(false, [&](int, int c0, float* s) {
#pragma unroll
      for (int t = 0; t < HC; ++t)
        if (c0 + t < limit) mx = fmaxf(mx, __fmul_rn(s[t], factor));
    });
    float o0, o1, unused;
    exchange(mx, 0.f, o0, unused);
    mx = fmaxf(mx, o0);
    float sum = 0.f;
    sweep(false, [&](int, int c0, float* s) {
#pragma unroll
      for (int t = 0; t < HC; ++t)
        if (c0 + t < limit) sum = __fadd_rn(sum, expf(__fsub_rn(__fmul_rn(s[t], factor), mx)));
    });
    exchange(sum, 0.f, o1, unused);
    sum = half == 0 ? __fadd_rn(sum, o1) : __fadd_rn(o1, sum);
    float* wrow = live ? weights_out + (((int64_t)blockIdx.z * n_q_heads + head) * sq.n_new + qi) * w_ld - w_col0
                       : nullptr;
    sweep(false, [&](int, int c0, float* s) {
      if (!wrow || c0 >= nb || c0 + HC <= w_col0) return;
      float p[HC];
#pragma unroll
      for (int t = 0; t < HC; ++t)
        p[t] = c0 + t < limit ? __fdiv_rn(expf(__fsub_rn(__fmul_rn(s[t], factor), mx)), sum) : 0.f;
      float* dst = wrow + c0;
      if (c0 >= w_col0 && c0 + HC <= nb && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
        for (int t = 0; t < HC / 4; ++t)
          reinterpret_cast<float4*>(dst)[t] = make_float4(p[4 * t], p[4 * t + 1], p[4 * t + 2], p[4 * t + 3]);
      } else {
#pragma unroll
        for (int t = 0; t < HC; ++t)
          if (c0 + t >= w_col0 && c0 + t < nb) dst[t] = p[t];
      }
    });
  } else {
    // Context rows: ONE sweep, online softmax in the log2 domain (MUFU ex2).
    // Per key tile the two column halves of a row agree on the tile max
    // through shared memory; the running max moves only when a tile raises
    // it by more than 2^8 (lazy rescale: O in TMEM and the partial sums are
    // scaled then), P = 2^(y - max) unnormalised feeds O += P V, and the
    // epilogue divides by the row sum.
    const float fl = factor * 1.4426950408889634f;
    float m_run = -INFINITY, l_half = 0.f;
    sweep(true, [&](int j, int c0, float* s) {
      float tm = -INFINITY;
#pragma unroll
      for (int t = 0; t < HC; ++t) {
        s[t] = c0 + t < limit ? s[t] * fl : -INFINITY;
        tm = fmaxf(tm, s[t]);
      }
      red[half * kBtRows + r] = tm;
      __syncthreads();
      tm = fmaxf(tm, red[(half ^ 1) * kBtRows + r]);
      float alpha = 1.f;
      bool resc = false;
      if (tm > m_run + 8.0f) {
        alpha = m_run == -INFINITY ? 0.f : ex2_approx(m_run - tm);
        m_run = tm;
        resc = true;
      }
      if (j > 0 && __any_sync(0xffffffffu, resc)) {
        // O is stable: the sweep waited for PV(j-1) before staging this tile
        const float a = resc ? alpha : 1.f;
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          float o[32];
          tmem_ld32(tl + Cfg::T_O + half * (HD / 2) + c * 32, o);
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] *= a;
          tmem_st32_f(tl + Cfg::T_O + half * (HD / 2) + c * 32, o);
        }
      }
      float ph[HC], ls = 0.f;
#pragma unroll
      for (int t = 0; t < HC; ++t) {
        const float pv = c0 + t < limit ? ex2_approx(s[t] - m_run) : 0.f;
        ls += pv;
        float lo;
        split_tf32_finite(pv, ph[t], lo);
        float l2;
        split_tf32_finite(lo, s[t], l2);
      }
      l_half = l_half * alpha + ls;
#pragma unroll
      for (int c = 0; c < HC; c += 16) {
        tmem_st16_f(tl + Cfg::T_PH + half * HC + c, ph + c);
        tmem_st16_f(tl + Cfg::T_PL + half * HC + c, s + c);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncthreads();
      tc_fence_after();
      if (warp == 0) {
#pragma unroll
        for (int k = 0; k < kBtKeys / 8; ++k) {
          // V^T [HD dims][keys]: 32-key (128-byte) K-blocks HD rows apart
          const uint32_t vo = ((k >> 2) * (HD * 128) + (k & 3) * 32) >> 4;
          const uint64_t bh = dv_h + vo, bl = dv_l + vo;
          tc_mma_ts_tf32_warp(tmem_u + Cfg::T_O, tmem_u + Cfg::T_PH + k * 8, bh, Cfg::IDESC_PV,
                              (j > 0 || k > 0) ? 1u : 0u);
          tc_mma_ts_tf32_warp(tmem_u + Cfg::T_O, tmem_u + Cfg::T_PH + k * 8, bl, Cfg::IDESC_PV, 1u);
          tc_mma_ts_tf32_warp(tmem_u + Cfg::T_O, tmem_u + Cfg::T_PL + k * 8, bh, Cfg::IDESC_PV, 1u);
        }
        tc_commit_warp(pv_bar);
      }
    });
    float l_other, unused;
    exchange(l_half, 0.f, l_other, unused);
    const float L = half == 0 ? l_half + l_other : l_other + l_half;
    const float inv = L > 0.f ? 1.0f / L : 0.f;
    mbar_wait(pv_bar, pv_phase);
    tc_fence_after();
#pragma unroll
    for (int c = 0; c < HD / 64; ++c) {
      float o[32];
      const int d0 = half * (HD / 2) + c * 32;
      tmem_ld32(tl + Cfg::T_O + d0, o);
      if (!live) continue;
#pragma unroll
      for (int e = 0; e < 32; ++e) o[e] *= inv;
      const int64_t row = sq.row0 + qi;
      const int64_t col0 = (int64_t)head * HD + d0;
      if (out_mode == CC_F32) {
        float4* p = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + row * qw + col0);
#pragma unroll
        for (int t = 0; t < 8; ++t) p[t] = make_float4(o[4 * t], o[4 * t + 1], o[4 * t + 2], o[4 * t + 3]);
      } else {  // [hi | hi | lo] (the o-proj A operand)
        float* p = reinterpret_cast<float*>(out) + row * qw * 3 + col0;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          float4 v = make_float4(o[4 * t], o[4 * t + 1], o[4 * t + 2], o[4 * t + 3]), hi, lo, lh, ll;
          split4(v, hi, lo);
          split4(lo, lh, ll);
          reinterpret_cast<float4*>(p)[t] = hi;  // (middle hi copy unread by the 3xTF32 GEMM)
          reinterpret_cast<float4*>(p + 2 * qw)[t] = lh;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, Cfg::TMEM_COLS);
  }
}

}  // namespace cc

using namespace cc;

extern "C" int cc_banked_attention_f32(const cc_bank_seq* seqs_dev, int32_t n_seqs, int32_t max_new,
                                      int64_t max_bank, const float* q, const float* k_new, const float* v_new,
                                      int32_t n_q_heads, int32_t n_kv_heads, int32_t head_dim, float factor,
                                      void* out, int32_t out_mode, float* weights_out, int64_t w_col0,
                                      int64_t w_ld, void* stream) {
  CC_CHECK_ARG(n_kv_heads > 0 && n_q_heads % n_kv_heads == 0, CC_ERR_DIMENSION, "bad head counts");
  CC_CHECK_ARG(head_dim == 64 || head_dim == 128, CC_ERR_UNSUPPORTED, "head_dim %d unsupported", head_dim);
  CC_CHECK_ARG(out_mode == CC_F32 || out_mode == CC_F32_SPLIT3, CC_ERR_UNSUPPORTED, "out mode");
  const int G = n_q_heads / n_kv_heads;
  CC_CHECK_ARG(G <= kBtRows, CC_ERR_UNSUPPORTED, "GQA group %d > %d", G, kBtRows);
  (void)max_bank;
  if (n_seqs <= 0 || max_new <= 0) return CC_OK;
  const int qpb = kBtRows / G;
  dim3 grid((max_new + qpb - 1) / qpb, n_kv_heads, n_seqs);
  cudaStream_t st = as_stream(stream);
  ProfScope ps(st, OP_BANKED, 0);
  if (head_dim == 64) {
    set_smem_once<banked_tc_kernel<64>>(BtCfg<64>::SMEM);
    launch_pdl(banked_tc_kernel<64>, grid, dim3(kBtThreads), BtCfg<64>::SMEM, st, seqs_dev, q, k_new, v_new,
               n_q_heads, n_kv_heads, factor, qpb, out, out_mode, weights_out, w_col0, w_ld);
  } else {
    set_smem_once<banked_tc_kernel<128>>(BtCfg<128>::SMEM);
    launch_pdl(banked_tc_kernel<128>, grid, dim3(kBtThreads), BtCfg<128>::SMEM, st, seqs_dev, q, k_new, v_new,
               n_q_heads, n_kv_heads, factor, qpb, out, out_mode, weights_out, w_col0, w_ld);
  }
  CC_LAUNCH_CHECK("banked_attention_tc");
  return CC_OK;
}
