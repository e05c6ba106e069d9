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
// The softmax keeps the reference's order exactly (tensor_core.py:88-96,
// 165-170): logits = S * factor (one fp32 multiply), masked, row max, e =
// exp(logit - max), row sum, p = e / sum, then p @ V. Since a row's 576
// logits do not fit TMEM, the key tiles are swept three times — max, sum,
// then p (stored as the last-layer weights, selector.py:157-165, or fed to
// the PV product); recomputing Q K^T is cheap next to the softmax.
//
// CTA = one sequence x one KV head x (128 / G) query rows; packed row r =
// query i0 + r / G, head kvh*G + r % G, so the K/V tiles are read once for
// all G heads. Thread r owns TMEM lane r (its packed row). K/V tiles are
// register-prefetched from global one tile ahead, split hi/lo and written
// into 128B-swizzled smem (V transposed: an MN-major tf32 B operand read back
// as zeros on this part, K-major V^T is exact); one thread issues the MMAs.
#include "cc_common.cuh"

namespace cc {

constexpr int kBtRows = 128;   // packed rows per CTA = TMEM lanes
constexpr int kBtKeys = 32;    // keys per tile
constexpr int kBtThreads = 128;

template <int HD>
struct BtCfg {
  static constexpr int Q_BYTES = kBtRows * HD * 4;  // one of Q_hi / Q_lo
  static constexpr int K_BYTES = kBtKeys * HD * 4;  // one of K_hi / K_lo / V_hi / V_lo
  static constexpr int SMEM = 2 * Q_BYTES + 4 * K_BYTES + 1024 + 64;
  static constexpr int T_S = 0, T_PH = kBtKeys, T_PL = 2 * kBtKeys, T_O = 3 * kBtKeys;
  static constexpr int TMEM_COLS = (3 * kBtKeys + HD) <= 256 ? 256 : 512;
  static constexpr int F4 = kBtKeys * HD / 4 / kBtThreads;  // float4 per thread per K (or V) tile
  static constexpr uint32_t IDESC_S = umma_idesc(128, kBtKeys, true);
  static constexpr uint32_t IDESC_PV = umma_idesc(128, HD, true);  // B = V^T, K-major
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

template <int HD>
__global__ void __launch_bounds__(kBtThreads) banked_tc_kernel(
    const cc_bank_seq* __restrict__ seqs, const float* __restrict__ q, const float* __restrict__ k_new,
    const float* __restrict__ v_new, int n_q_heads, int n_kv_heads, float factor, int qpb, void* __restrict__ out,
    int out_mode, float* __restrict__ weights_out, int64_t w_col0, int64_t w_ld) {
  using Cfg = BtCfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sQh = smem;
  uint8_t* sQl = sQh + Cfg::Q_BYTES;
  uint8_t* sKh = sQl + Cfg::Q_BYTES;
  uint8_t* sKl = sKh + Cfg::K_BYTES;
  uint8_t* sVh = sKl + Cfg::K_BYTES;
  uint8_t* sVl = sVh + Cfg::K_BYTES;
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(sVl + Cfg::K_BYTES);
  uint64_t* pv_bar = s_bar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_bar + 2);

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
  const int tid = threadIdx.x, warp = tid >> 5;
  const bool want_pv = weights_out == nullptr;

  if (tid == 0) {
    mbar_init(s_bar, 1);
    mbar_init(pv_bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);

  // ---- this thread's packed row: Q -> split hi/lo, swizzled K-major ----
  const int r = tid;
  const bool live = r < nrows;
  const int qi = i0 + (live ? r / G : 0);
  const int head = kvh * G + (live ? r % G : 0);
  const int limit = live ? (int)(nb + qi + 1) : 0;
  {
    const float4* src = reinterpret_cast<const float4*>(q + (sq.row0 + qi) * qw + (int64_t)head * HD);
#pragma unroll
    for (int c4 = 0; c4 < HD / 4; ++c4) {
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
        // V^T [HD dims][32 keys], K-major (one 128-byte block of keys per dim)
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
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);

  uint32_t s_phase = 0, pv_phase = 0;
  float mx = -INFINITY, sum = 0.f;
  float* wrow = nullptr;
  if (!want_pv && live)
    wrow = weights_out + (((int64_t)blockIdx.z * n_q_heads + head) * sq.n_new + qi) * w_ld - w_col0;

  for (int pass = 0; pass < 3; ++pass) {
    const bool pv = pass == 2 && want_pv;
    fetch(0, pv);
    for (int j = 0; j < n_tiles; ++j) {
      if (pv && j > 0) {  // PV(j-1) still reads V smem and P in TMEM
        mbar_wait(pv_bar, pv_phase);
        pv_phase ^= 1;
      }
      stage(pv);
      fence_proxy_async_bt();
      tc_fence_before();
      __syncthreads();
      tc_fence_after();
      if (tid == 0) {
        const uint32_t q0h = smem_u32(sQh), q0l = smem_u32(sQl), k0h = smem_u32(sKh), k0l = smem_u32(sKl);
#pragma unroll
        for (int k = 0; k < HD / 8; ++k) {
          const uint32_t qo = (k >> 2) * (kBtRows * 128) + (k & 3) * 32;
          const uint32_t ko = (k >> 2) * (kBtKeys * 128) + (k & 3) * 32;
          tc_mma<true>(tmem + Cfg::T_S, umma_desc_sw128(q0h + qo), umma_desc_sw128(k0h + ko), Cfg::IDESC_S,
                       k > 0 ? 1u : 0u);
          tc_mma<true>(tmem + Cfg::T_S, umma_desc_sw128(q0h + qo), umma_desc_sw128(k0l + ko), Cfg::IDESC_S, 1u);
          tc_mma<true>(tmem + Cfg::T_S, umma_desc_sw128(q0l + qo), umma_desc_sw128(k0h + ko), Cfg::IDESC_S, 1u);
        }
        tc_commit(s_bar);
      }
      if (j + 1 < n_tiles) fetch(j + 1, pv);  // in flight during the MMA and the softmax
      mbar_wait(s_bar, s_phase);
      s_phase ^= 1;
      tc_fence_after();
      float s[kBtKeys];
      tmem_ld32(trow + Cfg::T_S, s);
      const int c0 = j * kBtKeys;
      if (pass == 0) {
#pragma unroll
        for (int t = 0; t < kBtKeys; ++t)
          if (c0 + t < limit) mx = fmaxf(mx, __fmul_rn(s[t], factor));
      } else if (pass == 1) {
#pragma unroll
        for (int t = 0; t < kBtKeys; ++t)
          if (c0 + t < limit) sum = __fadd_rn(sum, expf(__fsub_rn(__fmul_rn(s[t], factor), mx)));
      } else {
#pragma unroll
        for (int t = 0; t < kBtKeys; ++t)
          s[t] = c0 + t < limit ? __fdiv_rn(expf(__fsub_rn(__fmul_rn(s[t], factor), mx)), sum) : 0.f;
        if (!pv) {
          if (wrow) {  // last-layer weights over bank columns [w_col0, nb)
#pragma unroll
            for (int t = 0; t < kBtKeys; ++t)
              if (c0 + t >= w_col0 && c0 + t < nb) wrow[c0 + t] = s[t];
          }
        } else {
          float ph[kBtKeys];
#pragma unroll
          for (int t = 0; t < kBtKeys; ++t) {
            float lo;
            split_tf32(s[t], ph[t], lo);
            float l2;
            split_tf32(lo, s[t], l2);
          }
          tmem_st32_f(trow + Cfg::T_PH, ph);
          tmem_st32_f(trow + Cfg::T_PL, s);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          __syncthreads();
          tc_fence_after();
          if (tid == 0) {
            const uint32_t v0h = smem_u32(sVh), v0l = smem_u32(sVl);
#pragma unroll
            for (int k = 0; k < kBtKeys / 8; ++k) {
              const uint64_t bh = umma_desc_sw128(v0h + k * 32), bl = umma_desc_sw128(v0l + k * 32);
              tc_mma_ts_tf32(tmem + Cfg::T_O, tmem + Cfg::T_PH + k * 8, bh, Cfg::IDESC_PV, (j > 0 || k > 0) ? 1u : 0u);
              tc_mma_ts_tf32(tmem + Cfg::T_O, tmem + Cfg::T_PH + k * 8, bl, Cfg::IDESC_PV, 1u);
              tc_mma_ts_tf32(tmem + Cfg::T_O, tmem + Cfg::T_PL + k * 8, bh, Cfg::IDESC_PV, 1u);
            }
            tc_commit(pv_bar);
          }
        }
      }
      if (!pv) {  // the next tile's S MMA overwrites S and K smem: everyone has read S
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
      }
    }
  }

  if (want_pv) {
    mbar_wait(pv_bar, pv_phase);
    tc_fence_after();
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      float o[32];
      tmem_ld32(trow + Cfg::T_O + c * 32, o);
      if (!live) continue;
      const int64_t row = sq.row0 + qi;
      const int64_t col0 = (int64_t)head * HD + c * 32;
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
          reinterpret_cast<float4*>(p)[t] = hi;
          reinterpret_cast<float4*>(p + qw)[t] = hi;
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
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(banked_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, BtCfg<64>::SMEM);
      set = true;
    }
    banked_tc_kernel<64><<<grid, kBtThreads, BtCfg<64>::SMEM, st>>>(seqs_dev, q, k_new, v_new, n_q_heads,
                                                                      n_kv_heads, factor, qpb, out, out_mode,
                                                                      weights_out, w_col0, w_ld);
  } else {
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(banked_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, BtCfg<128>::SMEM);
      set = true;
    }
    banked_tc_kernel<128><<<grid, kBtThreads, BtCfg<128>::SMEM, st>>>(seqs_dev, q, k_new, v_new, n_q_heads,
                                                                        n_kv_heads, factor, qpb, out, out_mode,
                                                                        weights_out, w_col0, w_ld);
  }
  CC_LAUNCH_CHECK("banked_attention_tc");
  return CC_OK;
}
