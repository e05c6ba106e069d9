// fp32-faithful banked attention of the scoring model.
//
// causal_attention of peek_forward (model.py:568-607 -> tensor_core.py:109-170)
// for many sequences at once: sequence s = one chunk cache (its rotated K/V
// bank of n_bank rows at local positions) plus the query rows, new row i
// seeing bank rows [0, n_bank) and new rows [0, i]. The reference's operation
// order is kept — logits = (q . k) * factor, masked, max-shifted exp, sum,
// true division, then weights @ v — with every product in fp32 FFMA, so the
// last-layer weights that become importance scores (selector.py:157-165)
// differ from numpy's only by fp32 rounding order.
//
// One CTA = one sequence x one KV head x up to 8 query rows, with all G query
// heads of that KV head packed as rows (the K/V tiles are read once for all
// of them). Logits live transposed in shared memory, S^T[col][row], so both
// matrix products run as 4x4 register micro-tiles fed by float4 smem loads.
#include "cc_common.cuh"

namespace cc {

constexpr int kBkRows = 64;    // packed rows per CTA (query rows x G heads)
constexpr int kBkKeys = 64;    // keys per K/V tile
constexpr int kBkThreads = 256;

template <int HD>
__global__ void __launch_bounds__(kBkThreads) banked_f32_kernel(
    const cc_bank_seq* __restrict__ seqs, const float* __restrict__ q, const float* __restrict__ k_new,
    const float* __restrict__ v_new, int n_q_heads, int n_kv_heads, float factor, int qpb, int ncols_cap,
    void* __restrict__ out, int out_mode, float* __restrict__ weights_out, int64_t w_col0, int64_t w_ld) {
  extern __shared__ __align__(16) float fsm[];
  const cc_bank_seq sq = seqs[blockIdx.z];
  const int kvh = blockIdx.y;
  const int G = n_q_heads / n_kv_heads;
  const int i0 = blockIdx.x * qpb;  // first query row of this CTA
  if (i0 >= sq.n_new) return;
  const int nq = min(qpb, (int)(sq.n_new - i0));
  const int nrows = nq * G;          // packed row r -> query i0 + r / G, head kvh*G + r % G
  const int64_t nb = sq.n_bank;
  const int ncols = (int)(nb + i0 + nq);
  const int64_t qw = (int64_t)n_q_heads * HD, kvw = (int64_t)n_kv_heads * HD;

  float* sT = fsm;                                  // S^T [ncols_cap][64]
  float* qT = sT + (size_t)ncols_cap * kBkRows;     // Q^T [HD][64]
  float* tile = qT + HD * kBkRows;                  // K^T [HD][64] or V [64][HD]
  const int tid = threadIdx.x;

  // Q^T (rows beyond nrows are zero)
  for (int idx = tid; idx < kBkRows * HD; idx += kBkThreads) {
    const int r = idx / HD, d = idx % HD;
    float v = 0.f;
    if (r < nrows) {
      const int64_t row = sq.row0 + i0 + r / G;
      v = q[row * qw + (int64_t)(kvh * G + r % G) * HD + d];
    }
    qT[d * kBkRows + r] = v;
  }

  auto kv_row = [&](const float* bank, const float* fresh, int64_t col) -> const float* {
    return col < nb ? bank + col * kvw + (int64_t)kvh * HD : fresh + (sq.row0 + (col - nb)) * kvw + (int64_t)kvh * HD;
  };
  const int tr = tid / 16, tc = tid % 16;  // 16 x 16 threads, 4 x 4 micro-tiles

  // Tiles are register double-buffered: the next tile's loads are in flight
  // while the current one is consumed from shared memory.
  constexpr int LPT = kBkKeys * (HD / 4) / kBkThreads;  // float4 per thread per tile
  float4 pre[LPT];
  auto fetch_k = [&](int c0) {
    const int nk = min(kBkKeys, ncols - c0);
#pragma unroll
    for (int e = 0; e < LPT; ++e) {
      const int idx = tid + e * kBkThreads;
      const int kk = idx % kBkKeys, d4 = idx / kBkKeys;
      pre[e] = kk < nk ? *reinterpret_cast<const float4*>(kv_row(sq.k, k_new, c0 + kk) + 4 * d4)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto fetch_v = [&](int c0) {
    const int nk = min(kBkKeys, ncols - c0);
#pragma unroll
    for (int e = 0; e < LPT; ++e) {
      const int idx = tid + e * kBkThreads;
      const int kk = idx / (HD / 4), d4 = idx % (HD / 4);
      pre[e] = kk < nk ? *reinterpret_cast<const float4*>(kv_row(sq.v, v_new, c0 + kk) + 4 * d4)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };

  // ---- phase 1: S^T = (K Q^T) * factor, masked (limit of row r = nb + i + 1)
  fetch_k(0);
  for (int c0 = 0; c0 < ncols; c0 += kBkKeys) {
    const int nk = min(kBkKeys, ncols - c0);
    __syncthreads();
#pragma unroll
    for (int e = 0; e < LPT; ++e) {
      const int idx = tid + e * kBkThreads;
      const int kk = idx % kBkKeys, d4 = idx / kBkKeys;
      tile[(4 * d4 + 0) * kBkKeys + kk] = pre[e].x;
      tile[(4 * d4 + 1) * kBkKeys + kk] = pre[e].y;
      tile[(4 * d4 + 2) * kBkKeys + kk] = pre[e].z;
      tile[(4 * d4 + 3) * kBkKeys + kk] = pre[e].w;
    }
    __syncthreads();
    if (c0 + kBkKeys < ncols) fetch_k(c0 + kBkKeys);
    float acc[4][4] = {};
#pragma unroll 8
    for (int d = 0; d < HD; ++d) {
      const float4 a = *reinterpret_cast<const float4*>(qT + d * kBkRows + 4 * tr);
      const float4 b = *reinterpret_cast<const float4*>(tile + d * kBkKeys + 4 * tc);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int kk = 4 * tc + j;
      if (kk >= nk) continue;
      const int col = c0 + kk;
      float o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = 4 * tr + i;
        const int limit = (int)(nb + i0 + r / G + 1);
        o[i] = col < limit ? __fmul_rn(acc[i][j], factor) : -INFINITY;
      }
      *reinterpret_cast<float4*>(sT + (size_t)col * kBkRows + 4 * tr) = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
  __syncthreads();

  if (!weights_out) fetch_v(0);  // first V tile in flight during the softmax

  // ---- phase 2: softmax per row (tensor_core.py:88-96): 4 threads per row,
  // columns interleaved, partial max / sum combined with quad shuffles -------
  {
    const int r = tid >> 2, part = tid & 3;  // 64 rows x 4 parts = 256 threads
    const bool live = r < nrows;
    const int limit = live ? (int)(nb + i0 + r / G + 1) : 0;
    float mx = -INFINITY;
    for (int c = part; c < limit; c += 4) mx = fmaxf(mx, sT[(size_t)c * kBkRows + r]);
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    float sum = 0.f;
    for (int c = part; c < limit; c += 4) {
      const float e = expf(__fsub_rn(sT[(size_t)c * kBkRows + r], mx));
      sT[(size_t)c * kBkRows + r] = e;
      sum = __fadd_rn(sum, e);
    }
    sum = __fadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, 1));
    sum = __fadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, 2));
    for (int c = part; c < ncols; c += 4) {
      float* p = sT + (size_t)c * kBkRows + r;
      *p = c < limit ? __fdiv_rn(*p, sum) : 0.f;
    }
  }
  if (weights_out) {  // last-layer map over bank columns [w_col0, nb): warp per row, coalesced stores
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31;
    for (int r = warp; r < nrows; r += kBkThreads / 32) {
      const int i = i0 + r / G, head = kvh * G + r % G;
      float* dst = weights_out + ((((int64_t)blockIdx.z * n_q_heads + head) * sq.n_new) + i) * w_ld;
      for (int64_t c = w_col0 + lane; c < nb; c += 32) dst[c - w_col0] = sT[(size_t)c * kBkRows + r];
    }
    return;
  }
  __syncthreads();

  // ---- phase 3: context = weights @ V (4 rows x 4*HD/64 dims per thread) ----
  constexpr int DPT = HD / 16;  // dims per thread
  float acc[4][DPT] = {};
  for (int c0 = 0; c0 < ncols; c0 += kBkKeys) {
    const int nk = min(kBkKeys, ncols - c0);
    __syncthreads();
#pragma unroll
    for (int e = 0; e < LPT; ++e) {
      const int idx = tid + e * kBkThreads;
      const int kk = idx / (HD / 4), d4 = idx % (HD / 4);
      *reinterpret_cast<float4*>(tile + kk * HD + 4 * d4) = pre[e];
    }
    __syncthreads();
    if (c0 + kBkKeys < ncols) fetch_v(c0 + kBkKeys);
    for (int kk = 0; kk < nk; ++kk) {
      const float4 w = *reinterpret_cast<const float4*>(sT + (size_t)(c0 + kk) * kBkRows + 4 * tr);
      const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int dq = 0; dq < DPT / 4; ++dq) {
        const float4 b = *reinterpret_cast<const float4*>(tile + kk * HD + 4 * (tc + 16 * dq));
        const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][4 * dq + j] = fmaf(wv[i], bv[j], acc[i][4 * dq + j]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = 4 * tr + i;
    if (r >= nrows) continue;
    const int64_t row = sq.row0 + i0 + r / G;
    const int head = kvh * G + r % G;
#pragma unroll
    for (int dq = 0; dq < DPT / 4; ++dq) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t col = (int64_t)head * HD + 4 * (tc + 16 * dq) + j;
        const float v = acc[i][4 * dq + j];
        if (out_mode == CC_F32) {
          reinterpret_cast<float*>(out)[row * qw + col] = v;
        } else {
          float hi, lo, lh, ll;
          split_tf32(v, hi, lo);
          split_tf32(lo, lh, ll);
          float* p = reinterpret_cast<float*>(out) + row * qw * 3;
          p[col] = hi;  // (middle hi copy unread by the 3xTF32 GEMM)
          p[2 * qw + col] = lh;
        }
      }
    }
  }
}

}  // namespace cc

using namespace cc;

extern "C" int cc_banked_attention_simt(const cc_bank_seq* seqs_dev, int32_t n_seqs, int32_t max_new,
                                       int64_t max_bank, const float* q, const float* k_new, const float* v_new,
                                       int32_t n_q_heads, int32_t n_kv_heads, int32_t head_dim, float factor,
                                       void* out, int32_t out_mode, float* weights_out, int64_t w_col0,
                                       int64_t w_ld, void* stream) {
  CC_CHECK_ARG(n_kv_heads > 0 && n_q_heads % n_kv_heads == 0, CC_ERR_DIMENSION, "bad head counts");
  CC_CHECK_ARG(head_dim == 64 || head_dim == 128, CC_ERR_UNSUPPORTED, "head_dim %d unsupported", head_dim);
  CC_CHECK_ARG(out_mode == CC_F32 || out_mode == CC_F32_SPLIT3, CC_ERR_UNSUPPORTED, "out mode");
  const int G = n_q_heads / n_kv_heads;
  CC_CHECK_ARG(G <= kBkRows, CC_ERR_UNSUPPORTED, "GQA group %d > %d", G, kBkRows);
  if (n_seqs <= 0 || max_new <= 0) return CC_OK;
  const int qpb = kBkRows / G < 8 ? kBkRows / G : 8;
  const int64_t ncols_cap = ((max_bank + max_new + 3) / 4) * 4;
  const size_t smem = ((size_t)ncols_cap * kBkRows + 2 * (size_t)head_dim * kBkRows) * sizeof(float);
  CC_CHECK_ARG(smem <= 227 * 1024, CC_ERR_UNSUPPORTED, "banked attention: %lld columns exceed shared memory",
               (long long)(max_bank + max_new));
  dim3 grid((max_new + qpb - 1) / qpb, n_kv_heads, n_seqs);
  cudaStream_t st = as_stream(stream);
  ProfScope ps(st, OP_OTHER, 0);
  if (head_dim == 64) {
    cudaFuncSetAttribute(banked_f32_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    banked_f32_kernel<64><<<grid, kBkThreads, smem, st>>>(seqs_dev, q, k_new, v_new, n_q_heads, n_kv_heads, factor,
                                                          qpb, (int)ncols_cap, out, out_mode, weights_out, w_col0,
                                                          w_ld);
  } else {
    cudaFuncSetAttribute(banked_f32_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    banked_f32_kernel<128><<<grid, kBkThreads, smem, st>>>(seqs_dev, q, k_new, v_new, n_q_heads, n_kv_heads,
                                                           factor, qpb, (int)ncols_cap, out, out_mode, weights_out,
                                                           w_col0, w_ld);
  }
  CC_LAUNCH_CHECK("banked_attention_f32");
  return CC_OK;
}
