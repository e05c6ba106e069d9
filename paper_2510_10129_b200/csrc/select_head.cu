// Importance reduction, grouped top-k selection, and the first-token head.
//
// reduce_scores_kernel     selector.py:163-165  (mean over heads, then queries;
//                           in-order fp32 sums and true division, bitwise the
//                           numpy reduction order given the same weights)
// select_topk_windows      selector.py:113-129 + 182-214 (exact stable top-k by
//                           MSB-first radix select on order-preserving keys,
//                           lower index first among equal scores; then the
//                           per-chunk window rule and an ordered compaction)
// lm_head_argmax           model.py:495-503 + cli.py:233 (RMSNorm of the last
//                           row, GEMV over the vocabulary, first-max argmax)
#include "cc_common.cuh"

namespace cc {

__global__ void reduce_scores_kernel(const float* __restrict__ w, int n_heads, int n_query, int64_t w_ld,
                                     const int64_t* __restrict__ chunk_lens, const int64_t* __restrict__ col_off,
                                     float* __restrict__ scores) {
  const int s = blockIdx.y;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= chunk_lens[s]) return;
  const float* base = w + (int64_t)s * n_heads * n_query * w_ld + j;
  float acc_q = 0.f;
  for (int qi = 0; qi < n_query; ++qi) {
    float acc_h = base[(int64_t)qi * w_ld];
    for (int h = 1; h < n_heads; ++h) acc_h = __fadd_rn(acc_h, base[((int64_t)h * n_query + qi) * w_ld]);
    const float mq = __fdiv_rn(acc_h, (float)n_heads);
    acc_q = qi == 0 ? mq : __fadd_rn(acc_q, mq);
  }
  scores[col_off[s] + j] = __fdiv_rn(acc_q, (float)n_query);
}

// ---------------------------------------------------------------------------
constexpr int kSelThreads = 1024;

__device__ __forceinline__ uint32_t order_key(float s) {
  uint32_t u = __float_as_uint(s == 0.f ? 0.f : s);  // -0 == +0 for argsort
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// exclusive block scan of one value per thread; returns (exclusive, total)
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* sh, int64_t& total) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < (kSelThreads / 32) ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    sh[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  const int64_t warp_prefix = warp == 0 ? 0 : sh[warp - 1];
  total = sh[kSelThreads / 32 - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

__global__ void __launch_bounds__(kSelThreads) select_topk_windows_kernel(
    const float* __restrict__ scores, int64_t n, const int64_t* __restrict__ chunk_lens, int n_chunks,
    int64_t n_windows, int64_t budget, int window_len, int threshold, int expand, int64_t index_offset,
    int64_t* __restrict__ out_idx, int64_t* __restrict__ out_count, int32_t* __restrict__ win_selected,
    int32_t* __restrict__ win_kept, uint8_t* __restrict__ cand, int64_t* __restrict__ tok_off,
    int64_t* __restrict__ win_off, int32_t* __restrict__ win_take) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t s_prefix, s_mask;
  __shared__ int64_t s_remaining;
  __shared__ int64_t scan_sh[32];
  const int tid = threadIdx.x;

  // ---- 1. radix select the budget-th largest key ------------------------
  if (tid == 0) {
    s_prefix = 0;
    s_mask = 0;
    s_remaining = budget;
  }
  __syncthreads();
  if (budget > 0) {
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int b = tid; b < 256; b += kSelThreads) hist[b] = 0;
      __syncthreads();
      const uint32_t pre = s_prefix, msk = s_mask;
      for (int64_t i = tid; i < n; i += kSelThreads) {
        const uint32_t k = order_key(scores[i]);
        if ((k & msk) == pre) atomicAdd(&hist[(k >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (tid == 0) {
        int64_t rem = s_remaining;
        int b = 255;
        for (; b > 0; --b) {
          if ((int64_t)hist[b] >= rem) break;
          rem -= hist[b];
        }
        s_prefix = pre | ((uint32_t)b << shift);
        s_mask = msk | (255u << shift);
        s_remaining = rem;  // elements still to take from the == prefix group
      }
      __syncthreads();
    }
  }
  const uint32_t thr = s_prefix;
  const int64_t take_eq = budget > 0 ? s_remaining : 0;

  // ---- 2. candidate flags; equal keys by ascending index ----------------
  const int64_t per = (n + kSelThreads - 1) / kSelThreads;
  const int64_t lo = tid * per, hi = min(n, lo + per);
  int64_t n_eq = 0;
  if (budget > 0)
    for (int64_t i = lo; i < hi; ++i) n_eq += order_key(scores[i]) == thr;
  int64_t tot;
  int64_t eq_rank = block_exclusive_scan(n_eq, scan_sh, tot);
  for (int64_t i = lo; i < hi; ++i) {
    uint8_t c = 0;
    if (budget > 0) {
      const uint32_t k = order_key(scores[i]);
      if (k > thr) c = 1;
      else if (k == thr) c = (eq_rank++ < take_eq) ? 1 : 0;
    }
    cand[i] = c;
  }
  // ---- 3. chunk / window offsets ----------------------------------------
  if (tid == 0) {
    int64_t t = 0, w = 0;
    for (int c = 0; c < n_chunks; ++c) {
      tok_off[c] = t;
      win_off[c] = w;
      t += chunk_lens[c];
      w += (chunk_lens[c] + window_len - 1) / window_len;
    }
    tok_off[n_chunks] = t;
    win_off[n_chunks] = w;
  }
  __syncthreads();
  __threadfence_block();
  // ---- 4. window rule -----------------------------------------------------
  const int64_t wper = (n_windows + kSelThreads - 1) / kSelThreads;
  const int64_t wlo = tid * wper, whi = min(n_windows, wlo + wper);
  int64_t my_take = 0;
  for (int64_t wi = wlo; wi < whi; ++wi) {
    int a = 0, b = n_chunks - 1;
    while (a < b) {
      int mid = (a + b + 1) >> 1;
      if (win_off[mid] <= wi) a = mid; else b = mid - 1;
    }
    const int64_t clen = chunk_lens[a];
    const int64_t ws = (wi - win_off[a]) * window_len;
    const int64_t we = min(ws + window_len, clen);
    const int64_t gs = tok_off[a] + ws, ge = tok_off[a] + we;
    int cnt = 0;
    for (int64_t i = gs; i < ge; ++i) cnt += cand[i];
    const bool partial = (we - ws) < window_len;
    const bool kept = cnt > 0 && (partial || cnt >= threshold);
    win_selected[wi] = cnt;
    win_kept[wi] = kept ? 1 : 0;
    const int take = kept ? (expand ? (int)(ge - gs) : cnt) : 0;
    win_take[wi] = take;
    my_take += take;
  }
  int64_t total;
  int64_t pos = block_exclusive_scan(my_take, scan_sh, total);
  __syncthreads();
  for (int64_t wi = wlo; wi < whi; ++wi) {
    if (!win_take[wi]) continue;
    int a = 0, b = n_chunks - 1;
    while (a < b) {
      int mid = (a + b + 1) >> 1;
      if (win_off[mid] <= wi) a = mid; else b = mid - 1;
    }
    const int64_t ws = (wi - win_off[a]) * window_len;
    const int64_t we = min(ws + window_len, chunk_lens[a]);
    const int64_t gs = tok_off[a] + ws, ge = tok_off[a] + we;
    for (int64_t i = gs; i < ge; ++i)
      if (expand || cand[i]) out_idx[pos++] = i + index_offset;
  }
  if (tid == 0) *out_count = total;
}

// ---------------------------------------------------------------------------
constexpr int kHeadThreads = 256;

__global__ void __launch_bounds__(kHeadThreads) lm_head_kernel(const float* __restrict__ h, const float* __restrict__ gain,
                                                             float eps, int d, const void* __restrict__ W, int dtype,
                                                             int64_t vocab, float* __restrict__ logits,
                                                             unsigned long long* __restrict__ best) {
  extern __shared__ float xs[];
  __shared__ float red[33];
  __shared__ unsigned long long s_best;
  // RMSNorm of the last row (recomputed per CTA: d floats)
  float ss = 0.f;
  for (int j = threadIdx.x; j < d; j += kHeadThreads) {
    const float v = h[j];
    ss = fmaf(v, v, ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = ss;
  if (threadIdx.x == 0) s_best = 0ull;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < kHeadThreads / 32; ++i) t += red[i];
    red[32] = __fsqrt_rn(__fadd_rn(__fdiv_rn(t, (float)d), eps));
  }
  __syncthreads();
  const float r = red[32];
  for (int j = threadIdx.x; j < d; j += kHeadThreads) xs[j] = __fmul_rn(__fdiv_rn(h[j], r), gain[j]);
  __syncthreads();
  // one warp per vocabulary row
  const int64_t row0 = ((int64_t)blockIdx.x * (kHeadThreads / 32) + warp);
  for (int64_t v = row0; v < vocab; v += (int64_t)gridDim.x * (kHeadThreads / 32)) {
    float acc = 0.f;
    if (dtype == CC_BF16) {
      // batches of 8 row segments per lane: all loads of a batch are in flight
      // before the first FMA (one load per lane at a time left HBM at ~0.6)
      const uint4* wr = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(W) + v * d);
      const int n8 = d / 8;
      for (int c0 = lane; c0 < n8; c0 += 32 * 8) {
        uint4 u[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const int c = c0 + 32 * b;
          u[b] = c < n8 ? __ldg(wr + c) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const int c = c0 + 32 * b;
          if (c >= n8) break;
          const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&u[b]);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float2 f = __bfloat1622float2(p[i]);
            acc = fmaf(xs[c * 8 + 2 * i], f.x, acc);
            acc = fmaf(xs[c * 8 + 2 * i + 1], f.y, acc);
          }
        }
      }
    } else {
      const float4* wr = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(W) + v * d);
      for (int c = lane; c < d / 4; c += 32) {
        float4 f = __ldg(wr + c);
        acc = fmaf(xs[c * 4], f.x, acc);
        acc = fmaf(xs[c * 4 + 1], f.y, acc);
        acc = fmaf(xs[c * 4 + 2], f.z, acc);
        acc = fmaf(xs[c * 4 + 3], f.w, acc);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      logits[v] = acc;
      const unsigned long long key = ((unsigned long long)order_key(acc) << 32) | (0xFFFFFFFFull - (uint32_t)v);
      atomicMax(&s_best, key);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(best, s_best);
}

__global__ void argmax_finish_kernel(const unsigned long long* best, int64_t* out) {
  *out = (int64_t)(0xFFFFFFFFull - (*best & 0xFFFFFFFFull));
}

}  // namespace cc

using namespace cc;

// CacheBlend discrepancy (selector.py:280-282): out[r] = ||a[r] - b[r]||_2,
// a the recomputed layer-1 values, b the cached ones (each CC_BF16 or
// CC_F32). One warp per row; each lane sums a fixed strided subset, then a
// fixed xor-tree: deterministic.
__device__ __forceinline__ float ld_any(const void* p, int dtype, int64_t i) {
  return dtype == CC_BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i])
                          : reinterpret_cast<const float*>(p)[i];
}
__global__ void row_l2_diff_kernel(const void* __restrict__ a, int a_dtype, int64_t lda, const void* __restrict__ b,
                                   int b_dtype, int64_t ldb, int64_t n, int width, float* __restrict__ out) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  float acc = 0.f;
  for (int j = lane; j < width; j += 32) {
    const float d = __fsub_rn(ld_any(a, a_dtype, row * lda + j), ld_any(b, b_dtype, row * ldb + j));
    acc = __fmaf_rn(d, d, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[row] = __fsqrt_rn(acc);
}

extern "C" {

int cc_reduce_scores(const float* weights, int32_t n_seqs, int32_t n_heads, int32_t n_query, int64_t w_ld,
                     const int64_t* chunk_lens_dev, const int64_t* col_offset_dev, int64_t max_chunk, float* scores,
                     void* stream) {
  if (n_seqs <= 0 || max_chunk <= 0) return CC_OK;
  CC_CHECK_ARG(n_heads > 0 && n_query > 0, CC_ERR_VALUE, "query must be non-empty");
  dim3 grid((unsigned)((max_chunk + 255) / 256), n_seqs);
  ProfScope ps(as_stream(stream), OP_SCORES, 0);
  reduce_scores_kernel<<<grid, 256, 0, as_stream(stream)>>>(weights, n_heads, n_query, w_ld, chunk_lens_dev,
                                                             col_offset_dev, scores);
  CC_LAUNCH_CHECK("reduce_scores");
  return CC_OK;
}

int cc_row_l2_diff(const void* a, int32_t a_dtype, int64_t lda, const void* b, int32_t b_dtype, int64_t ldb,
                   int64_t n, int32_t width, float* out, void* stream) {
  CC_CHECK_ARG(width > 0 && lda >= width && ldb >= width, CC_ERR_DIMENSION, "bad row width %d", width);
  CC_CHECK_ARG((a_dtype == CC_BF16 || a_dtype == CC_F32) && (b_dtype == CC_BF16 || b_dtype == CC_F32),
               CC_ERR_UNSUPPORTED, "dtypes %d / %d", a_dtype, b_dtype);
  if (n <= 0) return CC_OK;
  ProfScope ps(as_stream(stream), OP_OTHER, 0);
  row_l2_diff_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, as_stream(stream)>>>(a, a_dtype, lda, b, b_dtype,
                                                                                       ldb, n, width, out);
  CC_LAUNCH_CHECK("row_l2_diff");
  return CC_OK;
}

int64_t cc_select_workspace_bytes(int64_t n, int32_t n_chunks) {
  const int64_t windows = n + n_chunks;  // upper bound
  return ((n + 15) / 16) * 16 + 2 * 8 * (int64_t)(n_chunks + 1) + 4 * windows + 64;
}

int cc_select_topk_windows(const float* scores, int64_t n, const int64_t* chunk_lens_dev, int32_t n_chunks,
                           int64_t n_windows, int64_t budget, int32_t window_len, int32_t threshold, int32_t expand,
                           int64_t index_offset, int64_t* out_indices, int64_t* out_count, int32_t* win_selected,
                           int32_t* win_kept, void* workspace, void* stream) {
  CC_CHECK_ARG(n >= 0 && budget >= 0 && budget <= n, CC_ERR_VALUE, "budget %lld outside 0..%lld",
               (long long)budget, (long long)n);
  CC_CHECK_ARG(window_len >= 1 && threshold >= 0 && threshold <= window_len, CC_ERR_VALUE, "bad window rule");
  CC_CHECK_ARG(n_chunks >= 1 && workspace, CC_ERR_VALUE, "need chunks and a workspace");
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  uint8_t* cand = ws;
  int64_t* tok_off = reinterpret_cast<int64_t*>(ws + ((n + 15) / 16) * 16);
  int64_t* win_off = tok_off + (n_chunks + 1);
  int32_t* win_take = reinterpret_cast<int32_t*>(win_off + (n_chunks + 1));
  ProfScope ps(as_stream(stream), OP_SELECT, 0);
  select_topk_windows_kernel<<<1, kSelThreads, 0, as_stream(stream)>>>(
      scores, n, chunk_lens_dev, n_chunks, n_windows, budget, window_len, threshold, expand, index_offset,
      out_indices, out_count, win_selected, win_kept, cand, tok_off, win_off, win_take);
  CC_LAUNCH_CHECK("select_topk_windows");
  return CC_OK;
}

int64_t cc_lm_head_workspace_bytes(int64_t vocab) {
  (void)vocab;
  return 64;
}

int cc_lm_head_argmax(const float* h_row, const float* gain, float eps, int32_t d, const void* lm_head,
                      int32_t dtype, int64_t vocab, float* logits, int64_t* argmax_out, void* workspace,
                      void* stream) {
  CC_CHECK_ARG(d > 0 && d % 8 == 0 && d <= 16384, CC_ERR_UNSUPPORTED, "d_model %d unsupported", d);
  CC_CHECK_ARG(vocab > 0 && vocab < 0xFFFFFFFFll, CC_ERR_DIMENSION, "vocab %lld", (long long)vocab);
  cudaStream_t st = as_stream(stream);
  ProfScope ps(st, OP_HEAD, (double)vocab * d * (dtype == CC_BF16 ? 2 : 4));  // weight bytes read
  unsigned long long* best = reinterpret_cast<unsigned long long*>(workspace);
  cudaMemsetAsync(best, 0, sizeof(unsigned long long), st);
  const int rows_per_block = kHeadThreads / 32;
  int64_t blocks = (vocab + rows_per_block - 1) / rows_per_block;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  const size_t smem = (size_t)d * sizeof(float);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(lm_head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  lm_head_kernel<<<(unsigned)blocks, kHeadThreads, smem, st>>>(h_row, gain, eps, d, lm_head, dtype, vocab, logits,
                                                                best);
  CC_LAUNCH_CHECK("lm_head");
  if (argmax_out) {
    argmax_finish_kernel<<<1, 1, 0, st>>>(best, argmax_out);
    CC_LAUNCH_CHECK("argmax_finish");
  }
  return CC_OK;
}

}  // extern "C"
