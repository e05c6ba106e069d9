// Native layer executor: the per-layer loops of selective_forward /
// extend_cache / prefill_full (model.py:506-728) and of the scoring model's
// peek_forward (model.py:568-607), driven from C++ so a 28-layer pass is one
// C-ABI call instead of ~250 Python-side launches. Every launch goes through
// the same C-ABI entry points (cc_gemm, cc_sparse_row_attention, ...), so the
// validation, error codes and the launch profiler are shared.
#include "cc_common.cuh"

#include <algorithm>
#include <cstdint>
#include <vector>

extern thread_local double g_attn_flops;

namespace cc {

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Carve {
  uint8_t* base;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    T* p = reinterpret_cast<T*>(base + off);
    off = align256(off + count * sizeof(T));
    return p;
  }
};

// Rows of split-KV partials a pass of R rows needs: the full-layer launches
// (R rows, small grids) and the last layer's single head row, each at the
// largest split count any key count can ask for.
static int64_t split_part_rows(const cc_model_desc* md, int64_t R) {
  const int64_t a = cc_attention_splits(R, md->n_heads, md->n_kv_heads, INT64_MAX);
  const int64_t b = cc_attention_splits(1, md->n_heads, md->n_kv_heads, INT64_MAX);
  return std::max<int64_t>(a > 1 ? a * R : 0, b > 1 ? b : 0);
}

static size_t rows_ws_bytes(const cc_model_desc* md, int64_t R) {
  const size_t d = md->d_model, qw = (size_t)md->n_heads * md->head_dim, ff = md->d_ff;
  size_t s = 0;
  s += align256(R * d * 4);          // h
  s += align256(R * d * 2);          // x
  s += align256(R * qw * 2);         // q
  s += align256(R * qw * 2);         // ctx
  s += align256(R * ff * 2);         // act
  s += 2 * align256(R * (md->head_dim / 2) * 4);  // cos, sin
  s += align256(64);                 // head workspace
  s += align256((size_t)((d + 31) / 32) * R * 4);  // fused RMSNorm partial sums
  s += align256((size_t)R * 4);                     // and 1/rms per row
  // split-KV partials (small grids: decode, low ratios, the last layer's head row)
  const int64_t pr = split_part_rows(md, R);
  if (pr > 0) {
    s += align256((size_t)pr * qw * 4);
    s += align256((size_t)pr * md->n_heads * 4);
  }
  return s;
}

static size_t banked_ws_bytes(const cc_model_desc* md, int64_t R) {
  const size_t d = md->d_model, qw = (size_t)md->n_heads * md->head_dim, kw = (size_t)md->n_kv_heads * md->head_dim,
               ff = md->d_ff;
  size_t s = 0;
  s += align256(R * d * 4);       // h
  s += align256(R * 3 * d * 4);   // x split
  s += align256(R * qw * 4);      // q
  s += align256(R * kw * 4);      // k new
  s += align256(R * kw * 4);      // v scratch
  s += align256(R * 3 * qw * 4);  // ctx split
  s += align256(R * 3 * ff * 4);  // act split
  s += 2 * align256(R * (md->head_dim / 2) * 4);
  return s;
}

static int gemm_call(int kind, int epi, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, const void* B,
                     int64_t ldb, const float* bias, void* C, int64_t ldc, int c_mode, int act, int64_t n_out,
                     void* stream) {
  cc_gemm_args a{};
  a.kind = kind;
  a.epilogue = epi;
  a.M = M;
  a.N = N;
  a.K = K;
  a.A = A;
  a.lda = lda;
  a.B = B;
  a.ldb = ldb;
  a.bias = bias;
  a.C = C;
  a.ldc = ldc;
  a.c_mode = c_mode;
  a.act = act;
  a.glu_block = 128;
  a.n_out = n_out;
  return cc_gemm(&a, stream);
}

#define CC_TRY(x)          \
  do {                     \
    int rc_ = (x);         \
    if (rc_) return rc_;   \
  } while (0)

// Fused RMSNorm (bf16 pass): the residual epilogue that writes h also writes
// the next GEMM's operand bf16(h * gain) and per-row partial sums of h^2; the
// consumer's epilogue scales rows by 1/rms. CC_FUSED_NORM=0: standalone
// RMSNorm launches (A/B runs).
struct NormFuse {
  void* xn;         // bf16 [rows][d], row-aligned with h
  float* ssq;       // [d/32][ld]
  float* inv;       // [ld]: 1/rms per row (cc_norm_finalize)
  int64_t ld;       // rows of the pass
  int parts, d;
  float eps;
};

static bool fused_norm_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("CC_FUSED_NORM");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

static void norm_produce(cc_gemm_args& a, const NormFuse& nf, int64_t r0, const float* gain) {
  a.xn_out = (uint8_t*)nf.xn + (size_t)r0 * nf.d * 2;
  a.ldxn = nf.d;
  a.norm_gain = gain;
  a.ssq_out = nf.ssq + r0;
  a.ld_ssq = nf.ld;
}

// point the consumer GEMM at the partials of rows [r0, r0 + n): its epilogue
// forms 1/rms per row (cc_norm_finalize's arithmetic, no separate launch)
static int norm_consume(cc_gemm_args& a, const NormFuse& nf, int64_t r0, int64_t n, void* stream) {
  (void)n;
  (void)stream;
  a.ssq_in = nf.ssq + r0;
  a.n_ssq = nf.parts;
  a.ld_ssq_in = nf.ld;
  a.norm_eps = nf.eps;
  return CC_OK;
}

// gate/up on xn (written by the o-proj epilogue, rows scaled by 1/rms in the
// GLU epilogue) -> down + residual, whose epilogue prepares the next layer's
// QKV operand (next_gain = next layer's attn_norm; NULL after the last layer)
static int run_mlp_fused(const cc_model_desc* md, const cc_layer_weights& lw, float* h, void* act, int64_t R,
                         int64_t r0, const NormFuse& nf, const float* next_gain, void* stream) {
  const int64_t d = md->d_model, ff = md->d_ff;
  cc_gemm_args a{};
  a.kind = CC_GEMM_BF16;
  a.M = R;
  a.K = d;
  a.A = (uint8_t*)nf.xn + (size_t)r0 * d * 2;
  a.lda = d;
  a.B = lw.w_up;
  a.ldb = d;
  a.bias = lw.b_up;
  a.C = act;
  a.ldc = ff;
  a.c_mode = CC_BF16;
  a.act = md->act;
  a.glu_block = 128;
  if (md->mlp_gated) {
    a.epilogue = CC_EPI_GLU;
    a.N = lw.n_up;
    a.n_out = ff;
  } else {
    a.epilogue = CC_EPI_ACT;
    a.N = ff;
  }
  if (!md->mlp_gated) return fail(CC_ERR_UNSUPPORTED, "fused RMSNorm needs the gated MLP");
  CC_TRY(norm_consume(a, nf, r0, R, stream));
  CC_TRY(cc_gemm(&a, stream));
  cc_gemm_args b{};
  b.kind = CC_GEMM_BF16;
  b.epilogue = CC_EPI_RESIDUAL;
  b.M = R;
  b.N = d;
  b.K = ff;
  b.A = act;
  b.lda = ff;
  b.B = lw.w_down;
  b.ldb = ff;
  b.bias = lw.b_down;
  b.C = h;
  b.ldc = d;
  b.c_mode = CC_F32;
  if (next_gain) norm_produce(b, nf, r0, next_gain);
  return cc_gemm(&b, stream);
}

// RMSNorm -> gate/up (fused activation) -> down + residual
static int run_mlp(const cc_model_desc* md, const cc_layer_weights& lw, float* h, void* x, void* act, int64_t R,
                   int kind, int x_mode, void* stream) {
  const int64_t d = md->d_model, ff = md->d_ff;
  const int64_t kmul = kind == CC_GEMM_TF32X3 ? 3 : 1;
  CC_TRY(cc_rmsnorm(h, R, (int)d, d, lw.mlp_norm, md->norm_eps, x, x_mode, stream));
  if (md->mlp_gated) {
    CC_TRY(gemm_call(kind, CC_EPI_GLU, R, lw.n_up, d, x, kmul * d, lw.w_up, kmul * d, lw.b_up, act, ff, x_mode,
                     md->act, ff, stream));
  } else {
    CC_TRY(gemm_call(kind, CC_EPI_ACT, R, ff, d, x, kmul * d, lw.w_up, kmul * d, lw.b_up, act, ff, x_mode, md->act, 0,
                     stream));
  }
  return gemm_call(kind, CC_EPI_RESIDUAL, R, d, ff, act, kmul * ff, lw.w_down, kmul * ff, lw.b_down, h, d, CC_F32, 0,
                   0, stream);
}

}  // namespace cc

using namespace cc;

extern "C" {

int cc_fused_norm(void) { return fused_norm_enabled() ? 1 : 0; }

int64_t cc_forward_rows_workspace_bytes(const cc_model_desc* md, int64_t rows) {
  return (int64_t)rows_ws_bytes(md, rows);
}

int64_t cc_forward_banked_workspace_bytes(const cc_model_desc* md, int64_t rows) {
  return (int64_t)banked_ws_bytes(md, rows);
}

int cc_forward_rows(const cc_model_desc* md, const int64_t* ids, const int64_t* positions, int64_t R,
                    const cc_kv_plan* plan, int64_t n_keys, double attn_pairs, const float* row_factor,
                    int64_t tail_rows, void* workspace, float* logits, int64_t* argmax, void* stream) {
  CC_CHECK_ARG(md && plan && workspace, CC_ERR_VALUE, "null model / plan / workspace");
  CC_CHECK_ARG(md->dtype == CC_BF16, CC_ERR_UNSUPPORTED, "cc_forward_rows runs bf16 models");
  CC_CHECK_ARG(tail_rows == R || tail_rows == 1 || tail_rows == 0, CC_ERR_VALUE,
               "tail_rows must be 0, 1 or rows (got %lld)", (long long)tail_rows);
  CC_CHECK_ARG(!logits || tail_rows >= 1, CC_ERR_VALUE, "logits need the last row's final state (tail_rows >= 1)");
  if (R <= 0) return CC_OK;
  const int64_t d = md->d_model, qw = (int64_t)md->n_heads * md->head_dim;
  const int64_t kw = (int64_t)md->n_kv_heads * md->head_dim;
  Carve cv{reinterpret_cast<uint8_t*>(workspace)};
  float* h = cv.take<float>(R * d);
  __nv_bfloat16* x = cv.take<__nv_bfloat16>(R * d);
  __nv_bfloat16* q = cv.take<__nv_bfloat16>(R * qw);
  __nv_bfloat16* ctx = cv.take<__nv_bfloat16>(R * qw);
  __nv_bfloat16* act = cv.take<__nv_bfloat16>(R * md->d_ff);
  float* cs = cv.take<float>(R * (md->head_dim / 2));
  float* sn = cv.take<float>(R * (md->head_dim / 2));
  void* hws = cv.take<uint8_t>(64);
  float* ssq = cv.take<float>((size_t)((d + 31) / 32) * R);
  float* inv_rms = cv.take<float>((size_t)R);
  const bool fuse = fused_norm_enabled() && d % 32 == 0 && md->mlp_gated;
  const NormFuse nf{x, ssq, inv_rms, R, (int)(d / 32), (int)d, md->norm_eps};
  const int64_t part_rows = split_part_rows(md, R);
  float* o_parts = part_rows > 0 ? cv.take<float>((size_t)part_rows * qw) : nullptr;
  float* lse_parts = part_rows > 0 ? cv.take<float>((size_t)part_rows * md->n_heads) : nullptr;
  CC_TRY(cc_rope_table(positions, R, md->inv_freq, md->head_dim, cs, sn, stream));
  const float factor = (float)(1.0 / sqrt((double)md->head_dim));  // np.float32(1/sqrt(d))
  auto lp = [](const void* base, int64_t stride, int l) -> void* {
    return base ? (void*)((const uint8_t*)base + stride * l) : nullptr;
  };
  for (int l = 0; l < md->n_layers; ++l) {
    const cc_layer_weights& lw = md->layers[l];
    if (plan->layer_ready && plan->layer_ready[l]) {
      const cudaError_t e = cudaStreamWaitEvent(as_stream(stream), (cudaEvent_t)plan->layer_ready[l], 0);
      if (e != cudaSuccess) return fail(CC_ERR_CUDA, "cudaStreamWaitEvent: %s", cudaGetErrorString(e));
    }
    if (l == 0)
      CC_TRY(cc_embed_rmsnorm(ids, R, md->embed, CC_BF16, md->vocab, (int)d, h, lw.attn_norm, md->norm_eps, x,
                              CC_BF16, stream));
    else if (!fuse)
      CC_TRY(cc_rmsnorm(h, R, (int)d, d, lw.attn_norm, md->norm_eps, x, CC_BF16, stream));
    cc_gemm_args a{};
    a.kind = CC_GEMM_BF16;
    a.epilogue = CC_EPI_QKV_ROPE;
    a.M = R;
    a.N = lw.n_qkv;
    a.K = d;
    a.A = x;
    a.lda = d;
    a.B = lw.w_qkv;
    a.ldb = d;
    a.bias = lw.b_qkv;
    a.n_q_heads = md->n_heads;
    a.n_kv_heads = md->n_kv_heads;
    a.head_dim = md->head_dim;
    a.rope_cos = cs;
    a.rope_sin = sn;
    a.q_out = q;
    a.ldq = qw;
    a.q_mode = CC_BF16;
    a.k_cache = lp(plan->k_scatter, plan->k_scatter_stride, l);
    a.v_cache = lp(plan->v_scatter, plan->v_scatter_stride, l);
    a.cache_dtype = CC_BF16;
    a.dst_rows = plan->dst_rows;
    a.k_raw = lp(plan->k_raw, plan->k_raw_stride, l);
    a.raw_rows = plan->raw_rows;
    if (fuse && l > 0) CC_TRY(norm_consume(a, nf, 0, R, stream));  // x = bf16(h * attn_norm), previous down
    CC_TRY(cc_gemm(&a, stream));
    // Last layer: every row's K/V are in the cache now (the QKV epilogue
    // scattered them); its attention output, o-proj and MLP feed nothing but
    // the final state of the rows the caller reads (tail_rows: the head's last
    // row, all rows, or none), so only those rows continue.
    const int64_t r0 = (l == md->n_layers - 1) ? R - tail_rows : 0;
    const int64_t Rl = R - r0;
    if (Rl > 0) {
      // profiler work: the full layer's pairs (-1 = known only after the
      // selection read-back, filled in by cc_profile_fill_work); a last-layer
      // tail launch runs only the final row, which sees the whole bank
      g_attn_flops = 4.0 * md->n_heads * md->head_dim * (r0 == 0 ? attn_pairs : (double)n_keys * Rl);
      // never more part rows than the workspace holds
      const int n_splits =
          o_parts ? (int)std::max<int64_t>(1, std::min<int64_t>(cc_attention_splits(Rl, md->n_heads,
                                                                                     md->n_kv_heads, n_keys),
                                                                 part_rows / Rl))
                  : 1;
      CC_TRY(cc_sparse_row_attention_split(q + r0 * qw, qw, positions + r0,
                                           plan->key_start ? plan->key_start + r0 : nullptr, Rl,
                                           lp(plan->attn_k, plan->attn_k_stride, l),
                                           lp(plan->attn_v, plan->attn_v_stride, l), n_keys, md->n_heads,
                                           md->n_kv_heads, md->head_dim, factor,
                                           row_factor ? row_factor + r0 : nullptr, n_splits, o_parts, lse_parts,
                                           ctx + r0 * qw, qw, stream));
      g_attn_flops = 0.0;
      if (fuse) {
        cc_gemm_args o{};
        o.kind = CC_GEMM_BF16;
        o.epilogue = CC_EPI_RESIDUAL;
        o.M = Rl;
        o.N = d;
        o.K = qw;
        o.A = ctx + r0 * qw;
        o.lda = qw;
        o.B = lw.w_o;
        o.ldb = qw;
        o.bias = lw.b_o;
        o.C = h + r0 * d;
        o.ldc = d;
        o.c_mode = CC_F32;
        norm_produce(o, nf, r0, lw.mlp_norm);
        CC_TRY(cc_gemm(&o, stream));
        const float* next_gain = l + 1 < md->n_layers ? md->layers[l + 1].attn_norm : nullptr;
        CC_TRY(run_mlp_fused(md, lw, h + r0 * d, act, Rl, r0, nf, next_gain, stream));
      } else {
        CC_TRY(gemm_call(CC_GEMM_BF16, CC_EPI_RESIDUAL, Rl, d, qw, ctx + r0 * qw, qw, lw.w_o, qw, lw.b_o, h + r0 * d,
                         d, CC_F32, 0, 0, stream));
        CC_TRY(run_mlp(md, lw, h + r0 * d, x, act, Rl, CC_GEMM_BF16, CC_BF16, stream));
      }
    }
  }
  (void)kw;
  if (logits)
    CC_TRY(cc_lm_head_argmax(h + (R - 1) * d, md->final_norm, md->norm_eps, (int)d, md->lm_head, md->head_dtype,
                             md->vocab, logits, argmax, hws, stream));
  return CC_OK;
}

int cc_forward_banked(const cc_model_desc* md, const int64_t* ids, const int64_t* positions, int64_t R,
                      const cc_bank_seq* tables, int32_t n_seqs, int32_t max_new, int64_t max_bank, void* v_dst,
                      int64_t v_dst_stride, void* k_raw_dst, int64_t k_raw_stride, const cc_score_spec* score,
                      void* const* layer_ready, int32_t want_state, void* workspace, void* stream) {
  CC_CHECK_ARG(md && tables && workspace, CC_ERR_VALUE, "null model / tables / workspace");
  CC_CHECK_ARG(md->dtype == CC_F32, CC_ERR_UNSUPPORTED, "cc_forward_banked runs fp32 (3xTF32) models");
  if (R <= 0) return CC_OK;
  const int64_t d = md->d_model, qw = (int64_t)md->n_heads * md->head_dim;
  const int64_t kw = (int64_t)md->n_kv_heads * md->head_dim;
  Carve cv{reinterpret_cast<uint8_t*>(workspace)};
  float* h = cv.take<float>(R * d);
  float* x = cv.take<float>(R * 3 * d);
  float* q = cv.take<float>(R * qw);
  float* k_new = cv.take<float>(R * kw);
  float* v_scr = cv.take<float>(R * kw);
  float* ctx = cv.take<float>(R * 3 * qw);
  float* act = cv.take<float>(R * 3 * md->d_ff);
  float* cs = cv.take<float>(R * (md->head_dim / 2));
  float* sn = cv.take<float>(R * (md->head_dim / 2));
  CC_TRY(cc_rope_table(positions, R, md->inv_freq, md->head_dim, cs, sn, stream));
  const float factor = (float)(1.0 / sqrt((double)md->head_dim));  // np.float32(1/sqrt(d))
  const int L = md->n_layers;
  for (int l = 0; l < L; ++l) {
    const cc_layer_weights& lw = md->layers[l];
    if (layer_ready && layer_ready[l]) {  // this layer's banks still streaming in on another stream
      const cudaError_t e = cudaStreamWaitEvent(as_stream(stream), (cudaEvent_t)layer_ready[l], 0);
      if (e != cudaSuccess) return fail(CC_ERR_CUDA, "cudaStreamWaitEvent: %s", cudaGetErrorString(e));
    }
    if (l == 0)
      CC_TRY(cc_embed_rmsnorm(ids, R, md->embed, CC_F32, md->vocab, (int)d, h, lw.attn_norm, md->norm_eps, x,
                              CC_F32_SPLIT3, stream));
    else
      CC_TRY(cc_rmsnorm(h, R, (int)d, d, lw.attn_norm, md->norm_eps, x, CC_F32_SPLIT3, stream));
    const bool last_scoring = score && l == L - 1;
    float* vd = v_dst ? (float*)((uint8_t*)v_dst + v_dst_stride * l) : v_scr;
    cc_gemm_args a{};
    a.kind = CC_GEMM_TF32X3;
    a.epilogue = CC_EPI_QKV_ROPE;
    a.M = R;
    a.N = last_scoring ? (int64_t)(md->n_heads + md->n_kv_heads) * md->head_dim : lw.n_qkv;
    a.K = d;
    a.A = x;
    a.lda = 3 * d;
    a.B = lw.w_qkv;
    a.ldb = 3 * d;
    a.bias = lw.b_qkv;
    a.n_q_heads = md->n_heads;
    a.n_kv_heads = md->n_kv_heads;
    a.head_dim = md->head_dim;
    a.rope_cos = cs;
    a.rope_sin = sn;
    a.q_out = q;
    a.ldq = qw;
    a.q_mode = CC_F32;
    a.k_cache = k_new;
    a.v_cache = vd;
    a.cache_dtype = CC_F32;
    a.k_raw = k_raw_dst ? (void*)((uint8_t*)k_raw_dst + k_raw_stride * l) : nullptr;
    CC_TRY(cc_gemm(&a, stream));
    const cc_bank_seq* tl = tables + (int64_t)l * n_seqs;
    if (last_scoring) {
      CC_TRY(cc_banked_attention_f32(tl, n_seqs, max_new, max_bank, q, k_new, vd, md->n_heads, md->n_kv_heads,
                                     md->head_dim, factor, ctx, CC_F32_SPLIT3, score->weights, score->col0,
                                     score->max_chunk, stream));
      return cc_reduce_scores(score->weights, n_seqs, md->n_heads, max_new, score->max_chunk, score->chunk_lens,
                              score->col_off, score->max_chunk, score->scores, stream);
    }
    if (l == L - 1 && !want_state) break;  // cache-only prefill: the last layer's K/V are written, nothing reads h
    CC_TRY(cc_banked_attention_f32(tl, n_seqs, max_new, max_bank, q, k_new, vd, md->n_heads, md->n_kv_heads,
                                   md->head_dim, factor, ctx, CC_F32_SPLIT3, nullptr, 0, 0, stream));
    CC_TRY(gemm_call(CC_GEMM_TF32X3, CC_EPI_RESIDUAL, R, d, qw, ctx, 3 * qw, lw.w_o, 3 * qw, lw.b_o, h, d, CC_F32,
                     0, 0, stream));
    CC_TRY(run_mlp(md, lw, h, x, act, R, CC_GEMM_TF32X3, CC_F32_SPLIT3, stream));
  }
  return CC_OK;
}

}  // extern "C"
