/*
 * cacheclip_sm100.h — C-ABI of libcacheclip_sm100.so, the B200 (sm_100a)
 * kernels behind CacheClip's prefill hot path (arxiv 2510.10129).
 *
 * The reference (``cacheclip``, pure Python/numpy) has no FFI; its drop-in
 * boundary is the Python function API (pkg/src/cacheclip/__init__.py:9-133).
 * Each entry point below replaces the numpy body of one reference function;
 * the Python package ``paper_2510_10129_b200`` keeps the reference names and
 * signatures and calls these through ctypes.
 *
 * Conventions (all entry points):
 *   - plain device pointers, element counts / strides as int64, a cudaStream_t
 *     (passed as void*); no torch types, no allocation inside (caller-owned
 *     workspaces), no host synchronisation, stream-ordered and reentrant;
 *   - return 0 on success, otherwise a CC_ERR_* code; the message is
 *     available from cc_last_error() (thread-local). Arguments are validated
 *     before any launch, mirroring the reference's validate-before-mutate rule
 *     (model.py:688-701, kv_store.py:206-225).
 */
#ifndef CACHECLIP_SM100_H_
#define CACHECLIP_SM100_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CC_ABI_VERSION 1

/* status codes -> Python exceptions (paper_2510_10129_b200/_lib.py) */
#define CC_OK 0
#define CC_ERR_VALUE 1       /* ValueError (bad selection, ids, ...)          */
#define CC_ERR_DIMENSION 2   /* DimensionError (tensor_core.py:18)            */
#define CC_ERR_CONSISTENCY 3 /* CacheConsistencyError (kv_store.py:52)        */
#define CC_ERR_CUDA 4        /* RuntimeError: CUDA launch / driver failure    */
#define CC_ERR_UNSUPPORTED 5 /* DimensionError: shape outside kernel support  */

/* element types */
#define CC_F32 0
#define CC_BF16 1
/* activation-operand layout for the 3xTF32 GEMM: row r of a [rows, K] matrix
 * is stored as 3K floats [hi | hi | lo] with hi = tf32(x), lo = x - hi. */
#define CC_F32_SPLIT3 2

/* GEMM kinds */
#define CC_GEMM_BF16 0   /* A, B bf16, fp32 accumulate in TMEM (tcgen05 kind::f16) */
#define CC_GEMM_TF32X3 1 /* A = [hi|hi|lo], B = [hi|lo|hi] along K (kind::tf32)   */

/* GEMM epilogues */
#define CC_EPI_STORE 0    /* C = acc + bias                                      */
#define CC_EPI_RESIDUAL 1 /* H(f32) += acc + bias                                */
#define CC_EPI_GLU 2      /* C = act(gate + bg) * (up + bu), gate/up interleaved */
#define CC_EPI_ACT 3      /* C = act(acc + bias)                                 */
#define CC_EPI_QKV_ROPE 4 /* bias, RoPE q/k per row, q out, K/V scattered        */

#define CC_ACT_SILU 0
#define CC_ACT_GELU_TANH 1

/* Library identity / device check. */
int cc_abi_version(void);
const char* cc_last_error(void);
/* Returns CC_OK when device `dev` is sm_100 (B200) and the kernels load. */
int cc_device_check(int dev);
/* Self-check of the batched SiLU the GLU epilogues use (silu_n, cc_common.cuh)
 * against the per-element x / (1 + exp(-x)) with IEEE division: writes the
 * number of bitwise mismatches over x[0..n) to *mismatches (device int64). */
int cc_check_silu(const float* x, int64_t n, int64_t* mismatches, void* stream);

/* ------------------------------------------------------------------------
 * (1) KV assembly — replaces the per-layer concatenate + rope_apply in
 *     merge_caches (kv_store.py:237-248) and ChunkCache.attention_banks
 *     (kv_store.py:106-116, single segment, local positions).
 *
 * Destination row r (0 <= r < n_dst_rows) is copied from exactly one segment;
 * its key is rotated to position r (+ pos_offset), values pass through.
 * Angles: theta = pos * inv_freq[i] in float64 (inv_freq from the host,
 * computed as base ** (-2i/d) exactly like tensor_core.py:48-50), cos/sin
 * rounded to float32, products separately rounded (bitwise rope_apply).
 * Source/destination layout per tensor: [n_layers][rows][kv_heads][head_dim].
 * ---------------------------------------------------------------------- */
typedef struct {
  const void* k;     /* source keys (position-free), [n_layers][src_rows][H][D] */
  const void* v;     /* source values                                            */
  int64_t src_rows;  /* rows per layer in the source tensors                    */
  int64_t src_row0;  /* first source row copied                                 */
  int64_t dst_row0;  /* first destination row                                   */
  int64_t n_rows;    /* rows in this segment                                    */
  int64_t pos0;      /* RoPE position of the segment's first row (merge: dst_row0;
                        a sequence shard: the chunk's global position)          */
} cc_kv_segment;

int cc_assemble_kv(const cc_kv_segment* segs_dev, int32_t n_segs, int64_t n_dst_rows,
                   int32_t n_layers, int32_t kv_heads, int32_t head_dim, int32_t dtype,
                   const double* inv_freq_host, int64_t pos_offset,
                   void* dst_k, void* dst_v, int64_t dst_rows_cap, void* stream);

/* Small host -> device upload (tables, ids) read by the SMs straight from
 * pinned host memory (src_pinned: a pinned host pointer, 16-byte aligned),
 * stream-ordered. Keeps such uploads off the copy engines, which may be busy
 * with bulk cache DMA (cc_h2d_segments) for tens of milliseconds. */
int cc_upload(void* dst_dev, const void* src_pinned, int64_t bytes, void* stream);

/* Host-resident (pinned) chunk caches, transfer half: copy-engine DMA of
 * layers [layer0, layer0 + n_layers) of every segment (segs_host: a HOST
 * array whose k/v are pinned host pointers) into dst_k / dst_v
 * ([layers][dst_rows_cap][H][D]) at the segments' destination rows, keys still
 * position-free (dst_v = NULL: keys only). One cudaMemcpy2DAsync per
 * (segment, K|V): no SM is occupied
 * by the transfer, so it overlaps scoring and recompute kernels at full PCIe
 * rate. Replaces the per-chunk array reads of merge_caches / attention_banks
 * (kv_store.py:237-248, :106-116) when the caches live in host memory. */
int cc_h2d_segments(const cc_kv_segment* segs_host, int32_t n_segs, int32_t layer0, int32_t n_layers,
                    int32_t kv_heads, int32_t head_dim, int32_t dtype, void* dst_k, void* dst_v,
                    int64_t dst_rows_cap, void* stream);
/* Same transfer for a run of chunks stored at a constant host stride (slots of
 * a layer-major HostCachePool) that land back to back: one cudaMemcpy2DAsync
 * per (layer, K|V) moves `width` bytes of every chunk (rows = chunks, source
 * pitch src_chunk_pitch, destination pitch dst_chunk_pitch), layers
 * [layer0, layer0 + n_layers) at the given layer pitches (dst_v = NULL: keys
 * only). All sizes in bytes; src pointers are pinned host, dst device. */
int cc_h2d_uniform(const void* src_k, const void* src_v, int64_t src_chunk_pitch, int64_t src_layer_pitch,
                   void* dst_k, void* dst_v, int64_t width, int64_t dst_layer_pitch, int64_t dst_chunk_pitch,
                   int32_t n_chunks, int32_t layer0, int32_t n_layers, void* stream);
/* Rotation half: rotate the keys of rows [0, n_rows) in place over n_layers
 * layers (k points at the first layer; layer stride rows_cap rows); row r of
 * the segment containing it (by dst_row0) sits at position pos0 + r - dst_row0.
 * Same float64-angle / separately-rounded arithmetic as cc_assemble_kv. */
int cc_rope_rows_inplace(const cc_kv_segment* segs_dev, int32_t n_segs, int64_t n_rows, int32_t n_layers,
                         int32_t kv_heads, int32_t head_dim, int32_t dtype, const double* inv_freq_host,
                         void* k, int64_t rows_cap, void* stream);

/* Per-row float32 cos/sin tables [n][head_dim/2] for arbitrary positions
 * (float64 angle formation, tensor_core.py:41-51). */
int cc_rope_table(const int64_t* positions, int64_t n, const double* inv_freq_host,
                  int32_t head_dim, float* cos_out, float* sin_out, void* stream);

/* ------------------------------------------------------------------------
 * (2) Embedding gather + RMSNorm — _embed (model.py:484-492) and rms_norm
 *     (tensor_core.py:99-106) feeding attention_qkv / _mlp / _final_logits.
 * h_out (f32 residual stream, may be NULL): h = embed[ids[r]]
 * x_out: rmsnorm(h) * gain in x_mode (CC_BF16 / CC_F32 / CC_F32_SPLIT3).
 * ---------------------------------------------------------------------- */
int cc_embed_rmsnorm(const int64_t* ids, int64_t rows, const void* embed, int32_t embed_dtype,
                     int64_t vocab, int32_t d, float* h_out, const float* gain, float eps,
                     void* x_out, int32_t x_mode, void* stream);
int cc_rmsnorm(const float* h, int64_t rows, int32_t d, int64_t ld_h, const float* gain,
               float eps, void* x_out, int32_t x_mode, void* stream);
/* The fused-RMSNorm operand of cc_gemm_args (xn = bf16(h * gain) and per-32-
 * column partial sums of h^2 at ssq_out[(col/32) * ld_ssq + row]) for rows
 * whose producer GEMM did not emit it, bit-identical to the RESIDUAL
 * epilogue's; d % 32 == 0. */
int cc_norm_prep(const float* h, int64_t rows, int32_t d, int64_t ld_h, const float* gain, void* xn_out,
                 float* ssq_out, int64_t ld_ssq, void* stream);
/* inv_rms[m] = 1 / sqrt((sum over the d/32 partials in order) / d + eps). */
int cc_norm_finalize(const float* ssq, int64_t rows, int32_t d, int64_t ld_ssq, float eps, float* inv_rms,
                     void* stream);
/* 1 when the bf16 layer executor folds RMSNorm into its GEMMs (default; the
 * environment variable CC_FUSED_NORM=0 selects standalone RMSNorm launches). */
int cc_fused_norm(void);
/* Weight preparation: fp32 [rows, cols] -> CC_BF16 or split layout
 * (split_mode 0 = activation [hi|hi|lo], 1 = weight [hi|lo|hi]). */
int cc_convert_matrix(const float* src, int64_t rows, int64_t cols, void* dst, int32_t dst_mode,
                      int32_t split_weight, void* stream);

/* ------------------------------------------------------------------------
 * (3) tcgen05 GEMM with fused epilogues — every x @ W in attention_qkv,
 *     _attn_project_out and _mlp (model.py:340-432). C[M,N] = A[M,K]·B[N,K]^T,
 *     both operands K-major (weights stored transposed, [out, in]).
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t kind;      /* CC_GEMM_BF16 | CC_GEMM_TF32X3                            */
  int32_t epilogue;  /* CC_EPI_*                                                 */
  int64_t M, N, K;   /* logical sizes; operand row width is K (bf16) or 3K      */
  const void* A; int64_t lda;  /* elements                                       */
  const void* B; int64_t ldb;
  const float* bias;           /* [N] (GLU: interleaved like B) or NULL          */
  void* C; int64_t ldc; int32_t c_mode;  /* output (RESIDUAL: f32 H, in place)   */
  int32_t act;                 /* CC_ACT_* for GLU / ACT                          */
  int32_t glu_block;           /* GLU: gate/up interleave block (columns)         */
  int64_t n_out;               /* GLU: valid output columns (d_ff)                */
  /* QKV + RoPE epilogue */
  int32_t n_q_heads, n_kv_heads, head_dim;
  const float* rope_cos; const float* rope_sin;  /* [M][head_dim/2]              */
  void* q_out; int64_t ldq; int32_t q_mode;
  void* k_cache; void* v_cache; int32_t cache_dtype;   /* row = dst_rows[m]      */
  const int64_t* dst_rows;     /* [M] cache row per GEMM row (NULL: identity)    */
  void* k_raw;                 /* optional position-free K (chunk precompute)    */
  const int64_t* raw_rows;     /* [M] row in k_raw (NULL: identity)              */
  /* RMSNorm fused across GEMMs (bf16 kind only; rms_norm, tensor_core.py:99-106):
   * the RESIDUAL epilogue that writes h also writes the next GEMM's A operand
   * xn = bf16(h * norm_gain) and per-row partial sums of h^2, one per 32-column
   * chunk: ssq_out[(col / 32) * ld_ssq + m] (N % 32 == 0); cc_norm_finalize
   * reduces them to inv_rms[m] = 1 / sqrt(sum_p ssq / d + eps). A consumer
   * GEMM (QKV / GLU / STORE / ACT epilogue) given inv_rms scales each
   * accumulator row by it before the bias: (h * g) @ W / rms(h) ==
   * rms_norm(h) @ W. */
  void* xn_out; int64_t ldxn; const float* norm_gain;
  float* ssq_out;
  const float* inv_rms;
  int64_t ld_ssq;
  /* The consumer may instead take the producer's partial sums directly:
   * ssq_in[p * ld_ssq_in + m] for p < n_ssq (d = 32 * n_ssq); its epilogue
   * then forms 1/rms per row itself, with cc_norm_finalize's arithmetic and
   * summation order (bitwise the same scaling, one launch fewer). */
  const float* ssq_in;
  int32_t n_ssq;
  int64_t ld_ssq_in;
  float norm_eps;
} cc_gemm_args;

int cc_gemm(const cc_gemm_args* args, void* stream);

/* ------------------------------------------------------------------------
 * (4) Sparse-row attention — causal_attention(q, bank_k, bank_v,
 *     row_limits=idx+1) in selective_forward (model.py:715-720) and the
 *     mask_offset rule of layer_forward (model.py:467-476). Row i of q
 *     (packed [m][Hq][D], rotated) attends cache rows [0, positions[i]] of
 *     the bf16 bank [rows][Hkv][D]; GQA head h reads KV head h / (Hq/Hkv).
 *     factor = scale/(sqrt(D)*temperature) per row (row_factor, or uniform).
 * ---------------------------------------------------------------------- */
int cc_sparse_row_attention(const void* q, int64_t ldq, const int64_t* positions, int64_t m,
                            const void* k_cache, const void* v_cache, int64_t n_keys,
                            int32_t n_q_heads, int32_t n_kv_heads, int32_t head_dim,
                            float factor, const float* row_factor,
                            void* out, int64_t ldo, void* stream);
/* Same with a per-row first key (key_start NULL: 0): row i attends bank rows
 * [key_start[i], key_start[i] + positions[i]] — many independent sequences
 * in one bank (batched prefill_chunk, model.py:538-565, one pass for all
 * chunks). */
int cc_sparse_row_attention_ranged(const void* q, int64_t ldq, const int64_t* positions,
                                   const int64_t* key_start, int64_t m, const void* k_cache,
                                   const void* v_cache, int64_t n_keys, int32_t n_q_heads,
                                   int32_t n_kv_heads, int32_t head_dim, float factor,
                                   const float* row_factor, void* out, int64_t ldo, void* stream);
/* Split-KV partial attention for sequence-sharded caches:
 * same kernel, but row i attends local keys [0, limits[i]] (limits = local
 * index of its last visible key, -1 = none; cc_local_limits) and writes the
 * locally normalised context o_part[i][Hq][D] (part_dtype CC_F32 or CC_BF16:
 * bf16 halves the all_to_all and merge bytes) plus its log2-domain
 * log-sum-exp lse[i][Hq] (fp32, -inf when no key is visible). */
int cc_sparse_row_attention_partial(const void* q, int64_t ldq, const int64_t* limits, int64_t m,
                                    const void* k_cache, const void* v_cache, int64_t n_keys,
                                    int32_t n_q_heads, int32_t n_kv_heads, int32_t head_dim,
                                    float factor, const float* row_factor, void* o_part, int32_t part_dtype,
                                    float* lse, void* stream);
/* limits[i] = (number of sorted local key positions <= row_pos[i]) - 1. */
int cc_local_limits(const int64_t* row_pos, int64_t m, const int64_t* local_pos, int64_t n_local,
                    int64_t* limits, void* stream);
/* Split-KV attention on ONE GPU for launches of few rows over long key
 * ranges (a decode step, the last layer's head row): each CTA's key tiles
 * are cut into n_splits parts run as separate CTAs (partials in o_parts
 * [n_splits][m][Hq][D] fp32 and lse_parts [n_splits][m][Hq], caller-owned),
 * then merged by log-sum-exp into `out` (bf16). n_splits <= 1 is
 * cc_sparse_row_attention_ranged. */
int cc_sparse_row_attention_split(const void* q, int64_t ldq, const int64_t* positions, const int64_t* key_start,
                                  int64_t m, const void* k_cache, const void* v_cache, int64_t n_keys,
                                  int32_t n_q_heads, int32_t n_kv_heads, int32_t head_dim, float factor,
                                  const float* row_factor, int32_t n_splits, float* o_parts, float* lse_parts,
                                  void* out, int64_t ldo, void* stream);
/* The split count cc_forward_rows uses: > 1 only when the launch's
 * ceil(m * (Hq / Hkv) / 256) * Hkv CTAs are under one wave of the SMs and
 * the keys are >= 4096 (up to 32 parts, at least 1024 keys each); 1
 * otherwise. Inside the kernel a CTA uses one part per 8 key tiles of its
 * own range at most (unused parts report LSE = -inf). */
int32_t cc_attention_splits(int64_t m, int32_t n_q_heads, int32_t n_kv_heads, int64_t n_keys);
/* Log-sum-exp merge of n_parts partial attentions (parts stride
 * part_stride rows): out[i][h*D..] = sum_w 2^(lse_w - M) O_w / sum_w 2^(lse_w - M). */
int cc_lse_merge(const void* o_parts, int32_t part_dtype, const float* lse_parts, int32_t n_parts,
                 int64_t part_stride, int64_t m, int32_t n_q_heads, int32_t head_dim, void* out, int64_t ldo,
                 int32_t out_dtype, void* stream);
/* Same contract on legacy mma.sync tensor cores: the baseline the tcgen05
 * kernel above is measured against (kept for A/B tests and the bench). */
int cc_sparse_row_attention_mma(const void* q, int64_t ldq, const int64_t* positions, int64_t m,
                                const void* k_cache, const void* v_cache, int64_t n_keys,
                                int32_t n_q_heads, int32_t n_kv_heads, int32_t head_dim,
                                float factor, const float* row_factor,
                                void* out, int64_t ldo, void* stream);

/* Float32 banked causal attention (the fp32-faithful aux model path,
 * peek_forward / prefill of the scoring model): for sequence s, new row i
 * (global packed row row0[s] + i, i < n_new[s]) attends the sequence's bank
 * rows [0, n_bank[s]) and new rows [0, i]. out_mode CC_F32 / CC_F32_SPLIT3
 * writes the context; weights_out (optional, replaces the context) receives
 * the softmax weights of bank columns [w_col0, n_bank[s]) as
 * [s][head][i][col - w_col0] with row pitch w_ld (the last-layer scoring map,
 * selector.py:157-165). */
typedef struct {
  const float* k;   /* bank keys (rotated) for this layer, [n_bank][Hkv][D] */
  const float* v;
  int64_t n_bank;
  int64_t row0;     /* first packed new row */
  int64_t n_new;
} cc_bank_seq;

int cc_banked_attention_f32(const cc_bank_seq* seqs_dev, int32_t n_seqs, int32_t max_new,
                            int64_t max_bank, const float* q, const float* k_new,
                            const float* v_new, int32_t n_q_heads, int32_t n_kv_heads,
                            int32_t head_dim, float factor, void* out, int32_t out_mode,
                            float* weights_out, int64_t w_col0, int64_t w_ld, void* stream);
/* The same contract on the FP32 SIMT pipe (4x4 FFMA micro-tiles, logits in
 * shared memory; bank + new rows must fit ~800 columns). cc_banked_attention_f32
 * itself runs on tcgen05 (3xTF32, banked_tc.cu); this one is kept as an
 * independent cross-check of it. */
int cc_banked_attention_simt(const cc_bank_seq* seqs_dev, int32_t n_seqs, int32_t max_new,
                             int64_t max_bank, const float* q, const float* k_new,
                             const float* v_new, int32_t n_q_heads, int32_t n_kv_heads,
                             int32_t head_dim, float factor, void* out, int32_t out_mode,
                             float* weights_out, int64_t w_col0, int64_t w_ld, void* stream);

/* ------------------------------------------------------------------------
 * (5) Importance reduction + grouped top-k — aux_score_tokens' head/query
 *     mean (selector.py:163-165), selection_budget/top_candidates
 *     (selector.py:113-129) and the per-chunk window rule (selector.py:182-214).
 * ---------------------------------------------------------------------- */
/* CacheBlend discrepancy (selector.py:280-282): out[r] = || a[r] - b[r] ||_2
 * over `width` columns; a and b each CC_BF16 or CC_F32 (row pitches lda, ldb). */
int cc_row_l2_diff(const void* a, int32_t a_dtype, int64_t lda, const void* b, int32_t b_dtype, int64_t ldb,
                   int64_t n, int32_t width, float* out, void* stream);
/* weights [n_seqs][H][Q][w_ld] -> scores[col_offset[s] + j], j < chunk_len[s]:
 * in-order sum over heads / H, then in-order sum over queries / Q. */
int cc_reduce_scores(const float* weights, int32_t n_seqs, int32_t n_heads, int32_t n_query,
                     int64_t w_ld, const int64_t* chunk_lens_dev, const int64_t* col_offset_dev,
                     int64_t max_chunk, float* scores, void* stream);

/* Stable top-`budget` of scores (higher first, lower index on ties), then the
 * window rule per chunk. Outputs: out_indices[0..*out_count) ascending
 * (+ index_offset); win_selected / win_kept per window (windows enumerated
 * chunk by chunk, ceil(len/window_len) each). Single CTA; workspace >=
 * cc_select_workspace_bytes(n, n_chunks). */
int64_t cc_select_workspace_bytes(int64_t n, int32_t n_chunks);
int cc_select_topk_windows(const float* scores, int64_t n, const int64_t* chunk_lens_dev,
                           int32_t n_chunks, int64_t n_windows, int64_t budget,
                           int32_t window_len, int32_t threshold, int32_t expand,
                           int64_t index_offset, int64_t* out_indices, int64_t* out_count,
                           int32_t* win_selected, int32_t* win_kept, void* workspace,
                           void* stream);

/* ------------------------------------------------------------------------
 * (6) First token — _final_logits (model.py:495-503) + argmax
 *     (cli.py:233): RMSNorm of the last row, lm_head GEMV, argmax.
 * ---------------------------------------------------------------------- */
int64_t cc_lm_head_workspace_bytes(int64_t vocab);
int cc_lm_head_argmax(const float* h_row, const float* gain, float eps, int32_t d,
                      const void* lm_head, int32_t dtype, int64_t vocab, float* logits,
                      int64_t* argmax_out, void* workspace, void* stream);

/* Row gather for the residual stream (compaction helpers). */
int cc_gather_i64(const int64_t* src, const int64_t* idx, int64_t n, int64_t* dst, void* stream);
/* Rows of the fused selective_forward + extend_cache pass, built on device
 * from the selection kernel's output (no host round trip of the indices):
 * r < m: pos = sel[r], id = token_ids[sel[r]]; m <= r < m+nq: pos = base+r-m,
 * id = query_ids[r-m]. */
int cc_build_rows(const int64_t* sel, int64_t m, const int64_t* token_ids, const int64_t* query_ids, int64_t nq,
                  int64_t base, int64_t* ids_out, int64_t* pos_out, void* stream);

/* ------------------------------------------------------------------------
 * (7) Native layer executor — the per-layer loops of selective_forward,
 *     extend_cache, prefill_full (model.py:506-728) and the scoring model's
 *     peek_forward (model.py:568-607) as one call each. Weights are described
 *     by plain pointers (device layouts documented in weights.py).
 * ---------------------------------------------------------------------- */
typedef struct {
  const void* w_qkv; const float* b_qkv; int64_t n_qkv;  /* [(Hq+2Hkv)*D, d] */
  const void* w_o; const float* b_o;                     /* [d, Hq*D]        */
  const float* attn_norm; const float* mlp_norm;
  const void* w_up; const float* b_up; int64_t n_up;     /* GLU-interleaved or w_in */
  const void* w_down; const float* b_down;               /* [d, d_ff]        */
} cc_layer_weights;

typedef struct {
  int32_t n_layers, n_heads, n_kv_heads, head_dim, d_model, d_ff;
  int64_t vocab;
  int32_t dtype;       /* CC_BF16 (bf16 engine) or CC_F32 (3xTF32 banked engine) */
  int32_t mlp_gated, act;
  float norm_eps;
  const void* embed; const float* final_norm; const void* lm_head; int32_t head_dtype;
  const cc_layer_weights* layers;  /* host array [n_layers] */
  const double* inv_freq;          /* host [head_dim/2], tensor_core.py:48-50 */
} cc_model_desc;

/* Where the QKV epilogue writes K/V and what attention reads, per layer:
 * pointer(l) = base + l * stride (bytes; stride 0 = one shared buffer). */
typedef struct {
  void* k_scatter; int64_t k_scatter_stride;
  void* v_scatter; int64_t v_scatter_stride;
  const int64_t* dst_rows;              /* cache row per input row (NULL: identity) */
  void* k_raw; int64_t k_raw_stride;    /* optional position-free K (precompute)     */
  const int64_t* raw_rows;
  const void* attn_k; int64_t attn_k_stride;
  const void* attn_v; int64_t attn_v_stride;
  void* const* layer_ready;             /* optional host array of cudaEvent_t: layer l's
                                           QKV/attention wait for layer_ready[l] (a merge
                                           still streaming in on another stream) */
  const int64_t* key_start;             /* optional first visible key per row (NULL: 0):
                                           row r sees keys [key_start[r],
                                           key_start[r] + positions[r] + 1) — one bank
                                           holding many independent sequences (batched
                                           chunk precompute) */
} cc_kv_plan;

/* Last-layer scoring (selector.py:157-165): weights workspace
 * [n_seqs][Hq][Q][max_chunk] fp32, scores[col_off[s] + j]. */
typedef struct {
  int64_t col0; const int64_t* chunk_lens; const int64_t* col_off; int64_t max_chunk;
  float* weights; float* scores;
} cc_score_spec;

int64_t cc_forward_rows_workspace_bytes(const cc_model_desc* md, int64_t rows);
int64_t cc_forward_banked_workspace_bytes(const cc_model_desc* md, int64_t rows);
/* bf16 engine: rows (ids, positions) through every layer; logits of the last
 * row + argmax when logits != NULL. attn_pairs = sum of visible keys (for the
 * profiler's algorithmic FLOPs only). tail_rows (0, 1 or rows): how many
 * trailing rows' final states the caller reads. Every row's K/V are written
 * at every layer; in the LAST layer the attention, o-proj and MLP run only
 * for the tail rows (the reference computes them for all rows, but nothing
 * reads them: selective_forward returns the cache, extend_cache the last
 * row's logits). The residual stream stays at the start of the workspace
 * ([rows][d] fp32; after the call only the tail rows hold final states). */
int cc_forward_rows(const cc_model_desc* md, const int64_t* ids, const int64_t* positions, int64_t rows,
                    const cc_kv_plan* plan, int64_t n_keys, double attn_pairs, const float* row_factor,
                    int64_t tail_rows, void* workspace, float* logits, int64_t* argmax, void* stream);
/* fp32 engine over sequences with banks (tables: device cc_bank_seq[n_layers][n_seqs]).
 * layer_ready: optional host array of cudaEvent_t — layer l waits for
 * layer_ready[l] (banks streamed in from pinned host memory on another stream).
 * want_state = 0: the caller reads only the written K/V (cache-only prefill),
 * so the last layer stops after its QKV GEMM. */
int cc_forward_banked(const cc_model_desc* md, const int64_t* ids, const int64_t* positions, int64_t rows,
                      const cc_bank_seq* tables, int32_t n_seqs, int32_t max_new, int64_t max_bank,
                      void* v_dst, int64_t v_dst_stride, void* k_raw_dst, int64_t k_raw_stride,
                      const cc_score_spec* score, void* const* layer_ready, int32_t want_state,
                      void* workspace, void* stream);

/* Launch profiler: CUDA events around every launch while enabled; collect
 * returns (op id, algorithmic work, ms) per launch and clears. op ids:
 * 0 gemm bf16, 1 gemm 3xTF32, 2 attention (tcgen05), 3 attention (mma.sync),
 * 4 banked fp32 attention, 5 rmsnorm, 6 KV assembly, 7 select, 8 score
 * reduction, 9 lm_head, 10 rope table. */
void cc_profile_enable(int32_t on);
int64_t cc_profile_collect(int32_t* ops, double* work, float* ms, int64_t cap);
/* The same records as a timeline: start and end of each launch in ms after
 * the first record's start (idle gaps between launches, stream overlap).
 * Does not clear; call before cc_profile_collect. */
int64_t cc_profile_timeline(int32_t* ops, float* t0_ms, float* t1_ms, int64_t cap);
/* Set the algorithmic work of pending records of `op` launched with an
 * unknown (negative) work: cc_forward_rows with attn_pairs < 0, i.e. launched
 * before the host has read the selected positions. */
void cc_profile_fill_work(int32_t op, double work);

#ifdef __cplusplus
}
#endif

#endif /* CACHECLIP_SM100_H_ */
