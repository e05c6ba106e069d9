"""Layer-by-layer forward engine over device caches (one stream, no host syncs).

Two engines share the kernels of libcacheclip_sm100.so:

``forward_rows``   bf16 models. A set of rows at arbitrary global positions
                   (selected rows, query rows, or a whole prompt) runs every
                   layer: RMSNorm -> QKV GEMM whose epilogue adds bias, rotates
                   q/k and scatters K/V into the cache rows (model.py:708-714)
                   -> sparse-row attention over the cache with limit pos+1
                   (model.py:715-720) -> o-proj GEMM + residual -> RMSNorm ->
                   gate/up GEMM with fused activation -> down GEMM + residual.
                   Rows sharing a layer pass see each other's fresh K/V because
                   the scatter completes before the attention launch (H5).

``forward_banked`` fp32 models (the scoring model). Per sequence a bank of
                   cached rows plus causal new rows (peek_forward over chunk
                   caches, model.py:568-607, or a dense prefill with an empty
                   bank); 3xTF32 GEMMs and fp32 attention. In scoring mode the
                   last layer stops after the attention weights, which are
                   reduced into per-token importance (selector.py:157-165).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch

from . import _lib
from .weights import GLU_BLOCK, Model


def _s() -> int:
    return torch.cuda.current_stream().cuda_stream


def _p(t) -> int | None:
    return None if t is None else t.data_ptr()


def gemm(kind: int, epilogue: int, M: int, N: int, K: int, A: torch.Tensor, B: torch.Tensor, *,
         bias=None, C=None, ldc: int = 0, c_mode: int = _lib.CC_BF16, act: int = 0, n_out: int = 0,
         lda: int | None = None, rope=None, q_out=None, ldq: int = 0, q_mode: int = _lib.CC_BF16,
         k_cache=None, v_cache=None, cache_dtype: int = _lib.CC_BF16, dst_rows=None, k_raw=None,
         raw_rows=None, heads=(0, 0, 0)) -> None:
    a = _lib.GemmArgs()
    a.kind, a.epilogue = kind, epilogue
    a.M, a.N, a.K = M, N, K
    a.A, a.lda = A.data_ptr(), lda if lda is not None else A.shape[-1]
    a.B, a.ldb = B.data_ptr(), B.shape[-1]
    a.bias = _p(bias)
    a.C, a.ldc, a.c_mode = _p(C), ldc, c_mode
    a.act, a.glu_block, a.n_out = act, GLU_BLOCK, n_out
    a.n_q_heads, a.n_kv_heads, a.head_dim = heads
    if rope is not None:
        a.rope_cos, a.rope_sin = rope[0].data_ptr(), rope[1].data_ptr()
    a.q_out, a.ldq, a.q_mode = _p(q_out), ldq, q_mode
    a.k_cache, a.v_cache, a.cache_dtype = _p(k_cache), _p(v_cache), cache_dtype
    a.dst_rows, a.k_raw, a.raw_rows = _p(dst_rows), _p(k_raw), _p(raw_rows)
    _lib.call("cc_gemm", ctypes.byref(a), _s(), meta={"flops": 2.0 * M * N * K, "kind": kind})


def rope_table(model: Model, positions: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    c = model.config
    n = positions.numel()
    cos = torch.empty(n, c.d_head // 2, dtype=torch.float32, device=positions.device)
    sin = torch.empty_like(cos)
    inv = c.rope.inv_freq
    _lib.call("cc_rope_table", positions.data_ptr(), n, inv.ctypes.data, c.d_head, cos.data_ptr(),
              sin.data_ptr(), _s())
    return cos, sin


def _act_code(model: Model) -> int:
    return _lib.CC_ACT_SILU if model.config.activation == "silu" else _lib.CC_ACT_GELU_TANH


def _mlp(model: Model, lw, h: torch.Tensor, x: torch.Tensor, act_buf: torch.Tensor, kind: int,
         x_mode: int) -> None:
    """RMSNorm(h) -> up/gate GEMM (fused activation) -> down GEMM + residual."""
    c = model.config
    R, d = h.shape
    _lib.call("cc_rmsnorm", h.data_ptr(), R, d, d, lw.mlp_norm.data_ptr(), c.norm_eps, x.data_ptr(), x_mode, _s())
    if c.mlp_gated:
        gemm(kind, _lib.CC_EPI_GLU, R, lw.w_up.shape[0], d, x, lw.w_up, bias=lw.b_up, C=act_buf,
             ldc=c.d_ff, c_mode=x_mode, act=_act_code(model), n_out=c.d_ff)
    else:
        gemm(kind, _lib.CC_EPI_ACT, R, c.d_ff, d, x, lw.w_up, bias=lw.b_up, C=act_buf, ldc=c.d_ff,
             c_mode=x_mode, act=_act_code(model))
    gemm(kind, _lib.CC_EPI_RESIDUAL, R, d, c.d_ff, act_buf, lw.w_down, bias=lw.b_down, C=h, ldc=d,
         c_mode=_lib.CC_F32)


@dataclass
class RowsResult:
    h: torch.Tensor                 # final residual stream [R, d] fp32
    logits: torch.Tensor | None     # [V] fp32 (last row)
    argmax: torch.Tensor | None     # [1] int64


def forward_rows(model: Model, ids: torch.Tensor, positions: torch.Tensor,
                 kv: Callable[[int], tuple], n_keys: int, *, row_factor: torch.Tensor | None = None,
                 want_logits: bool = True, logits_out: torch.Tensor | None = None,
                 pairs: int = 0) -> RowsResult:
    """bf16 engine. kv(layer) -> (k_scatter, v_scatter, dst_rows, k_raw, raw_rows,
    attn_k, attn_v): where the QKV epilogue writes and what attention reads."""
    c = model.config
    if c.dtype != "bf16":
        raise ValueError("forward_rows runs bf16 models; fp32 models use forward_banked")
    dev = ids.device
    R, d = ids.numel(), c.d_model
    qw, kvw = c.attn_width, c.kv_width
    h = torch.empty(R, d, dtype=torch.float32, device=dev)
    x = torch.empty(R, d, dtype=torch.bfloat16, device=dev)
    q = torch.empty(R, qw, dtype=torch.bfloat16, device=dev)
    ctx = torch.empty(R, qw, dtype=torch.bfloat16, device=dev)
    act = torch.empty(R, c.d_ff, dtype=torch.bfloat16, device=dev)
    cos_sin = rope_table(model, positions)
    factor = float(np.float32(1.0 / math.sqrt(c.d_head)))
    BF = _lib.CC_GEMM_BF16
    for li, lw in enumerate(model.layers):
        if li == 0:
            _lib.call("cc_embed_rmsnorm", ids.data_ptr(), R, model.embed.data_ptr(), _lib.CC_BF16,
                      c.vocab_size, d, h.data_ptr(), lw.attn_norm.data_ptr(), c.norm_eps, x.data_ptr(),
                      _lib.CC_BF16, _s())
        else:
            _lib.call("cc_rmsnorm", h.data_ptr(), R, d, d, lw.attn_norm.data_ptr(), c.norm_eps, x.data_ptr(),
                      _lib.CC_BF16, _s())
        ks, vs, dst, kraw, rrows, ak, av = kv(li)
        gemm(BF, _lib.CC_EPI_QKV_ROPE, R, lw.w_qkv.shape[0], d, x, lw.w_qkv, bias=lw.b_qkv, rope=cos_sin,
             q_out=q, ldq=qw, q_mode=_lib.CC_BF16, k_cache=ks, v_cache=vs, cache_dtype=_lib.CC_BF16,
             dst_rows=dst, k_raw=kraw, raw_rows=rrows, heads=(c.n_heads, c.kv_heads, c.d_head))
        _lib.call("cc_sparse_row_attention", q.data_ptr(), qw, positions.data_ptr(), R, ak.data_ptr(),
                  av.data_ptr(), n_keys, c.n_heads, c.kv_heads, c.d_head, factor, _p(row_factor),
                  ctx.data_ptr(), qw, _s(), meta={"flops": 4.0 * c.n_heads * c.d_head * pairs})
        gemm(BF, _lib.CC_EPI_RESIDUAL, R, d, qw, ctx, lw.w_o, bias=lw.b_o, C=h, ldc=d, c_mode=_lib.CC_F32)
        _mlp(model, lw, h, x, act, BF, _lib.CC_BF16)
    logits = argmax = None
    if want_logits:
        logits, argmax = final_logits(model, h[R - 1], logits_out)
    return RowsResult(h, logits, argmax)


def final_logits(model: Model, h_row: torch.Tensor, logits_out=None):
    """_final_logits (model.py:495-503) + argmax on device."""
    c = model.config
    if model.lm_head is None:
        raise ValueError("model has no output head")
    dev = h_row.device
    logits = logits_out if logits_out is not None else torch.empty(c.vocab_size, dtype=torch.float32, device=dev)
    argmax = torch.empty(1, dtype=torch.int64, device=dev)
    ws = torch.empty(64, dtype=torch.uint8, device=dev)
    dt = _lib.CC_BF16 if model.lm_head.dtype == torch.bfloat16 else _lib.CC_F32
    _lib.call("cc_lm_head_argmax", h_row.data_ptr(), model.final_norm.data_ptr(), c.norm_eps, c.d_model,
              model.lm_head.data_ptr(), dt, c.vocab_size, logits.data_ptr(), argmax.data_ptr(), ws.data_ptr(),
              _s())
    return logits, argmax


# ---------------------------------------------------------------------------
# fp32 (3xTF32) banked engine — the scoring model
# ---------------------------------------------------------------------------
@dataclass
class ScoreSpec:
    """Last-layer scoring: weights of bank columns [col0, n_bank) per sequence,
    reduced to scores[col_off[s] + j]."""
    col0: int
    chunk_lens: torch.Tensor     # int64 [S] (device)
    col_off: torch.Tensor        # int64 [S] (device)
    max_chunk: int
    scores: torch.Tensor         # fp32 [sum chunk_lens]


def forward_banked(model: Model, ids: torch.Tensor, positions: torch.Tensor, seq_tables: list[torch.Tensor],
                   n_seqs: int, max_new: int, max_bank: int, *, v_dst=None, k_raw_dst=None,
                   score: ScoreSpec | None = None) -> torch.Tensor:
    """fp32 engine. seq_tables[l]: device cc_bank_seq[S] for layer l (bank
    pointers of that layer). v_dst(l)/k_raw_dst(l): optional per-layer
    destinations for the new rows' values / position-free keys (dense
    precompute); otherwise they land in scratch. Returns the residual stream."""
    c = model.config
    if c.dtype != "fp32":
        raise ValueError("forward_banked runs fp32 models")
    dev = ids.device
    R, d = ids.numel(), c.d_model
    qw, kvw = c.attn_width, c.kv_width
    SP = _lib.CC_F32_SPLIT3
    TF = _lib.CC_GEMM_TF32X3
    h = torch.empty(R, d, dtype=torch.float32, device=dev)
    x = torch.empty(R, 3 * d, dtype=torch.float32, device=dev)
    q = torch.empty(R, qw, dtype=torch.float32, device=dev)
    k_new = torch.empty(R, kvw, dtype=torch.float32, device=dev)
    v_scratch = torch.empty(R, kvw, dtype=torch.float32, device=dev) if v_dst is None else None
    ctx = torch.empty(R, 3 * qw, dtype=torch.float32, device=dev)
    act = torch.empty(R, 3 * c.d_ff, dtype=torch.float32, device=dev)
    cos_sin = rope_table(model, positions)
    factor = float(np.float32(1.0 / math.sqrt(c.d_head)))
    L = c.n_layers
    for li, lw in enumerate(model.layers):
        if li == 0:
            _lib.call("cc_embed_rmsnorm", ids.data_ptr(), R, model.embed.data_ptr(), _lib.CC_F32, c.vocab_size,
                      d, h.data_ptr(), lw.attn_norm.data_ptr(), c.norm_eps, x.data_ptr(), SP, _s())
        else:
            _lib.call("cc_rmsnorm", h.data_ptr(), R, d, d, lw.attn_norm.data_ptr(), c.norm_eps, x.data_ptr(),
                      SP, _s())
        last_scoring = score is not None and li == L - 1
        vd = v_dst(li) if v_dst is not None else v_scratch
        kraw = k_raw_dst(li) if k_raw_dst is not None else None
        n_qkv = (c.n_heads + c.kv_heads) * c.d_head if last_scoring else lw.w_qkv.shape[0]
        gemm(TF, _lib.CC_EPI_QKV_ROPE, R, n_qkv, d, x, lw.w_qkv, bias=lw.b_qkv, rope=cos_sin, q_out=q,
             ldq=qw, q_mode=_lib.CC_F32, k_cache=k_new, v_cache=vd if vd is not None else k_new,
             cache_dtype=_lib.CC_F32, k_raw=kraw, heads=(c.n_heads, c.kv_heads, c.d_head))
        table = seq_tables[li]
        if last_scoring:
            w = torch.empty(n_seqs, c.n_heads, max_new, score.max_chunk, dtype=torch.float32, device=dev)
            _lib.call("cc_banked_attention_f32", table.data_ptr(), n_seqs, max_new, max_bank, q.data_ptr(),
                      k_new.data_ptr(), vd.data_ptr(), c.n_heads, c.kv_heads, c.d_head, factor, ctx.data_ptr(),
                      _lib.CC_F32_SPLIT3, w.data_ptr(), score.col0, score.max_chunk, _s())
            _lib.call("cc_reduce_scores", w.data_ptr(), n_seqs, c.n_heads, max_new, score.max_chunk,
                      score.chunk_lens.data_ptr(), score.col_off.data_ptr(), score.max_chunk,
                      score.scores.data_ptr(), _s())
            return h
        _lib.call("cc_banked_attention_f32", table.data_ptr(), n_seqs, max_new, max_bank, q.data_ptr(),
                  k_new.data_ptr(), vd.data_ptr(), c.n_heads, c.kv_heads, c.d_head, factor, ctx.data_ptr(),
                  _lib.CC_F32_SPLIT3, None, 0, 0, _s())
        gemm(TF, _lib.CC_EPI_RESIDUAL, R, d, qw, ctx, lw.w_o, bias=lw.b_o, C=h, ldc=d, c_mode=_lib.CC_F32)
        _mlp(model, lw, h, x, act, TF, SP)
    return h


def bank_tables(layers: int, seqs: list[tuple], device) -> list[torch.Tensor]:
    """seqs: [(k [L,n,H,D] or None, v or None, n_bank, row0, n_new)] ->
    one device cc_bank_seq table per layer (single H2D copy)."""
    n = len(seqs)
    arr = (_lib.BankSeq * (n * layers))()
    for li in range(layers):
        for si, (k, v, nb, row0, nn) in enumerate(seqs):
            kp = k[li].data_ptr() if k is not None else 0
            vp = v[li].data_ptr() if v is not None else 0
            arr[li * n + si] = _lib.BankSeq(kp, vp, nb, row0, nn)
    raw = np.frombuffer(bytes(arr), dtype=np.uint8).copy()
    dev = torch.from_numpy(raw).pin_memory().to(device, non_blocking=True)
    stride = n * ctypes.sizeof(_lib.BankSeq)
    return [dev[li * stride:(li + 1) * stride] for li in range(layers)]
