"""Layer-by-layer forward engines over device caches (one stream, no host syncs).

Both engines are single calls into the native executor of
libcacheclip_sm100.so (csrc/executor.cu), which launches the sm_100a kernels:

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
from dataclasses import dataclass

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
         raw_rows=None, heads=(0, 0, 0), inv_rms=None, ld_ssq: int = 0, xn_out=None, ldxn: int = 0,
         norm_gain=None, ssq_out=None, ssq_in=None, n_ssq: int = 0, ld_ssq_in: int = 0,
         norm_eps: float = 0.0) -> None:
    """Direct cc_gemm call (kernel tests and one-off GEMMs). ``ssq_in`` /
    ``n_ssq`` / ``ld_ssq_in`` / ``norm_eps``: a fused-norm consumer forming
    1/rms per row from a producer's per-32-column partial sums."""
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
    a.xn_out, a.ldxn, a.norm_gain, a.ssq_out = _p(xn_out), ldxn, _p(norm_gain), _p(ssq_out)
    a.inv_rms, a.ld_ssq = _p(inv_rms), ld_ssq
    a.ssq_in, a.n_ssq, a.ld_ssq_in, a.norm_eps = _p(ssq_in), n_ssq, ld_ssq_in, norm_eps
    _lib.call("cc_gemm", ctypes.byref(a), _s())


def rope_table(model: Model, positions: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Per-row fp32 cos/sin tables (float64 angles, tensor_core.py:41-51)."""
    c = model.config
    n = positions.numel()
    cos = torch.empty(n, c.d_head // 2, dtype=torch.float32, device=positions.device)
    sin = torch.empty_like(cos)
    inv = c.rope.inv_freq
    _lib.call("cc_rope_table", positions.data_ptr(), n, inv.ctypes.data, c.d_head, cos.data_ptr(), sin.data_ptr(),
              _s())
    return cos, sin


def _mlp(model: Model, lw, h: torch.Tensor, x: torch.Tensor, act_buf: torch.Tensor, kind: int, x_mode: int) -> None:
    """RMSNorm(h) -> gate/up GEMM (fused activation) -> down GEMM + residual, for
    Python-driven layer loops (the sequence-sharded path)."""
    c = model.config
    R, d = h.shape
    if R == 0:
        return
    _lib.call("cc_rmsnorm", h.data_ptr(), R, d, d, lw.mlp_norm.data_ptr(), c.norm_eps, x.data_ptr(), x_mode, _s())
    act = _lib.CC_ACT_SILU if c.activation == "silu" else _lib.CC_ACT_GELU_TANH
    if c.mlp_gated:
        gemm(kind, _lib.CC_EPI_GLU, R, lw.w_up.shape[0], d, x, lw.w_up, bias=lw.b_up, C=act_buf, ldc=c.d_ff,
             c_mode=x_mode, act=act, n_out=c.d_ff)
    else:
        gemm(kind, _lib.CC_EPI_ACT, R, c.d_ff, d, x, lw.w_up, bias=lw.b_up, C=act_buf, ldc=c.d_ff, c_mode=x_mode,
             act=act)
    gemm(kind, _lib.CC_EPI_RESIDUAL, R, d, c.d_ff, act_buf, lw.w_down, bias=lw.b_down, C=h, ldc=d,
         c_mode=_lib.CC_F32)


def _layer_stride(t: torch.Tensor | None) -> int:
    """Bytes between consecutive layers of a [L, rows, H, D] tensor (0 for a
    single shared [rows, H, D] buffer)."""
    if t is None or t.dim() < 4:
        return 0
    return t.stride(0) * t.element_size()


@dataclass
class KvPlan:
    """Where the QKV epilogue writes K/V and what attention reads; tensors are
    [L, rows, Hkv, D] (per layer) or [rows, Hkv, D] (one shared buffer)."""
    k_scatter: torch.Tensor
    v_scatter: torch.Tensor
    attn_k: torch.Tensor
    attn_v: torch.Tensor
    dst_rows: torch.Tensor | None = None
    k_raw: torch.Tensor | None = None
    raw_rows: torch.Tensor | None = None
    layer_ready: list | None = None   # torch.cuda.Event per layer (streamed merge) or None
    key_start: torch.Tensor | None = None  # int64 [rows]: first visible bank row (batched sequences)

    def to_c(self) -> _lib.KvPlan:
        ready = None
        if self.layer_ready:
            self._ready_arr = (ctypes.c_void_p * len(self.layer_ready))(*[e.cuda_event for e in self.layer_ready])
            ready = ctypes.cast(self._ready_arr, ctypes.POINTER(ctypes.c_void_p))
        return _lib.KvPlan(_p(self.k_scatter), _layer_stride(self.k_scatter), _p(self.v_scatter),
                           _layer_stride(self.v_scatter), _p(self.dst_rows), _p(self.k_raw),
                           _layer_stride(self.k_raw), _p(self.raw_rows), _p(self.attn_k), _layer_stride(self.attn_k),
                           _p(self.attn_v), _layer_stride(self.attn_v), ready, _p(self.key_start))


@dataclass
class RowsResult:
    h: torch.Tensor                 # final residual stream [R, d] fp32 (workspace view)
    logits: torch.Tensor | None     # [V] fp32 (last row)
    argmax: torch.Tensor | None     # [1] int64


def forward_rows(model: Model, ids: torch.Tensor, positions: torch.Tensor, plan: KvPlan, n_keys: int, *,
                 row_factor: torch.Tensor | None = None, want_logits: bool = True, pairs: int = 0,
                 layers: int | None = None) -> RowsResult:
    """``layers``: run only the first `layers` layers (no head); the residual
    stream of every row after them is returned (CacheBlend's layer-0 pass).
    A full pass keeps only what its outputs read: K/V of every row at every
    layer, and the last layer's attention / o-proj / MLP for the head's last
    row (want_logits) or for no row (cache-only prefill) — RowsResult.h then
    holds final states for those rows only."""
    c = model.config
    if c.dtype != "bf16":
        raise ValueError("forward_rows runs bf16 models; fp32 models use forward_banked")
    dev = ids.device
    R = ids.numel()
    md = model.desc()
    if layers is not None:
        if not 1 <= layers <= c.n_layers:
            raise ValueError(f"layers={layers} outside 1..{c.n_layers}")
        md = _lib.ModelDesc.from_buffer_copy(md)
        md.n_layers = layers
        want_logits = want_logits and layers == c.n_layers
    lib = _lib.load()
    ws = torch.empty(int(lib.cc_forward_rows_workspace_bytes(ctypes.byref(md), R)), dtype=torch.uint8, device=dev)
    logits = argmax = None
    if want_logits:
        logits = torch.empty(c.vocab_size, dtype=torch.float32, device=dev)
        argmax = torch.empty(1, dtype=torch.int64, device=dev)
    cplan = plan.to_c()
    tail = R if layers is not None else (1 if want_logits else 0)
    _lib.check(lib.cc_forward_rows(ctypes.byref(md), ids.data_ptr(), positions.data_ptr(), R, ctypes.byref(cplan),
                                   n_keys, float(pairs), _p(row_factor), tail, ws.data_ptr(), _p(logits),
                                   _p(argmax), _s()))
    h = ws[: R * c.d_model * 4].view(torch.float32).view(R, c.d_model)
    return RowsResult(h, logits, argmax)


def final_logits(model: Model, h_row: torch.Tensor):
    """_final_logits (model.py:495-503) + argmax on device."""
    c = model.config
    if model.lm_head is None:
        raise ValueError("model has no output head")
    dev = h_row.device
    logits = torch.empty(c.vocab_size, dtype=torch.float32, device=dev)
    argmax = torch.empty(1, dtype=torch.int64, device=dev)
    ws = torch.empty(64, dtype=torch.uint8, device=dev)
    dt = _lib.CC_BF16 if model.lm_head.dtype == torch.bfloat16 else _lib.CC_F32
    _lib.call("cc_lm_head_argmax", h_row.data_ptr(), model.final_norm.data_ptr(), c.norm_eps, c.d_model,
              model.lm_head.data_ptr(), dt, c.vocab_size, logits.data_ptr(), argmax.data_ptr(), ws.data_ptr(), _s())
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


def forward_banked(model: Model, ids: torch.Tensor, positions: torch.Tensor, tables: torch.Tensor,
                   n_seqs: int, max_new: int, max_bank: int, *, v_dst: torch.Tensor | None = None,
                   k_raw_dst: torch.Tensor | None = None, score: ScoreSpec | None = None,
                   layer_ready: list | None = None, want_state: bool = True) -> torch.Tensor:
    """fp32 engine. tables: device cc_bank_seq[n_layers][n_seqs]. v_dst /
    k_raw_dst: optional [L, rows, Hkv, D] destinations of the new rows' values
    and position-free keys (dense precompute). Returns the residual stream
    (meaningless with want_state=False: the last layer then stops after its
    QKV GEMM, K/V being all the caller reads)."""
    c = model.config
    if c.dtype != "fp32":
        raise ValueError("forward_banked runs fp32 models")
    dev = ids.device
    R = ids.numel()
    md = model.desc()
    lib = _lib.load()
    ws = torch.empty(int(lib.cc_forward_banked_workspace_bytes(ctypes.byref(md), R)), dtype=torch.uint8,
                     device=dev)
    spec_c = None
    w = None
    if score is not None:
        w = torch.empty(n_seqs, c.n_heads, max_new, score.max_chunk, dtype=torch.float32, device=dev)
        spec_c = _lib.ScoreSpec(score.col0, score.chunk_lens.data_ptr(), score.col_off.data_ptr(), score.max_chunk,
                                w.data_ptr(), score.scores.data_ptr())
    ready = None
    if layer_ready:
        ready = (ctypes.c_void_p * len(layer_ready))(*[e.cuda_event for e in layer_ready])
    _lib.check(lib.cc_forward_banked(ctypes.byref(md), ids.data_ptr(), positions.data_ptr(), R, tables.data_ptr(),
                                     n_seqs, max_new, max_bank, _p(v_dst), _layer_stride(v_dst), _p(k_raw_dst),
                                     _layer_stride(k_raw_dst), ctypes.byref(spec_c) if spec_c is not None else None,
                                     ctypes.cast(ready, ctypes.POINTER(ctypes.c_void_p)) if ready else None,
                                     1 if want_state else 0, ws.data_ptr(), _s()))
    return ws[: R * c.d_model * 4].view(torch.float32).view(R, c.d_model)


def bank_tables(layers: int, seqs: list[tuple], device) -> torch.Tensor:
    """seqs: [(k [L,n,H,D] or None, v or None, n_bank, row0, n_new)] -> device
    cc_bank_seq[layers][len(seqs)] (single pinned H2D copy)."""
    n = len(seqs)
    per = np.empty((n, 5), dtype=np.int64)     # (k base, v base, n_bank, row0, n_new)
    stride = np.zeros((n, 2), dtype=np.int64)  # layer strides of k, v in bytes
    for si, (k, v, nb, row0, nn) in enumerate(seqs):
        per[si] = (k.data_ptr() if k is not None else 0, v.data_ptr() if v is not None else 0, nb, row0, nn)
        if k is not None:
            stride[si] = (k.stride(0) * k.element_size(), v.stride(0) * v.element_size())
    arr = np.repeat(per[None], layers, axis=0)  # [L, S, 5] == cc_bank_seq[L][S]
    lidx = np.arange(layers, dtype=np.int64)[:, None]
    arr[:, :, 0] += lidx * stride[None, :, 0] * (per[None, :, 0] != 0)
    arr[:, :, 1] += lidx * stride[None, :, 1] * (per[None, :, 1] != 0)
    from .kv_store import host_to_device
    return host_to_device(arr.reshape(-1).view(np.uint8), device)
