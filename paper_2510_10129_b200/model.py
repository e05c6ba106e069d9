"""Model-level entry points with the reference's names and signatures
(pkg/src/cacheclip/model.py:506-728), running on the device engine.

Returned logits are host float32 numpy arrays like the reference's; the
device copies stay available (``last_device_logits``) for callers that want
to avoid the D2H read.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .config import ModelConfig
from .errors import DimensionError
from .flops import PipelineTrace, trace_layer
from .kv_store import ChunkCache, MergedCache, host_to_device, require_cache_dtype
from .runtime import KvPlan, bank_tables, final_logits, forward_banked, forward_rows
from .weights import Model, from_params, init_model  # noqa: F401  (re-export)


def visible_pairs(n_new: int, n_past: int = 0) -> int:
    """tensor_core.py:173-179."""
    return n_new * n_past + n_new * (n_new + 1) // 2


def _ids_tensor(model: Model, token_ids: Sequence[int]) -> torch.Tensor:
    """_embed's validation (model.py:484-492), then the ids on device."""
    ids = np.asarray(list(token_ids), dtype=np.int64)
    if ids.ndim != 1 or ids.size == 0:
        raise ValueError("token ids must be a non-empty 1-D sequence")
    if ids.min() < 0 or ids.max() >= model.config.vocab_size:
        raise ValueError(f"token id outside vocab of size {model.config.vocab_size}")
    return host_to_device(ids, model.device)


def _p(t):
    return None if t is None else t.data_ptr()


def _positions(start: int, n: int, device) -> torch.Tensor:
    return torch.arange(start, start + n, dtype=torch.int64, device=device)


@dataclass
class LayerCache:
    """Plain forward cache of prefill_full: keys position-free (model.py:285-304)."""

    k: torch.Tensor
    v: torch.Tensor
    token_ids: list[int]
    KEYS_ROTATED = False

    @property
    def keys(self):
        return list(self.k.unbind(0))

    @property
    def values(self):
        return list(self.v.unbind(0))

    @property
    def n_rows(self) -> int:
        return self.k.shape[1]


@dataclass
class PrefillResult:
    cache: LayerCache
    logits: np.ndarray | None
    maps: None = None
    first_token: int | None = None
    logits_device: torch.Tensor | None = None


def _dense(model: Model, ids: torch.Tensor, want_logits: bool):
    """Causal forward over rows 0..n-1; returns (K position-free, V, logits, argmax)."""
    c = model.config
    n = ids.numel()
    dev = model.device
    K = torch.empty(c.n_layers, n, c.kv_heads, c.d_head, dtype=model.wdtype, device=dev)
    V = torch.empty_like(K)
    pos = _positions(0, n, dev)
    if c.dtype == "bf16":
        bank = torch.empty(n, c.kv_heads, c.d_head, dtype=torch.bfloat16, device=dev)  # rotated K, reused per layer
        plan = KvPlan(k_scatter=bank, v_scatter=V, attn_k=bank, attn_v=V, k_raw=K)
        res = forward_rows(model, ids, pos, plan, n, want_logits=want_logits, pairs=visible_pairs(n))
        return K, V, res.logits, res.argmax
    tables = bank_tables(c.n_layers, [(None, None, 0, 0, n)], dev)
    h = forward_banked(model, ids, pos, tables, 1, n, 0, v_dst=V, k_raw_dst=K, want_state=want_logits)
    logits = argmax = None
    if want_logits:
        logits, argmax = final_logits(model, h[n - 1])
    return K, V, logits, argmax


def prefill_full(model: Model, token_ids: Sequence[int], *, capture_maps: bool = False,
                 trace: PipelineTrace | None = None, stage: str = "decode") -> PrefillResult:
    """Causal forward over the whole sequence at positions 0..n-1 (model.py:506-535)."""
    if capture_maps:
        raise NotImplementedError("attention-map capture is not materialised on the device path")
    ids = _ids_tensor(model, token_ids)
    K, V, logits, argmax = _dense(model, ids, True)
    n = ids.numel()
    trace_layer(trace, model.config, stage, n, visible_pairs(n), times=model.config.n_layers)
    if trace is not None:
        trace.matmul(stage, 1, model.config.d_model, model.config.vocab_size)
    host = logits.cpu().numpy()
    return PrefillResult(LayerCache(K, V, list(token_ids)), host, None, int(host.argmax()), logits)


def prefill_chunk(model: Model, prefix_ids: Sequence[int], chunk_ids: Sequence[int], *,
                  trace: PipelineTrace | None = None) -> ChunkCache:
    """Precompute one chunk behind the shared prefix at local positions;
    position-free keys (model.py:538-565). The logits the reference computes
    and discards are skipped."""
    prefix_ids, chunk_ids = list(prefix_ids), list(chunk_ids)
    if not chunk_ids:
        raise ValueError("chunk must contain at least one token")
    ids = _ids_tensor(model, prefix_ids + chunk_ids)
    K, V, _, _ = _dense(model, ids, False)
    n = ids.numel()
    trace_layer(trace, model.config, "chunk_precompute", n, visible_pairs(n), times=model.config.n_layers)
    if trace is not None:
        trace.matmul("chunk_precompute", 1, model.config.d_model, model.config.vocab_size)
    return ChunkCache(K, V, prefix_ids + chunk_ids, len(prefix_ids), model.config.tokenizer_id,
                      model.fingerprint)


def _dense_batched(model: Model, seqs: list[list[int]]):
    """Independent causal forwards of many sequences in ONE layer-wise pass
    (every GEMM sees all rows). bf16: one key bank holding every sequence at a
    128-row-aligned base, so each row attends [base, base + pos] over the same
    key tiles a lone prefill would (bitwise-equal results); fp32: the banked
    engine with one empty-bank sequence each. Returns per-sequence (K, V)."""
    c = model.config
    dev = model.device
    lens = np.array([len(x) for x in seqs], dtype=np.int64)
    R = int(lens.sum())
    ids_h = np.concatenate([np.asarray(x, dtype=np.int64) for x in seqs])
    if ids_h.min() < 0 or ids_h.max() >= c.vocab_size:
        raise ValueError(f"token id outside vocab of size {c.vocab_size}")
    pos_h = np.concatenate([np.arange(n, dtype=np.int64) for n in lens])
    row0 = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    if c.dtype == "bf16":
        padded = -(-lens // 128) * 128
        base = np.concatenate([[0], np.cumsum(padded)[:-1]]).astype(np.int64)
        n_bank = int(padded.sum())
        kstart_h = np.repeat(base, lens)
        dst_h = kstart_h + pos_h
        buf = host_to_device(np.concatenate([ids_h, pos_h, kstart_h, dst_h]), dev)
        ids, pos, kstart, dst = buf[:R], buf[R:2 * R], buf[2 * R:3 * R], buf[3 * R:]
        K = torch.empty(c.n_layers, n_bank, c.kv_heads, c.d_head, dtype=torch.bfloat16, device=dev)
        V = torch.zeros_like(K)  # padding rows are read (masked, P = 0) by attention: must be finite
        bank = torch.zeros(n_bank, c.kv_heads, c.d_head, dtype=torch.bfloat16, device=dev)
        plan = KvPlan(k_scatter=bank, v_scatter=V, attn_k=bank, attn_v=V, dst_rows=dst, k_raw=K, raw_rows=dst,
                      key_start=kstart)
        pairs = int(sum(visible_pairs(int(n)) for n in lens))
        forward_rows(model, ids, pos, plan, n_bank, want_logits=False, pairs=pairs)
        return [(K[:, b:b + n], V[:, b:b + n]) for b, n in zip(base.tolist(), lens.tolist())]
    buf = host_to_device(np.concatenate([ids_h, pos_h]), dev)
    ids, pos = buf[:R], buf[R:]
    K = torch.empty(c.n_layers, R, c.kv_heads, c.d_head, dtype=torch.float32, device=dev)
    V = torch.empty_like(K)
    tables = bank_tables(c.n_layers, [(None, None, 0, int(r0), int(n)) for r0, n in zip(row0, lens)], dev)
    forward_banked(model, ids, pos, tables, len(seqs), int(lens.max()), 0, v_dst=V, k_raw_dst=K, want_state=False)
    return [(K[:, b:b + n], V[:, b:b + n]) for b, n in zip(row0.tolist(), lens.tolist())]


def prefill_chunks(model: Model, prefix_ids: Sequence[int], chunks: Sequence[Sequence[int]], *,
                   trace: PipelineTrace | None = None, max_rows: int = 65536) -> list[ChunkCache]:
    """Batched ``prefill_chunk``: every chunk behind the shared prefix at local
    positions, position-free keys, in as few layer-wise passes as fit
    ``max_rows`` rows (model.py:538-565 applied to each chunk; the results are
    the per-chunk ones). One pass feeds the GEMMs tens of thousands of rows
    instead of a few hundred per chunk."""
    prefix_ids = list(prefix_ids)
    chunks = [list(x) for x in chunks]
    if not chunks:
        return []
    if any(not x for x in chunks):
        raise ValueError("chunk must contain at least one token")
    out: list[ChunkCache] = []
    i = 0
    while i < len(chunks):
        batch, rows = [], 0
        while i < len(chunks) and (not batch or rows + len(prefix_ids) + len(chunks[i]) <= max_rows):
            batch.append(prefix_ids + chunks[i])
            rows += len(batch[-1])
            i += 1
        for seq, (k, v) in zip(batch, _dense_batched(model, batch)):
            out.append(ChunkCache(k, v, seq, len(prefix_ids), model.config.tokenizer_id, model.fingerprint))
            n = len(seq)
            trace_layer(trace, model.config, "chunk_precompute", n, visible_pairs(n), times=model.config.n_layers)
            if trace is not None:
                trace.matmul("chunk_precompute", 1, model.config.d_model, model.config.vocab_size)
    return out


def _check_cache(model: Model, cache) -> None:
    if getattr(cache, "model_fingerprint", model.fingerprint) != model.fingerprint:
        raise ValueError("cache was built by a different model")
    if not isinstance(cache, MergedCache):
        raise TypeError("the device path extends merged caches (rotated keys); got "
                        f"{type(cache).__name__}")
    if cache.k_store.shape[0] != model.config.n_layers:
        raise DimensionError(f"cache has {cache.k_store.shape[0]} layers, model has {model.config.n_layers}")
    require_cache_dtype([cache], model.wdtype, "merged cache")


def _row_factor(model: Model, knobs, n: int, n_plain: int = 0, device=None):
    if knobs is None:
        return None
    import math
    t, s = knobs
    f = np.float32(s / (math.sqrt(model.config.d_head) * t))
    plain = np.float32(1.0 / math.sqrt(model.config.d_head))
    arr = np.full(n_plain + n, f, dtype=np.float32)
    arr[:n_plain] = plain
    return host_to_device(arr, device)


def forward_on_merged(model: Model, cache: MergedCache, sel_idx: np.ndarray | None, sel_idx_dev,
                      query_ids: Sequence[int] | None, *, knobs=None, append: bool = True,
                      want_logits: bool = True, trace: PipelineTrace | None = None,
                      sel_stage: str = "recompute", query_stage: str = "decode", n_sel: int | None = None):
    """One layer-wise pass over selected rows (recomputed in place, causal by
    global position) followed by query rows appended at n_rows.. — the fused
    form of selective_forward + extend_cache (bit-identical composition in the
    reference's algebra: selected rows never see query positions).

    ``n_sel``: the selected rows are known only on the device (``sel_idx`` is
    None, ``sel_idx_dev`` holds ``n_sel`` sorted indices still being written
    by the selection kernel on this stream): the pass is launched without a
    host sync and the caller completes the host bookkeeping with
    ``finish_selection`` once the indices are read back."""
    c = model.config
    dev = model.device
    require_cache_dtype([cache], model.wdtype, "merged cache")
    deferred = sel_idx is None and n_sel is not None
    m = int(n_sel) if deferred else (0 if sel_idx is None else int(sel_idx.size))
    nq = 0 if query_ids is None else len(query_ids)
    base = cache.n_rows
    R = m + nq
    if R == 0:
        return None, None
    cache.ensure_capacity(base + nq)
    q_dev = None
    if nq:
        q = np.asarray(list(query_ids), dtype=np.int64)
        if q.min() < 0 or q.max() >= c.vocab_size:
            raise ValueError(f"token id outside vocab of size {c.vocab_size}")
        q_dev = host_to_device(q, dev)
    if m and sel_idx_dev is None:
        sel_idx_dev = host_to_device(np.ascontiguousarray(sel_idx, dtype=np.int64), dev)
    # rows assembled on device: selected rows (id gathered from the merged ids)
    # then the query rows at base.. (cc_build_rows)
    rows = torch.empty(2, R, dtype=torch.int64, device=dev)
    ids, pos = rows[0], rows[1]
    _lib.call("cc_build_rows", _p(sel_idx_dev), m, cache.token_ids_device().data_ptr() if m else None, _p(q_dev),
              nq, base, ids.data_ptr(), pos.data_ptr(), torch.cuda.current_stream().cuda_stream)
    rf = _row_factor(model, knobs, nq, m, dev)
    ks, vs = cache.k_store, cache.v_store
    # attention work, for the launch profiler only: unknown (-1) until the
    # deferred indices are read back (finish_selection fills it in)
    pairs = -1 if deferred and m else (int(np.sum(sel_idx + 1)) if m else 0) + (visible_pairs(nq, base) if nq else 0)
    plan = KvPlan(k_scatter=ks, v_scatter=vs, attn_k=ks, attn_v=vs, dst_rows=pos,
                  layer_ready=getattr(cache, "layer_ready", None))
    res = forward_rows(model, ids, pos, plan, base + nq, row_factor=rf, want_logits=want_logits and nq > 0,
                       pairs=pairs)
    cache.layer_ready = None  # every layer is now ordered before this stream's work
    if trace is not None:
        if nq:
            trace_layer(trace, c, query_stage, nq, visible_pairs(nq, base), times=c.n_layers)
        if nq and want_logits:
            trace.matmul(query_stage, 1, c.d_model, c.vocab_size)
    if append and nq:
        cache._append_rows(query_ids, q_dev)
    if m and not deferred:
        finish_selection(model, cache, sel_idx, base, nq, trace=trace, sel_stage=sel_stage)
    return res.logits, res.argmax


def finish_selection(model: Model, cache: MergedCache, sel_idx: np.ndarray, base: int, nq: int, *,
                     trace: PipelineTrace | None = None, sel_stage: str = "recompute", deferred: bool = False):
    """Host bookkeeping of a recompute pass once the selected indices are on
    the host: recomputed_rows, the reference's MAC trace and (deferred
    launches) the attention work of the launch profiler."""
    c = model.config
    pairs_sel = int(np.sum(np.asarray(sel_idx, dtype=np.int64) + 1))
    if trace is not None:
        trace_layer(trace, c, sel_stage, int(sel_idx.size), pairs_sel, times=c.n_layers)
    cache.recomputed_rows = tuple(np.asarray(sel_idx, dtype=np.int64).tolist())
    if deferred:
        pairs = pairs_sel + (visible_pairs(nq, base) if nq else 0)
        _lib.load().cc_profile_fill_work(_lib.PROFILE_OPS.index("attention_tcgen05"),
                                         4.0 * c.n_heads * c.d_head * pairs)


last_device_logits: torch.Tensor | None = None


def _host_logits(logits_dev):
    global last_device_logits
    last_device_logits = logits_dev
    return logits_dev.cpu().numpy()


def extend_cache(model: Model, cache, token_ids: Sequence[int], *, knobs=None, capture_maps: bool = False,
                 trace: PipelineTrace | None = None, stage: str = "decode"):
    """Append token rows to a merged cache; return last-row logits (model.py:610-629)."""
    if capture_maps:
        raise NotImplementedError("attention-map capture is not materialised on the device path")
    _check_cache(model, cache)
    if len(list(token_ids)) == 0:
        raise ValueError("token ids must be a non-empty 1-D sequence")
    logits, _ = forward_on_merged(model, cache, None, None, list(token_ids), knobs=knobs, trace=trace,
                                  query_stage=stage)
    return _host_logits(logits), None


def peek_forward(model: Model, cache, token_ids: Sequence[int], *, knobs=None, capture_maps: bool = False,
                 trace: PipelineTrace | None = None, stage: str = "decode"):
    """Like extend_cache but leaves the cache's rows untouched (model.py:632-646):
    the new rows' K/V land in spare capacity past n_rows and are not adopted."""
    if capture_maps:
        raise NotImplementedError("attention-map capture is not materialised on the device path")
    _check_cache(model, cache)
    logits, _ = forward_on_merged(model, cache, None, None, list(token_ids), knobs=knobs, append=False,
                                  trace=trace, query_stage=stage)
    return _host_logits(logits), None


def decode_step(model: Model, cache, token_id: int, position: int | None = None):
    """model.py:649-666."""
    expected = cache.n_rows
    if position is not None and position != expected:
        raise ValueError(f"non-contiguous position {position}; cache continues at {expected}")
    logits, _ = extend_cache(model, cache, [token_id])
    return logits, cache


def validate_selection(cache: MergedCache, selection) -> np.ndarray:
    """model.py:686-701: sorted unique merged-row indices outside the sink."""
    indices = getattr(selection, "indices", selection)
    idx = np.asarray(sorted(int(i) for i in indices), dtype=np.int64)
    if idx.size == 0:
        return idx
    if len(np.unique(idx)) != idx.size:
        raise ValueError("selection contains duplicate indices")
    sink = cache.layout.sink_len
    total = cache.layout.total
    if idx[0] < sink:
        raise ValueError(f"selection index {idx[0]} inside the retained shared prefix (< {sink})")
    if idx[-1] >= total:
        raise ValueError(f"selection index {int(idx[-1])} out of range (>= {total})")
    return idx


def selective_forward(model: Model, cache: MergedCache, selection, *, trace: PipelineTrace | None = None,
                      stage: str = "recompute") -> MergedCache:
    """Recompute the selected rows' K/V with merged (global) context, in place
    (model.py:669-728). Empty selection is a no-op."""
    _check_cache(model, cache)
    idx = validate_selection(cache, selection)
    if idx.size == 0:
        return cache
    forward_on_merged(model, cache, idx, None, None, want_logits=False, trace=trace, sel_stage=stage)
    return cache
