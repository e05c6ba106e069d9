"""Token-importance scoring and recompute-set selection on the device
(pkg/src/cacheclip/selector.py).

aux_score_tokens runs the scoring model (fp32, 3xTF32 GEMMs) for every chunk
in ONE batched pass: each chunk is a sequence whose bank is its cached rows at
local positions and whose new rows are the query (model.py:568-607); the last
layer stops at the attention weights over chunk columns, reduced in the
reference's order into per-token scores (selector.py:157-179).

select_tokens runs budget -> exact stable top-k -> per-chunk window rule in a
single-CTA kernel; one host read brings back the selection.
"""

from __future__ import annotations

import math
from dataclasses import asdict, dataclass
from fractions import Fraction
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .flops import PipelineTrace, trace_layer
from .kv_store import ChunkCache, host_to_device, require_cache_dtype
from .runtime import KvPlan, ScoreSpec, bank_tables, forward_banked, forward_rows
from .tokenizers import TokenSpan, align_spans
from .weights import Model


@dataclass(frozen=True)
class SelectionConfig:
    recomp_ratio: float
    window_len: int = 8
    window_threshold: int = 5
    expand_full_window: bool = False

    def __post_init__(self) -> None:
        if not 0.0 <= self.recomp_ratio <= 1.0:
            raise ValueError(f"recomp_ratio must be in [0, 1], got {self.recomp_ratio}")
        if self.window_len < 1:
            raise ValueError(f"window_len must be >= 1, got {self.window_len}")
        if not 0 <= self.window_threshold <= self.window_len:
            raise ValueError(f"window_threshold must be in 0..window_len, got {self.window_threshold}")


class ImportanceScores:
    """Concatenated per-token scores (device fp32) with their chunk lengths."""

    def __init__(self, scores, chunk_lens) -> None:
        if isinstance(scores, torch.Tensor):
            self.device_scores = scores.float().contiguous()
        else:
            arr = np.asarray(scores, dtype=np.float32)
            if arr.ndim != 1:
                raise ValueError("scores must be 1-D")
            self.device_scores = torch.from_numpy(arr.copy())
        self.chunk_lens = tuple(int(c) for c in chunk_lens)
        if self.device_scores.dim() != 1 or self.device_scores.numel() != sum(self.chunk_lens):
            raise ValueError(f"{self.device_scores.numel()} scores for chunk lengths {self.chunk_lens}")

    @property
    def scores(self) -> np.ndarray:
        return self.device_scores.detach().cpu().numpy()


@dataclass(frozen=True)
class WindowRecord:
    window_id: int
    chunk: int
    start: int
    end: int
    selected: int
    kept: bool
    partial: bool


@dataclass(frozen=True)
class AuxSelection:
    indices: tuple[int, ...]
    windows: tuple[WindowRecord, ...]
    n_tokens: int
    requested_ratio: float

    @property
    def effective_ratio(self) -> float:
        return len(self.indices) / self.n_tokens if self.n_tokens else 0.0


@dataclass(frozen=True)
class SelectionPlan:
    indices: tuple[int, ...]
    windows: tuple[WindowRecord, ...]
    requested_ratio: float
    effective_ratio: float

    def to_json_dict(self) -> dict:
        return {"indices": list(self.indices), "windows": [asdict(w) for w in self.windows],
                "requested_ratio": self.requested_ratio, "effective_ratio": self.effective_ratio}

    @classmethod
    def from_json_dict(cls, data: dict) -> "SelectionPlan":
        return cls(tuple(int(i) for i in data["indices"]), tuple(WindowRecord(**w) for w in data["windows"]),
                   float(data["requested_ratio"]), float(data["effective_ratio"]))


def selection_budget(ratio: float, n_tokens: int) -> int:
    """ceil(ratio * n) on the ratio's decimal rendering (selector.py:113-123)."""
    if n_tokens < 0:
        raise ValueError("token count must be non-negative")
    return max(0, min(n_tokens, math.ceil(Fraction(str(float(ratio))) * n_tokens)))


# ---------------------------------------------------------------------------
def _device_of(t: torch.Tensor) -> torch.device:
    return t.device if t.is_cuda else torch.device("cuda")


def _run_select(scores: torch.Tensor, chunk_lens: Sequence[int], budget: int, window_len: int, threshold: int,
                expand: bool, index_offset: int = 0):
    """Launch the top-k/window kernel; returns device (indices, count, win_sel, win_kept)."""
    dev = _device_of(scores)
    s = scores.to(dev, dtype=torch.float32).contiguous()
    n = s.numel()
    lens = np.asarray(chunk_lens, dtype=np.int64)
    n_win = int(sum(-(-int(c) // window_len) for c in lens))
    lib = _lib.load()
    ws_bytes = int(lib.cc_select_workspace_bytes(n, len(lens)))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    out_idx = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    out_cnt = torch.empty(1, dtype=torch.int64, device=dev)
    win_sel = torch.empty(max(n_win, 1), dtype=torch.int32, device=dev)
    win_kept = torch.empty(max(n_win, 1), dtype=torch.int32, device=dev)
    lens_dev = host_to_device(lens, dev)
    _lib.call("cc_select_topk_windows", s.data_ptr(), n, lens_dev.data_ptr(), len(lens), n_win, budget,
              window_len, threshold, int(expand), index_offset, out_idx.data_ptr(), out_cnt.data_ptr(),
              win_sel.data_ptr(), win_kept.data_ptr(), ws.data_ptr(), torch.cuda.current_stream().cuda_stream)
    return out_idx, out_cnt, win_sel[:n_win], win_kept[:n_win]


def top_candidates(scores, budget: int) -> np.ndarray:
    """Indices of the `budget` highest scores, lower index first on ties,
    returned ascending (selector.py:126-129) — the window kernel with 1-token
    windows and threshold 1 keeps exactly the candidates."""
    t = scores if isinstance(scores, torch.Tensor) else torch.from_numpy(np.asarray(scores, np.float32).copy())
    n = t.numel()
    budget = max(0, min(int(budget), n))
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    idx, cnt, _, _ = _run_select(t, [n], budget, 1, 1, False)
    k = int(cnt.item())
    return idx[:k].cpu().numpy()


def select_tokens(scores: ImportanceScores, config: SelectionConfig) -> AuxSelection:
    """Budgeted top-k filtered by the window rule, aux-token space (selector.py:182-214)."""
    return select_tokens_device(scores, config).aux_selection()


@dataclass
class DeviceSelection:
    """Selection kernel output after the pipeline's single host sync: the
    count, indices and window flags came back in one D2H copy; the device
    indices feed the recompute launch directly. Python objects (windows,
    tuples) are built afterwards, while the GPU runs."""
    count: int
    idx_dev: torch.Tensor          # [count] int64, index_offset applied
    idx_host: np.ndarray           # [count] int64, index_offset applied
    win_selected: np.ndarray
    win_kept: np.ndarray
    n_tokens: int
    chunk_lens: tuple[int, ...]
    config: SelectionConfig
    index_offset: int

    def windows(self) -> tuple[WindowRecord, ...]:
        wl = self.config.window_len
        out = []
        wid, base = 0, 0
        ws_sel, ws_kept = self.win_selected.tolist(), self.win_kept.tolist()
        for ci, clen in enumerate(self.chunk_lens):
            for ws in range(0, clen, wl):
                we = min(ws + wl, clen)
                out.append(WindowRecord(wid, ci, base + ws, base + we, ws_sel[wid], bool(ws_kept[wid]),
                                        (we - ws) < wl))
                wid += 1
            base += clen
        return tuple(out)

    def aux_selection(self) -> AuxSelection:
        aux_idx = tuple((self.idx_host - self.index_offset).tolist())
        return AuxSelection(aux_idx, self.windows(), self.n_tokens, self.config.recomp_ratio)


@dataclass
class PendingSelection:
    """The selection kernel's device outputs, launched but not yet read back."""
    idx: torch.Tensor
    cnt: torch.Tensor
    win_sel: torch.Tensor
    win_kept: torch.Tensor
    budget: int
    n_tokens: int
    chunk_lens: tuple[int, ...]
    config: SelectionConfig
    index_offset: int
    done: torch.cuda.Event  # recorded right behind the selection kernel

    @property
    def count_known(self) -> bool:
        """With threshold <= 1 and no expansion every candidate's window is
        kept (count >= 1 >= threshold), so exactly `budget` rows are selected
        (selector.py:199-207): the host knows the count without reading it."""
        return self.config.window_threshold <= 1 and not self.config.expand_full_window

    def read_back(self, stream: torch.cuda.Stream | None = None) -> DeviceSelection:
        """One D2H read: count | window counts | kept flags | indices. On a
        side `stream` (waiting for the kernel) it does not wait for work
        queued on the launching stream after the selection."""
        if stream is None:
            flags = torch.cat([self.cnt, self.win_sel.long(), self.win_kept.long(), self.idx]).cpu().numpy()
        else:
            stream.wait_event(self.done)
            with torch.cuda.stream(stream):
                dev = torch.cat([self.cnt, self.win_sel.long(), self.win_kept.long(), self.idx])
                host = torch.empty(dev.shape, dtype=dev.dtype, pin_memory=True)
                host.copy_(dev, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record()
            for t in (self.cnt, self.win_sel, self.win_kept, self.idx):
                t.record_stream(stream)
            ev.synchronize()
            flags = host.numpy()
        k = int(flags[0])
        n_win = self.win_sel.numel()
        return DeviceSelection(k, self.idx[:k], flags[1 + 2 * n_win:1 + 2 * n_win + k].astype(np.int64),
                               flags[1:1 + n_win], flags[1 + n_win:1 + 2 * n_win], self.n_tokens, self.chunk_lens,
                               self.config, self.index_offset)


def launch_select(scores: ImportanceScores, config: SelectionConfig, index_offset: int = 0) -> PendingSelection:
    n = int(scores.device_scores.numel())
    budget = selection_budget(config.recomp_ratio, n)
    idx, cnt, wsel, wkept = _run_select(scores.device_scores, scores.chunk_lens, budget, config.window_len,
                                        config.window_threshold, config.expand_full_window, index_offset)
    done = torch.cuda.Event()
    done.record()
    return PendingSelection(idx, cnt, wsel, wkept, budget, n, tuple(scores.chunk_lens), config, index_offset, done)


def select_tokens_device(scores: ImportanceScores, config: SelectionConfig, index_offset: int = 0) -> DeviceSelection:
    return launch_select(scores, config, index_offset).read_back()


def map_selection(aux_selection: AuxSelection, aux_spans: Sequence[TokenSpan], primary_spans: Sequence[TokenSpan],
                  *, index_offset: int = 0) -> SelectionPlan:
    """Project aux-space selection onto primary tokens (selector.py:217-245)."""
    if len(aux_spans) != aux_selection.n_tokens:
        raise ValueError(f"{len(aux_spans)} aux spans for a selection over {aux_selection.n_tokens} tokens")
    if _same_spans(aux_spans, primary_spans):
        primary = list(aux_selection.indices)
    else:
        primary = align_spans(aux_spans, primary_spans).project(aux_selection.indices)
    return SelectionPlan(tuple(p + index_offset for p in primary), aux_selection.windows,
                         aux_selection.requested_ratio,
                         len(primary) / len(primary_spans) if primary_spans else 0.0)


def _same_spans(a, b) -> bool:
    if a is b:
        return True
    if len(a) != len(b):
        return False
    return all(x.start == y.start and x.end == y.end for x, y in zip(a, b))


# ---------------------------------------------------------------------------
def aux_score_tokens(aux_model: Model, aux_chunk_caches: Sequence[ChunkCache], query_ids: Sequence[int], *,
                     trace: PipelineTrace | None = None, workers: int = 1, _banks=None) -> ImportanceScores:
    """Score chunk tokens by last-layer query attention (selector.py:132-179).

    All chunks run as one batch of sequences; ``workers`` is accepted for
    signature parity (the result is invariant to it, as in the reference)."""
    if not aux_chunk_caches:
        raise ValueError("no chunk caches to score")
    if not query_ids:
        raise ValueError("query must be non-empty")
    for i, cache in enumerate(aux_chunk_caches):
        if cache.model_fingerprint != aux_model.fingerprint:
            raise ValueError(f"aux chunk {i} was built by a different model")
    c = aux_model.config
    if c.dtype != "fp32":
        raise ValueError("the scoring model must run in fp32 mode (exact selection)")
    require_cache_dtype(aux_chunk_caches, aux_model.wdtype, "aux chunk")
    q = np.asarray(list(query_ids), dtype=np.int64)
    if q.min() < 0 or q.max() >= c.vocab_size:
        raise ValueError(f"token id outside vocab of size {c.vocab_size}")
    dev = aux_model.device
    S, Q = len(aux_chunk_caches), q.size
    n_rows = np.array([ch.n_rows for ch in aux_chunk_caches], dtype=np.int64)
    prefix = aux_chunk_caches[0].prefix_len
    chunk_lens = n_rows - np.array([ch.prefix_len for ch in aux_chunk_caches], dtype=np.int64)
    if any(ch.prefix_len != prefix for ch in aux_chunk_caches):
        # the reference scores each chunk against its own prefix_len; one
        # banked launch takes one score column offset, so chunks are scored in
        # groups of equal prefix length (a chunk's scores depend on that chunk
        # and the query only) and reassembled in chunk order
        if _banks is not None:
            raise ValueError("streamed aux banks must share one prefix length")
        groups: dict[int, list[int]] = {}
        for i, ch in enumerate(aux_chunk_caches):
            groups.setdefault(ch.prefix_len, []).append(i)
        parts: list = [None] * len(aux_chunk_caches)
        for idxs in groups.values():
            sub = aux_score_tokens(aux_model, [aux_chunk_caches[i] for i in idxs], query_ids, trace=trace)
            offs = np.concatenate([[0], np.cumsum(sub.chunk_lens)])
            for k, i in enumerate(idxs):
                parts[i] = sub.device_scores[int(offs[k]):int(offs[k + 1])]
        return ImportanceScores(torch.cat(parts), tuple(int(x) for x in chunk_lens))
    ids = np.tile(q, S)
    pos = (n_rows[:, None] + np.arange(Q, dtype=np.int64)[None, :]).reshape(-1)
    col_off = np.concatenate([[0], np.cumsum(chunk_lens)[:-1]]).astype(np.int64)
    host = np.concatenate([ids, pos, chunk_lens, col_off])
    buf = host_to_device(host, dev)
    R = S * Q
    ids_d, pos_d = buf[:R], buf[R:2 * R]
    lens_d, off_d = buf[2 * R:2 * R + S], buf[2 * R + S:]
    ready = None
    if _banks is not None:  # host caches streamed in per layer (kv_store.stream_local_banks)
        kb, vb, offs, ready = _banks
        seqs = [(kb[:, o:o + ch.n_rows], vb[:, o:o + ch.n_rows], ch.n_rows, si * Q, Q)
                for si, (ch, o) in enumerate(zip(aux_chunk_caches, offs.tolist()))]
    else:
        seqs = [(ch.local_rotated_keys(c.rope), ch.v, ch.n_rows, si * Q, Q)
                for si, ch in enumerate(aux_chunk_caches)]
    tables = bank_tables(c.n_layers, seqs, dev)
    scores = torch.empty(int(chunk_lens.sum()), dtype=torch.float32, device=dev)
    spec = ScoreSpec(prefix, lens_d, off_d, int(chunk_lens.max()), scores)
    forward_banked(aux_model, ids_d, pos_d, tables, S, Q, int(n_rows.max()), score=spec, layer_ready=ready)
    if trace is not None:  # the reference's per-chunk peek events, folded (linear counts)
        rows_total = int(n_rows.sum())
        trace.rope("selection", c.n_layers * rows_total * c.kv_heads, c.d_head)
        trace_layer(trace, c, "selection", Q * S, Q * rows_total + S * (Q * (Q + 1) // 2), times=c.n_layers)
        trace.matmul("selection", S, c.d_model, c.vocab_size)
    return ImportanceScores(scores, tuple(int(x) for x in chunk_lens))


def cacheblend_select(primary_model: Model, merged, ratio: float, *, trace: PipelineTrace | None = None,
                      return_scores: bool = False):
    """selector.py:248-291 (see _cacheblend_device)."""
    plan, _, disc = _cacheblend_device(primary_model, merged, ratio, trace)
    if return_scores:
        return plan, disc.cpu().numpy()
    return plan


def _cacheblend_device(primary_model: Model, merged, ratio: float, trace: PipelineTrace | None = None):
    """CacheBlend-style discrepancy selection (selector.py:248-291) on the
    device: layer 0 of every merged row recomputed with global context (one
    dense causal pass, the cache untouched), layer 1's value projection of
    those states (RMSNorm + the V rows of the fused QKV weight), the per-row
    L2 drift against the cached layer-1 values (cc_row_l2_diff), then the
    exact stable top-ceil(ratio*N) with no windows."""
    c = primary_model.config
    if c.n_layers < 2:
        raise ValueError("discrepancy selection needs at least two layers")
    if not 0.0 <= ratio <= 1.0:
        raise ValueError(f"ratio must be in [0, 1], got {ratio}")
    if c.dtype != "bf16":
        raise ValueError("device CacheBlend runs the bf16 primary engine")
    dev = primary_model.device
    sink, total = merged.layout.sink_len, merged.layout.total
    n = total - sink
    if n <= 0:
        return SelectionPlan((), (), float(ratio), 0.0), None, torch.zeros(0, device=dev)
    ids = merged.token_ids_device()[:total]
    pos = torch.arange(total, dtype=torch.int64, device=dev)
    bank_k = torch.empty(total, c.kv_heads, c.d_head, dtype=torch.bfloat16, device=dev)
    bank_v = torch.empty_like(bank_k)
    res = forward_rows(primary_model, ids, pos, KvPlan(k_scatter=bank_k, v_scatter=bank_v, attn_k=bank_k,
                                                       attn_v=bank_v), total, want_logits=False,
                       pairs=total * (total + 1) // 2, layers=1)
    lw = primary_model.layers[1]
    s = torch.cuda.current_stream().cuda_stream
    x = torch.empty(total, c.d_model, dtype=torch.bfloat16, device=dev)
    qw, kw = c.attn_width, c.kv_width
    from .runtime import gemm
    # layer 1's values in the arithmetic of the executor that built the
    # caches: with fused RMSNorm, bf16(h * gain) with per-row 1/rms applied in
    # the GEMM epilogue (cc_norm_prep = the residual epilogue's operand); the
    # cache's own precision (bf16 rounding, as the QKV epilogue stores them),
    # so a row whose context did not change drifts by exactly 0
    norm = {}
    if _lib.load().cc_fused_norm() and c.d_model % 32 == 0 and c.mlp_gated:
        ssq = torch.empty(c.d_model // 32, total, dtype=torch.float32, device=dev)
        inv = torch.empty(total, dtype=torch.float32, device=dev)
        _lib.call("cc_norm_prep", res.h.data_ptr(), total, c.d_model, c.d_model, lw.attn_norm.data_ptr(),
                  x.data_ptr(), ssq.data_ptr(), total, s)
        _lib.call("cc_norm_finalize", ssq.data_ptr(), total, c.d_model, total, c.norm_eps, inv.data_ptr(), s)
        norm = dict(inv_rms=inv)
    else:
        _lib.call("cc_rmsnorm", res.h.data_ptr(), total, c.d_model, c.d_model, lw.attn_norm.data_ptr(), c.norm_eps,
                  x.data_ptr(), _lib.CC_BF16, s)
    cached = merged.v_store[1][sink:total]
    v_global = torch.empty(total, kw, dtype=cached.dtype, device=dev)
    vmode = _lib.CC_BF16 if cached.dtype == torch.bfloat16 else _lib.CC_F32
    gemm(_lib.CC_GEMM_BF16, _lib.CC_EPI_STORE, total, kw, c.d_model, x, lw.w_qkv[qw + kw:qw + 2 * kw],
         bias=None if lw.b_qkv is None else lw.b_qkv[qw + kw:qw + 2 * kw], C=v_global, ldc=kw, c_mode=vmode,
         **norm)
    disc = torch.empty(n, dtype=torch.float32, device=dev)
    _lib.call("cc_row_l2_diff", v_global[sink:].data_ptr(), vmode, kw, cached.data_ptr(), vmode, kw, n, kw,
              disc.data_ptr(), s)
    if trace is not None:
        trace_layer(trace, c, "selection", total, total * (total + 1) // 2, times=1)
        trace.matmul("selection", total, c.d_model, kw)
    # one "chunk" and threshold 1: the window rule keeps exactly the candidates
    dsel = select_tokens_device(ImportanceScores(disc, (n,)), SelectionConfig(ratio, 8, 1), index_offset=sink)
    plan = SelectionPlan(tuple(dsel.idx_host.tolist()), (), float(ratio), dsel.count / n)
    return plan, dsel, disc


def random_select(n_tokens: int, ratio: float, seed: int, *, index_offset: int = 0) -> SelectionPlan:
    """Seeded uniform sample without replacement; ablation control (selector.py:294-312)."""
    if n_tokens < 0:
        raise ValueError("token count must be non-negative")
    budget = selection_budget(ratio, n_tokens)
    rng = np.random.default_rng(seed)
    chosen = np.sort(rng.choice(n_tokens, size=budget, replace=False))
    return SelectionPlan(tuple(int(i) + index_offset for i in chosen), (), float(ratio),
                         budget / n_tokens if n_tokens else 0.0)
