"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of CacheClip's prefill hot path (reference package
``cacheclip`` under ``/root/reference/pkg/src/cacheclip``), generalised to
grouped-query attention. Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module, and only as the checker or the reported CPU baseline.

Parity status: PINNED. ``tests/golden/make_golden.py`` runs the reference
itself (imported from /root/reference, MHA-expanded weights for GQA models)
and commits its outputs under ``tests/golden/``; ``tests/test_oracle_golden.py``
checks this module against them (bitwise for MHA models, within 1e-6 for GQA),
plus the reference's own known-answer tests (frozen RoPE/softmax values,
selection worked examples).

Every arithmetic step keeps the reference's float32 operation order so that
an MHA model reproduces the reference bit for bit:
  * RoPE angles formed in float64, tables cast to float32, adjacent-pair
    rotation with separately rounded products (tensor_core.py:41-85);
  * RMSNorm as x / sqrt(mean(x^2) + eps) * gain (tensor_core.py:99-106);
  * attention logits (q @ k^T) * factor, masked, max-shifted softmax, then
    weights @ v (tensor_core.py:109-170).
GQA: query head h reads key/value head h // (n_heads // n_kv_heads); the
key/value banks are repeated to MHA width before the batched matmul, which is
exactly what the reference computes on column-replicated weights.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Sequence

import numpy as np

F32 = np.float32


# --------------------------------------------------------------------------
# configuration and weights
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class OracleConfig:
    """ModelConfig (model.py:62-106) plus ``n_kv_heads`` for GQA."""

    n_layers: int
    n_heads: int
    d_model: int
    d_head: int
    d_ff: int
    vocab_size: int
    n_kv_heads: int = 0  # 0 -> n_heads (MHA, the reference's only mode)
    rope_base: float = 10000.0
    norm_eps: float = 1e-5
    activation: str = "gelu"
    mlp_gated: bool = False
    attn_bias: bool = False
    mlp_bias: bool = False

    @property
    def kv_heads(self) -> int:
        return self.n_kv_heads or self.n_heads

    @property
    def group(self) -> int:
        return self.n_heads // self.kv_heads

    @property
    def q_width(self) -> int:
        return self.n_heads * self.d_head

    @property
    def kv_width(self) -> int:
        return self.kv_heads * self.d_head


def tensor_shapes(cfg: OracleConfig) -> list[tuple[str, tuple[int, ...]]]:
    """Tensor table in the reference's manifest order (model.py:109-137)."""
    dm, qw, kw, ff = cfg.d_model, cfg.q_width, cfg.kv_width, cfg.d_ff
    table: list[tuple[str, tuple[int, ...]]] = [("embed.weight", (cfg.vocab_size, dm))]
    for i in range(cfg.n_layers):
        p = f"layers.{i}"
        table.append((f"{p}.attn_norm.gain", (dm,)))
        table += [
            (f"{p}.attn.wq.weight", (dm, qw)),
            (f"{p}.attn.wk.weight", (dm, kw)),
            (f"{p}.attn.wv.weight", (dm, kw)),
            (f"{p}.attn.wo.weight", (qw, dm)),
        ]
        if cfg.attn_bias:
            table += [
                (f"{p}.attn.wq.bias", (qw,)),
                (f"{p}.attn.wk.bias", (kw,)),
                (f"{p}.attn.wv.bias", (kw,)),
                (f"{p}.attn.wo.bias", (dm,)),
            ]
        table.append((f"{p}.mlp_norm.gain", (dm,)))
        if cfg.mlp_gated:
            table.append((f"{p}.mlp.w_gate.weight", (dm, ff)))
        table.append((f"{p}.mlp.w_in.weight", (dm, ff)))
        table.append((f"{p}.mlp.w_out.weight", (ff, dm)))
        if cfg.mlp_bias:
            if cfg.mlp_gated:
                table.append((f"{p}.mlp.w_gate.bias", (ff,)))
            table.append((f"{p}.mlp.w_in.bias", (ff,)))
            table.append((f"{p}.mlp.w_out.bias", (dm,)))
    table.append(("final_norm.gain", (dm,)))
    table.append(("lm_head.weight", (cfg.vocab_size, dm)))
    return table


def seeded_params(cfg: OracleConfig, seed: int, bias_std: float = 0.0, *,
                  fast: bool = False) -> dict[str, np.ndarray]:
    """The reference's init recipe (model.py:178-201): N(0, 1/fan_in) weights,
    N(0,1) embedding, N(0, 1/d_model) lm_head, unit gains, zero biases.
    ``bias_std`` > 0 draws non-zero biases afterwards (a test-only knob so the
    bias path is actually exercised). ``fast`` draws float32 standard normals
    scaled in float32 (same distribution, different stream; ~2x faster, used
    for the full-size golden workloads that the GPU box must regenerate)."""
    rng = np.random.default_rng(seed)
    if fast:
        def normal(_mean, std, shape):
            return rng.standard_normal(shape, dtype=F32) * F32(std)
        rng_normal = normal
    else:
        def rng_normal(mean, std, shape):
            return rng.normal(mean, std, shape).astype(F32)
    fan_in = {"wq": cfg.d_model, "wk": cfg.d_model, "wv": cfg.d_model, "wo": cfg.q_width,
              "w_gate": cfg.d_model, "w_in": cfg.d_model, "w_out": cfg.d_ff}
    params: dict[str, np.ndarray] = {}
    for name, shape in tensor_shapes(cfg):
        parts = name.split(".")
        if name.endswith(".gain"):
            params[name] = np.ones(shape, F32)
        elif name.endswith(".bias"):
            params[name] = np.zeros(shape, F32)
        elif name == "embed.weight":
            params[name] = rng_normal(0.0, 1.0, shape)
        elif name == "lm_head.weight":
            params[name] = rng_normal(0.0, cfg.d_model ** -0.5, shape)
        else:
            params[name] = rng_normal(0.0, fan_in[parts[-2]] ** -0.5, shape)
    if bias_std > 0:
        brng = np.random.default_rng(seed + 1_000_003)
        for name in sorted(params):
            if name.endswith(".bias"):
                params[name] = brng.normal(0.0, bias_std, params[name].shape).astype(F32)
    return params


def round_to_bf16(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16, returned as float32 values."""
    u = np.ascontiguousarray(a, dtype=F32).view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    out = rounded.astype(np.uint32).view(F32)
    nan = np.isnan(a)
    if nan.any():
        out = out.copy()
        out[nan] = np.nan
    return out.reshape(np.shape(a))


def mha_expand(cfg: OracleConfig, params: dict[str, np.ndarray]) -> dict[str, np.ndarray]:
    """GQA -> MHA column replication for feeding the reference."""
    g = cfg.group
    if g == 1:
        return dict(params)
    out = dict(params)
    dh = cfg.d_head
    src_cols = np.concatenate(
        [np.arange((h // g) * dh, (h // g + 1) * dh) for h in range(cfg.n_heads)]
    )
    for i in range(cfg.n_layers):
        for w in ("wk", "wv"):
            key = f"layers.{i}.attn.{w}.weight"
            out[key] = np.ascontiguousarray(params[key][:, src_cols])
            bkey = f"layers.{i}.attn.{w}.bias"
            if bkey in params:
                out[bkey] = np.ascontiguousarray(params[bkey][src_cols])
    return out


# --------------------------------------------------------------------------
# numeric core (tensor_core.py)
# --------------------------------------------------------------------------


def rope_inv_freq(head_dim: int, base: float) -> np.ndarray:
    """base ** (-2i/d) in float64 (tensor_core.py:48-50)."""
    return base ** (-np.arange(0, head_dim, 2, dtype=np.float64) / head_dim)


def rope_tables(positions, head_dim: int, base: float) -> tuple[np.ndarray, np.ndarray]:
    """(cos, sin) float32 tables, angles formed in float64 (tensor_core.py:41-51)."""
    theta = np.asarray(positions, dtype=np.float64)[..., None] * rope_inv_freq(head_dim, base)
    return np.cos(theta).astype(F32), np.sin(theta).astype(F32)


def rope_rotate(x: np.ndarray, positions, head_dim: int, base: float) -> np.ndarray:
    """Adjacent-pair rotation of x (rows, [heads,] head_dim) by per-row
    position; separately rounded float32 products (tensor_core.py:54-85)."""
    x = np.asarray(x, dtype=F32)
    pos = np.asarray(positions)
    cos, sin = rope_tables(pos, head_dim, base)
    extra = x.ndim - 1 - pos.ndim
    cos = cos.reshape(pos.shape + (1,) * extra + (head_dim // 2,))
    sin = sin.reshape(cos.shape)
    ev, od = x[..., 0::2], x[..., 1::2]
    out = np.empty_like(x)
    out[..., 0::2] = ev * cos - od * sin
    out[..., 1::2] = ev * sin + od * cos
    return out


def rmsnorm(x: np.ndarray, gain: np.ndarray, eps: float) -> np.ndarray:
    """tensor_core.py:99-106."""
    x = np.asarray(x, dtype=F32)
    ms = np.mean(np.square(x), axis=-1, keepdims=True)
    return x / np.sqrt(ms + F32(eps)) * gain


def softmax_last(x: np.ndarray) -> np.ndarray:
    """Max-shifted softmax along the last axis (tensor_core.py:88-96)."""
    e = np.exp(x - np.max(x, axis=-1, keepdims=True))
    return e / np.sum(e, axis=-1, keepdims=True)


def attend(q: np.ndarray, k: np.ndarray, v: np.ndarray, limits: np.ndarray,
           *, temperature: float = 1.0, scale: float = 1.0) -> tuple[np.ndarray, np.ndarray]:
    """Masked attention of q (H, m, d) over k, v (Hkv, n, d).

    Row i sees key columns [0, limits[i]) (tensor_core.py:155-170). Returns
    (context (H, m, d), weights (H, m, n))."""
    h = q.shape[0]
    g = h // k.shape[0]
    if g > 1:
        k = np.repeat(k, g, axis=0)
        v = np.repeat(v, g, axis=0)
    n, d = k.shape[-2], q.shape[-1]
    limits = np.minimum(np.asarray(limits, dtype=np.int64), n)
    if np.any(limits < 1):
        raise ValueError("attention row with no visible keys")
    factor = F32(scale / (math.sqrt(d) * temperature))
    logits = (q @ np.swapaxes(k, -1, -2)) * factor
    visible = np.arange(n, dtype=np.int64)[None, :] < limits[:, None]
    logits = np.where(visible, logits, F32(-np.inf))
    w = softmax_last(logits)
    return w @ v, w


def activation(cfg: OracleConfig, x: np.ndarray) -> np.ndarray:
    """model.py:323-328."""
    if cfg.activation == "silu":
        return x / (F32(1.0) + np.exp(-x))
    c = F32(math.sqrt(2.0 / math.pi))
    return F32(0.5) * x * (F32(1.0) + np.tanh(c * (x + F32(0.044715) * x * x * x)))


# --------------------------------------------------------------------------
# model forward (model.py)
# --------------------------------------------------------------------------


@dataclass
class OracleModel:
    cfg: OracleConfig
    p: dict[str, np.ndarray]

    def w(self, layer: int, name: str) -> np.ndarray:
        return self.p[f"layers.{layer}.{name}"]


def qkv_project(m: OracleModel, layer: int, h: np.ndarray):
    """RMSNorm then three projections (+bias), model.py:340-364."""
    cfg = m.cfg
    rows = h.shape[0]
    x = rmsnorm(h, m.w(layer, "attn_norm.gain"), cfg.norm_eps)
    outs = []
    for name, heads in (("wq", cfg.n_heads), ("wk", cfg.kv_heads), ("wv", cfg.kv_heads)):
        y = x @ m.w(layer, f"attn.{name}.weight")
        if cfg.attn_bias:
            y = y + m.w(layer, f"attn.{name}.bias")
        outs.append(y.reshape(rows, heads, cfg.d_head))
    return outs[0], outs[1], outs[2]


def out_project(m: OracleModel, layer: int, ctx: np.ndarray) -> np.ndarray:
    """model.py:392-403; ctx (rows, H, d)."""
    y = ctx.reshape(ctx.shape[0], m.cfg.q_width) @ m.w(layer, "attn.wo.weight")
    if m.cfg.attn_bias:
        y = y + m.w(layer, "attn.wo.bias")
    return y


def mlp(m: OracleModel, layer: int, h: np.ndarray) -> np.ndarray:
    """model.py:406-432."""
    cfg = m.cfg
    x = rmsnorm(h, m.w(layer, "mlp_norm.gain"), cfg.norm_eps)
    up = x @ m.w(layer, "mlp.w_in.weight")
    if cfg.mlp_bias:
        up = up + m.w(layer, "mlp.w_in.bias")
    if cfg.mlp_gated:
        gate = x @ m.w(layer, "mlp.w_gate.weight")
        if cfg.mlp_bias:
            gate = gate + m.w(layer, "mlp.w_gate.bias")
        hidden = activation(cfg, gate) * up
    else:
        hidden = activation(cfg, up)
    y = hidden @ m.w(layer, "mlp.w_out.weight")
    if cfg.mlp_bias:
        y = y + m.w(layer, "mlp.w_out.bias")
    return y


def block(m: OracleModel, layer: int, h: np.ndarray, positions: np.ndarray,
          past: tuple[np.ndarray, np.ndarray] | None, *, knobs=None):
    """One pre-norm block over new rows against an optional rotated past bank
    (model.py:435-481). Returns (h, k_raw, k_rot, v, weights)."""
    cfg = m.cfg
    q, k, v = qkv_project(m, layer, h)
    q_rot = rope_rotate(q, positions, cfg.d_head, cfg.rope_base)
    k_rot = rope_rotate(k, positions, cfg.d_head, cfg.rope_base)
    if past is not None:
        bank_k = np.concatenate([past[0], k_rot], axis=0)
        bank_v = np.concatenate([past[1], v], axis=0)
    else:
        bank_k, bank_v = k_rot, v
    rows = h.shape[0]
    n_past = bank_k.shape[0] - rows
    temperature, scale = knobs if knobs is not None else (1.0, 1.0)
    limits = np.minimum(np.arange(rows) + 1 + n_past, bank_k.shape[0])
    ctx, w = attend(q_rot.transpose(1, 0, 2), bank_k.transpose(1, 0, 2),
                    bank_v.transpose(1, 0, 2), limits, temperature=temperature, scale=scale)
    h = h + out_project(m, layer, ctx.transpose(1, 0, 2))
    h = h + mlp(m, layer, h)
    return h, k, k_rot, v, w


def embed(m: OracleModel, ids: Sequence[int]) -> np.ndarray:
    """model.py:484-492."""
    arr = np.asarray(list(ids), dtype=np.int64)
    if arr.ndim != 1 or arr.size == 0:
        raise ValueError("token ids must be a non-empty 1-D sequence")
    if arr.min() < 0 or arr.max() >= m.cfg.vocab_size:
        raise ValueError("token id outside vocab")
    return m.p["embed.weight"][arr]


def final_logits(m: OracleModel, h: np.ndarray) -> np.ndarray:
    """Last-row RMSNorm then untied head (model.py:495-503)."""
    x = rmsnorm(h[-1:], m.p["final_norm.gain"], m.cfg.norm_eps)
    return (x @ m.p["lm_head.weight"].T)[0]


@dataclass
class Prefill:
    keys: list[np.ndarray]   # position-free keys per layer (rows, Hkv, d)
    values: list[np.ndarray]
    logits: np.ndarray
    maps: list[np.ndarray] | None = None


def prefill_full(m: OracleModel, ids: Sequence[int], capture: bool = False) -> Prefill:
    """model.py:506-535."""
    h = embed(m, ids)
    pos = np.arange(h.shape[0], dtype=np.int64)
    keys, values, maps = [], [], []
    for layer in range(m.cfg.n_layers):
        h, k, _, v, w = block(m, layer, h, pos, None)
        keys.append(k)
        values.append(v)
        if capture:
            maps.append(w)
    return Prefill(keys, values, final_logits(m, h), maps if capture else None)


@dataclass
class Chunk:
    """ChunkCache (kv_store.py:70-116): position-free keys, prefix_len."""
    keys: list[np.ndarray]
    values: list[np.ndarray]
    token_ids: list[int]
    prefix_len: int

    @property
    def n_rows(self) -> int:
        return self.keys[0].shape[0]

    @property
    def chunk_len(self) -> int:
        return self.n_rows - self.prefix_len

    @property
    def chunk_ids(self) -> list[int]:
        return self.token_ids[self.prefix_len:]


def prefill_chunk(m: OracleModel, prefix_ids, chunk_ids) -> Chunk:
    """model.py:538-565."""
    ids = list(prefix_ids) + list(chunk_ids)
    r = prefill_full(m, ids)
    return Chunk(r.keys, r.values, ids, len(list(prefix_ids)))


@dataclass
class Merged:
    """MergedCache (kv_store.py:133-183): rotated keys at global positions."""
    keys: list[np.ndarray]
    values: list[np.ndarray]
    token_ids: list[int]
    sink_len: int
    chunk_lens: tuple[int, ...]
    source: list[tuple[int, int]]
    recomputed_rows: tuple[int, ...] = ()

    @property
    def n_rows(self) -> int:
        return self.keys[0].shape[0]

    @property
    def total(self) -> int:
        return self.sink_len + sum(self.chunk_lens)


def merge(chunks: Sequence[Chunk], head_dim: int, base: float) -> Merged:
    """Keep chunk 0's prefix, concatenate every chunk's body, rotate keys to
    global positions 0..L-1, copy values (kv_store.py:193-258)."""
    first = chunks[0]
    sink = first.prefix_len
    for i, c in enumerate(chunks):
        if c.prefix_len != sink or c.token_ids[:sink] != first.token_ids[:sink]:
            raise ValueError(f"chunk {i} prefix mismatch")
    lens = tuple(c.chunk_len for c in chunks)
    pos = np.arange(sink + sum(lens), dtype=np.int64)
    ids = list(first.token_ids[:sink])
    src = [(0, r) for r in range(sink)]
    for ci, c in enumerate(chunks):
        ids += c.chunk_ids
        src += [(ci, sink + j) for j in range(c.chunk_len)]
    keys, values = [], []
    for layer in range(len(first.keys)):
        kr = np.concatenate([first.keys[layer][:sink]] + [c.keys[layer][sink:] for c in chunks])
        vr = np.concatenate([first.values[layer][:sink]] + [c.values[layer][sink:] for c in chunks])
        keys.append(rope_rotate(kr, pos, head_dim, base))
        values.append(np.ascontiguousarray(vr))
    return Merged(keys, values, ids, sink, lens, src)


def forward_on_cache(m: OracleModel, banks, n_past: int, ids, *, knobs=None, capture=False):
    """_forward_against_cache (model.py:568-607) without mutation; banks are
    (rotated keys, values) per layer. Returns (logits, maps, new k_rot, new v)."""
    h = embed(m, ids)
    pos = np.arange(n_past, n_past + h.shape[0], dtype=np.int64)
    maps, ks, vs = [], [], []
    for layer in range(m.cfg.n_layers):
        h, _, k_rot, v, w = block(m, layer, h, pos, banks[layer], knobs=knobs)
        ks.append(k_rot)
        vs.append(v)
        if capture:
            maps.append(w)
    return final_logits(m, h), (maps if capture else None), ks, vs


def extend(m: OracleModel, cache: Merged, ids, *, knobs=None) -> np.ndarray:
    """extend_cache on a merged cache (model.py:610-629): appends rows."""
    n_past = cache.n_rows
    logits, _, ks, vs = forward_on_cache(
        m, list(zip(cache.keys, cache.values)), n_past, ids, knobs=knobs)
    for layer in range(m.cfg.n_layers):
        cache.keys[layer] = np.concatenate([cache.keys[layer], ks[layer]])
        cache.values[layer] = np.concatenate([cache.values[layer], vs[layer]])
    cache.token_ids += [int(t) for t in ids]
    cache.source += [(-1, n_past + i) for i in range(len(ids))]
    return logits


def selective(m: OracleModel, cache: Merged, indices) -> Merged:
    """Selective recompute (model.py:669-728): selected rows restart from
    embeddings; per layer their fresh K/V overwrite the bank first, then they
    attend over the hybrid bank with row limit = own position + 1."""
    idx = np.asarray(sorted(int(i) for i in indices), dtype=np.int64)
    if idx.size == 0:
        return cache
    if len(np.unique(idx)) != idx.size:
        raise ValueError("selection contains duplicate indices")
    if idx[0] < cache.sink_len:
        raise ValueError("selection index inside the retained shared prefix")
    if idx[-1] >= cache.total:
        raise ValueError("selection index out of range")
    cfg = m.cfg
    h = embed(m, [cache.token_ids[i] for i in idx])
    for layer in range(cfg.n_layers):
        q, k, v = qkv_project(m, layer, h)
        q_rot = rope_rotate(q, idx, cfg.d_head, cfg.rope_base)
        k_rot = rope_rotate(k, idx, cfg.d_head, cfg.rope_base)
        cache.keys[layer][idx] = k_rot
        cache.values[layer][idx] = v
        ctx, _ = attend(q_rot.transpose(1, 0, 2), cache.keys[layer].transpose(1, 0, 2),
                        cache.values[layer].transpose(1, 0, 2), idx + 1)
        h = h + out_project(m, layer, ctx.transpose(1, 0, 2))
        h = h + mlp(m, layer, h)
    cache.recomputed_rows = tuple(int(i) for i in idx)
    return cache


# --------------------------------------------------------------------------
# selection (selector.py)
# --------------------------------------------------------------------------


def aux_scores(aux: OracleModel, aux_chunks: Sequence[Chunk], query_ids) -> np.ndarray:
    """Per chunk: forward the query over the chunk cache at local positions,
    take the last layer's weights on chunk columns [prefix_len, n_rows), mean
    over heads then over query rows (selector.py:132-179)."""
    cfg = aux.cfg
    out = []
    for c in aux_chunks:
        pos = np.arange(c.n_rows, dtype=np.int64)
        banks = [(rope_rotate(k, pos, cfg.d_head, cfg.rope_base), v)
                 for k, v in zip(c.keys, c.values)]
        _, maps, _, _ = forward_on_cache(aux, banks, c.n_rows, query_ids, capture=True)
        last = maps[-1]
        out.append(last[:, :, c.prefix_len:c.n_rows].mean(axis=0).mean(axis=0))
    return np.concatenate(out).astype(F32)


def budget(ratio: float, n: int) -> int:
    """ceil(ratio*n) from the ratio's decimal rendering (selector.py:113-123)."""
    if n < 0:
        raise ValueError("token count must be non-negative")
    return max(0, min(n, math.ceil(Fraction(str(float(ratio))) * n)))


def top_k_stable(scores: np.ndarray, k: int) -> np.ndarray:
    """Highest scores first, lower index on ties (selector.py:126-129)."""
    return np.sort(np.argsort(-np.asarray(scores), kind="stable")[:k])


@dataclass(frozen=True)
class Window:
    window_id: int
    chunk: int
    start: int
    end: int
    selected: int
    kept: bool
    partial: bool


def select(scores: np.ndarray, chunk_lens: Sequence[int], ratio: float,
           window_len: int = 8, threshold: int = 5, expand: bool = False):
    """Budgeted top-k then the per-chunk window rule (selector.py:182-214).
    Returns (indices tuple, windows tuple)."""
    n = int(scores.size)
    cand = np.zeros(n, dtype=bool)
    b = budget(ratio, n)
    if b:
        cand[top_k_stable(scores, b)] = True
    picked: list[int] = []
    windows: list[Window] = []
    base = 0
    for ci, clen in enumerate(chunk_lens):
        for ws in range(0, clen, window_len):
            we = min(ws + window_len, clen)
            lo, hi = base + ws, base + we
            cnt = int(cand[lo:hi].sum())
            partial = (we - ws) < window_len
            kept = cnt > 0 and (partial or cnt >= threshold)
            if kept:
                picked += list(range(lo, hi)) if expand else [int(i) + lo for i in np.flatnonzero(cand[lo:hi])]
            windows.append(Window(len(windows), ci, lo, hi, cnt, kept, partial))
        base += clen
    return tuple(picked), tuple(windows)


# --------------------------------------------------------------------------
# strategies (pipeline.py)
# --------------------------------------------------------------------------


@dataclass
class Outcome:
    cache: Merged
    logits: np.ndarray
    indices: tuple[int, ...]
    windows: tuple[Window, ...] = ()
    scores: np.ndarray | None = None


def cacheclip(primary: OracleModel, aux: OracleModel, chunks: Sequence[Chunk],
              aux_chunks: Sequence[Chunk], query_ids, ratio: float, *,
              window_len: int = 8, threshold: int = 5, expand: bool = False,
              knobs=None) -> Outcome:
    """cacheclip_prefill (pipeline.py:156-226) for a shared tokenizer, where
    the span alignment is the identity and the plan is the aux selection
    shifted by the sink length (selector.py:217-245)."""
    merged = merge(chunks, primary.cfg.d_head, primary.cfg.rope_base)
    s = aux_scores(aux, aux_chunks, query_ids)
    idx, wins = select(s, [c.chunk_len for c in aux_chunks], ratio, window_len, threshold, expand)
    plan = tuple(i + merged.sink_len for i in idx)
    selective(primary, merged, plan)
    logits = extend(primary, merged, query_ids, knobs=knobs)
    return Outcome(merged, logits, plan, wins, s)


def cacheblend_select(m: OracleModel, merged: Merged, ratio: float):
    """CacheBlend-style discrepancy selection (selector.py:248-291): layer 0
    recomputed for every merged row with global context, then the L2 drift
    of layer 1's value projection against the cached values, top
    ceil(ratio*N) with no windows. GQA: the L2 runs over the KV heads (the
    reference's MHA-expanded values give sqrt(G) x this, same order).
    Returns (indices, discrepancy)."""
    if m.cfg.n_layers < 2:
        raise ValueError("discrepancy selection needs at least two layers")
    if not 0.0 <= ratio <= 1.0:
        raise ValueError(f"ratio must be in [0, 1], got {ratio}")
    sink, total = merged.sink_len, merged.total
    n = total - sink
    h = embed(m, merged.token_ids[:total])
    h1 = block(m, 0, h, np.arange(total, dtype=np.int64), None)[0]
    _, _, v1 = qkv_project(m, 1, h1)   # == value_projection (model.py:367-389)
    diff = v1[sink:] - merged.values[1][sink:total]
    disc = np.sqrt(np.sum(np.square(diff.reshape(n, -1)), axis=1))
    chosen = top_k_stable(disc, budget(ratio, n))
    return tuple(int(i) + sink for i in chosen), disc


def cacheblend(m: OracleModel, chunks: Sequence[Chunk], query_ids, ratio: float) -> Outcome:
    """cacheblend_prefill (pipeline.py:229-255): prefix-less chunk caches,
    discrepancy selection, selective recompute, then the query."""
    for i, c in enumerate(chunks):
        if c.prefix_len != 0:
            raise ValueError(f"chunk {i} carries a shared prefix; this baseline concatenates raw chunks")
    merged = merge(chunks, m.cfg.d_head, m.cfg.rope_base)
    plan, disc = cacheblend_select(m, merged, ratio)
    selective(m, merged, plan)
    logits = extend(m, merged, query_ids)
    return Outcome(merged, logits, plan, (), disc)


def full_prefill(m: OracleModel, ids) -> Prefill:
    """full_attention_prefill (pipeline.py:77-84)."""
    return prefill_full(m, ids)


def context_ids(chunks: Sequence[Chunk], query_ids) -> list[int]:
    """reuse_context_ids (pipeline.py:66-74)."""
    ids = list(chunks[0].token_ids[:chunks[0].prefix_len])
    for c in chunks:
        ids += c.chunk_ids
    return ids + [int(t) for t in query_ids]
