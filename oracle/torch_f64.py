"""FLOAT64 RESTATEMENT (torch, any device) — test infrastructure only.

The scoring chain of the reference in float64 — ``prefill_chunk``
(model.py:538-565 via prefill_full / layer_forward, model.py:435-535) and
``aux_score_tokens`` (selector.py:132-179) — GQA-native. It is the "exact
math" yardstick for the fp32 parity question: how far the reference's own
fp32 scores and the device's fp32-faithful scores each sit from the exact
values, and which budget-boundary ties are decided below fp32 resolution.
Used only by tests/ and scripts/ diagnostics, never by the product.

Semantics follow the reference: RMSNorm x / sqrt(mean(x^2) + eps) * gain;
Q/K/V with biases; adjacent-pair RoPE with angles p * base^(-2i/d); keys
cached position-free and rotated at local positions 0..n-1 for scoring;
softmax over prefix + chunk + causal query columns with factor 1/sqrt(d);
score = mean over heads, then over queries, of the last layer's weights on
the chunk columns.
"""

from __future__ import annotations

import numpy as np
import torch

F64 = torch.float64


class F64Model:
    def __init__(self, cfg, params: dict, device):
        self.cfg = cfg
        self.dev = torch.device(device)
        self.p = {k: torch.as_tensor(np.asarray(v), dtype=F64, device=self.dev) for k, v in params.items()}
        c = cfg
        i = torch.arange(c.d_head // 2, dtype=F64, device=self.dev)
        self.inv_freq = c.rope_base ** (-2.0 * i / c.d_head)

    def w(self, layer, name):
        return self.p[f"layers.{layer}.{name}"]

    def rope(self, x, pos):  # x [n, H, D], pos [n]
        ang = pos.to(F64)[:, None] * self.inv_freq[None, :]
        cos, sin = ang.cos()[:, None, :], ang.sin()[:, None, :]
        e, o = x[..., 0::2], x[..., 1::2]
        out = torch.empty_like(x)
        out[..., 0::2] = e * cos - o * sin
        out[..., 1::2] = e * sin + o * cos
        return out

    def rms(self, x, gain):
        return x / torch.sqrt((x * x).mean(-1, keepdim=True) + self.cfg.norm_eps) * gain

    def qkv(self, layer, x):
        c = self.cfg
        out = []
        for n in ("wq", "wk", "wv"):
            y = x @ self.w(layer, f"attn.{n}.weight")
            b = self.p.get(f"layers.{layer}.attn.{n}.bias")
            out.append(y if b is None else y + b)
        q, k, v = out
        return (q.view(-1, c.n_heads, c.d_head), k.view(-1, c.kv_heads, c.d_head), v.view(-1, c.kv_heads, c.d_head))

    def attend(self, q, k, v, q_pos, k_pos, want_weights=False):
        """q [m, Hq, D] at positions q_pos over k/v [n, Hkv, D] (rotated) at
        k_pos, causal by position."""
        c = self.cfg
        g = c.n_heads // c.kv_heads
        kk = k.repeat_interleave(g, 1).transpose(0, 1)   # [Hq, n, D]
        vv = v.repeat_interleave(g, 1).transpose(0, 1)
        s = torch.matmul(q.transpose(0, 1), kk.transpose(1, 2)) / np.sqrt(c.d_head)  # [Hq, m, n]
        mask = k_pos[None, :] > q_pos[:, None]
        s = s.masked_fill(mask[None], float("-inf"))
        w = torch.softmax(s, dim=-1)
        ctx = torch.matmul(w, vv).transpose(0, 1).reshape(q.shape[0], -1)
        return ctx, (w if want_weights else None)

    def mlp(self, layer, x):
        c = self.cfg
        up = x @ self.w(layer, "mlp.w_in.weight")
        b = self.p.get(f"layers.{layer}.mlp.w_in.bias")
        if b is not None:
            up = up + b
        if c.mlp_gated:
            gt = x @ self.w(layer, "mlp.w_gate.weight")
            gb = self.p.get(f"layers.{layer}.mlp.w_gate.bias")
            if gb is not None:
                gt = gt + gb
            a = torch.nn.functional.silu(gt) * up if c.activation == "silu" else \
                torch.nn.functional.gelu(gt, approximate="tanh") * up
        else:
            a = torch.nn.functional.silu(up) if c.activation == "silu" else \
                torch.nn.functional.gelu(up, approximate="tanh")
        y = a @ self.w(layer, "mlp.w_out.weight")
        b = self.p.get(f"layers.{layer}.mlp.w_out.bias")
        return y if b is None else y + b

    def out_proj(self, layer, ctx):
        y = ctx @ self.w(layer, "attn.wo.weight")
        b = self.p.get(f"layers.{layer}.attn.wo.bias")
        return y if b is None else y + b

    def prefill(self, ids):
        """Position-free K/V [L][n][Hkv][D] of a causal prefill at 0..n-1."""
        c = self.cfg
        ids_t = torch.as_tensor(ids, device=self.dev)
        pos = torch.arange(len(ids), device=self.dev)
        h = self.p["embed.weight"][ids_t]
        ks, vs = [], []
        for l in range(c.n_layers):
            x = self.rms(h, self.w(l, "attn_norm.gain"))
            q, k, v = self.qkv(l, x)
            ks.append(k)
            vs.append(v)
            ctx, _ = self.attend(self.rope(q, pos), self.rope(k, pos), v, pos, pos)
            h = h + self.out_proj(l, ctx)
            x = self.rms(h, self.w(l, "mlp_norm.gain"))
            h = h + self.mlp(l, x)
        return torch.stack(ks), torch.stack(vs)

    def score_chunk(self, k_cache, v_cache, prefix_len, query_ids):
        """aux_score_tokens for one chunk: its cache (position-free) extended
        by the query rows; last layer's weights on the chunk columns."""
        c = self.cfg
        n = k_cache.shape[1]
        Q = len(query_ids)
        ids_t = torch.as_tensor(query_ids, device=self.dev)
        cpos = torch.arange(n, device=self.dev)
        qpos = torch.arange(n, n + Q, device=self.dev)
        allpos = torch.arange(n + Q, device=self.dev)
        h = self.p["embed.weight"][ids_t]
        for l in range(c.n_layers):
            x = self.rms(h, self.w(l, "attn_norm.gain"))
            q, k, v = self.qkv(l, x)
            kb = torch.cat([self.rope(k_cache[l], cpos), self.rope(k, qpos)])
            vb = torch.cat([v_cache[l], v])
            last = l == c.n_layers - 1
            ctx, w = self.attend(self.rope(q, qpos), kb, vb, qpos, allpos, want_weights=last)
            if last:
                return w[:, :, prefix_len:n].mean(0).mean(0)
            h = h + self.out_proj(l, ctx)
            x = self.rms(h, self.w(l, "mlp_norm.gain"))
            h = h + self.mlp(l, x)


def scores_f64(model: F64Model, prefix, chunk_ids, query, caches=None):
    """float64 scores of every chunk (concatenated), and the f64 caches."""
    out, kept = [], []
    for i, c in enumerate(chunk_ids):
        k, v = caches[i] if caches is not None else model.prefill(list(prefix) + list(c))
        kept.append((k, v))
        out.append(model.score_chunk(k, v, len(prefix), query))
    return torch.cat(out), kept
