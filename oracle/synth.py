"""Seeded synthetic RAG workloads shared by the oracle, the golden-fixture
generator and the parity tests (test infrastructure; see cacheclip_oracle.py).

Value distributions follow SURVEY.md §8: token ids uniform in [0, V) from
``np.random.default_rng(seed)``; weights from the reference init recipe.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .cacheclip_oracle import OracleConfig


@dataclass(frozen=True)
class Workload:
    name: str
    primary: OracleConfig
    aux: OracleConfig
    prefix_len: int
    n_chunks: int
    chunk_len: int
    query_len: int
    ratio: float = 0.2
    window_len: int = 8
    window_threshold: int = 5
    primary_seed: int = 0
    aux_seed: int = 1
    bias_std: float = 0.0
    chunk_lens: tuple = ()   # ragged chunks (overrides n_chunks x chunk_len)

    def token_ids(self, seed: int = 0):
        """(prefix, [chunk ids], query) drawn from one generator; aux shares
        the tokenizer (Qwen pair), so ids are valid for both vocabularies."""
        v = min(self.primary.vocab_size, self.aux.vocab_size)
        rng = np.random.default_rng(seed)
        prefix = rng.integers(0, v, self.prefix_len).tolist()
        lens = self.chunk_lens or (self.chunk_len,) * self.n_chunks
        chunks = [rng.integers(0, v, n).tolist() for n in lens]
        query = rng.integers(0, v, self.query_len).tolist()
        return prefix, chunks, query


# BASELINE.json configs[0]: tiny Llama-style primary (4 layers, d=256, GQA
# 4/2) + 2-layer auxiliary, 8 chunks x 128 tokens + 32-token query, recomp 20%.
C1_PRIMARY = OracleConfig(n_layers=4, n_heads=4, n_kv_heads=2, d_model=256, d_head=64,
                          d_ff=1024, vocab_size=512, rope_base=1e4, norm_eps=1e-5,
                          activation="silu", mlp_gated=True)
C1_AUX = OracleConfig(n_layers=2, n_heads=2, n_kv_heads=2, d_model=128, d_head=64,
                      d_ff=512, vocab_size=512, rope_base=1e4, norm_eps=1e-5,
                      activation="silu", mlp_gated=True)
C1 = Workload("c1", C1_PRIMARY, C1_AUX, prefix_len=16, n_chunks=8, chunk_len=128, query_len=32)

# Same shapes, exact-budget window mode (H2): |plan| == ceil(0.2 * N).
C1_EXACT = Workload("c1_exact", C1_PRIMARY, C1_AUX, prefix_len=16, n_chunks=8, chunk_len=128,
                    query_len=32, window_threshold=1)

# MHA primary with Qwen-style QKV bias (non-zero so the path is exercised),
# base 1e6, eps 1e-6, non-gated gelu MLP and ragged-free small chunks: pins
# the bias / gelu / MHA paths bit for bit against the reference.
B1_PRIMARY = OracleConfig(n_layers=2, n_heads=2, n_kv_heads=2, d_model=128, d_head=64,
                          d_ff=256, vocab_size=300, rope_base=1e6, norm_eps=1e-6,
                          activation="gelu", mlp_gated=False, attn_bias=True, mlp_bias=True)
B1_AUX = OracleConfig(n_layers=2, n_heads=2, n_kv_heads=1, d_model=128, d_head=64,
                      d_ff=256, vocab_size=300, rope_base=1e6, norm_eps=1e-6,
                      activation="silu", mlp_gated=True, attn_bias=True)
B1 = Workload("b1", B1_PRIMARY, B1_AUX, prefix_len=8, n_chunks=3, chunk_len=64, query_len=16,
              ratio=0.4, window_threshold=3, bias_std=0.05)

# Ragged chunks (1-token, sub-window, tile-straddling lengths), GQA primary,
# MHA aux with QKV bias, window threshold 3, ratio 0.3: pins partial windows
# and per-chunk window restarts against the reference.
R1 = Workload("r1", C1_PRIMARY, B1_AUX, prefix_len=5, n_chunks=6, chunk_len=0, query_len=9, ratio=0.3,
              window_threshold=3, bias_std=0.05, chunk_lens=(37, 1, 130, 8, 64, 7))

# Cross-tokenizer pair (selector.py:217-245 +
# tokenizers.py:151-177): the primary tokenizes single characters, the
# scoring model's tokenizer adds 64 two-character merges, so an aux token may
# cover two primary tokens and the plan is projected through the spans.
X1_AUX = OracleConfig(n_layers=2, n_heads=2, n_kv_heads=2, d_model=128, d_head=64,
                      d_ff=512, vocab_size=512 + 64, rope_base=1e4, norm_eps=1e-5,
                      activation="silu", mlp_gated=True)
X1_RATIO, X1_WINDOW_THRESHOLD = 0.25, 2


def cross_tokenizer_case(seed: int = 0, n_chunks: int = 5, chunk_chars: int = 96, prefix_chars: int = 11,
                         query_chars: int = 20):
    """(primary vocab, aux vocab, prefix text, [chunk texts], query text).
    Texts are random characters of the primary vocab with frequent merge
    pairs, so both tokenizations differ in length and alignment."""
    base = [chr(0x4E00 + i) for i in range(C1_PRIMARY.vocab_size)]
    merges = [base[2 * k] + base[2 * k + 1] for k in range(X1_AUX.vocab_size - len(base))]
    rng = np.random.default_rng(seed)

    def text(n):
        out = []
        while len(out) < n:
            if rng.random() < 0.4:
                out.extend(merges[int(rng.integers(0, len(merges)))])
            else:
                out.append(base[int(rng.integers(0, len(base)))])
        return "".join(out[:n])

    return base, base + merges, text(prefix_chars), [text(chunk_chars) for _ in range(n_chunks)], text(query_chars)


# Qwen2.5-7B / 0.5B shapes (BASELINE configs[1..2]); GPU-only sizes.
QWEN7B = OracleConfig(n_layers=28, n_heads=28, n_kv_heads=4, d_model=3584, d_head=128,
                      d_ff=18944, vocab_size=152064, rope_base=1e6, norm_eps=1e-6,
                      activation="silu", mlp_gated=True, attn_bias=True)
QWEN05B = OracleConfig(n_layers=24, n_heads=14, n_kv_heads=2, d_model=896, d_head=64,
                       d_ff=4864, vocab_size=151936, rope_base=1e6, norm_eps=1e-6,
                       activation="silu", mlp_gated=True, attn_bias=True)
QWEN14B = OracleConfig(n_layers=48, n_heads=40, n_kv_heads=8, d_model=5120, d_head=128,
                       d_ff=13824, vocab_size=152064, rope_base=1e6, norm_eps=1e-6,
                       activation="silu", mlp_gated=True, attn_bias=True)
C2 = Workload("c2", QWEN7B, QWEN05B, prefix_len=32, n_chunks=16, chunk_len=512, query_len=32)
C3 = Workload("c3", QWEN7B, QWEN05B, prefix_len=32, n_chunks=64, chunk_len=512, query_len=32)
C4 = Workload("c4", QWEN14B, QWEN05B, prefix_len=32, n_chunks=400, chunk_len=500, query_len=32)
C5 = Workload("c5", QWEN7B, QWEN05B, prefix_len=32, n_chunks=32, chunk_len=512, query_len=32)

WORKLOADS = {w.name: w for w in (C1, C1_EXACT, B1, R1, C2, C3, C4, C5)}


# Full-size parity (VERDICT r1 "What's missing" #1): the reference itself is
# run at the benchmarked scoring shapes (24-layer 0.5B-shape scoring model at
# C2 and C3) and with a depth-truncated 7B-shape primary at C2
# (tests/golden/make_golden_scale.py). Weights come from
# ``seeded_params(..., fast=True)`` so the GPU box regenerates them in seconds.
P2_PRIMARY = OracleConfig(n_layers=2, n_heads=28, n_kv_heads=4, d_model=3584, d_head=128,
                          d_ff=18944, vocab_size=152064, rope_base=1e6, norm_eps=1e-6,
                          activation="silu", mlp_gated=True, attn_bias=True)
P2 = Workload("p2", P2_PRIMARY, QWEN05B, prefix_len=32, n_chunks=16, chunk_len=512, query_len=32,
              window_threshold=1)
# the same request under the paper's default 8/5 window rule: a few hundred
# recomputed rows, the launches that take the small-grid split-KV attention
# and the split-K GEMMs
P2D = Workload("p2d", P2_PRIMARY, QWEN05B, prefix_len=32, n_chunks=16, chunk_len=512, query_len=32,
               window_threshold=5)
SCALE_RATIOS = (0.05, 0.2, 0.4)
SCALE_THRESHOLDS = (5, 1)   # the paper's default 8/5 rule and the exact-budget rule (H2)
