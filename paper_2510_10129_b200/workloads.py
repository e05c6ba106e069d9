"""Synthetic RAG workloads of BASELINE.json (shapes from SURVEY.md §8).

Random-init weights of the named architectures (no checkpoints offline) and
uniform random token ids: prefix P, n chunks x C tokens, query Q.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import ModelConfig

QWEN25_7B = ModelConfig(n_layers=28, n_heads=28, n_kv_heads=4, d_model=3584, d_head=128, d_ff=18944,
                        vocab_size=152064, rope_base=1e6, norm_eps=1e-6, activation="silu", mlp_gated=True,
                        attn_bias=True, tokenizer_id="qwen2.5", dtype="bf16")
QWEN25_05B = ModelConfig(n_layers=24, n_heads=14, n_kv_heads=2, d_model=896, d_head=64, d_ff=4864,
                         vocab_size=151936, rope_base=1e6, norm_eps=1e-6, activation="silu", mlp_gated=True,
                         attn_bias=True, tokenizer_id="qwen2.5", dtype="fp32")
QWEN25_14B = ModelConfig(n_layers=48, n_heads=40, n_kv_heads=8, d_model=5120, d_head=128, d_ff=13824,
                         vocab_size=152064, rope_base=1e6, norm_eps=1e-6, activation="silu", mlp_gated=True,
                         attn_bias=True, tokenizer_id="qwen2.5", dtype="bf16")
TINY_PRIMARY = ModelConfig(n_layers=4, n_heads=4, n_kv_heads=2, d_model=256, d_head=64, d_ff=1024, vocab_size=512,
                           rope_base=1e4, norm_eps=1e-5, activation="silu", mlp_gated=True, tokenizer_id="tiny",
                           dtype="bf16")
TINY_AUX = ModelConfig(n_layers=2, n_heads=2, n_kv_heads=2, d_model=128, d_head=64, d_ff=512, vocab_size=512,
                       rope_base=1e4, norm_eps=1e-5, activation="silu", mlp_gated=True, tokenizer_id="tiny",
                       dtype="fp32")


@dataclass(frozen=True)
class RagWorkload:
    name: str
    primary: ModelConfig
    aux: ModelConfig
    prefix_len: int
    n_chunks: int
    chunk_len: int
    query_len: int
    requests: int = 1
    description: str = ""

    @property
    def context_rows(self) -> int:
        return self.prefix_len + self.n_chunks * self.chunk_len

    @property
    def n_tokens(self) -> int:
        return self.n_chunks * self.chunk_len

    def token_ids(self, seed: int):
        v = min(self.primary.vocab_size, self.aux.vocab_size)
        rng = np.random.default_rng(seed)
        prefix = rng.integers(0, v, self.prefix_len).tolist()
        chunks = [rng.integers(0, v, self.chunk_len).tolist() for _ in range(self.n_chunks)]
        query = rng.integers(0, v, self.query_len).tolist()
        return prefix, chunks, query


WORKLOADS = {
    "c1": RagWorkload("c1", TINY_PRIMARY, TINY_AUX, 16, 8, 128, 32,
                      description="tiny Llama-style primary (4L d=256) + 2L aux, 8x128 + 32-token query"),
    "c2": RagWorkload("c2", QWEN25_7B, QWEN25_05B, 32, 16, 512, 32,
                      description="Qwen2.5-7B-shape primary + 0.5B-shape aux, 16x512 chunks (8K ctx)"),
    "c3": RagWorkload("c3", QWEN25_7B, QWEN25_05B, 32, 64, 512, 32,
                      description="Qwen2.5-7B-shape primary + 0.5B-shape aux, 64x512 chunks (32K ctx)"),
    "c4": RagWorkload("c4", QWEN25_14B, QWEN25_05B, 32, 400, 500, 32,
                      description="Qwen2.5-14B-shape primary + 0.5B aux, 400x500 chunks (200K ctx)"),
    "c5": RagWorkload("c5", QWEN25_7B, QWEN25_05B, 32, 32, 512, 32, requests=64,
                      description="64 concurrent RAG requests x 16K ctx, Qwen2.5-7B/0.5B shapes"),
}
