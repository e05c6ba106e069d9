"""Model configuration and rotary geometry (model.py:62-106, tensor_core.py:23-51).

``ModelConfig`` keeps every reference field and adds two: ``n_kv_heads``
(grouped-query attention; 0 means n_heads, the reference's MHA) and
``dtype`` — the arithmetic the device path runs the model in:
  * "bf16": bf16 weights and K/V cache, fp32 accumulation and residual stream
    (tcgen05 kind::f16). The primary model's throughput mode.
  * "fp32": fp32 weights/cache with 3xTF32 GEMMs (kind::tf32 on hi/lo splits)
    and fp32 attention — fp32-faithful, used by the scoring model so that
    token selection reproduces the reference's fp32 scores.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, fields

import numpy as np

from .errors import DimensionError, WeightFormatError

_ACTIVATIONS = ("gelu", "silu")
_DTYPES = ("bf16", "fp32")


@dataclass(frozen=True)
class RopeParams:
    head_dim: int
    base: float = 10000.0

    def __post_init__(self) -> None:
        if self.head_dim <= 0 or self.head_dim % 2:
            raise DimensionError(f"rotary head_dim must be positive and even, got {self.head_dim}")
        if self.base <= 1.0:
            raise ValueError(f"rotary base must exceed 1, got {self.base}")

    @property
    def inv_freq(self) -> np.ndarray:
        """base ** (-2i/d) in float64, formed exactly as tensor_core.py:48-50."""
        exponent = -np.arange(0, self.head_dim, 2, dtype=np.float64) / self.head_dim
        return np.ascontiguousarray(self.base ** exponent, dtype=np.float64)

    def angles(self, positions) -> tuple[np.ndarray, np.ndarray]:
        theta = np.asarray(positions, dtype=np.float64)[..., None] * self.inv_freq
        return np.cos(theta).astype(np.float32), np.sin(theta).astype(np.float32)


@dataclass(frozen=True)
class ModelConfig:
    n_layers: int
    n_heads: int
    d_model: int
    d_head: int
    d_ff: int
    vocab_size: int
    rope_base: float = 10000.0
    norm_eps: float = 1e-5
    activation: str = "gelu"
    mlp_gated: bool = False
    attn_bias: bool = False
    mlp_bias: bool = False
    tokenizer_id: str = ""
    n_kv_heads: int = 0
    dtype: str = "bf16"

    def __post_init__(self) -> None:
        for name in ("n_layers", "n_heads", "d_model", "d_head", "d_ff", "vocab_size"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        if self.activation not in _ACTIVATIONS:
            raise ValueError(f"activation must be one of {_ACTIVATIONS}")
        if self.dtype not in _DTYPES:
            raise ValueError(f"dtype must be one of {_DTYPES}")
        if self.n_kv_heads < 0 or self.n_heads % self.kv_heads:
            raise DimensionError(f"n_heads {self.n_heads} not a multiple of n_kv_heads {self.kv_heads}")
        self.rope  # validates head_dim / base

    @property
    def kv_heads(self) -> int:
        return self.n_kv_heads or self.n_heads

    @property
    def group(self) -> int:
        return self.n_heads // self.kv_heads

    @property
    def rope(self) -> RopeParams:
        return RopeParams(self.d_head, self.rope_base)

    @property
    def attn_width(self) -> int:
        return self.n_heads * self.d_head

    @property
    def kv_width(self) -> int:
        return self.kv_heads * self.d_head

    def to_dict(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}

    @classmethod
    def from_dict(cls, data: dict) -> "ModelConfig":
        known = {f.name for f in fields(cls)}
        unknown = set(data) - known
        if unknown:
            raise WeightFormatError(f"unknown config fields: {sorted(unknown)}")
        try:
            return cls(**data)
        except TypeError as exc:
            raise WeightFormatError(f"bad config block: {exc}") from exc

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), sort_keys=True)


def expected_tensors(config: ModelConfig) -> list[tuple[str, tuple[int, ...]]]:
    """Tensor table in manifest order (model.py:109-137), GQA-aware."""
    dm, qw, kw, ff = config.d_model, config.attn_width, config.kv_width, config.d_ff
    out: list[tuple[str, tuple[int, ...]]] = [("embed.weight", (config.vocab_size, dm))]
    for i in range(config.n_layers):
        p = f"layers.{i}"
        out.append((f"{p}.attn_norm.gain", (dm,)))
        out += [(f"{p}.attn.wq.weight", (dm, qw)), (f"{p}.attn.wk.weight", (dm, kw)),
                (f"{p}.attn.wv.weight", (dm, kw)), (f"{p}.attn.wo.weight", (qw, dm))]
        if config.attn_bias:
            out += [(f"{p}.attn.wq.bias", (qw,)), (f"{p}.attn.wk.bias", (kw,)),
                    (f"{p}.attn.wv.bias", (kw,)), (f"{p}.attn.wo.bias", (dm,))]
        out.append((f"{p}.mlp_norm.gain", (dm,)))
        if config.mlp_gated:
            out.append((f"{p}.mlp.w_gate.weight", (dm, ff)))
        out.append((f"{p}.mlp.w_in.weight", (dm, ff)))
        out.append((f"{p}.mlp.w_out.weight", (ff, dm)))
        if config.mlp_bias:
            if config.mlp_gated:
                out.append((f"{p}.mlp.w_gate.bias", (ff,)))
            out.append((f"{p}.mlp.w_in.bias", (ff,)))
            out.append((f"{p}.mlp.w_out.bias", (dm,)))
    out.append(("final_norm.gain", (dm,)))
    out.append(("lm_head.weight", (config.vocab_size, dm)))
    return out
