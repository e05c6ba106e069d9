"""Device-resident model weights in the layouts the sm_100a kernels consume.

Reference params are input-major (x @ W, model.py:12-14). On device every
projection is stored transposed, [out, in] (K-major for the tcgen05 GEMM):
  w_qkv  [(Hq + 2 Hkv) * dh, d]   q | k | v rows (one GEMM, RoPE+scatter epilogue)
  w_o    [d, Hq * dh]
  w_gu   [2 * ff_pad, d]          gate/up interleaved in 128-row blocks (GLU epilogue)
         or w_in [ff, d] for non-gated MLPs
  w_down [d, ff]
bf16 models store bf16 matrices; fp32 models store the 3xTF32 weight split
[hi | lo | hi] along K (3*in columns). Norm gains and biases stay fp32.
"""

from __future__ import annotations

import ctypes
import hashlib
import json
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .config import ModelConfig, expected_tensors
from .errors import MissingTensorError, TensorShapeError, WeightFormatError

GLU_BLOCK = 128


def _ptr(t):
    return None if t is None else t.data_ptr()


@dataclass
class LayerWeights:
    attn_norm: torch.Tensor
    w_qkv: torch.Tensor
    b_qkv: torch.Tensor | None
    w_o: torch.Tensor
    b_o: torch.Tensor | None
    mlp_norm: torch.Tensor
    w_up: torch.Tensor          # interleaved gate/up (gated) or w_in (plain)
    b_up: torch.Tensor | None
    w_down: torch.Tensor
    b_down: torch.Tensor | None


@dataclass
class Model:
    """A model whose forward runs on one B200 (see config.ModelConfig.dtype)."""

    config: ModelConfig
    embed: torch.Tensor
    layers: list[LayerWeights]
    final_norm: torch.Tensor
    lm_head: torch.Tensor | None
    fingerprint: str = ""
    device: torch.device = field(default_factory=lambda: torch.device("cuda"))
    _desc: object = field(default=None, repr=False, compare=False)

    def desc(self):
        """C-ABI description (cc_model_desc) of this model's device weights;
        built once, kept alive with the model."""
        if self._desc is None:
            c = self.config
            arr = (_lib.LayerWeightsDesc * c.n_layers)()
            for i, lw in enumerate(self.layers):
                arr[i] = _lib.LayerWeightsDesc(
                    lw.w_qkv.data_ptr(), _ptr(lw.b_qkv), lw.w_qkv.shape[0], lw.w_o.data_ptr(), _ptr(lw.b_o),
                    lw.attn_norm.data_ptr(), lw.mlp_norm.data_ptr(), lw.w_up.data_ptr(), _ptr(lw.b_up),
                    lw.w_up.shape[0], lw.w_down.data_ptr(), _ptr(lw.b_down))
            inv = (ctypes.c_double * (c.d_head // 2))(*c.rope.inv_freq.tolist())
            act = _lib.CC_ACT_SILU if c.activation == "silu" else _lib.CC_ACT_GELU_TANH
            head = self.lm_head
            d = _lib.ModelDesc(
                c.n_layers, c.n_heads, c.kv_heads, c.d_head, c.d_model, c.d_ff, c.vocab_size,
                _lib.CC_BF16 if c.dtype == "bf16" else _lib.CC_F32, int(c.mlp_gated), act, c.norm_eps,
                self.embed.data_ptr(), self.final_norm.data_ptr(), _ptr(head),
                _lib.CC_BF16 if head is not None and head.dtype == torch.bfloat16 else _lib.CC_F32,
                ctypes.cast(arr, ctypes.POINTER(_lib.LayerWeightsDesc)),
                ctypes.cast(inv, ctypes.POINTER(ctypes.c_double)))
            self._desc = (d, arr, inv)
        return self._desc[0]

    @property
    def wdtype(self) -> torch.dtype:
        return torch.bfloat16 if self.config.dtype == "bf16" else torch.float32

    @property
    def ff_pad(self) -> int:
        c = self.config
        return -(-c.d_ff // GLU_BLOCK) * GLU_BLOCK if c.mlp_gated else c.d_ff

    def nbytes(self) -> int:
        tot = self.embed.numel() * self.embed.element_size() + self.final_norm.numel() * 4
        if self.lm_head is not None:
            tot += self.lm_head.numel() * self.lm_head.element_size()
        for lw in self.layers:
            for t in vars(lw).values():
                if isinstance(t, torch.Tensor):
                    tot += t.numel() * t.element_size()
        return tot


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _matrix(w_in_out: torch.Tensor, dtype: str) -> torch.Tensor:
    """[in, out] fp32 -> device [out, in] in the model's operand format."""
    wt = w_in_out.t().contiguous().float()
    if dtype == "bf16":
        return wt.to(torch.bfloat16)
    rows, cols = wt.shape
    out = torch.empty(rows, 3 * cols, dtype=torch.float32, device=wt.device)
    _lib.call("cc_convert_matrix", wt.data_ptr(), rows, cols, out.data_ptr(), _lib.CC_F32_SPLIT3, 1, _stream())
    return out


def _interleave_glu(gate_t: torch.Tensor, up_t: torch.Tensor) -> torch.Tensor:
    """[ff, K] gate and up rows -> [2*ff_pad, K] in 128-row blocks g|u|g|u."""
    ff, k = gate_t.shape
    nb = -(-ff // GLU_BLOCK)
    pad = nb * GLU_BLOCK - ff
    if pad:
        z = torch.zeros(pad, k, dtype=gate_t.dtype, device=gate_t.device)
        gate_t = torch.cat([gate_t, z])
        up_t = torch.cat([up_t, z])
    g = gate_t.view(nb, GLU_BLOCK, k)
    u = up_t.view(nb, GLU_BLOCK, k)
    return torch.stack([g, u], dim=1).reshape(2 * nb * GLU_BLOCK, k).contiguous()


def _interleave_bias(bg: torch.Tensor, bu: torch.Tensor) -> torch.Tensor:
    ff = bg.numel()
    nb = -(-ff // GLU_BLOCK)
    pad = nb * GLU_BLOCK - ff
    if pad:
        z = torch.zeros(pad, dtype=bg.dtype, device=bg.device)
        bg, bu = torch.cat([bg, z]), torch.cat([bu, z])
    return torch.stack([bg.view(nb, GLU_BLOCK), bu.view(nb, GLU_BLOCK)], 1).reshape(-1).contiguous()


def fingerprint_params(config: ModelConfig, params: dict[str, np.ndarray]) -> str:
    """sha256 over config + float32 tensors in name order (model.py:140-147)."""
    h = hashlib.sha256()
    cfg = config.to_dict()
    cfg.pop("dtype", None)
    cfg.pop("n_kv_heads", None)
    h.update(json.dumps(cfg, sort_keys=True).encode("utf-8"))
    for name in sorted(params):
        arr = np.asarray(params[name])
        h.update(name.encode("utf-8"))
        h.update(str(arr.shape).encode("utf-8"))
        h.update(np.ascontiguousarray(arr, dtype="<f4").tobytes())
    return h.hexdigest()


def from_params(config: ModelConfig, params: dict, *, device=None, fingerprint: str | None = None) -> Model:
    """Upload reference-layout params (numpy or torch, [in, out]) to the device."""
    dev = torch.device(device if device is not None else "cuda")
    _lib.require_device(dev.index if dev.index is not None else torch.cuda.current_device())
    expected = dict(expected_tensors(config))
    for name, shape in expected.items():
        if name not in params:
            raise MissingTensorError(f"missing tensor: {name}")
        if tuple(params[name].shape) != shape:
            raise TensorShapeError(f"{name}: shape {tuple(params[name].shape)}, expected {shape}")
    extra = set(params) - set(expected)
    if extra:
        raise WeightFormatError(f"unexpected tensors: {sorted(extra)}")

    def T(name):
        v = params[name]
        if isinstance(v, np.ndarray):
            v = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32))
        return v.to(dev, dtype=torch.float32)

    c = config
    dt = c.dtype
    with torch.cuda.device(dev):
        layers = []
        for i in range(c.n_layers):
            p = f"layers.{i}"
            wq, wk, wv = T(f"{p}.attn.wq.weight"), T(f"{p}.attn.wk.weight"), T(f"{p}.attn.wv.weight")
            w_qkv = _matrix(torch.cat([wq, wk, wv], dim=1), dt)
            b_qkv = b_o = None
            if c.attn_bias:
                b_qkv = torch.cat([T(f"{p}.attn.wq.bias"), T(f"{p}.attn.wk.bias"), T(f"{p}.attn.wv.bias")])
                b_o = T(f"{p}.attn.wo.bias")
            w_o = _matrix(T(f"{p}.attn.wo.weight"), dt)
            if c.mlp_gated:
                g_t = T(f"{p}.mlp.w_gate.weight").t().contiguous()
                u_t = T(f"{p}.mlp.w_in.weight").t().contiguous()
                w_up = _matrix(_interleave_glu(g_t, u_t).t(), dt)
                b_up = (_interleave_bias(T(f"{p}.mlp.w_gate.bias"), T(f"{p}.mlp.w_in.bias"))
                        if c.mlp_bias else None)
            else:
                w_up = _matrix(T(f"{p}.mlp.w_in.weight"), dt)
                b_up = T(f"{p}.mlp.w_in.bias") if c.mlp_bias else None
            w_down = _matrix(T(f"{p}.mlp.w_out.weight"), dt)
            b_down = T(f"{p}.mlp.w_out.bias") if c.mlp_bias else None
            layers.append(LayerWeights(T(f"{p}.attn_norm.gain"), w_qkv, b_qkv, w_o, b_o,
                                       T(f"{p}.mlp_norm.gain"), w_up, b_up, w_down, b_down))
        emb = T("embed.weight")
        embed = emb.to(torch.bfloat16) if dt == "bf16" else emb
        head = T("lm_head.weight")
        lm_head = head.to(torch.bfloat16) if dt == "bf16" else head
        final_norm = T("final_norm.gain")
    if fingerprint is None:
        host = {k: (v if isinstance(v, np.ndarray) else v.detach().float().cpu().numpy())
                for k, v in params.items()}
        fingerprint = fingerprint_params(config, host)
    return Model(config, embed, layers, final_norm, lm_head, fingerprint, dev)


def reference_init_params(config: ModelConfig, seed: int) -> dict[str, np.ndarray]:
    """The reference init recipe (model.py:178-201) in numpy: N(0, 1/fan_in)
    weights in manifest order, N(0,1) embedding, N(0, 1/d) head, unit gains,
    zero biases. Bitwise what ``cacheclip.init_model`` draws for MHA."""
    rng = np.random.default_rng(seed)
    fan_in = {"wq": config.d_model, "wk": config.d_model, "wv": config.d_model, "wo": config.attn_width,
              "w_gate": config.d_model, "w_in": config.d_model, "w_out": config.d_ff}
    out: dict[str, np.ndarray] = {}
    for name, shape in expected_tensors(config):
        if name.endswith(".gain"):
            out[name] = np.ones(shape, np.float32)
        elif name.endswith(".bias"):
            out[name] = np.zeros(shape, np.float32)
        elif name == "embed.weight":
            out[name] = rng.normal(0.0, 1.0, shape).astype(np.float32)
        elif name == "lm_head.weight":
            out[name] = rng.normal(0.0, config.d_model ** -0.5, shape).astype(np.float32)
        else:
            out[name] = rng.normal(0.0, fan_in[name.split(".")[-2]] ** -0.5, shape).astype(np.float32)
    return out


def device_init_params(config: ModelConfig, seed: int, device=None) -> dict[str, torch.Tensor]:
    """Same distributions drawn on the GPU with torch (multi-billion-parameter
    synthetic models; not bitwise the numpy stream)."""
    dev = torch.device(device if device is not None else "cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    fan_in = {"wq": config.d_model, "wk": config.d_model, "wv": config.d_model, "wo": config.attn_width,
              "w_gate": config.d_model, "w_in": config.d_model, "w_out": config.d_ff}
    out: dict[str, torch.Tensor] = {}
    for name, shape in expected_tensors(config):
        if name.endswith(".gain"):
            out[name] = torch.ones(shape, device=dev)
        elif name.endswith(".bias"):
            out[name] = torch.zeros(shape, device=dev)
        else:
            if name == "embed.weight":
                std = 1.0
            elif name == "lm_head.weight":
                std = config.d_model ** -0.5
            else:
                std = fan_in[name.split(".")[-2]] ** -0.5
            out[name] = torch.randn(shape, generator=g, device=dev).mul_(std)
    return out


def init_model(config: ModelConfig, seed: int, *, device=None, source: str = "auto") -> Model:
    """Seeded random-init model (model.py:178-201) uploaded to the device.

    source="numpy" draws the reference's exact numpy stream (parity tests);
    "torch" draws on the GPU (large synthetic models); "auto" picks numpy
    below ~50M parameters."""
    n_params = sum(int(np.prod(s)) for _, s in expected_tensors(config))
    if source == "auto":
        source = "numpy" if n_params < 50_000_000 else "torch"
    if source == "numpy":
        return from_params(config, reference_init_params(config, seed), device=device)
    params = device_init_params(config, seed, device)
    fp = hashlib.sha256((config.to_json() + f"|torch-init|{seed}").encode()).hexdigest()
    model = from_params(config, params, device=device, fingerprint=fp)
    del params
    return model
