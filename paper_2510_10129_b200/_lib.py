"""ctypes binding of libcacheclip_sm100.so (the C-ABI in include/cacheclip_sm100.h).

There is deliberately no fallback: if the shared library is missing or the
device is not sm_100, every hot-path call raises. Status codes map to the
reference's exception classes (tensor_core.py:18, kv_store.py:36-52).
"""

from __future__ import annotations

import ctypes
import os

from .errors import CacheConsistencyError, DimensionError

LIB_NAME = "libcacheclip_sm100.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)
# tuning builds (same ABI, different compile-time knobs) can be swapped in by
# naming another in-tree build of the library
if os.environ.get("CACHECLIP_SM100_LIB"):
    LIB_PATH = os.path.abspath(os.environ["CACHECLIP_SM100_LIB"])

CC_OK, CC_ERR_VALUE, CC_ERR_DIMENSION, CC_ERR_CONSISTENCY, CC_ERR_CUDA, CC_ERR_UNSUPPORTED = range(6)
CC_F32, CC_BF16, CC_F32_SPLIT3 = 0, 1, 2
CC_GEMM_BF16, CC_GEMM_TF32X3 = 0, 1
CC_EPI_STORE, CC_EPI_RESIDUAL, CC_EPI_GLU, CC_EPI_ACT, CC_EPI_QKV_ROPE = range(5)
CC_ACT_SILU, CC_ACT_GELU_TANH = 0, 1

i32, i64, f32, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p


class KvSegment(ctypes.Structure):
    _fields_ = [("k", vp), ("v", vp), ("src_rows", i64), ("src_row0", i64),
                ("dst_row0", i64), ("n_rows", i64), ("pos0", i64)]


class BankSeq(ctypes.Structure):
    _fields_ = [("k", vp), ("v", vp), ("n_bank", i64), ("row0", i64), ("n_new", i64)]


class GemmArgs(ctypes.Structure):
    _fields_ = [
        ("kind", i32), ("epilogue", i32),
        ("M", i64), ("N", i64), ("K", i64),
        ("A", vp), ("lda", i64),
        ("B", vp), ("ldb", i64),
        ("bias", vp),
        ("C", vp), ("ldc", i64), ("c_mode", i32),
        ("act", i32), ("glu_block", i32), ("n_out", i64),
        ("n_q_heads", i32), ("n_kv_heads", i32), ("head_dim", i32),
        ("rope_cos", vp), ("rope_sin", vp),
        ("q_out", vp), ("ldq", i64), ("q_mode", i32),
        ("k_cache", vp), ("v_cache", vp), ("cache_dtype", i32),
        ("dst_rows", vp),
        ("k_raw", vp),
        ("raw_rows", vp),
        ("xn_out", vp), ("ldxn", i64), ("norm_gain", vp),
        ("ssq_out", vp),
        ("inv_rms", vp),
        ("ld_ssq", i64),
        ("ssq_in", vp), ("n_ssq", i32), ("ld_ssq_in", i64), ("norm_eps", ctypes.c_float),
    ]


class LayerWeightsDesc(ctypes.Structure):
    _fields_ = [("w_qkv", vp), ("b_qkv", vp), ("n_qkv", i64), ("w_o", vp), ("b_o", vp),
                ("attn_norm", vp), ("mlp_norm", vp), ("w_up", vp), ("b_up", vp), ("n_up", i64),
                ("w_down", vp), ("b_down", vp)]


class ModelDesc(ctypes.Structure):
    _fields_ = [("n_layers", i32), ("n_heads", i32), ("n_kv_heads", i32), ("head_dim", i32),
                ("d_model", i32), ("d_ff", i32), ("vocab", i64), ("dtype", i32), ("mlp_gated", i32),
                ("act", i32), ("norm_eps", f32), ("embed", vp), ("final_norm", vp), ("lm_head", vp),
                ("head_dtype", i32), ("layers", ctypes.POINTER(LayerWeightsDesc)),
                ("inv_freq", ctypes.POINTER(ctypes.c_double))]


class KvPlan(ctypes.Structure):
    _fields_ = [("k_scatter", vp), ("k_scatter_stride", i64), ("v_scatter", vp), ("v_scatter_stride", i64),
                ("dst_rows", vp), ("k_raw", vp), ("k_raw_stride", i64), ("raw_rows", vp),
                ("attn_k", vp), ("attn_k_stride", i64), ("attn_v", vp), ("attn_v_stride", i64),
                ("layer_ready", ctypes.POINTER(vp)), ("key_start", vp)]


class ScoreSpec(ctypes.Structure):
    _fields_ = [("col0", i64), ("chunk_lens", vp), ("col_off", vp), ("max_chunk", i64),
                ("weights", vp), ("scores", vp)]


_SIGS = {
    "cc_abi_version": ([], i32),
    "cc_last_error": ([], ctypes.c_char_p),
    "cc_device_check": ([i32], i32),
    "cc_check_silu": ([vp, i64, vp, vp], i32),
    "cc_assemble_kv": ([vp, i32, i64, i32, i32, i32, i32, vp, i64, vp, vp, i64, vp], i32),
    "cc_upload": ([vp, vp, i64, vp], i32),
    "cc_h2d_uniform": ([vp, vp, i64, i64, vp, vp, i64, i64, i64, i32, i32, i32, vp], i32),
    "cc_h2d_segments": ([vp, i32, i32, i32, i32, i32, i32, vp, vp, i64, vp], i32),
    "cc_rope_rows_inplace": ([vp, i32, i64, i32, i32, i32, i32, vp, vp, i64, vp], i32),
    "cc_rope_table": ([vp, i64, vp, i32, vp, vp, vp], i32),
    "cc_embed_rmsnorm": ([vp, i64, vp, i32, i64, i32, vp, vp, f32, vp, i32, vp], i32),
    "cc_rmsnorm": ([vp, i64, i32, i64, vp, f32, vp, i32, vp], i32),
    "cc_norm_prep": ([vp, i64, i32, i64, vp, vp, vp, i64, vp], i32),
    "cc_norm_finalize": ([vp, i64, i32, i64, f32, vp, vp], i32),
    "cc_fused_norm": ([], i32),
    "cc_convert_matrix": ([vp, i64, i64, vp, i32, i32, vp], i32),
    "cc_gemm": ([ctypes.POINTER(GemmArgs), vp], i32),
    "cc_sparse_row_attention": ([vp, i64, vp, i64, vp, vp, i64, i32, i32, i32, f32, vp, vp, i64, vp], i32),
    "cc_sparse_row_attention_ranged": ([vp, i64, vp, vp, i64, vp, vp, i64, i32, i32, i32, f32, vp, vp, i64, vp],
                                       i32),
    "cc_sparse_row_attention_split": ([vp, i64, vp, vp, i64, vp, vp, i64, i32, i32, i32, f32, vp, i32, vp, vp, vp,
                                       i64, vp], i32),
    "cc_attention_splits": ([i64, i32, i32, i64], i32),
    "cc_sparse_row_attention_partial": ([vp, i64, vp, i64, vp, vp, i64, i32, i32, i32, f32, vp, vp, i32, vp, vp],
                                        i32),
    "cc_row_l2_diff": ([vp, i32, i64, vp, i32, i64, i64, i32, vp, vp], i32),
    "cc_local_limits": ([vp, i64, vp, i64, vp, vp], i32),
    "cc_lse_merge": ([vp, i32, vp, i32, i64, i64, i32, i32, vp, i64, i32, vp], i32),
    "cc_sparse_row_attention_mma": ([vp, i64, vp, i64, vp, vp, i64, i32, i32, i32, f32, vp, vp, i64, vp], i32),
    "cc_banked_attention_f32": ([vp, i32, i32, i64, vp, vp, vp, i32, i32, i32, f32, vp, i32, vp, i64, i64, vp], i32),
    "cc_banked_attention_simt": ([vp, i32, i32, i64, vp, vp, vp, i32, i32, i32, f32, vp, i32, vp, i64, i64, vp], i32),
    "cc_reduce_scores": ([vp, i32, i32, i32, i64, vp, vp, i64, vp, vp], i32),
    "cc_select_workspace_bytes": ([i64, i32], i64),
    "cc_select_topk_windows": ([vp, i64, vp, i32, i64, i64, i32, i32, i32, i64, vp, vp, vp, vp, vp, vp], i32),
    "cc_lm_head_workspace_bytes": ([i64], i64),
    "cc_lm_head_argmax": ([vp, vp, f32, i32, vp, i32, i64, vp, vp, vp, vp], i32),
    "cc_gather_i64": ([vp, vp, i64, vp, vp], i32),
    "cc_build_rows": ([vp, i64, vp, vp, i64, i64, vp, vp, vp], i32),
    "cc_forward_rows_workspace_bytes": ([ctypes.POINTER(ModelDesc), i64], i64),
    "cc_forward_banked_workspace_bytes": ([ctypes.POINTER(ModelDesc), i64], i64),
    "cc_forward_rows": ([ctypes.POINTER(ModelDesc), vp, vp, i64, ctypes.POINTER(KvPlan), i64, ctypes.c_double,
                         vp, i64, vp, vp, vp, vp], i32),
    "cc_forward_banked": ([ctypes.POINTER(ModelDesc), vp, vp, i64, vp, i32, i32, i64, vp, i64, vp, i64,
                           ctypes.POINTER(ScoreSpec), ctypes.POINTER(vp), i32, vp, vp], i32),
    "cc_profile_enable": ([i32], None),
    "cc_profile_collect": ([vp, vp, vp, i64], i64),
    "cc_profile_fill_work": ([i32, ctypes.c_double], None),
    "cc_profile_timeline": ([vp, vp, vp, i64], i64),
}

PROFILE_OPS = ("gemm_bf16", "gemm_3xtf32", "attention_tcgen05", "attention_mma", "banked_attention_f32",
               "rmsnorm", "assemble_kv", "select_topk", "score_reduce", "lm_head", "rope_table", "other",
               "lse_merge")


def profile_enable(on: bool) -> None:
    load().cc_profile_enable(1 if on else 0)


def profile_collect():
    """[(op name, algorithmic work, ms)] for every launch since enable; clears."""
    import numpy as np
    lib = load()
    cap = 1 << 16
    ops = np.zeros(cap, np.int32)
    work = np.zeros(cap, np.float64)
    ms = np.zeros(cap, np.float32)
    n = int(lib.cc_profile_collect(ops.ctypes.data, work.ctypes.data, ms.ctypes.data, cap))
    n = min(n, cap)
    return [(PROFILE_OPS[o] if 0 <= o < len(PROFILE_OPS) else f"op{o}", float(w), float(t))
            for o, w, t in zip(ops[:n], work[:n], ms[:n])]

def profile_timeline():
    """[(op name, start ms, end ms)] of every launch recorded since enable,
    relative to the first start; does not clear (profile_collect does)."""
    import numpy as np
    lib = load()
    cap = 1 << 16
    ops = np.zeros(cap, np.int32)
    t0 = np.zeros(cap, np.float32)
    t1 = np.zeros(cap, np.float32)
    n = min(int(lib.cc_profile_timeline(ops.ctypes.data, t0.ctypes.data, t1.ctypes.data, cap)), cap)
    return [(PROFILE_OPS[o] if 0 <= o < len(PROFILE_OPS) else f"op{o}", float(a), float(b))
            for o, a, b in zip(ops[:n], t0[:n], t1[:n])]


EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the C-ABI library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{LIB_NAME} not built ({path}); run `python -c 'import __graft_entry__ as g; g.build()'` "
            "— there is no CPU fallback for the CacheClip hot path")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == CC_OK:
        return
    msg = load().cc_last_error().decode("utf-8", "replace")
    if rc == CC_ERR_VALUE:
        raise ValueError(msg)
    if rc in (CC_ERR_DIMENSION, CC_ERR_UNSUPPORTED):
        raise DimensionError(msg)
    if rc == CC_ERR_CONSISTENCY:
        raise CacheConsistencyError(msg)
    raise RuntimeError(f"libcacheclip_sm100: {msg}")


class KernelTimer:
    """Optional per-launch CUDA-event timing (bench roofline). Each record is
    (entry point, start event, end event, meta dict) on the launching stream."""

    def __init__(self) -> None:
        self.records: list = []

    def summary(self) -> dict:
        import torch
        torch.cuda.synchronize()
        out: dict = {}
        for name, e0, e1, meta in self.records:
            d = out.setdefault(name, {"launches": 0, "ms": 0.0, "flops": 0.0, "bytes": 0.0})
            d["launches"] += 1
            d["ms"] += e0.elapsed_time(e1)
            d["flops"] += meta.get("flops", 0.0)
            d["bytes"] += meta.get("bytes", 0.0)
        return out


_timer: KernelTimer | None = None


def set_timer(timer: KernelTimer | None) -> None:
    global _timer
    _timer = timer


def call(name: str, *args, meta: dict | None = None) -> None:
    fn = getattr(load(), name)
    t = _timer
    if t is None:
        check(fn(*args))
        return
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    check(fn(*args))
    e1.record()
    t.records.append((name, e0, e1, meta or {}))


_device_ok: set[int] = set()


def require_device(dev: int) -> None:
    """Fail loudly unless `dev` is a B200 (sm_100) the kernels can run on."""
    if dev in _device_ok:
        return
    call("cc_device_check", dev)
    _device_ok.add(dev)
