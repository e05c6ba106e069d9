"""Time the tcgen05 GEMMs alone on the C3 layer shapes, with their real epilogues.

    python scripts/bench_gemm.py [--lib path/to/variant.so] [--reps 20]

Primary (bf16, M = 6586 recomputed + query rows of a Qwen2.5-7B layer):
qkv (RoPE + K/V scatter), o-proj (+residual), gate/up (GLU), down (+residual).
Scoring model (3xTF32, M = 2048 = 64 chunks x 32 query rows of the 0.5B
shape): the same four. CUDA events around `reps` back-to-back launches.
"""
import argparse
import os
import sys

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--only", default="")
ap.add_argument("--trials", type=int, default=5)
args = ap.parse_args()
if args.lib:
    os.environ["CACHECLIP_SM100_LIB"] = args.lib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2510_10129_b200 import _lib as L  # noqa: E402
from paper_2510_10129_b200.runtime import gemm  # noqa: E402

DEV = "cuda:0"
torch.cuda.set_device(0)


def timed(fn, flops, label):
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(args.trials):  # best of `trials` batches (clock / power noise)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / args.reps)
    ms = best
    print(f"{label:34s} {ms * 1e3:9.1f} us  {flops / ms / 1e9:8.1f} TFLOP/s", flush=True)
    return ms


def shapes(kind, M, d, hq, hkv, dh, ff):
    f32 = kind == L.CC_GEMM_TF32X3
    km = 3 if f32 else 1
    wdt = torch.float32 if f32 else torch.bfloat16
    qw, kw = hq * dh, hkv * dh
    n_qkv = qw + 2 * kw
    g = torch.Generator(device=DEV).manual_seed(0)

    def rnd(r, c):
        return (torch.randn(r, c, device=DEV, generator=g) * 0.05).to(wdt)

    x = rnd(M, km * d)
    ctx = rnd(M, km * qw)
    act = rnd(M, km * ff)
    w_qkv, w_o, w_up, w_down = rnd(n_qkv, km * d), rnd(d, km * qw), rnd(2 * ff, km * d), rnd(d, km * ff)
    b_qkv = torch.zeros(n_qkv, device=DEV)
    h = torch.zeros(M, d, device=DEV)
    cos = torch.ones(M, dh // 2, device=DEV)
    sin = torch.zeros(M, dh // 2, device=DEV)
    q = torch.empty(M, qw, device=DEV, dtype=torch.float32 if f32 else torch.bfloat16)
    kc = torch.empty(M, kw, device=DEV, dtype=q.dtype)
    vc = torch.empty(M, kw, device=DEV, dtype=q.dtype)
    rows = torch.arange(M, device=DEV, dtype=torch.int64)
    mode = L.CC_F32 if f32 else L.CC_BF16
    amode = L.CC_F32_SPLIT3 if f32 else L.CC_BF16
    tag = "tf32x3" if f32 else "bf16"
    out = {}
    out[f"{tag} qkv  M={M} N={n_qkv} K={d}"] = (lambda: gemm(
        kind, L.CC_EPI_QKV_ROPE, M, n_qkv, d, x, w_qkv, bias=b_qkv, rope=(cos, sin), q_out=q, ldq=qw, q_mode=mode,
        k_cache=kc, v_cache=vc, cache_dtype=mode, dst_rows=rows, heads=(hq, hkv, dh)), 2.0 * M * n_qkv * d)
    out[f"{tag} o    M={M} N={d} K={qw}"] = (lambda: gemm(
        kind, L.CC_EPI_RESIDUAL, M, d, qw, ctx, w_o, C=h, ldc=d, c_mode=L.CC_F32), 2.0 * M * d * qw)
    out[f"{tag} up   M={M} N={2 * ff} K={d}"] = (lambda: gemm(
        kind, L.CC_EPI_GLU, M, 2 * ff, d, x, w_up, C=act, ldc=ff, c_mode=amode, n_out=ff), 2.0 * M * 2 * ff * d)
    out[f"{tag} down M={M} N={d} K={ff}"] = (lambda: gemm(
        kind, L.CC_EPI_RESIDUAL, M, d, ff, act, w_down, C=h, ldc=d, c_mode=L.CC_F32), 2.0 * M * d * ff)
    if not f32:  # the fused-RMSNorm epilogues of the layer executor
        xn = torch.empty(M, d, device=DEV, dtype=torch.bfloat16)
        ssq = torch.zeros(d // 32, M, device=DEV)
        inv = torch.ones(M, device=DEV)
        gain = torch.ones(d, device=DEV)
        nrm = dict(xn_out=xn, ldxn=d, norm_gain=gain, ssq_out=ssq, ld_ssq=M)
        out[f"{tag} qkv+rms M={M} N={n_qkv} K={d}"] = (lambda: gemm(
            kind, L.CC_EPI_QKV_ROPE, M, n_qkv, d, x, w_qkv, bias=b_qkv, rope=(cos, sin), q_out=q, ldq=qw,
            q_mode=mode, k_cache=kc, v_cache=vc, cache_dtype=mode, dst_rows=rows, heads=(hq, hkv, dh),
            inv_rms=inv), 2.0 * M * n_qkv * d)
        out[f"{tag} o+norm M={M} N={d} K={qw}"] = (lambda: gemm(
            kind, L.CC_EPI_RESIDUAL, M, d, qw, ctx, w_o, C=h, ldc=d, c_mode=L.CC_F32, **nrm), 2.0 * M * d * qw)
        out[f"{tag} up+rms M={M} N={2 * ff} K={d}"] = (lambda: gemm(
            kind, L.CC_EPI_GLU, M, 2 * ff, d, x, w_up, C=act, ldc=ff, c_mode=amode, n_out=ff, inv_rms=inv),
            2.0 * M * 2 * ff * d)
        out[f"{tag} down+norm M={M} N={d} K={ff}"] = (lambda: gemm(
            kind, L.CC_EPI_RESIDUAL, M, d, ff, act, w_down, C=h, ldc=d, c_mode=L.CC_F32, **nrm), 2.0 * M * d * ff)
        out[f"{tag} finalize M={M}"] = (lambda: L.call(
            "cc_norm_finalize", ssq.data_ptr(), M, d, M, 1e-6, inv.data_ptr(),
            torch.cuda.current_stream().cuda_stream), 1.0)
    return out


total = {}
for kind, M, cfg in ((L.CC_GEMM_BF16, 6586, (3584, 28, 4, 128, 18944)),
                     (L.CC_GEMM_TF32X3, 2048, (896, 14, 2, 64, 4864))):
    for label, (fn, fl) in shapes(kind, M, *cfg).items():
        if args.only and args.only not in label:
            continue
        total[label] = timed(fn, fl, label)
for tag, layers in (("bf16", 28), ("tf32x3", 24)):
    s = sum(v for k, v in total.items() if k.startswith(tag + " "))
    print(f"{tag}: {s * 1e3:.1f} us per layer -> {s * layers:.2f} ms per pass ({layers} layers)")
