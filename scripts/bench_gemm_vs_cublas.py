"""Plain bf16 GEMM throughput: our tcgen05 kernel (STORE epilogue, bf16 out)
vs cuBLAS (torch.matmul) on the same shapes, interleaved to share clock state.

    python scripts/bench_gemm_vs_cublas.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_10129_b200 import _lib as L  # noqa: E402
from paper_2510_10129_b200.runtime import gemm  # noqa: E402

torch.cuda.set_device(0)
DEV = "cuda:0"


def t(fn, reps=10, trials=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(trials):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best


for M, N, K in ((8192, 8192, 8192), (6586, 37888, 3584), (6586, 3584, 18944), (6586, 4608, 3584)):
    A = torch.randn(M, K, device=DEV).to(torch.bfloat16)
    B = torch.randn(N, K, device=DEV).to(torch.bfloat16)
    C = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    fl = 2.0 * M * N * K
    ours = t(lambda: gemm(L.CC_GEMM_BF16, L.CC_EPI_STORE, M, N, K, A, B, C=C, ldc=N, c_mode=L.CC_BF16))
    cub = t(lambda: torch.matmul(A, B.t(), out=C))
    ours2 = t(lambda: gemm(L.CC_GEMM_BF16, L.CC_EPI_STORE, M, N, K, A, B, C=C, ldc=N, c_mode=L.CC_BF16))
    print(f"M={M} N={N} K={K}: ours {fl / ours / 1e9:7.1f} / {fl / ours2 / 1e9:7.1f} TFLOP/s, "
          f"cuBLAS {fl / cub / 1e9:7.1f} TFLOP/s", flush=True)
