"""MMA-warp wait timeline of the 3xTF32 GEMM (block 0) for the scoring model's
up projection (M=2048, N=9728, K=896): where the tensor core's issue thread
waits — for a free accumulator (tempty: the epilogue's phase fold) or for
operands (full: TMA) — and how long the epilogue takes per phase.

    make -C paper_2510_10129_b200/csrc variant VFLAGS=-DCC_GEMM_TRACE VOUT=../variants/libcc_gtrace.so
    python scripts/dbg_gemm_trace.py paper_2510_10129_b200/variants/libcc_gtrace.so [qkv|o|up|down]
"""
import ctypes
import os
import sys

os.environ["CACHECLIP_SM100_LIB"] = sys.argv[1]
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_10129_b200 import _lib as L  # noqa: E402
from paper_2510_10129_b200.runtime import gemm  # noqa: E402

which = sys.argv[2] if len(sys.argv) > 2 else "up"
DEV = "cuda"
M, d, ff = 2048, 896, 4864
g = torch.Generator(device=DEV).manual_seed(0)
rnd = lambda r, c: (torch.randn(r, c, device=DEV, generator=g) * 0.05)  # noqa: E731
x = rnd(M, 3 * d)
act = torch.empty(M, 3 * ff, device=DEV)
h = torch.zeros(M, d, device=DEV)
if which == "up":
    w = rnd(2 * ff, 3 * d)
    run = lambda: gemm(L.CC_GEMM_TF32X3, L.CC_EPI_GLU, M, 2 * ff, d, x, w, C=act, ldc=ff,  # noqa: E731
                       c_mode=L.CC_F32_SPLIT3, n_out=ff)
    num_kb = d // 32
else:
    a = rnd(M, 3 * ff)
    w = rnd(d, 3 * ff)
    run = lambda: gemm(L.CC_GEMM_TF32X3, L.CC_EPI_RESIDUAL, M, d, ff, a, w, C=h, ldc=d, c_mode=L.CC_F32)  # noqa: E731
    num_kb = ff // 32
run()
torch.cuda.synchronize()
run()
torch.cuda.synchronize()
lib = L.load()
buf = (ctypes.c_longlong * (5 * 4096))()
assert lib.cc_debug_gemm_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(5, 4096).astype(np.float64)
n = int(np.count_nonzero(t[2]))
t0 = t[0, 0]
start, after_tempty, after_full = t[0, :n] - t0, t[1, :n] - t0, t[2, :n] - t0
w_tempty = after_tempty - start
w_full = after_full - after_tempty
issue = np.diff(start)
print(f"{which}: {n} K-blocks traced on block 0, {num_kb} per tile, span {after_full[-1]:.0f} clk "
      f"= {after_full[-1] / n:.0f} clk per K-block (MMA ideal 768)")
print(f"  wait tempty: total {w_tempty.sum():.0f} clk ({100 * w_tempty.sum() / after_full[-1]:.1f} %), "
      f"max {w_tempty.max():.0f}")
print(f"  wait full  : total {w_full.sum():.0f} clk ({100 * w_full.sum() / after_full[-1]:.1f} %), "
      f"max {w_full.max():.0f}")
print(f"  issue step : median {np.median(issue):.0f} clk")
ne = int(np.count_nonzero(t[3])) // 2
e = t[3, :2 * ne].reshape(ne, 2) - t0
fold = e[1:, 0] - e[:-1, 1]  # from tfull seen to the next phase's wait start: fold (+ tile epilogue)
print(f"  epilogue phases {ne}: fold+epilogue per phase median {np.median(fold):.0f}, max {fold.max():.0f} clk")
nt = int(np.count_nonzero(t[4])) // 3
if nt:
    fe = t[4, :3 * nt].reshape(nt, 3)
    print(f"  final epilogue per tile ({nt} tiles): median {np.median(fe[:, 2] - fe[:, 0]):.0f} clk "
          f"(GLU math {np.median(fe[:, 1] - fe[:, 0]):.0f}, store tail {np.median(fe[:, 2] - fe[:, 1]):.0f})")
for i in range(min(n, 40)):
    print(f"    kb {i:3d}: start {start[i]:9.0f}  tempty {w_tempty[i]:6.0f}  full {w_full[i]:6.0f}")
