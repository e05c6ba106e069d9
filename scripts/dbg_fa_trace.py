"""Per-tile SM-clock timeline of the heaviest attention CTA (debug build).

    make -C paper_2510_10129_b200/csrc variant VFLAGS=-DCC_FA_TRACE VOUT=../variants/libcc_trace.so
    python scripts/dbg_fa_trace.py paper_2510_10129_b200/variants/libcc_trace.so
"""
import ctypes
import math
import os
import sys

os.environ["CACHECLIP_SM100_LIB"] = sys.argv[1]
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_10129_b200 import _lib as L  # noqa: E402

DEV = "cuda:0"
Hq, Hkv, D = 28, 4, 128
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
m = n
q = torch.randn(m, Hq, D, device=DEV).to(torch.bfloat16)
k = torch.randn(n, Hkv, D, device=DEV).to(torch.bfloat16)
v = torch.randn(n, Hkv, D, device=DEV).to(torch.bfloat16)
pos = torch.arange(n, device=DEV)
out = torch.empty(m, Hq * D, device=DEV, dtype=torch.bfloat16)
for _ in range(2):
    L.call("cc_sparse_row_attention", q.data_ptr(), Hq * D, pos.data_ptr(), m, k.data_ptr(), v.data_ptr(), n,
           Hq, Hkv, D, 1.0 / math.sqrt(D), None, out.data_ptr(), Hq * D, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (16 * 128))()
assert L.load().cc_debug_fa_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(16, 128).astype(np.float64)
t0 = t[0, 0]
names = ["A_wake", "A_P", "B_wake", "B_P", "PV_A", "S_A+", "PV_B", "S_B+"]
print("j   " + " ".join(f"{x:>8s}" for x in names) + "   A_soft   B_soft   period")
for j in range(min(40, 128)):
    row = t[:8, j] - t0
    if t[0, j] == 0:
        break
    per = t[0, j + 1] - t[0, j] if t[0, j + 1] else float("nan")
    print(f"{j:3d} " + " ".join(f"{x:8.0f}" for x in row) +
          f" {t[1, j] - t[0, j]:8.0f} {t[3, j] - t[2, j]:8.0f} {per:8.0f}")
