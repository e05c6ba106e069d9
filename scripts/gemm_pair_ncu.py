"""One 8192^3 bf16 GEMM through our CTA-pair kernel and one through cuBLAS,
for an ncu --set full side-by-side (run under ncu; numbers here are not timed)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_10129_b200 import _lib as L  # noqa: E402
from paper_2510_10129_b200.runtime import gemm  # noqa: E402

torch.cuda.set_device(0)
M = N = K = 8192
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
gemm(L.CC_GEMM_BF16, L.CC_EPI_STORE, M, N, K, A, B, C=C, ldc=N, c_mode=L.CC_BF16)
torch.matmul(A, B.t(), out=C)
torch.cuda.synchronize()
