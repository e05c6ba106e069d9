"""Time the tcgen05 sparse-row attention alone on the C3 recompute shape.

    python scripts/bench_attention.py [--lib path/to/variant.so] [--dense N]

m selected rows (sorted, uniform over the context) of a Qwen2.5-7B layer
(28 query heads, 4 KV heads, d 128) attending to their causal prefix of an
n-row bank; FLOPs = 4 * d * Hq * sum(pos + 1). CUDA events, median of reps.
"""
import argparse
import math
import os
import sys

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None)
ap.add_argument("--m", type=int, default=6586)
ap.add_argument("--n", type=int, default=32832)
ap.add_argument("--dense", type=int, default=0, help="also time a dense causal prefill of this many rows")
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
if args.lib:
    os.environ["CACHECLIP_SM100_LIB"] = args.lib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2510_10129_b200 import _lib as L  # noqa: E402

DEV = "cuda:0"
Hq, Hkv, D = 28, 4, 128


def run(m, n, pos, label):
    g = torch.Generator(device=DEV).manual_seed(0)
    q = torch.randn(m, Hq, D, device=DEV, generator=g).to(torch.bfloat16)
    k = torch.randn(n, Hkv, D, device=DEV, generator=g).to(torch.bfloat16)
    v = torch.randn(n, Hkv, D, device=DEV, generator=g).to(torch.bfloat16)
    out = torch.empty(m, Hq * D, device=DEV, dtype=torch.bfloat16)
    st = torch.cuda.current_stream()
    flops = 4.0 * D * Hq * float((pos + 1).sum().item())

    def once():
        L.call("cc_sparse_row_attention", q.data_ptr(), Hq * D, pos.data_ptr(), m, k.data_ptr(), v.data_ptr(), n,
               Hq, Hkv, D, 1.0 / math.sqrt(D), None, out.data_ptr(), Hq * D, st.cuda_stream)

    for _ in range(3):
        once()
    times = []
    for _ in range(args.reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        once()
        b.record(st)
        b.synchronize()
        times.append(a.elapsed_time(b))
    times.sort()
    t = times[len(times) // 2]
    print(f"{label}: {t * 1e3:.1f} us  {flops / t / 1e9:.1f} TFLOP/s  (lib {os.path.basename(L.LIB_PATH)})")


pos = torch.sort(torch.randperm(args.n, generator=torch.Generator().manual_seed(1))[:args.m]).values.to(DEV)
run(args.m, args.n, pos, f"sparse m={args.m} n={args.n}")
if args.dense:
    run(args.dense, args.dense, torch.arange(args.dense, device=DEV), f"dense causal n={args.dense}")
