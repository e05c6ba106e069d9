"""Decode after the first token (model.decode_step on the merged C3 cache,
32K context): ms per generated token, CUDA events, median of 20."""
import argparse
import os
import sys

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None)
args = ap.parse_args()
if args.lib:
    os.environ["CACHECLIP_SM100_LIB"] = args.lib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2510_10129_b200 as cc
from paper_2510_10129_b200 import _lib
from paper_2510_10129_b200.workloads import WORKLOADS

w = WORKLOADS["c3"]
dev = torch.device("cuda")
primary = cc.init_model(w.primary, 0, device=dev, source="torch")
aux = cc.init_model(w.aux, 1, device=dev, source="torch")
prefix, chunk_ids, query = w.token_ids(1000)
chunks = cc.prefill_chunks(primary, prefix, chunk_ids)
aux_chunks = cc.prefill_chunks(aux, prefix, chunk_ids)
out = cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query, cc.SelectionConfig(0.2, 8, 1))
cache, tok = out.cache, out.first_token
ts = []
for i in range(25):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    logits, cache = cc.decode_step(primary, cache, tok)
    b.record()
    torch.cuda.synchronize()
    tok = int(np.argmax(logits))
    if i >= 5:
        ts.append(a.elapsed_time(b))
print(f"decode at {cache.n_rows} rows: {np.median(ts):.2f} ms/token (lib {os.path.basename(_lib.LIB_PATH)})")
# one token under the launch profiler: where the step goes
_lib.profile_collect()
_lib.profile_enable(True)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
logits, cache = cc.decode_step(primary, cache, tok)
b.record()
torch.cuda.synchronize()
_lib.profile_enable(False)
tl = _lib.profile_timeline()
recs = _lib.profile_collect()
ops = {}
for op, _, ms in recs:
    n, t = ops.get(op, (0, 0.0))
    ops[op] = (n + 1, t + ms)
span = max(t1 for _, _, t1 in tl) - min(t0 for _, t0, _ in tl)
print(f"profiled token: wall {a.elapsed_time(b):.2f} ms, first..last launch {span:.2f} ms, "
      f"kernel sum {sum(t for _, t in ops.values()):.2f} ms over {len(recs)} launches")
for op, (n, t) in sorted(ops.items(), key=lambda kv: -kv[1][1]):
    print(f"   {op:24s} {n:4d} launches {t:7.3f} ms")
print("first layer, per launch (op, work, us; GEMM work 2*M*N*K):")
for (op, wk, ms), (_, t0, t1) in list(zip(recs, tl))[:12]:
    print(f"   {op:20s} work {wk:12.4g}  {ms * 1e3:7.1f} us  start {t0 * 1e3:8.1f} us")
