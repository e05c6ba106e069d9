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
