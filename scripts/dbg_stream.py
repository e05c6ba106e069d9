import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2510_10129_b200 as cc
from paper_2510_10129_b200.workloads import WORKLOADS
w = WORKLOADS["c3"]
dev = torch.device("cuda")
primary = cc.init_model(w.primary, 0, device=dev, source="torch")
prefix, chunk_ids, query = w.token_ids(1000)
chunks = [cc.prefill_chunk(primary, prefix, c) for c in chunk_ids]
host = [cc.ChunkCache(c.k.cpu().pin_memory(), c.v.cpu().pin_memory(), c.token_ids, c.prefix_len, c.tokenizer_id, c.model_fingerprint) for c in chunks]
nbytes = sum(c.k.numel() * 2 * 2 for c in chunks)
def t(fn, n=3):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
print("bytes", nbytes / 1e9, "GB")
ms = t(lambda: cc.merge_caches(chunks, primary.config.rope, capacity=33000))
print(f"device merge {ms:.2f} ms")
ms = t(lambda: cc.merge_caches(host, primary.config.rope, capacity=33000, device=dev))
print(f"streamed merge {ms:.2f} ms -> {nbytes/ms/1e6:.1f} GB/s")
def h2d():
    for c in host:
        c.k.to(dev, non_blocking=True); c.v.to(dev, non_blocking=True)
ms = t(h2d)
print(f"copy-engine H2D {ms:.2f} ms -> {nbytes/ms/1e6:.1f} GB/s")
