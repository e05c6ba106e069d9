import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_10129_b200 as cc
from paper_2510_10129_b200 import kv_store
from paper_2510_10129_b200.workloads import WORKLOADS
w = WORKLOADS["c3"]
dev = torch.device("cuda")
primary = cc.init_model(w.primary, 0, device=dev, source="torch")
prefix, chunk_ids, query = w.token_ids(1000)
chunks = [cc.prefill_chunk(primary, prefix, c) for c in chunk_ids]
host = [cc.ChunkCache(c.k.cpu().pin_memory(), c.v.cpu().pin_memory(), c.token_ids, c.prefix_len, c.tokenizer_id, c.model_fingerprint) for c in chunks]
nbytes = sum(c.k.numel() * 2 * 2 for c in chunks)
for ctas in (4, 8, 16, 24, 48, 148, 0):
    kv_store.STREAM_CTAS = ctas
    f = lambda: cc.merge_caches(host, primary.config.rope, capacity=33000, device=dev)
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); f(); f(); b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 2
    print(f"ctas={ctas}: {ms:.2f} ms -> {nbytes/ms/1e6:.1f} GB/s")
