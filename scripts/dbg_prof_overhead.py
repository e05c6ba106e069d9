"""TTFT of the C3 step with the in-library launch profiler on vs off."""
import os
import sys

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
cfg = cc.SelectionConfig(0.2, 8, 1)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query, cfg)
for rep in range(3):
    for on in (True, False):
        ts = []
        _lib.profile_enable(on)
        for _ in range(8):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query, cfg)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        _lib.profile_enable(False)
        _lib.profile_collect()
        print(f"profiler {'on ' if on else 'off'}: {np.mean(ts):.2f} ms (min {np.min(ts):.2f})", flush=True)
