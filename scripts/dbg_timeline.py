"""Host/GPU timeline of one C3 cacheclip_prefill: where is the GPU idle?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2510_10129_b200 as cc
from paper_2510_10129_b200 import pipeline, selector, model as mdl
from paper_2510_10129_b200.workloads import WORKLOADS
w = WORKLOADS["c3"]
dev = torch.device("cuda")
primary = cc.init_model(w.primary, 0, device=dev, source="torch")
aux = cc.init_model(w.aux, 1, device=dev, source="torch")
prefix, chunk_ids, query = w.token_ids(1000)
chunks = [cc.prefill_chunk(primary, prefix, c) for c in chunk_ids]
aux_chunks = [cc.prefill_chunk(aux, prefix, c) for c in chunk_ids]
config = cc.SelectionConfig(0.2, 8, 1)
marks = []
def mark(name):
    e = torch.cuda.Event(enable_timing=True); e.record(); marks.append((name, time.perf_counter(), e))
# monkeypatch stage boundaries
orig_score, orig_sel, orig_fwd = pipeline.aux_score_tokens, pipeline.select_tokens_device, pipeline.forward_on_merged
def score(*a, **k):
    mark("score_begin"); r = orig_score(*a, **k); mark("score_launched"); return r
def sel(*a, **k):
    mark("select_begin"); r = orig_sel(*a, **k); mark("select_synced"); return r
def fwd(*a, **k):
    mark("recompute_begin"); r = orig_fwd(*a, **k); mark("recompute_launched"); return r
pipeline.aux_score_tokens, pipeline.select_tokens_device, pipeline.forward_on_merged = score, sel, fwd
for it in range(4):
    marks.clear()
    torch.cuda.synchronize()
    mark("start")
    out = cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query, config)
    mark("end")
    torch.cuda.synchronize()
t0h, e0 = marks[0][1], marks[0][2]
print(f"{'stage':22s} {'host ms':>9s} {'gpu ms':>9s}")
for name, th, e in marks:
    print(f"{name:22s} {1e3*(th-t0h):9.2f} {e0.elapsed_time(e):9.2f}")
