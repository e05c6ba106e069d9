"""Host-side cProfile of one C3 cacheclip_prefill (device-resident caches):
which Python work precedes the first kernel launch, and (argv[1] = 5: the
default 8/5 window rule) what runs between the selection read-back and the
recompute launch."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2510_10129_b200 as cc
from paper_2510_10129_b200.workloads import WORKLOADS

w = WORKLOADS["c3"]
dev = torch.device("cuda")
primary = cc.init_model(w.primary, 0, device=dev, source="torch")
aux = cc.init_model(w.aux, 1, device=dev, source="torch")
prefix, chunk_ids, query = w.token_ids(1000)
chunks = cc.prefill_chunks(primary, prefix, chunk_ids)
aux_chunks = cc.prefill_chunks(aux, prefix, chunk_ids)
thr = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = cc.SelectionConfig(0.2, 8, thr)
for _ in range(3):
    cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query, cfg)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(30)
st.sort_stats("tottime").print_stats(20)
