"""Scores of the scoring pass (C2 / C3 shapes) written to a .npy, for bitwise
A/B of library variants: python scripts/bt_bitwise.py OUT.npy [c2|c3]
(CACHECLIP_SM100_LIB selects the library)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_10129_b200 as cc  # noqa: E402
from paper_2510_10129_b200.workloads import WORKLOADS  # noqa: E402

out, name = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "c2")
w = WORKLOADS[name]
dev = torch.device("cuda", 0)
aux = cc.init_model(w.aux, 1, device=dev, source="torch")
prefix, chunk_ids, query = w.token_ids(1000)
ac = cc.prefill_chunks(aux, prefix, chunk_ids)
sc = cc.aux_score_tokens(aux, ac, query)
arr = sc.device_scores.cpu().numpy()
np.save(out, arr)
print(out, arr.shape, float(arr.sum()))
