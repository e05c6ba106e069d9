import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_10129_b200 as cc
from oracle import cacheclip_oracle as orc
from oracle.synth import C1 as w
oc = w.aux
cfg = cc.ModelConfig(n_layers=oc.n_layers, n_heads=oc.n_heads, d_model=oc.d_model, d_head=oc.d_head, d_ff=oc.d_ff,
                     vocab_size=oc.vocab_size, rope_base=oc.rope_base, norm_eps=oc.norm_eps, activation=oc.activation,
                     mlp_gated=oc.mlp_gated, n_kv_heads=oc.kv_heads, dtype="fp32", tokenizer_id="chars")
aux = cc.from_params(cfg, orc.seeded_params(oc, 1))
prefix, chunks, query = w.token_ids(0)
c = cc.prefill_chunk(aux, prefix, chunks[0]); torch.cuda.synchronize(); print("prefill ok", c.k.shape)
k = c.local_rotated_keys(aux.config.rope); torch.cuda.synchronize(); print("rot ok")
s = cc.aux_score_tokens(aux, [c], query); torch.cuda.synchronize(); print("score ok", s.scores[:4])
