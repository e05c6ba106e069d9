"""Stress the request pipeline on one GPU: many C1/R1-shaped requests with
varying ratios, window rules, device / pinned-pool caches and worker counts,
each compared bitwise with a first run of the same request (determinism
across streams, the no-sync launch, the pinned staging ring wrap-around and
the copy-engine streaming). Prints one line per config and a total."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2510_10129_b200 as cc
from oracle import cacheclip_oracle as orc
from oracle.synth import C1, R1


def cfg(oc, dtype):
    return cc.ModelConfig(n_layers=oc.n_layers, n_heads=oc.n_heads, d_model=oc.d_model, d_head=oc.d_head,
                          d_ff=oc.d_ff, vocab_size=oc.vocab_size, rope_base=oc.rope_base, norm_eps=oc.norm_eps,
                          activation=oc.activation, mlp_gated=oc.mlp_gated, attn_bias=oc.attn_bias,
                          mlp_bias=oc.mlp_bias, tokenizer_id="chars", n_kv_heads=oc.kv_heads, dtype=dtype)


def pool_of(caches):
    L, _, H, D = caches[0].k.shape
    pool = cc.HostCachePool(len(caches), max(c.n_rows for c in caches), L, H, D, caches[0].k.dtype)
    return [pool.store(c) for c in caches]


t0 = time.time()
n_runs = 0
for w in (C1, R1):
    primary = cc.from_params(cfg(w.primary, "bf16"), orc.seeded_params(w.primary, 0, w.bias_std))
    aux = cc.from_params(cfg(w.aux, "fp32"), orc.seeded_params(w.aux, 1, w.bias_std))
    for seed in range(3):
        prefix, chunk_ids, query = w.token_ids(seed)
        pc = cc.prefill_chunks(primary, prefix, chunk_ids)
        ac = cc.prefill_chunks(aux, prefix, chunk_ids)
        hp, ha = pool_of(pc), pool_of(ac)
        for ratio in (0.0, 0.05, 0.2, 0.5, 1.0):
            for thr in (1, 3, 5):
                config = cc.SelectionConfig(ratio, 8, thr)
                ref = cc.cacheclip_prefill(primary, aux, pc, ac, query, config)
                for caches, workers in (((pc, ac), 2), ((hp, ha), 2), ((hp, ha), 1), ((pc, ac), 1)):
                    for _ in range(2):
                        out = cc.cacheclip_prefill(primary, aux, caches[0], caches[1], query, config,
                                                   workers=workers)
                        n_runs += 1
                        assert out.plan == ref.plan, (w.name, seed, ratio, thr, workers)
                        assert np.array_equal(out.logits, ref.logits), (w.name, seed, ratio, thr, workers)
                        assert out.first_token == ref.first_token
        print(f"{w.name} seed {seed}: ok ({n_runs} requests so far, {time.time() - t0:.1f} s)", flush=True)
torch.cuda.synchronize()
print(f"stress ok: {n_runs} requests bitwise equal to their first run")

if len(sys.argv) > 1 and sys.argv[1] == "c3":
    # full size: device-resident vs HostCachePool caches, exact-budget and
    # default rules, bitwise equal
    from paper_2510_10129_b200.workloads import WORKLOADS
    wl = WORKLOADS["c3"]
    dev = torch.device("cuda")
    primary = cc.init_model(wl.primary, 0, device=dev, source="torch")
    aux = cc.init_model(wl.aux, 1, device=dev, source="torch")
    for seed in (11, 12):
        prefix, chunk_ids, query = wl.token_ids(seed)
        pc = cc.prefill_chunks(primary, prefix, chunk_ids)
        ac = cc.prefill_chunks(aux, prefix, chunk_ids)
        hp, ha = pool_of(pc), pool_of(ac)
        for config in (cc.SelectionConfig(0.2, 8, 1), cc.SelectionConfig(0.2)):
            ref = cc.cacheclip_prefill(primary, aux, pc, ac, query, config)
            for _ in range(3):
                out = cc.cacheclip_prefill(primary, aux, hp, ha, query, config)
                assert out.plan == ref.plan and np.array_equal(out.logits, ref.logits)
        print(f"c3 seed {seed}: device == pool (bitwise), {len(ref.plan.indices)} rows", flush=True)
    print("stress c3 ok")
