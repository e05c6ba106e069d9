"""Where the scoring model's fp32 error comes from at the benchmarked sizes
(GPU diagnostic; writes gpurun_out/diag_scoring_<w>.json).

Four score vectors for the same seeded C2 / C3 workload:
  ref     the unmodified reference (tests/golden/<w>_scoring.npz)
  f64     float64 torch restatement (oracle/torch_f64.py): caches + scoring
  dev     device chain: prefill_chunks + aux_score_tokens (3xTF32)
  dev64   device scoring pass on the float64 caches rounded to fp32
          (isolates the scoring pass from the chunk precompute)
and the selections each produces at ratios 0.05/0.2/0.4 x thresholds 5/1.
"""

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2510_10129_b200 as cc  # noqa: E402
from oracle import cacheclip_oracle as orc  # noqa: E402
from oracle.synth import C2, C3, SCALE_RATIOS, SCALE_THRESHOLDS  # noqa: E402
from oracle.torch_f64 import F64Model, scores_f64  # noqa: E402


def cfg_of(oc, dtype):
    return cc.ModelConfig(n_layers=oc.n_layers, n_heads=oc.n_heads, d_model=oc.d_model, d_head=oc.d_head,
                          d_ff=oc.d_ff, vocab_size=oc.vocab_size, rope_base=oc.rope_base, norm_eps=oc.norm_eps,
                          activation=oc.activation, mlp_gated=oc.mlp_gated, attn_bias=oc.attn_bias,
                          mlp_bias=oc.mlp_bias, tokenizer_id="chars", n_kv_heads=oc.kv_heads, dtype=dtype)


def rel(a, b):
    r = np.abs(a - b) / np.maximum(np.abs(b), 1e-30)
    return {"max": float(r.max()), "median": float(np.median(r)), "p99": float(np.percentile(r, 99))}


def main(names):
    dev = torch.device("cuda", 0)
    params = orc.seeded_params(C2.aux, C2.aux_seed, fast=True)
    aux = cc.from_params(cfg_of(C2.aux, "fp32"), params)
    f64 = F64Model(C2.aux, params, dev)
    del params
    for w in [x for x in (C2, C3) if x.name in names]:
        t0 = time.time()
        g = dict(np.load(os.path.join(ROOT, "tests", "golden", f"{w.name}_scoring.npz")))
        prefix, chunk_ids, query = w.token_ids(0)
        s64, caches = scores_f64(f64, prefix, chunk_ids, query)
        s64 = s64.cpu().numpy()
        dchunks = cc.prefill_chunks(aux, prefix, chunk_ids)
        sdev = np.asarray(cc.aux_score_tokens(aux, dchunks, query).scores, dtype=np.float32)
        # device-cache error vs f64 caches (layer-wise rel L2 of K, first chunk)
        kerr = [float(torch.linalg.norm(dchunks[0].k[l].double() - caches[0][0][l]) /
                      torch.linalg.norm(caches[0][0][l])) for l in range(w.aux.n_layers)]
        del dchunks
        c64 = [cc.ChunkCache(k.float().contiguous(), v.float().contiguous(), list(prefix) + list(c), len(prefix),
                             "chars", aux.fingerprint) for (k, v), c in zip(caches, chunk_ids)]
        sdev64 = np.asarray(cc.aux_score_tokens(aux, c64, query).scores, dtype=np.float32)
        del c64, caches
        ref = g["scores"]
        lens = [len(c) for c in chunk_ids]
        out = {"workload": w.name, "n": int(ref.size),
               "rel_ref_vs_f64": rel(ref, s64), "rel_dev_vs_f64": rel(sdev, s64), "rel_dev_vs_ref": rel(sdev, ref),
               "rel_dev64_vs_f64": rel(sdev64, s64), "k_rel_l2_dev_vs_f64_by_layer": kerr, "selection": {}}
        for ratio in SCALE_RATIOS:
            for thr in SCALE_THRESHOLDS:
                want = g[f"idx_{ratio}_{thr}"].astype(np.int64)
                row = {}
                for tag, s in (("f64", s64), ("dev", sdev), ("dev64", sdev64)):
                    idx, _ = orc.select(s.astype(np.float32), lens, ratio, 8, thr)
                    got = np.asarray(idx, dtype=np.int64)
                    diff = np.setxor1d(got, want)
                    row[tag] = {"n_diff_vs_ref": int(diff.size), "diff": diff[:10].tolist(),
                                "ref_scores": ref[diff[:10]].tolist(), "f64_scores": s64[diff[:10]].tolist(),
                                "this_scores": s[diff[:10]].tolist()}
                out["selection"][f"{ratio}_{thr}"] = row
        out["seconds"] = time.time() - t0
        print(json.dumps(out))
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", f"diag_scoring_{w.name}.json"), "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3"])
