"""Full-size golden fixtures from the REFERENCE itself (VERDICT r1 "What's
missing" #1): the benchmarked scoring model and a depth-truncated 7B primary.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden_scale.py            # c2, c3, p2, p2d
    python tests/golden/make_golden_scale.py c3         # one of them

* ``c2_scoring.npz`` / ``c3_scoring.npz`` — the 24-layer Qwen2.5-0.5B-shape
  scoring model (GQA 14/2, MHA-expanded for the reference),
  32-token prefix and query, 16 / 64 chunks x 512 tokens. The reference's
  ``prefill_chunk`` builds every scoring cache, ``aux_score_tokens``
  (selector.py:132-179) scores them, and ``select_tokens``
  (selector.py:182-214) selects at ratios 0.05 / 0.2 / 0.4 under the default
  8/5 window rule and the exact-budget rule (threshold 1). Stored: the
  scores, and per (ratio, threshold) the selected indices and window records,
  plus the relative score gap at each budget boundary (near-tie diagnostic).
* ``p2_primary.npz`` — a 2-layer Qwen2.5-7B-shape primary (bf16-rounded
  weights, fp32 arithmetic in the reference) + the same scoring model at C2:
  the reference's ``cacheclip_prefill`` (pipeline.py:156-226) at ratio 0.2,
  exact-budget rule, and ``full_attention_prefill`` (pipeline.py:77-84).
  Stored: plan indices, first-token logits of both, and recomputed K/V of
  every 8th selected row and of the query rows.

Weights are NOT stored: ``oracle.cacheclip_oracle.seeded_params(fast=True)``
regenerates them from the seed on the GPU box.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)
sys.path.insert(0, REF_SRC)

import cacheclip as ref  # noqa: E402  (the reference, read-only)

from oracle import cacheclip_oracle as orc  # noqa: E402
from oracle.synth import C2, C3, P2, P2D, SCALE_RATIOS, SCALE_THRESHOLDS  # noqa: E402

sys.path.insert(0, HERE)
from make_golden import char_vocab, ref_config  # noqa: E402

SEL_STRIDE = 8


def _bf16_2d(params):
    return {k: (orc.round_to_bf16(v) if v.ndim == 2 else v) for k, v in params.items()}


def _aux_model(w):
    a_params = orc.seeded_params(w.aux, w.aux_seed, w.bias_std, fast=True)
    return ref.Model(ref_config(w.aux, "chars"), orc.mha_expand(w.aux, a_params))


def _windows(sel) -> np.ndarray:
    return np.array([[x.window_id, x.chunk, x.start, x.end, x.selected, int(x.kept), int(x.partial)]
                     for x in sel.windows], dtype=np.int32).reshape(-1, 7)


def scoring(w, aux=None):
    t0 = time.perf_counter()
    aux = aux or _aux_model(w)
    prefix, chunk_ids, query = w.token_ids(0)
    aux_chunks = [ref.prefill_chunk(aux, prefix, c) for c in chunk_ids]
    t1 = time.perf_counter()
    scores = ref.aux_score_tokens(aux, aux_chunks, query)
    t2 = time.perf_counter()
    out = dict(scores=scores.scores, chunk_lens=np.asarray(scores.chunk_lens, dtype=np.int64),
               ratios=np.asarray(SCALE_RATIOS), thresholds=np.asarray(SCALE_THRESHOLDS))
    s = np.asarray(scores.scores, dtype=np.float32)
    order = np.argsort(-s, kind="stable")
    for ratio in SCALE_RATIOS:
        k = ref.selection_budget(ratio, s.size)
        gap = (s[order[k - 1]] - s[order[k]]) / max(abs(float(s[order[k - 1]])), 1e-30) if k < s.size else np.inf
        out[f"gap_{ratio}"] = np.float64(gap)
        for thr in SCALE_THRESHOLDS:
            cfg = ref.SelectionConfig(recomp_ratio=ratio, window_threshold=thr)
            sel = ref.select_tokens(scores, cfg)
            out[f"idx_{ratio}_{thr}"] = np.asarray(sel.indices, dtype=np.int32)
            out[f"win_{ratio}_{thr}"] = _windows(sel)
            print(f"  {w.name} ratio {ratio} thr {thr}: {len(sel.indices)} selected, boundary gap {gap:.3e}")
    print(f"{w.name}: chunk precompute {t1 - t0:.1f} s, scoring {t2 - t1:.1f} s")
    return out, aux, aux_chunks


def primary(w, aux, aux_chunks, full_prefill: bool = True, prim_chunks=None):
    t0 = time.perf_counter()
    if prim_chunks is None:
        p_params = _bf16_2d(orc.seeded_params(w.primary, w.primary_seed, w.bias_std, fast=True))
        prim = ref.Model(ref_config(w.primary, "chars"), orc.mha_expand(w.primary, p_params))
        del p_params
        prefix, chunk_ids, query = w.token_ids(0)
        chunks = [ref.prefill_chunk(prim, prefix, c) for c in chunk_ids]
    else:
        prim, chunks = prim_chunks
        prefix, chunk_ids, query = w.token_ids(0)
    t1 = time.perf_counter()
    tok = ref.GreedyTokenizer(char_vocab(max(w.primary.vocab_size, w.aux.vocab_size)), "chars")
    cfg = ref.SelectionConfig(recomp_ratio=w.ratio, window_len=w.window_len, window_threshold=w.window_threshold)
    clip = ref.cacheclip_prefill(prim, aux, chunks, aux_chunks, tok.decode(query), cfg,
                                 primary_tokenizer=tok, aux_tokenizer=tok)
    t2 = time.perf_counter()
    g = w.primary.group
    head_sel = np.arange(w.primary.kv_heads) * g
    sel = np.asarray(clip.plan.indices, dtype=np.int64)
    srows = sel[::SEL_STRIDE]
    qrows = np.arange(clip.cache.n_rows - len(query), clip.cache.n_rows)
    out = dict(indices=sel.astype(np.int32), clip_logits=clip.logits, sel_rows=srows.astype(np.int32),
               q_rows=qrows.astype(np.int32),
               sel_k=np.stack([k[srows][:, head_sel] for k in clip.cache.keys]),
               sel_v=np.stack([v[srows][:, head_sel] for v in clip.cache.values]),
               q_k=np.stack([k[qrows][:, head_sel] for k in clip.cache.keys]),
               q_v=np.stack([v[qrows][:, head_sel] for v in clip.cache.values]))
    del clip
    if full_prefill:
        full = ref.full_attention_prefill(prim, ref.reuse_context_ids(chunks, query))
        out["full_logits"] = full.logits
    t3 = time.perf_counter()
    print(f"{w.name}: chunk precompute {t1 - t0:.1f} s, cacheclip_prefill {t2 - t1:.1f} s, full prefill "
          f"{t3 - t2:.1f} s; {len(sel)} rows, top1 clip={int(np.argmax(out['clip_logits']))}")
    return out, (prim, chunks)


def main(names) -> None:
    aux = aux_c2 = None
    if "c2" in names or "p2" in names or "p2d" in names:
        out, aux, aux_c2 = scoring(C2)
        np.savez_compressed(os.path.join(HERE, "c2_scoring.npz"), **out)
    pc = None
    if "p2" in names:
        out, pc = primary(P2, aux, aux_c2)
        np.savez_compressed(os.path.join(HERE, "p2_primary.npz"), **out)
    if "p2d" in names:  # same model and chunks, default 8/5 rule (no full prefill: p2 holds it)
        out, pc = primary(P2D, aux, aux_c2, full_prefill=False, prim_chunks=pc)
        np.savez_compressed(os.path.join(HERE, "p2d_primary.npz"), **out)
    del pc
    del aux_c2
    if "c3" in names:
        out, _, _ = scoring(C3, aux)
        np.savez_compressed(os.path.join(HERE, "c3_scoring.npz"), **out)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "p2", "p2d", "c3"])
