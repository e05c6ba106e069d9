"""Parity at the BENCHMARKED sizes against the reference's own outputs
(tests/golden/make_golden_scale.py ran the unmodified reference; VERDICT r1
"What's missing" #1).

* Scoring + selection at C2 (16 x 512) and C3 (64 x 512): the 24-layer
  Qwen2.5-0.5B-shape scoring model (fp32-faithful, 3xTF32 tcgen05) scores
  chunk caches that the DEVICE precomputed (``prefill_chunks``); the device
  top-k + window kernel then selects at ratios 0.05 / 0.2 / 0.4 under the
  default 8/5 rule and the exact-budget rule. Selected indices and window
  records: EXACT vs the reference. Scores: rtol 1e-5 (the budget-boundary
  gaps the reference's scores leave are 4e-5..1.2e-4 relative, printed by
  the generator).
* The 7B-shape primary, depth-truncated to 2 layers (P2, C2 context): the
  full ``cacheclip_prefill`` request (exact-budget rule, ratio 0.2, 1,639
  recomputed rows). Plan: EXACT. Recomputed K/V of sampled selected rows and
  of the query rows: relative L2 < 2e-2 per layer. First-token logits: within
  5e-2 x std and within 2x the error of the device's own dense bf16 full
  prefill against the reference's full prefill (SURVEY §8(c) calibration).

Weights are regenerated from the seed (``seeded_params(fast=True)``), the
same generator the reference was fed; the bf16 primary rounds them to bf16
(round-to-nearest-even) exactly as the reference's copy was rounded.
"""

import os

import numpy as np
import pytest
import torch

from oracle import cacheclip_oracle as orc
from oracle.synth import C2, C3, P2, P2D, SCALE_RATIOS, SCALE_THRESHOLDS

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SCORE_RTOL = 1e-5
KV_RTOL = 2e-2
LOGIT_TOL = 5e-2


def _cfg(oc, dtype):
    from paper_2510_10129_b200 import ModelConfig
    return ModelConfig(n_layers=oc.n_layers, n_heads=oc.n_heads, d_model=oc.d_model, d_head=oc.d_head,
                       d_ff=oc.d_ff, vocab_size=oc.vocab_size, rope_base=oc.rope_base, norm_eps=oc.norm_eps,
                       activation=oc.activation, mlp_gated=oc.mlp_gated, attn_bias=oc.attn_bias,
                       mlp_bias=oc.mlp_bias, tokenizer_id="chars", n_kv_heads=oc.kv_heads, dtype=dtype)


_AUX = {}


def _aux():
    import paper_2510_10129_b200 as cc
    if "m" not in _AUX:
        _AUX["m"] = cc.from_params(_cfg(C2.aux, "fp32"), orc.seeded_params(C2.aux, C2.aux_seed, fast=True))
    return _AUX["m"]


def _windows(sel):
    return np.array([[x.window_id, x.chunk, x.start, x.end, x.selected, int(x.kept), int(x.partial)]
                     for x in sel.windows], dtype=np.int32).reshape(-1, 7)


@pytest.mark.parametrize("w", [C2, C3], ids=lambda w: w.name)
def test_scoring_selection_matches_reference_at_scale(w):
    import paper_2510_10129_b200 as cc
    path = os.path.join(GOLDEN, f"{w.name}_scoring.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    g = dict(np.load(path))
    aux = _aux()
    prefix, chunk_ids, query = w.token_ids(0)
    aux_chunks = cc.prefill_chunks(aux, prefix, chunk_ids)
    scores = cc.aux_score_tokens(aux, aux_chunks, query)
    del aux_chunks
    s = np.asarray(scores.scores, dtype=np.float32)
    ref = g["scores"]
    rel = np.abs(s - ref) / np.maximum(np.abs(ref), 1e-30)
    print(f"{w.name}: {s.size} scores, max rel err {rel.max():.3e}, median {np.median(rel):.3e}")
    assert tuple(scores.chunk_lens) == tuple(int(x) for x in g["chunk_lens"])
    bad = []
    for ratio in SCALE_RATIOS:
        for thr in SCALE_THRESHOLDS:
            sel = cc.select_tokens(scores, cc.SelectionConfig(ratio, 8, thr))
            want = g[f"idx_{ratio}_{thr}"]
            got = np.asarray(sel.indices, dtype=np.int64)
            if got.shape != want.shape or not np.array_equal(got, want):
                diff = np.setxor1d(got, want)
                bad.append(f"ratio {ratio} thr {thr}: {diff.size} indices differ (boundary gap "
                           f"{float(g[f'gap_{ratio}']):.3e}); first {diff[:8].tolist()}")
                continue
            np.testing.assert_array_equal(_windows(sel), g[f"win_{ratio}_{thr}"])
    assert not bad, f"{w.name}: " + "; ".join(bad)
    np.testing.assert_allclose(s, ref, rtol=SCORE_RTOL, atol=0)


@pytest.mark.parametrize("w", [P2, P2D], ids=lambda w: w.name)
def test_truncated_7b_primary_request_matches_reference(w):
    """P2: the exact-budget rule (1,639 rows). P2D: the paper's default 8/5
    rule (a few hundred rows), whose launches take the small-grid paths: the
    work-aware split-KV attention + LSE merge and the split-K bf16 GEMMs
    (asserted below), against the same reference logits tolerance; the dense
    error bound comes from P2's reference full prefill (same model, context)."""
    import paper_2510_10129_b200 as cc
    from paper_2510_10129_b200 import _lib
    path = os.path.join(GOLDEN, f"{w.name}_primary.npz")
    full_path = os.path.join(GOLDEN, "p2_primary.npz")
    if not os.path.exists(path) or not os.path.exists(full_path):
        pytest.skip(f"{path} not generated")
    g = dict(np.load(path))
    g_full = np.load(full_path)["full_logits"]
    aux = _aux()
    primary = cc.from_params(_cfg(w.primary, "bf16"), orc.seeded_params(w.primary, w.primary_seed, fast=True))
    prefix, chunk_ids, query = w.token_ids(0)
    chunks = cc.prefill_chunks(primary, prefix, chunk_ids)
    aux_chunks = cc.prefill_chunks(aux, prefix, chunk_ids)
    out = cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query,
                               cc.SelectionConfig(w.ratio, w.window_len, w.window_threshold))
    assert out.plan.indices == tuple(int(i) for i in g["indices"])
    if w is P2D:  # the launches of this request really are the small-grid kinds
        lib = _lib.load()
        rows = len(out.plan.indices) + len(query)
        c = w.primary
        assert lib.cc_attention_splits(rows, c.n_heads, c.kv_heads, out.cache.n_rows) > 1
    assert out.cache.recomputed_rows == out.plan.indices
    for l in range(w.primary.n_layers):
        for rows_key, pre in (("sel_rows", "sel"), ("q_rows", "q")):
            rows = torch.from_numpy(g[rows_key].astype(np.int64)).to(out.cache.keys[l].device)
            for t, name in ((out.cache.keys[l], "k"), (out.cache.values[l], "v")):
                got = t.index_select(0, rows).float().cpu().numpy()
                ref = g[f"{pre}_{name}"][l]
                rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
                print(f"layer {l} {pre} {name}: rel L2 {rel:.3e}")
                assert rel < KV_RTOL, (l, pre, name, rel)
    ref_logits = g["clip_logits"]
    std = float(ref_logits.std())
    dl = float(np.abs(out.logits - ref_logits).max())
    full = cc.full_attention_prefill(primary, cc.reuse_context_ids(chunks, query))
    dense = float(np.abs(full.logits - g_full).max())
    print(f"{w.name}: {len(out.plan.indices)} rows, |dlogits| clip {dl:.3e}, dense {dense:.3e}, std {std:.3f}; "
          f"top1 {out.first_token} "
          f"(ref {int(np.argmax(ref_logits))})")
    assert dl < LOGIT_TOL * std
    assert dl <= 2 * dense + 1e-3 * std
