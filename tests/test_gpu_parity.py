"""End-to-end parity of the device hot path against the CPU oracle and the
reference's own golden outputs (tests/golden/*.npz).

Tolerances (stated here, measured on B200):
  * token selection (indices, window records), merged layout: EXACT;
  * importance scores: rtol 1e-5 (fp32-faithful 3xTF32 scoring model);
  * merged keys/values from identical chunk caches: BITWISE (fp32 rotation
    with separately rounded products, then bf16 rounding);
  * recomputed K/V and first-token logits of the bf16 primary: within
    BF16_KV_RTOL relative L2 / BF16_LOGIT_TOL x std(logits), and never more
    than 2x the error of the device's own dense bf16 full prefill on the same
    inputs (SURVEY §8(c) calibration rule).
"""

import os

import numpy as np
import pytest
import torch

from oracle import cacheclip_oracle as orc
from oracle.synth import B1, C1, C1_EXACT, R1

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
DEV = "cuda"
BF16_KV_RTOL = 2e-2
BF16_LOGIT_TOL = 5e-2


def _cfg(oc: orc.OracleConfig, dtype: str, tokenizer_id: str = "chars"):
    from paper_2510_10129_b200 import ModelConfig
    return ModelConfig(n_layers=oc.n_layers, n_heads=oc.n_heads, d_model=oc.d_model, d_head=oc.d_head,
                       d_ff=oc.d_ff, vocab_size=oc.vocab_size, rope_base=oc.rope_base, norm_eps=oc.norm_eps,
                       activation=oc.activation, mlp_gated=oc.mlp_gated, attn_bias=oc.attn_bias,
                       mlp_bias=oc.mlp_bias, tokenizer_id=tokenizer_id, n_kv_heads=oc.kv_heads, dtype=dtype)


def _bf16_params(p):
    out = {}
    for k, v in p.items():
        out[k] = orc.round_to_bf16(v) if v.ndim == 2 else v
    return out


class Case:
    def __init__(self, w):
        import paper_2510_10129_b200 as cc
        self.w = w
        self.g = dict(np.load(os.path.join(GOLDEN, f"{w.name}.npz")))
        self.p_params = orc.seeded_params(w.primary, w.primary_seed, w.bias_std)
        self.a_params = orc.seeded_params(w.aux, w.aux_seed, w.bias_std)
        self.primary = cc.from_params(_cfg(w.primary, "bf16"), self.p_params)
        self.aux = cc.from_params(_cfg(w.aux, "fp32"), self.a_params)
        self.o_primary = orc.OracleModel(w.primary, _bf16_params(self.p_params))   # same bf16 weights
        self.o_aux = orc.OracleModel(w.aux, self.a_params)
        self.prefix, self.chunk_ids, self.query = w.token_ids(0)
        self.config = cc.SelectionConfig(w.ratio, w.window_len, w.window_threshold)


@pytest.fixture(scope="module", params=[C1, C1_EXACT, B1, R1], ids=lambda w: w.name)
def case(request):
    return Case(request.param)


def _upload_chunk(o: orc.Chunk, dtype, fp):
    import paper_2510_10129_b200 as cc
    k = np.stack(o.keys)
    v = np.stack(o.values)
    return cc.ChunkCache(torch.from_numpy(k).to(DEV, dtype), torch.from_numpy(v).to(DEV, dtype), o.token_ids,
                         o.prefix_len, "chars", fp)


def test_chain_selection_matches_reference(case):
    """Device chunk precompute + scoring + selection reproduce the REFERENCE's
    selected indices and window records exactly (golden fixture)."""
    import paper_2510_10129_b200 as cc
    aux_chunks = [cc.prefill_chunk(case.aux, case.prefix, c) for c in case.chunk_ids]
    scores = cc.aux_score_tokens(case.aux, aux_chunks, case.query)
    np.testing.assert_allclose(scores.scores, case.g["scores"], rtol=1e-5, atol=1e-9)
    sel = cc.select_tokens(scores, case.config)
    sink = case.w.prefix_len
    assert tuple(i + sink for i in sel.indices) == tuple(int(i) for i in case.g["indices"])
    win = np.array([[x.window_id, x.chunk, x.start, x.end, x.selected, int(x.kept), int(x.partial)]
                    for x in sel.windows], dtype=np.int64).reshape(-1, 7)
    np.testing.assert_array_equal(win, case.g["windows"])


def test_stage_parity_from_identical_caches(case):
    """Feed the oracle's own chunk caches to the device path: merge bitwise,
    scores rtol 1e-5, selection exact, recompute + logits within bf16 tolerance."""
    import paper_2510_10129_b200 as cc
    w = case.w
    o_chunks = [orc.prefill_chunk(case.o_primary, case.prefix, c) for c in case.chunk_ids]
    # the device primary stores bf16 caches: round the oracle caches identically
    for ch in o_chunks:
        ch.keys = [orc.round_to_bf16(k) for k in ch.keys]
        ch.values = [orc.round_to_bf16(v) for v in ch.values]
    o_aux_chunks = [orc.prefill_chunk(case.o_aux, case.prefix, c) for c in case.chunk_ids]
    d_chunks = [_upload_chunk(c, torch.bfloat16, case.primary.fingerprint) for c in o_chunks]
    d_aux = [_upload_chunk(c, torch.float32, case.aux.fingerprint) for c in o_aux_chunks]

    # merge: bitwise after bf16 rounding
    merged = cc.merge_caches(d_chunks, case.primary.config.rope, capacity=10_000)
    o_merged = orc.merge(o_chunks, w.primary.d_head, w.primary.rope_base)
    for l in range(w.primary.n_layers):
        np.testing.assert_array_equal(merged.keys[l].float().cpu().numpy(), orc.round_to_bf16(o_merged.keys[l]))
        np.testing.assert_array_equal(merged.values[l].float().cpu().numpy(), o_merged.values[l])
    assert merged.token_ids == o_merged.token_ids and merged.source == o_merged.source

    # scoring + selection
    o_scores = orc.aux_scores(case.o_aux, o_aux_chunks, case.query)
    scores = cc.aux_score_tokens(case.aux, d_aux, case.query)
    np.testing.assert_allclose(scores.scores, o_scores, rtol=1e-5, atol=1e-9)
    o_idx, o_win = orc.select(o_scores, [c.chunk_len for c in o_aux_chunks], w.ratio, w.window_len,
                              w.window_threshold)
    sel = cc.select_tokens(scores, case.config)
    assert sel.indices == o_idx

    # full pipeline from identical caches
    tok = cc.GreedyTokenizer(cc.char_vocab(max(w.primary.vocab_size, w.aux.vocab_size)), "chars")
    out = cc.cacheclip_prefill(case.primary, case.aux, d_chunks, d_aux, tok.decode(case.query), case.config,
                               primary_tokenizer=tok, aux_tokenizer=tok)
    o_out = orc.cacheclip(case.o_primary, case.o_aux, o_chunks, o_aux_chunks, case.query, w.ratio,
                          window_len=w.window_len, threshold=w.window_threshold)
    assert out.plan.indices == o_out.indices
    assert out.cache.recomputed_rows == o_out.cache.recomputed_rows
    assert out.cache.token_ids == o_out.cache.token_ids
    sel_rows = np.asarray(o_out.indices, dtype=np.int64)
    q_rows = np.arange(o_out.cache.n_rows - len(case.query), o_out.cache.n_rows)
    rows = np.concatenate([sel_rows, q_rows])
    for l in range(w.primary.n_layers):
        for got_t, want in ((out.cache.keys[l], o_out.cache.keys[l]), (out.cache.values[l], o_out.cache.values[l])):
            got = got_t.float().cpu().numpy()[rows]
            ref = want[rows]
            rel = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-12)
            assert rel < BF16_KV_RTOL, (l, rel)
    dl = np.abs(out.logits - o_out.logits).max()
    assert dl < BF16_LOGIT_TOL * o_out.logits.std(), dl
    # calibration: the device's dense bf16 full prefill on the same context
    full = cc.full_attention_prefill(case.primary, orc.context_ids(o_chunks, case.query))
    o_full = orc.full_prefill(case.o_primary, orc.context_ids(o_chunks, case.query))
    dense_err = np.abs(full.logits - o_full.logits).max()
    print(f"{w.name}: |dlogits| clip={dl:.3e} dense={dense_err:.3e} std={o_out.logits.std():.3f} "
          f"m={len(out.plan.indices)}")
    assert dl <= 2 * dense_err + 1e-3 * o_out.logits.std()


def test_full_prefill_and_ratio_identities(case):
    import paper_2510_10129_b200 as cc
    w = case.w
    chunks = [cc.prefill_chunk(case.primary, case.prefix, c) for c in case.chunk_ids]
    aux_chunks = [cc.prefill_chunk(case.aux, case.prefix, c) for c in case.chunk_ids]
    ids = cc.reuse_context_ids(chunks, case.query)
    full = cc.full_attention_prefill(case.primary, ids)
    std = case.g["full_logits"].std()
    assert np.abs(full.logits - case.g["full_logits"]).max() < BF16_LOGIT_TOL * std
    # ratio 0 == direct reuse, bitwise on device (test_pipeline.py:124-133)
    clip0 = cc.cacheclip_prefill(case.primary, case.aux, chunks, aux_chunks, case.query,
                                 cc.SelectionConfig(0.0))
    direct = cc.direct_reuse_prefill(case.primary, chunks, case.query)
    assert clip0.plan.indices == ()
    np.testing.assert_array_equal(clip0.logits, direct.logits)
    # ratio 1 == full prefill within the bf16 tolerance (test_pipeline.py:144-150)
    clip1 = cc.cacheclip_prefill(case.primary, case.aux, chunks, aux_chunks, case.query,
                                 cc.SelectionConfig(1.0))
    assert clip1.plan.indices == tuple(range(w.prefix_len, clip1.cache.layout.total))
    assert np.abs(clip1.logits - full.logits).max() < BF16_LOGIT_TOL * std
    # the same two edges through the exact-budget (threshold 1, no host sync)
    # launch: identical results to the synced launch
    for ratio, ref in ((0.0, clip0), (1.0, clip1)):
        d = cc.cacheclip_prefill(case.primary, case.aux, chunks, aux_chunks, case.query,
                                 cc.SelectionConfig(ratio, 8, 1))
        assert d.plan.indices == ref.plan.indices and d.plan.windows == ref.plan.windows
        assert d.cache.recomputed_rows == ref.cache.recomputed_rows
        np.testing.assert_array_equal(d.logits, ref.logits)
    # the CacheClip strategy vs the reference's own first-token logits
    clip = cc.cacheclip_prefill(case.primary, case.aux, chunks, aux_chunks, case.query, case.config)
    assert clip.plan.indices == tuple(int(i) for i in case.g["indices"])
    assert np.abs(clip.logits - case.g["clip_logits"]).max() < BF16_LOGIT_TOL * std
    assert clip.first_token == int(np.argmax(clip.logits))


_SEED_CASES: dict = {}


@pytest.mark.parametrize("wname", ["r1", "c1_exact"])
@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6])
def test_selection_exact_across_seeds(wname, seed):
    """SURVEY §8(d) seeds: for fresh inputs the device chain (chunk precompute
    -> batched scoring -> top-k + windows) selects exactly the oracle chain's
    tokens (the oracle being pinned to the reference above)."""
    import paper_2510_10129_b200 as cc
    from oracle.synth import WORKLOADS
    w = WORKLOADS[wname]
    if wname not in _SEED_CASES:
        _SEED_CASES[wname] = Case(w)
    case = _SEED_CASES[wname]
    prefix, chunk_ids, query = w.token_ids(seed)
    aux_chunks = cc.prefill_chunks(case.aux, prefix, chunk_ids)
    scores = cc.aux_score_tokens(case.aux, aux_chunks, query)
    o_aux = [orc.prefill_chunk(case.o_aux, prefix, c) for c in chunk_ids]
    o_scores = orc.aux_scores(case.o_aux, o_aux, query)
    np.testing.assert_allclose(scores.scores, o_scores, rtol=1e-5, atol=1e-9)
    o_idx, o_win = orc.select(o_scores, [len(c) for c in chunk_ids], w.ratio, w.window_len, w.window_threshold)
    sel = cc.select_tokens(scores, case.config)
    assert sel.indices == o_idx
    assert [(x.start, x.end, x.selected, x.kept, x.partial) for x in sel.windows] == \
        [(x.start, x.end, x.selected, x.kept, x.partial) for x in o_win]


def test_cross_tokenizer_prefill_matches_reference():
    """cacheclip_prefill with different primary / scoring tokenizers
    (pipeline.py:118-226): chunk texts re-encoded by both, the device
    selection projected onto primary rows through the character spans
    (selector.py:217-245). Plan: exact vs the reference's own run; logits:
    bf16 tolerance."""
    import paper_2510_10129_b200 as cc
    from oracle.synth import C1_PRIMARY, X1_AUX, X1_RATIO, X1_WINDOW_THRESHOLD, cross_tokenizer_case
    g = dict(np.load(os.path.join(GOLDEN, "c1.npz")))
    pv, av, prefix_t, chunk_ts, query_t = cross_tokenizer_case(0)
    tp, ta = cc.GreedyTokenizer(pv, "chars"), cc.GreedyTokenizer(av, "chars+merges")
    primary = cc.from_params(_cfg(C1_PRIMARY, "bf16"), orc.seeded_params(C1_PRIMARY, 0))
    aux = cc.from_params(_cfg(X1_AUX, "fp32", "chars+merges"), orc.seeded_params(X1_AUX, 1))
    chunks = [cc.prefill_chunk(primary, tp.encode(prefix_t), tp.encode(t)) for t in chunk_ts]
    aux_chunks = [cc.prefill_chunk(aux, ta.encode(prefix_t), ta.encode(t)) for t in chunk_ts]
    cfg = cc.SelectionConfig(X1_RATIO, 8, X1_WINDOW_THRESHOLD)
    scores = cc.aux_score_tokens(aux, aux_chunks, ta.encode(query_t))
    np.testing.assert_allclose(scores.scores, g["x_scores"], rtol=1e-5, atol=1e-9)
    out = cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query_t, cfg,
                               primary_tokenizer=tp, aux_tokenizer=ta)
    assert out.plan.indices == tuple(int(i) for i in g["x_indices"])
    assert out.plan.effective_ratio == float(g["x_effective_ratio"])
    assert out.cache.recomputed_rows == out.plan.indices
    ref = g["x_clip_logits"]
    assert np.abs(out.logits - ref).max() < BF16_LOGIT_TOL * ref.std()
    assert out.first_token == int(np.argmax(out.logits))


def test_scoring_mixed_prefix_lengths():
    """Chunks precomputed behind different prefixes are each scored against
    their own prefix_len, as the reference does (selector.py:132-179):
    grouped banked launches reassembled in chunk order, rtol 1e-5 vs the oracle."""
    import paper_2510_10129_b200 as cc
    w = C1
    a_params = orc.seeded_params(w.aux, w.aux_seed, w.bias_std)
    aux = cc.from_params(_cfg(w.aux, "fp32"), a_params)
    o_aux = orc.OracleModel(w.aux, a_params)
    prefix, chunk_ids, query = w.token_ids(0)
    prefixes = [prefix, prefix[: max(1, len(prefix) // 2)], prefix, list(prefix) + list(prefix[:3])]
    chunks = chunk_ids[: len(prefixes)]
    d = [cc.prefill_chunk(aux, p, c) for p, c in zip(prefixes, chunks)]
    o = [orc.prefill_chunk(o_aux, p, c) for p, c in zip(prefixes, chunks)]
    got = cc.aux_score_tokens(aux, d, query)
    want = orc.aux_scores(o_aux, o, query)
    assert got.chunk_lens == tuple(len(c) for c in chunks)
    np.testing.assert_allclose(got.scores, want, rtol=1e-5, atol=1e-9)
