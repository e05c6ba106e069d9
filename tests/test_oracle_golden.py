"""Pin the CPU oracle to the reference's own outputs (tests/golden/*.npz,
made by tests/golden/make_golden.py from the unmodified reference) and to the
reference tests' frozen known-answer values."""

import hashlib
import os

import numpy as np
import pytest

from oracle import cacheclip_oracle as orc
from oracle.synth import B1, C1, C1_EXACT, R1

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _digest(arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, dtype="<f4").tobytes())
    return h.hexdigest()


def _run(w, seed=0):
    prim = orc.OracleModel(w.primary, orc.seeded_params(w.primary, w.primary_seed, w.bias_std))
    aux = orc.OracleModel(w.aux, orc.seeded_params(w.aux, w.aux_seed, w.bias_std))
    prefix, chunk_ids, query = w.token_ids(seed)
    chunks = [orc.prefill_chunk(prim, prefix, c) for c in chunk_ids]
    aux_chunks = [orc.prefill_chunk(aux, prefix, c) for c in chunk_ids]
    direct = orc.merge(chunks, w.primary.d_head, w.primary.rope_base)
    direct_kv = [k.copy() for k in direct.keys] + [v.copy() for v in direct.values]
    out = orc.cacheclip(prim, aux, chunks, aux_chunks, query, w.ratio,
                        window_len=w.window_len, threshold=w.window_threshold)
    full = orc.full_prefill(prim, orc.context_ids(chunks, query))
    return dict(prim=prim, chunks=chunks, direct=direct, direct_kv=direct_kv, out=out, full=full)


@pytest.fixture(scope="module", params=[C1, C1_EXACT, B1, R1], ids=lambda w: w.name)
def case(request):
    w = request.param
    g = dict(np.load(os.path.join(GOLDEN, f"{w.name}.npz")))
    return w, g, _run(w)


def test_selection_is_exact(case):
    w, g, r = case
    out = r["out"]
    assert out.indices == tuple(int(i) for i in g["indices"])
    win = np.array([[x.window_id, x.chunk, x.start, x.end, x.selected, int(x.kept), int(x.partial)]
                    for x in out.windows], dtype=np.int64).reshape(-1, 7)
    np.testing.assert_array_equal(win, g["windows"])
    assert out.cache.recomputed_rows == tuple(int(i) for i in g["recomputed_rows"])
    assert out.cache.token_ids == g["token_ids"].tolist()
    assert [tuple(s) for s in out.cache.source] == [tuple(s) for s in g["source"].tolist()]


def test_scores(case):
    w, g, r = case
    s = r["out"].scores
    if w.aux.group == 1:  # MHA aux: same op sequence as the reference -> bitwise
        assert _digest([s]) == str(g["digest_scores"])
    np.testing.assert_allclose(s, g["scores"], rtol=1e-6, atol=1e-9)


def test_merge_layout_and_rotation(case):
    w, g, r = case
    d = r["direct"]
    rows = g["direct_rows"]
    ks = np.stack([k[rows] for k in d.keys])
    vs = np.stack([v[rows] for v in d.values])
    if w.primary.group == 1:
        assert _digest(r["direct_kv"]) == str(g["digest_direct_kv"])
    np.testing.assert_allclose(ks, g["direct_k"], rtol=0, atol=2e-5)
    np.testing.assert_allclose(vs, g["direct_v"], rtol=0, atol=2e-5)


def test_logits_and_recomputed_kv(case):
    w, g, r = case
    out, full = r["out"], r["full"]
    if w.primary.group == 1:
        assert _digest([out.logits]) == str(g["digest_clip_logits"])
        assert _digest([full.logits]) == str(g["digest_full_logits"])
        assert _digest(list(out.cache.keys) + list(out.cache.values)) == str(g["digest_clip_kv"])
    np.testing.assert_allclose(out.logits, g["clip_logits"], rtol=0, atol=2e-5)
    np.testing.assert_allclose(full.logits, g["full_logits"], rtol=0, atol=2e-5)
    rows = g["rows"]
    np.testing.assert_allclose(np.stack([k[rows] for k in out.cache.keys]), g["clip_k"], rtol=0, atol=2e-5)
    np.testing.assert_allclose(np.stack([v[rows] for v in out.cache.values]), g["clip_v"], rtol=0, atol=2e-5)


# ---- the reference tests' frozen known-answer values -----------------------

COS_1 = 0.5403023058681398   # test_tensor_core.py:18-21
SIN_1 = 0.8414709848078965
SOFTMAX_TEMPERED = (0.24766380113907163, 0.7523361988609285)  # test_tensor_core.py:113


def test_rope_frozen_radian():
    cos, sin = orc.rope_tables(np.array([1]), 2, 10000.0)
    assert cos.dtype == np.float32
    np.testing.assert_allclose([cos[0, 0], sin[0, 0]], [COS_1, SIN_1], rtol=0, atol=1e-7)
    out = orc.rope_rotate(np.array([[1.0, 0.0]], np.float32), np.array([1]), 2, 10000.0)
    np.testing.assert_allclose(out[0], [COS_1, SIN_1], rtol=0, atol=1e-7)


def test_softmax_frozen_pair():
    out = orc.softmax_last(np.array([[0.0, 1.0 / 0.9]], dtype=np.float32))
    np.testing.assert_allclose(out[0], SOFTMAX_TEMPERED, rtol=0, atol=1e-6)


def test_budget_kats():  # test_selector.py:26-34
    assert orc.budget(0.2, 125) == 25
    assert orc.budget(0.2, 16) == 4
    assert orc.budget(0.3, 10) == 3
    assert orc.budget(1.0, 7) == 7
    assert orc.budget(0.0, 7) == 0
    assert orc.budget(0.5, 0) == 0


def test_window_worked_example():  # test_selector.py:49-58
    s = np.array([10, 9, 8, 7, 6, 5, 0, 0, 4, 3, 0, 0, 0, 0, 0, 0], np.float32)
    idx, wins = orc.select(s, [16], 0.5)
    assert idx == (0, 1, 2, 3, 4, 5)
    assert (wins[0].selected, wins[0].kept, wins[1].selected, wins[1].kept) == (6, True, 2, False)


def test_stable_ties():  # test_selector.py:37-41
    np.testing.assert_array_equal(orc.top_k_stable(np.array([1, 3, 3, .5], np.float32), 2), [1, 2])
    np.testing.assert_array_equal(orc.top_k_stable(np.ones(5, np.float32), 3), [0, 1, 2])


def test_full_selection_equals_full_prefill():
    """test_model.py:231-249 on the GQA C1 primary (truncated sizes)."""
    w = C1
    prim = orc.OracleModel(w.primary, orc.seeded_params(w.primary, 0))
    rng = np.random.default_rng(3)
    prefix = rng.integers(0, 512, 4).tolist()
    chunk_ids = [rng.integers(0, 512, n).tolist() for n in (9, 14, 5)]
    chunks = [orc.prefill_chunk(prim, prefix, c) for c in chunk_ids]
    merged = orc.merge(chunks, 64, w.primary.rope_base)
    orc.selective(prim, merged, range(merged.sink_len, merged.n_rows))
    ids = orc.context_ids(chunks, [])
    full = orc.prefill_full(prim, ids)
    pos = np.arange(len(ids))
    for layer in range(w.primary.n_layers):
        np.testing.assert_allclose(merged.keys[layer],
                                   orc.rope_rotate(full.keys[layer], pos, 64, w.primary.rope_base),
                                   rtol=0, atol=1e-4)
        np.testing.assert_allclose(merged.values[layer], full.values[layer], rtol=0, atol=1e-4)


@pytest.mark.parametrize("w", [C1, B1, R1], ids=lambda w: w.name)
def test_cacheblend_matches_reference(w):
    """cacheblend_select / cacheblend_prefill (selector.py:248-291,
    pipeline.py:229-255) against the reference's own run (make_golden.py)."""
    g = dict(np.load(os.path.join(GOLDEN, f"{w.name}.npz")))
    prim = orc.OracleModel(w.primary, orc.seeded_params(w.primary, w.primary_seed, w.bias_std))
    _, chunk_ids, query = w.token_ids(0)
    chunks = [orc.prefill_chunk(prim, [], c) for c in chunk_ids]
    out = orc.cacheblend(prim, chunks, query, w.ratio)
    assert out.indices == tuple(int(i) for i in g["cb_indices"])
    assert out.indices == tuple(int(i) for i in g["cb_select_indices"])
    # the reference L2 runs over MHA-expanded values: sqrt(G) x the GQA norm
    np.testing.assert_allclose(out.scores * np.sqrt(w.primary.group), g["cb_discrepancy"], rtol=1e-5, atol=1e-6)
    if w.primary.group == 1:
        assert _digest([out.logits]) == str(g["digest_cb_logits"])
    np.testing.assert_allclose(out.logits, g["cb_logits"], rtol=0, atol=2e-5)


def test_cacheblend_rejects_prefixed_chunks_and_shallow_models():
    w = B1
    prim = orc.OracleModel(w.primary, orc.seeded_params(w.primary, 0, w.bias_std))
    chunks = [orc.prefill_chunk(prim, [1, 2], [3, 4, 5])]
    with pytest.raises(ValueError):
        orc.cacheblend(prim, chunks, [7], 0.5)
    with pytest.raises(ValueError):
        orc.cacheblend_select(prim, orc.merge(chunks, 64, w.primary.rope_base), 1.5)


def _cross_spans(tok_p, tok_a, chunk_texts):
    """pipeline.py:118-153: per-chunk spans shifted by the running offset."""
    p_spans, a_spans, off = [], [], 0
    for t in chunk_texts:
        p_spans += [type(s)(s.token_id, s.start + off, s.end + off) for s in tok_p.encode_with_offsets(t)]
        a_spans += [type(s)(s.token_id, s.start + off, s.end + off) for s in tok_a.encode_with_offsets(t)]
        off += len(t)
    return p_spans, a_spans


def test_cross_tokenizer_selection_and_projection():
    """Two tokenizers (selector.py:217-245, tokenizers.py:151-177): the
    oracle's aux scores / selection and the package's host-side span
    projection reproduce the reference's own run (tests/golden/c1.npz x_*)."""
    from oracle.synth import C1_PRIMARY, X1_AUX, X1_RATIO, X1_WINDOW_THRESHOLD, cross_tokenizer_case
    from paper_2510_10129_b200 import AuxSelection, GreedyTokenizer
    from paper_2510_10129_b200.selector import map_selection

    g = np.load(os.path.join(GOLDEN, "c1.npz"))
    pv, av, prefix_t, chunk_ts, query_t = cross_tokenizer_case(0)
    tp, ta = GreedyTokenizer(pv, "chars"), GreedyTokenizer(av, "chars+merges")
    aux = orc.OracleModel(X1_AUX, orc.seeded_params(X1_AUX, 1))
    aux_chunks = [orc.prefill_chunk(aux, ta.encode(prefix_t), ta.encode(t)) for t in chunk_ts]
    scores = orc.aux_scores(aux, aux_chunks, ta.encode(query_t))
    np.testing.assert_allclose(scores, g["x_scores"], rtol=1e-6, atol=0)
    idx, _ = orc.select(scores, [len(ta.encode(t)) for t in chunk_ts], X1_RATIO, 8, X1_WINDOW_THRESHOLD)
    assert idx == tuple(int(i) for i in g["x_aux_indices"])
    p_spans, a_spans = _cross_spans(tp, ta, chunk_ts)
    assert len(a_spans) == int(g["x_n_aux"]) and len(p_spans) == int(g["x_n_primary"])
    assert len(a_spans) < len(p_spans)  # merges make the aux tokenization shorter
    plan = map_selection(AuxSelection(idx, (), len(a_spans), X1_RATIO), a_spans, p_spans,
                         index_offset=len(tp.encode(prefix_t)))
    assert plan.indices == tuple(int(i) for i in g["x_indices"])
    assert plan.effective_ratio == float(g["x_effective_ratio"])
