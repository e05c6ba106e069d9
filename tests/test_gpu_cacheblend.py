"""CacheBlend baseline on the device (selector.py:248-291, pipeline.py:229-255)
against the oracle restatement, which is pinned to the reference's own run
(test_oracle_golden.py::test_cacheblend_matches_reference)."""

import numpy as np
import pytest
import torch

from oracle import cacheclip_oracle as orc
from oracle.synth import C1

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import paper_2510_10129_b200 as cc
    oc = C1.primary
    cfg = cc.ModelConfig(n_layers=oc.n_layers, n_heads=oc.n_heads, d_model=oc.d_model, d_head=oc.d_head,
                         d_ff=oc.d_ff, vocab_size=oc.vocab_size, rope_base=oc.rope_base, norm_eps=oc.norm_eps,
                         activation=oc.activation, mlp_gated=oc.mlp_gated, n_kv_heads=oc.kv_heads, dtype="bf16",
                         tokenizer_id="chars")
    params = orc.seeded_params(oc, 0)
    model = cc.from_params(cfg, params)
    o_model = orc.OracleModel(oc, {k: (orc.round_to_bf16(v) if v.ndim == 2 else v) for k, v in params.items()})
    _, chunk_ids, query = C1.token_ids(0)
    chunks = [cc.prefill_chunk(model, [], c) for c in chunk_ids]
    o_chunks = [orc.prefill_chunk(o_model, [], c) for c in chunk_ids]
    return cc, model, o_model, chunk_ids, query, chunks, o_chunks


def test_discrepancy_and_selection_track_the_oracle(env):
    cc, model, o_model, _, _, chunks, o_chunks = env
    merged = cc.merge_caches(chunks, model.config.rope)
    plan, disc = cc.cacheblend_select(model, merged, 0.2, return_scores=True)
    o_merged = orc.merge(o_chunks, o_model.cfg.d_head, o_model.cfg.rope_base)
    o_idx, o_disc = orc.cacheblend_select(o_model, o_merged, 0.2)
    n = len(o_disc)
    assert disc.shape == (n,) and len(plan.indices) == orc.budget(0.2, n) == len(o_idx)
    assert plan.windows == () and plan.effective_ratio == pytest.approx(len(o_idx) / n)
    # chunk 0 sees no other chunk: its layer-0 recompute equals its cache bit for bit
    assert np.all(disc[:len(chunks[0].chunk_ids)] == 0.0)
    assert np.abs(disc - o_disc).max() <= 0.05 * o_disc.max()
    overlap = len(set(plan.indices) & set(o_idx)) / len(o_idx)
    assert overlap >= 0.85, overlap
    # selection is the exact stable top-k of the device discrepancies
    assert plan.indices == tuple(int(i) for i in orc.top_k_stable(disc, len(o_idx)))


def test_cacheblend_prefill_logits(env):
    cc, model, o_model, _, query, chunks, o_chunks = env
    out = cc.cacheblend_prefill(model, chunks, query, 0.2)
    # the oracle run with the device's selection isolates the recompute numerics
    o_merged = orc.merge(o_chunks, o_model.cfg.d_head, o_model.cfg.rope_base)
    orc.selective(o_model, o_merged, out.plan.indices)
    ref = orc.extend(o_model, o_merged, query)
    assert np.abs(out.logits - ref).max() < 5e-2 * ref.std()
    assert out.first_token == int(np.argmax(out.logits))
    assert out.cache.recomputed_rows == out.plan.indices


def test_cacheblend_ratio_edges_and_errors(env):
    cc, model, _, chunk_ids, query, chunks, _ = env
    none = cc.cacheblend_prefill(model, chunks, query, 0.0)
    direct = cc.direct_reuse_prefill(model, chunks, query)
    assert none.plan.indices == () and np.array_equal(none.logits, direct.logits)
    every = cc.cacheblend_prefill(model, chunks, query, 1.0)
    full = cc.full_attention_prefill(model, cc.reuse_context_ids(chunks, query))
    assert np.abs(every.logits - full.logits).max() < 5e-2 * full.logits.std()
    with pytest.raises(ValueError):
        cc.cacheblend_prefill(model, [cc.prefill_chunk(model, [1, 2], chunk_ids[0])], query, 0.2)
    merged = cc.merge_caches(chunks, model.config.rope)
    with pytest.raises(ValueError):
        cc.cacheblend_select(model, merged, 1.5)
    torch.cuda.synchronize()
