"""Batched chunk precompute (prefill_chunks) against the per-chunk path
(prefill_chunk, model.py:538-565, itself pinned to the oracle in
test_gpu_parity.py): the same caches, bit for bit, for ragged chunk lengths
(tile-aligned, one row over, single token), several passes (max_rows), the
bf16 primary engine (head_dim 64 and 128, GQA) and the fp32 scoring engine."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

LENS = (40, 57, 33, 128, 129, 1, 255)


def _model(dtype, d_head, n_heads, kv, d_model, layers=2, vocab=512):
    import paper_2510_10129_b200 as cc
    cfg = cc.ModelConfig(n_layers=layers, n_heads=n_heads, n_kv_heads=kv, d_model=d_model, d_head=d_head,
                         d_ff=4 * d_model, vocab_size=vocab, rope_base=1e4, norm_eps=1e-5, activation="silu",
                         mlp_gated=True, attn_bias=True, tokenizer_id="tiny", dtype=dtype)
    return cc.init_model(cfg, 3, device=torch.device("cuda", 0), source="torch")


def _check(model, max_rows):
    import paper_2510_10129_b200 as cc
    rng = np.random.default_rng(11)
    prefix = rng.integers(0, 512, 16).tolist()
    chunks = [rng.integers(0, 512, n).tolist() for n in LENS]
    one = [cc.prefill_chunk(model, prefix, c) for c in chunks]
    many = cc.prefill_chunks(model, prefix, chunks, max_rows=max_rows)
    torch.cuda.synchronize()
    assert len(many) == len(one)
    for a, b in zip(one, many):
        assert a.token_ids == b.token_ids and a.prefix_len == b.prefix_len
        assert a.model_fingerprint == b.model_fingerprint
        assert a.k.shape == b.k.shape and b.k.is_contiguous()
        assert torch.equal(a.k, b.k), (a.k.float() - b.k.float()).abs().max().item()
        assert torch.equal(a.v, b.v), (a.v.float() - b.v.float()).abs().max().item()


@pytest.mark.parametrize("d_head,n_heads,kv,d_model", [(64, 4, 2, 256), (128, 8, 2, 512)])
@pytest.mark.parametrize("max_rows", [1 << 16, 300])
def test_prefill_chunks_bf16_equals_per_chunk(d_head, n_heads, kv, d_model, max_rows):
    _check(_model("bf16", d_head, n_heads, kv, d_model), max_rows)


@pytest.mark.parametrize("max_rows", [1 << 16, 300])
def test_prefill_chunks_fp32_equals_per_chunk(max_rows):
    _check(_model("fp32", 64, 2, 2, 128), max_rows)


def test_prefill_chunks_feeds_cacheclip_prefill():
    """The batched caches drop into the hot path: same selection and logits."""
    import paper_2510_10129_b200 as cc
    primary = _model("bf16", 64, 4, 2, 256)
    aux = _model("fp32", 64, 2, 2, 128)
    rng = np.random.default_rng(4)
    prefix = rng.integers(0, 512, 16).tolist()
    chunks = [rng.integers(0, 512, 96).tolist() for _ in range(6)]
    query = rng.integers(0, 512, 12).tolist()
    cfg = cc.SelectionConfig(0.25, 8, 1)
    ref = cc.cacheclip_prefill(primary, aux, [cc.prefill_chunk(primary, prefix, c) for c in chunks],
                               [cc.prefill_chunk(aux, prefix, c) for c in chunks], query, cfg)
    out = cc.cacheclip_prefill(primary, aux, cc.prefill_chunks(primary, prefix, chunks),
                               cc.prefill_chunks(aux, prefix, chunks), query, cfg)
    assert out.plan.indices == ref.plan.indices
    assert np.array_equal(out.logits, ref.logits)


def test_prefill_chunks_rejects_empty_chunk():
    import paper_2510_10129_b200 as cc
    model = _model("bf16", 64, 4, 2, 256)
    with pytest.raises(ValueError):
        cc.prefill_chunks(model, [1, 2], [[3, 4], []])
    assert cc.prefill_chunks(model, [1, 2], []) == []


def test_host_pinned_caches_equal_device_caches():
    """e2e path: pinned host chunk caches (scoring caches streamed in per
    layer and rotated on the way, primary caches streamed into the merge)
    give bit-identical scores, selection and logits to device caches."""
    import paper_2510_10129_b200 as cc
    primary = _model("bf16", 64, 4, 2, 256)
    aux = _model("fp32", 64, 2, 2, 128)
    rng = np.random.default_rng(8)
    prefix = rng.integers(0, 512, 16).tolist()
    chunks_ids = [rng.integers(0, 512, n).tolist() for n in (96, 40, 130, 7)]
    query = rng.integers(0, 512, 12).tolist()
    cfg = cc.SelectionConfig(0.3, 8, 2)
    pc = cc.prefill_chunks(primary, prefix, chunks_ids)
    ac = cc.prefill_chunks(aux, prefix, chunks_ids)

    def host(c, m):
        return cc.ChunkCache(c.k.cpu().pin_memory(), c.v.cpu().pin_memory(), c.token_ids, c.prefix_len,
                             m.config.tokenizer_id, m.fingerprint)

    dev_out = cc.cacheclip_prefill(primary, aux, pc, ac, query, cfg)
    host_out = cc.cacheclip_prefill(primary, aux, [host(c, primary) for c in pc], [host(c, aux) for c in ac],
                                    query, cfg)
    torch.cuda.synchronize()
    assert host_out.plan.indices == dev_out.plan.indices
    assert host_out.plan.windows == dev_out.plan.windows
    assert np.array_equal(host_out.logits, dev_out.logits)
    s_dev = cc.aux_score_tokens(aux, ac, query).scores
    from paper_2510_10129_b200.kv_store import stream_local_banks
    banks = stream_local_banks([host(c, aux) for c in ac], aux.config.rope, aux.device)
    s_host = cc.aux_score_tokens(aux, [host(c, aux) for c in ac], query, _banks=banks).scores
    assert np.array_equal(s_dev, s_host)


@pytest.mark.parametrize("lens", [(64, 64, 64, 64, 64), (96, 40, 130, 7, 40, 40)])
def test_host_cache_pool_equals_device_caches(lens):
    """Chunk caches in a layer-major pinned HostCachePool (runs of same-length
    chunks in consecutive slots stream as one 2-D DMA per layer; ragged ones
    per chunk) give bit-identical merged caches, scores, selection and logits
    to device-resident caches."""
    import paper_2510_10129_b200 as cc
    from paper_2510_10129_b200.kv_store import _uniform_runs
    primary = _model("bf16", 64, 4, 2, 256)
    aux = _model("fp32", 64, 2, 2, 128)
    rng = np.random.default_rng(9)
    prefix = rng.integers(0, 512, 16).tolist()
    chunks_ids = [rng.integers(0, 512, n).tolist() for n in lens]
    query = rng.integers(0, 512, 12).tolist()
    cfg = cc.SelectionConfig(0.3, 8, 1)
    pc = cc.prefill_chunks(primary, prefix, chunks_ids)
    ac = cc.prefill_chunks(aux, prefix, chunks_ids)
    rows = max(c.n_rows for c in pc)
    ppool = cc.HostCachePool(len(pc), rows, 2, 2, 64, torch.bfloat16)
    apool = cc.HostCachePool(len(ac), rows, 2, 2, 64, torch.float32)
    hp = [ppool.store(c) for c in pc]
    ha = [apool.store(c) for c in ac]
    assert all(c.k.is_pinned() and not c.k.is_contiguous() for c in hp)
    if len(set(lens)) == 1:  # body rows of chunks 1.. are one run; the scoring banks one run
        rb = 2 * 64 * 2
        spec = [(c, 0 if i == 0 else 16, 0, c.n_rows if i == 0 else c.chunk_len) for i, c in enumerate(hp)]
        spec = [(c, s0, sum(x[3] for x in spec[:i]), n) for i, (c, s0, _, n) in enumerate(spec)]
        assert _uniform_runs(spec, rb) == [(0, 1), (1, len(hp))]
    a = cc.merge_caches(pc, primary.config.rope, capacity=1000)
    b = cc.merge_caches(hp, primary.config.rope, capacity=1000, device=primary.device)
    torch.cuda.synchronize()
    assert torch.equal(a.k_store[:, :a.n_rows], b.k_store[:, :b.n_rows])
    assert torch.equal(a.v_store[:, :a.n_rows], b.v_store[:, :b.n_rows])
    dev_out = cc.cacheclip_prefill(primary, aux, pc, ac, query, cfg)
    host_out = cc.cacheclip_prefill(primary, aux, hp, ha, query, cfg)
    serial_out = cc.cacheclip_prefill(primary, aux, hp, ha, query, cfg, workers=1)  # plain uploads, one stream
    torch.cuda.synchronize()
    assert host_out.plan == dev_out.plan == serial_out.plan
    assert np.array_equal(host_out.logits, dev_out.logits)
    assert np.array_equal(serial_out.logits, dev_out.logits)
