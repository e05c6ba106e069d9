"""Public API semantics on the device, mirroring the reference tests
(test_model.py:161-305, test_pipeline.py): extend / peek / decode_step,
selective_forward's validation-before-mutation rules, merge-layout fields."""

import numpy as np
import pytest
import torch

from oracle import cacheclip_oracle as orc
from oracle.synth import C1

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import paper_2510_10129_b200 as cc
    w = C1
    oc = w.primary
    cfg = cc.ModelConfig(n_layers=oc.n_layers, n_heads=oc.n_heads, d_model=oc.d_model, d_head=oc.d_head,
                         d_ff=oc.d_ff, vocab_size=oc.vocab_size, rope_base=oc.rope_base, norm_eps=oc.norm_eps,
                         activation=oc.activation, mlp_gated=oc.mlp_gated, n_kv_heads=oc.kv_heads, dtype="bf16",
                         tokenizer_id="chars")
    params = orc.seeded_params(oc, 0)
    model = cc.from_params(cfg, params)
    o_model = orc.OracleModel(oc, {k: (orc.round_to_bf16(v) if v.ndim == 2 else v) for k, v in params.items()})
    rng = np.random.default_rng(5)
    prefix = rng.integers(0, 512, 6).tolist()
    chunk_ids = [rng.integers(0, 512, n).tolist() for n in (40, 57, 33)]
    chunks = [cc.prefill_chunk(model, prefix, c) for c in chunk_ids]
    return cc, model, o_model, prefix, chunk_ids, chunks


def test_selective_forward_rejects_bad_selections(env):
    cc, model, _, prefix, _, chunks = env
    merged = cc.merge_caches(chunks, model.config.rope)
    before = merged.keys[0].clone()
    for bad in ((8, 8), (0,), (merged.n_rows,)):
        with pytest.raises(ValueError):
            cc.selective_forward(model, merged, bad)
    assert torch.equal(merged.keys[0], before)  # nothing mutated
    assert cc.selective_forward(model, merged, ()) is merged  # empty selection is a no-op


def test_selective_forward_touches_only_selected_rows(env):
    cc, model, _, _, _, chunks = env
    merged = cc.merge_caches(chunks, model.config.rope)
    untouched = [k.clone() for k in merged.keys]
    picked = (7, 30, 61)
    cc.selective_forward(model, merged, picked)
    mask = torch.ones(merged.n_rows, dtype=torch.bool, device=untouched[0].device)
    mask[list(picked)] = False
    for layer in range(model.config.n_layers):
        assert torch.equal(merged.keys[layer][mask], untouched[layer][mask])
        assert not torch.equal(merged.keys[layer][~mask], untouched[layer][~mask])
    assert merged.recomputed_rows == picked


def test_extend_peek_decode(env):
    cc, model, o_model, prefix, chunk_ids, chunks = env
    merged = cc.merge_caches(chunks, model.config.rope)
    n0 = merged.n_rows
    peek, _ = cc.peek_forward(model, merged, [5, 7])
    assert merged.n_rows == n0
    logits, _ = cc.extend_cache(model, merged, [5, 7])
    np.testing.assert_array_equal(peek, logits)
    assert merged.n_rows == n0 + 2 and merged.token_ids[-2:] == [5, 7]
    assert merged.source[-2:] == [(-1, n0), (-1, n0 + 1)]
    np.testing.assert_array_equal(merged.positions, np.arange(n0 + 2))
    # decode: contiguous positions only (model.py:649-666)
    tok = int(np.argmax(logits))
    l2, same = cc.decode_step(model, merged, tok, position=n0 + 2)
    assert same is merged and merged.n_rows == n0 + 3
    with pytest.raises(ValueError):
        cc.decode_step(model, merged, tok, position=n0 + 9)
    # against the oracle's direct-reuse + decode on the same bf16 weights
    o_chunks = [orc.prefill_chunk(o_model, prefix, c) for c in chunk_ids]
    o_merged = orc.merge(o_chunks, model.config.d_head, model.config.rope_base)
    o_logits = orc.extend(o_model, o_merged, [5, 7])
    o_l2 = orc.extend(o_model, o_merged, [tok])
    std = o_logits.std()
    assert np.abs(logits - o_logits).max() < 5e-2 * std
    assert np.abs(l2 - o_l2).max() < 5e-2 * std


def test_single_chunk_extend_equals_full_prefill(env):
    """Merging one chunk then extending equals a full prefill of the same ids
    (test_model.py:161-174, within the bf16 tolerance)."""
    cc, model, _, prefix, chunk_ids, _ = env
    one = cc.prefill_chunk(model, prefix, chunk_ids[0])
    merged = cc.merge_caches([one], model.config.rope)
    tail = [3, 1, 4, 1, 5]
    logits, _ = cc.extend_cache(model, merged, tail)
    full = cc.prefill_full(model, prefix + chunk_ids[0] + tail)
    assert np.abs(logits - full.logits).max() < 5e-2 * full.logits.std()


def test_merge_layout_fields(env):
    cc, model, _, prefix, chunk_ids, chunks = env
    merged = cc.merge_caches(chunks, model.config.rope)
    assert merged.layout.sink_len == len(prefix)
    assert merged.layout.chunk_lens == tuple(len(c) for c in chunk_ids)
    assert merged.token_ids == prefix + [t for c in chunk_ids for t in c]
    assert merged.source[:len(prefix)] == [(0, r) for r in range(len(prefix))]
    assert merged.source[len(prefix)] == (0, len(prefix))
    assert merged.source[-1] == (2, len(prefix) + len(chunk_ids[2]) - 1)
    bad = cc.ChunkCache(chunks[1].k, chunks[1].v, chunks[1].token_ids, chunks[1].prefix_len, "other",
                        chunks[1].model_fingerprint)
    with pytest.raises(cc.CacheConsistencyError):
        cc.merge_caches([chunks[0], bad], model.config.rope)


def test_cache_dtype_must_match_model(env, tmp_path):
    """fp32 chunk caches (a reference v1 .cclp file) given to
    the bf16 primary raise CacheConsistencyError before any device work, and
    bf16 caches given to the fp32 scoring model are rejected the same way;
    ``load_cache(dtype=torch.bfloat16)`` makes the v1 file usable, bitwise
    equal to the original bf16 caches (bf16 -> fp32 -> bf16 is lossless)."""
    cc, model, _, prefix, chunk_ids, chunks = env
    path = tmp_path / "c0.cclp"
    c0 = chunks[0]
    cc.save_cache(cc.ChunkCache(c0.k.float().cpu(), c0.v.float().cpu(), c0.token_ids, c0.prefix_len,
                                c0.tokenizer_id, c0.model_fingerprint), path)
    assert int.from_bytes(path.read_bytes()[4:8], "little") == 1  # reference format v1 (fp32)
    v1 = cc.load_cache(path, device="cuda")
    with pytest.raises(cc.CacheConsistencyError):
        cc.direct_reuse_prefill(model, [v1] + list(chunks[1:]), [1, 2, 3])
    with pytest.raises(cc.CacheConsistencyError):
        cc.cacheclip_prefill(model, model, [v1], [v1], [1, 2, 3], cc.SelectionConfig(0.2))
    conv = cc.load_cache(path, device="cuda", dtype=torch.bfloat16)
    assert torch.equal(conv.k, c0.k) and torch.equal(conv.v, c0.v)
    a = cc.direct_reuse_prefill(model, [conv] + list(chunks[1:]), [1, 2, 3])
    b = cc.direct_reuse_prefill(model, list(chunks), [1, 2, 3])
    np.testing.assert_array_equal(a.logits, b.logits)


_FUSE_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2510_10129_b200 as cc
from oracle import cacheclip_oracle as orc
from oracle.synth import C1
w = C1
oc = w.primary
cfg = cc.ModelConfig(n_layers=oc.n_layers, n_heads=oc.n_heads, d_model=oc.d_model, d_head=oc.d_head, d_ff=oc.d_ff,
                     vocab_size=oc.vocab_size, rope_base=oc.rope_base, norm_eps=oc.norm_eps,
                     activation=oc.activation, mlp_gated=oc.mlp_gated, n_kv_heads=oc.kv_heads, dtype="bf16",
                     tokenizer_id="chars")
p = orc.seeded_params(oc, 0)
rng = np.random.default_rng(3)
for k in p:   # non-trivial norm gains so the folding is exercised
    if k.endswith(".gain"):
        p[k] = (1.0 + 0.25 * rng.standard_normal(p[k].shape)).astype(np.float32)
model = cc.from_params(cfg, p)
prefix, chunk_ids, query = w.token_ids(0)
ids = prefix + sum(chunk_ids, []) + query
out = cc.full_attention_prefill(model, ids)
np.save(sys.argv[2], out.logits)
"""


def test_fused_rmsnorm_matches_standalone(tmp_path):
    """The bf16 pass folds RMSNorm into the GEMMs (the residual epilogue writes
    bf16(h * gain) and per-row partial sums of h^2, the QKV / GLU epilogues
    scale rows by 1/rms). Against standalone RMSNorm launches
    (CC_FUSED_NORM=0) the dense prefill's logits agree within bf16 rounding,
    and both agree with the fp32 oracle at the same tolerance."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for flag in ("1", "0"):
        f = tmp_path / f"logits_{flag}.npy"
        r = subprocess.run([sys.executable, "-c", _FUSE_SCRIPT, root, str(f)], env=dict(os.environ, CC_FUSED_NORM=flag),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[flag] = np.load(f)
    fused, plain = outs["1"], outs["0"]
    std = plain.std()
    d = np.abs(fused - plain).max()
    print(f"fused vs standalone RMSNorm: max|dlogits| {d:.3e} (std {std:.3f})")
    assert d < 2e-2 * std
    assert not np.array_equal(fused, plain)  # the fused path really ran


_SMALL_GRID_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2510_10129_b200 as cc
from oracle import cacheclip_oracle as orc
# d_model 1024 (16 K-blocks: the few-row GEMMs split along K), 8K-key bank
# (the few-row attention launches split along keys), fused RMSNorm on
oc = orc.OracleConfig(n_layers=2, n_heads=16, n_kv_heads=2, d_model=1024, d_head=128, d_ff=2048,
                      vocab_size=512, rope_base=1e6, norm_eps=1e-6, activation="silu", mlp_gated=True,
                      attn_bias=True)
ac = orc.OracleConfig(n_layers=2, n_heads=4, n_kv_heads=2, d_model=256, d_head=64, d_ff=512, vocab_size=512,
                      rope_base=1e6, norm_eps=1e-6, activation="silu", mlp_gated=True, attn_bias=True)
def cfg(o, dt):
    return cc.ModelConfig(n_layers=o.n_layers, n_heads=o.n_heads, d_model=o.d_model, d_head=o.d_head, d_ff=o.d_ff,
                          vocab_size=o.vocab_size, rope_base=o.rope_base, norm_eps=o.norm_eps, activation=o.activation,
                          mlp_gated=o.mlp_gated, attn_bias=o.attn_bias, n_kv_heads=o.kv_heads, dtype=dt,
                          tokenizer_id="chars")
primary = cc.from_params(cfg(oc, "bf16"), orc.seeded_params(oc, 0, 0.05))
aux = cc.from_params(cfg(ac, "fp32"), orc.seeded_params(ac, 1, 0.05))
rng = np.random.default_rng(5)
prefix = rng.integers(0, 512, 32).tolist()
chunk_ids = [rng.integers(0, 512, 512).tolist() for _ in range(16)]
query = rng.integers(0, 512, 32).tolist()
chunks = cc.prefill_chunks(primary, prefix, chunk_ids)
aux_chunks = cc.prefill_chunks(aux, prefix, chunk_ids)
out = cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query, cc.SelectionConfig(0.2))  # default 8/5 rule
tok = out.first_token
dec, _ = cc.decode_step(primary, out.cache, tok)
np.savez(sys.argv[2], logits=out.logits, decode=np.asarray(dec), rows=len(out.plan.indices))
"""


def test_small_grid_paths_match_whole_grid_paths(tmp_path):
    """Few-row launches (the default 8/5 rule's recompute, a decode step) take
    the split-K bf16 GEMMs and the split-KV attention; against the same
    request with both disabled (CC_GEMM_SPLITK=0, CC_ATTN_SPLIT=0: the
    whole-grid kernels) the logits agree within bf16 rounding, and the split
    run really differs (it ran)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for flag in ("1", "0"):
        f = tmp_path / f"out_{flag}.npz"
        env = dict(os.environ, CC_GEMM_SPLITK=flag, CC_ATTN_SPLIT=flag)
        r = subprocess.run([sys.executable, "-c", _SMALL_GRID_SCRIPT, root, str(f)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[flag] = dict(np.load(f))
    on, off = outs["1"], outs["0"]
    assert int(on["rows"]) == int(off["rows"]) and int(on["rows"]) < 400
    for key in ("logits", "decode"):
        std = off[key].std()
        d = np.abs(on[key] - off[key]).max()
        print(f"{key}: split vs whole-grid max|d| {d:.3e} (std {std:.3f}), rows {int(on['rows'])}")
        assert d < 2e-2 * std
    assert not np.array_equal(on["logits"], off["logits"])
