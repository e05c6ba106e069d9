"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src,
feeds it the seeded workloads of ``oracle/synth.py`` (GQA weights expanded to
MHA by column replication), and stores the outputs the hot path
must reproduce in ``tests/golden/<name>.npz``: aux importance scores, the
selected merged-row indices and window records, first-token logits of the
CacheClip strategy and of full-attention prefill, sampled merged K/V rows,
and SHA-256 digests of the full float32 arrays (for bitwise MHA checks).
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)
sys.path.insert(0, REF_SRC)

import cacheclip as ref  # noqa: E402  (the reference, read-only)

from oracle import cacheclip_oracle as orc  # noqa: E402
from oracle.synth import (B1, C1, C1_EXACT, C1_PRIMARY, R1, X1_AUX, X1_RATIO,  # noqa: E402
                          X1_WINDOW_THRESHOLD, Workload, cross_tokenizer_case)

ROW_STRIDE = 16  # sampled rows kept in the fixture (keeps files small)


def char_vocab(v: int) -> list[str]:
    """V distinct single characters: greedy matching is the identity, so any
    random id sequence round-trips through text."""
    return [chr(0x4E00 + i) for i in range(v)]


def ref_config(cfg: orc.OracleConfig, tokenizer_id: str) -> "ref.ModelConfig":
    return ref.ModelConfig(
        n_layers=cfg.n_layers, n_heads=cfg.n_heads, d_model=cfg.d_model, d_head=cfg.d_head,
        d_ff=cfg.d_ff, vocab_size=cfg.vocab_size, rope_base=cfg.rope_base,
        norm_eps=cfg.norm_eps, activation=cfg.activation, mlp_gated=cfg.mlp_gated,
        attn_bias=cfg.attn_bias, mlp_bias=cfg.mlp_bias, tokenizer_id=tokenizer_id)


def digest(arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, dtype="<f4").tobytes())
    return h.hexdigest()


def run(w: Workload, seed: int = 0) -> dict:
    vocab = char_vocab(max(w.primary.vocab_size, w.aux.vocab_size))
    tok = ref.GreedyTokenizer(vocab, "chars")
    p_params = orc.seeded_params(w.primary, w.primary_seed, w.bias_std)
    a_params = orc.seeded_params(w.aux, w.aux_seed, w.bias_std)
    primary = ref.Model(ref_config(w.primary, "chars"), orc.mha_expand(w.primary, p_params))
    aux = ref.Model(ref_config(w.aux, "chars"), orc.mha_expand(w.aux, a_params))
    prefix, chunk_ids, query = w.token_ids(seed)

    chunks = [ref.prefill_chunk(primary, prefix, c) for c in chunk_ids]
    aux_chunks = [ref.prefill_chunk(aux, prefix, c) for c in chunk_ids]
    scores = ref.aux_score_tokens(aux, aux_chunks, query)
    cfg = ref.SelectionConfig(recomp_ratio=w.ratio, window_len=w.window_len,
                              window_threshold=w.window_threshold)
    merged_direct = ref.merge_caches(chunks, primary.config.rope)
    direct_keys = [k.copy() for k in merged_direct.keys]
    direct_values = [v.copy() for v in merged_direct.values]

    query_text = tok.decode(query)
    clip = ref.cacheclip_prefill(primary, aux, chunks, aux_chunks, query_text, cfg,
                                 primary_tokenizer=tok, aux_tokenizer=tok)
    full = ref.full_attention_prefill(primary, ref.reuse_context_ids(chunks, query))

    kv_heads = w.primary.kv_heads
    g = w.primary.group
    # the reference holds MHA-expanded K/V: take one head per KV group
    head_sel = np.arange(kv_heads) * g
    rows = np.arange(0, clip.cache.n_rows, ROW_STRIDE)
    drows = np.arange(0, merged_direct.n_rows, ROW_STRIDE)
    sel = np.asarray(clip.plan.indices, dtype=np.int64)
    win = np.array([[x.window_id, x.chunk, x.start, x.end, x.selected, int(x.kept), int(x.partial)]
                    for x in clip.plan.windows], dtype=np.int64).reshape(-1, 7)
    pchunk_k = np.stack([chunks[1].keys[l][:, head_sel] for l in range(w.primary.n_layers)])
    return dict(
        scores=scores.scores,
        chunk_lens=np.asarray(scores.chunk_lens, dtype=np.int64),
        indices=sel,
        windows=win,
        effective_ratio=np.float64(clip.plan.effective_ratio),
        clip_logits=clip.logits,
        full_logits=full.logits,
        rows=rows,
        direct_rows=drows,
        direct_k=np.stack([k[drows][:, head_sel] for k in direct_keys]),
        direct_v=np.stack([v[drows][:, head_sel] for v in direct_values]),
        clip_k=np.stack([k[rows][:, head_sel] for k in clip.cache.keys]),
        clip_v=np.stack([v[rows][:, head_sel] for v in clip.cache.values]),
        sel_k=np.stack([k[sel][:, head_sel] for k in clip.cache.keys]) if sel.size else np.zeros(0, np.float32),
        chunk1_k=pchunk_k,
        digest_direct_kv=np.array(digest(direct_keys + direct_values)),
        digest_clip_kv=np.array(digest(list(clip.cache.keys) + list(clip.cache.values))),
        digest_clip_logits=np.array(digest([clip.logits])),
        digest_full_logits=np.array(digest([full.logits])),
        digest_scores=np.array(digest([scores.scores])),
        mac_report=np.array([clip.report.selection, clip.report.recompute,
                             clip.report.merge_overhead, clip.report.decode,
                             clip.report.full_prefill_reference], dtype=np.int64),
        token_ids=np.asarray(clip.cache.token_ids, dtype=np.int64),
        source=np.asarray(clip.cache.source, dtype=np.int64),
        recomputed_rows=np.asarray(clip.cache.recomputed_rows, dtype=np.int64),
    )


def run_cacheblend(w: Workload, seed: int = 0) -> dict:
    """cacheblend_prefill (pipeline.py:229-255) on prefix-less chunk caches of
    the workload's chunks (the baseline concatenates raw chunks)."""
    p_params = orc.seeded_params(w.primary, w.primary_seed, w.bias_std)
    primary = ref.Model(ref_config(w.primary, "chars"), orc.mha_expand(w.primary, p_params))
    _, chunk_ids, query = w.token_ids(seed)
    chunks = [ref.prefill_chunk(primary, [], c) for c in chunk_ids]
    merged = ref.merge_caches(chunks, primary.config.rope)
    plan, disc = ref.cacheblend_select(primary, merged, w.ratio, return_scores=True)
    out = ref.cacheblend_prefill(primary, chunks, query, w.ratio)
    return dict(cb_indices=np.asarray(out.plan.indices, dtype=np.int64),
                cb_select_indices=np.asarray(plan.indices, dtype=np.int64),
                cb_discrepancy=np.asarray(disc, dtype=np.float32), cb_logits=out.logits,
                digest_cb_logits=np.array(digest([out.logits])))


def run_cross_tokenizer(seed: int = 0) -> dict:
    """cacheclip_prefill with two different tokenizers (pipeline.py:118-226):
    chunk texts re-encoded by both, the aux selection projected onto primary
    tokens through the character spans (selector.py:217-245)."""
    pv, av, prefix_t, chunk_ts, query_t = cross_tokenizer_case(seed)
    tp, ta = ref.GreedyTokenizer(pv, "chars"), ref.GreedyTokenizer(av, "chars+merges")
    p_params = orc.seeded_params(C1_PRIMARY, 0)
    a_params = orc.seeded_params(X1_AUX, 1)
    primary = ref.Model(ref_config(C1_PRIMARY, "chars"), orc.mha_expand(C1_PRIMARY, p_params))
    aux = ref.Model(ref_config(X1_AUX, "chars+merges"), orc.mha_expand(X1_AUX, a_params))
    chunks = [ref.prefill_chunk(primary, tp.encode(prefix_t), tp.encode(t)) for t in chunk_ts]
    aux_chunks = [ref.prefill_chunk(aux, ta.encode(prefix_t), ta.encode(t)) for t in chunk_ts]
    cfg = ref.SelectionConfig(recomp_ratio=X1_RATIO, window_threshold=X1_WINDOW_THRESHOLD)
    scores = ref.aux_score_tokens(aux, aux_chunks, ta.encode(query_t))
    aux_sel = ref.select_tokens(scores, cfg)
    clip = ref.cacheclip_prefill(primary, aux, chunks, aux_chunks, query_t, cfg,
                                 primary_tokenizer=tp, aux_tokenizer=ta)
    return dict(x_scores=scores.scores, x_aux_indices=np.asarray(aux_sel.indices, dtype=np.int64),
                x_indices=np.asarray(clip.plan.indices, dtype=np.int64),
                x_effective_ratio=np.float64(clip.plan.effective_ratio), x_clip_logits=clip.logits,
                x_n_aux=np.int64(scores.scores.size),
                x_n_primary=np.int64(sum(len(tp.encode(t)) for t in chunk_ts)))


def write_reference_files() -> None:
    """Small .cclp files written by the reference's own save_cache (format v1)."""
    rng = np.random.default_rng(42)
    heads, d_head, layers = 2, 4, 2
    prefix = [1, 2]

    def chunk(body):
        n = len(prefix) + len(body)
        return ref.ChunkCache(
            keys=[rng.standard_normal((n, heads, d_head), dtype=np.float32) for _ in range(layers)],
            values=[rng.standard_normal((n, heads, d_head), dtype=np.float32) for _ in range(layers)],
            token_ids=prefix + list(body), prefix_len=len(prefix), tokenizer_id="t", model_fingerprint="m")

    c0, c1 = chunk([10, 11, 12]), chunk([20, 21])
    for c in (c1,):
        for layer in range(layers):
            c.keys[layer][:2] = c0.keys[layer][:2]
            c.values[layer][:2] = c0.values[layer][:2]
    ref.save_cache(c0, os.path.join(HERE, "ref_chunk.cclp"))
    merged = ref.merge_caches([c0, c1], ref.RopeParams(d_head))
    merged.recomputed_rows = (3,)
    ref.save_cache(merged, os.path.join(HERE, "ref_merged.cclp"))
    np.savez_compressed(os.path.join(HERE, "ref_files.npz"), chunk_token_ids=np.asarray(c0.token_ids),
                        chunk_prefix_len=np.int64(c0.prefix_len), chunk_k=np.stack(c0.keys),
                        chunk_v=np.stack(c0.values), merged_sink=np.int64(merged.layout.sink_len),
                        merged_lens=np.asarray(merged.layout.chunk_lens), merged_k=np.stack(merged.keys))


def main() -> None:
    write_reference_files()
    for w in (C1, C1_EXACT, B1, R1):
        out = run(w)
        if w is not C1_EXACT:
            out.update(run_cacheblend(w))
        if w is C1:
            out.update(run_cross_tokenizer())
        path = os.path.join(HERE, f"{w.name}.npz")
        np.savez_compressed(path, **out)
        print(f"{w.name}: {len(out['indices'])} selected of {out['scores'].size}, "
              f"top1 clip={int(np.argmax(out['clip_logits']))} full={int(np.argmax(out['full_logits']))} -> {path}")


if __name__ == "__main__":
    main()
