"""CPU REFERENCE ARM — test/measurement infrastructure only, never the product.

Times the UNMODIFIED reference package (``cacheclip``, pure Python/numpy,
SURVEY F1) on the host cores for a RAG request of a bench workload. Only
``bench.py`` (its ``--impl reference`` arm and the ``cpu_baseline`` leg) calls
this module.

The reference is installed, not copied, into ``oracle/_ref`` by
``oracle/build_ref.sh`` (``pip install --no-deps --target oracle/_ref
/root/reference/pkg``; git-ignored, it travels to the GPU box with the
snapshot like the built ``.so``). Without it this module raises and bench.py
falls back to the numpy oracle port (``cpu_baseline.kind = "port"``).

A full C3 request does not fit a CPU sample: the reference materialises dense
``(H, m, n)`` fp32 attention maps (~360 GB peak at C3) and
needs ~10^2 TFLOP. So each step runs every stage of ``cacheclip_prefill``
(pipeline.py:156-226) through the reference's own public functions on a
bounded sample of the SAME workload shape, and the request time is
extrapolated stage by stage:

  merge      ``merge_caches`` of all chunks, 1 of L primary layers      x L
  score      ``aux_score_tokens`` of S of n chunks, FULL scoring depth   x n/S
  select     ``select_tokens`` + ``map_selection`` over all N tokens     x 1
  recompute  ``selective_forward`` of r1 and of r2 of m rows (spread like
             the selection), 1 of L layers; the call's fixed cost (the
             bank transposes) and per-row cost are fitted from the two
             samples: (a + b m) x L
  query      ``extend_cache`` of the Q query rows, 1 of L layers,
             minus the head, + the head once (``_final_logits``)

  TTFT_ref = max(merge, score + select) + recompute + query

``max`` because the reference runs merge and scoring on two workers
(pipeline.py:204-214) — the conservative (faster-for-the-reference) choice.
Tokenisation and span alignment (``_chunk_text_and_spans``) are excluded on
both sides. The estimate is validated at C1, where the real
``cacheclip_prefill`` runs in full: ``c1_check`` reports both.

Weights are the reference init recipe's shapes (GQA expanded to MHA,
SURVEY F5) filled by tiling one seeded random block: BLAS timing does not
depend on the values, and 5+ GB of fresh normals would cost the box a minute.
"""

from __future__ import annotations

import os
import sys
import time
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")


def load_reference():
    """The stock ``cacheclip`` package from oracle/_ref (raises if absent)."""
    if not os.path.isdir(os.path.join(REF_DIR, "cacheclip")):
        raise ImportError(f"reference not installed under {REF_DIR} (run oracle/build_ref.sh)")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import cacheclip
    if not os.path.abspath(cacheclip.__file__).startswith(REF_DIR):
        raise ImportError(f"cacheclip resolved to {cacheclip.__file__}, not {REF_DIR}")
    return cacheclip


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        n = [d.get("num_threads", 0) for d in threadpool_info() if d.get("user_api") == "blas"]
        return max(n) if n else os.cpu_count()
    except Exception:  # pragma: no cover
        return os.cpu_count()


def _tiled(rng, shape, std, block=1 << 20):
    """An array of `shape` filled with one tiled N(0, std^2) block (float32)."""
    n = int(np.prod(shape))
    b = (rng.standard_normal(min(n, block), dtype=np.float32) * np.float32(std))
    reps = -(-n // b.size)
    return np.tile(b, reps)[:n].reshape(shape)


def ref_model(ref, cfg, n_layers: int, seed: int, tokenizer_id: str = "chars"):
    """A stock ``cacheclip.Model`` of ``cfg``'s shape with ``n_layers`` layers,
    MHA-expanded (the reference has no GQA)."""
    mc = ref.ModelConfig(n_layers=n_layers, n_heads=cfg.n_heads, d_model=cfg.d_model, d_head=cfg.d_head,
                         d_ff=cfg.d_ff, vocab_size=cfg.vocab_size, rope_base=cfg.rope_base, norm_eps=cfg.norm_eps,
                         activation=cfg.activation, mlp_gated=cfg.mlp_gated, attn_bias=cfg.attn_bias,
                         mlp_bias=getattr(cfg, "mlp_bias", False), tokenizer_id=tokenizer_id)
    rng = np.random.default_rng(seed)
    fan = {"wq": mc.d_model, "wk": mc.d_model, "wv": mc.d_model, "wo": mc.attn_width, "w_gate": mc.d_model,
           "w_in": mc.d_model, "w_out": mc.d_ff}
    params = {}
    for name, shape in ref.model.expected_tensors(mc):
        if name.endswith(".gain"):
            params[name] = np.ones(shape, np.float32)
        elif name.endswith(".bias"):
            params[name] = np.zeros(shape, np.float32)
        elif name == "embed.weight":
            params[name] = _tiled(rng, shape, 1.0)
        elif name == "lm_head.weight":
            params[name] = _tiled(rng, shape, mc.d_model ** -0.5)
        else:
            params[name] = _tiled(rng, shape, fan[name.split(".")[-2]] ** -0.5)
    # a fixed fingerprint skips hashing gigabytes of weights (setup only)
    return ref.Model(mc, params, fingerprint=f"bench-{seed}-{n_layers}")


def _chunk_caches(ref, rng, model, prefix_len, lens, vocab):
    mc = model.config
    prefix = rng.integers(0, vocab, prefix_len).tolist()
    out = []
    shared = None
    for n in lens:
        rows = prefix_len + n
        ks = [rng.standard_normal((rows, mc.n_heads, mc.d_head), dtype=np.float32) for _ in range(mc.n_layers)]
        vs = [rng.standard_normal((rows, mc.n_heads, mc.d_head), dtype=np.float32) for _ in range(mc.n_layers)]
        if shared is None:
            shared = ([k[:prefix_len].copy() for k in ks], [v[:prefix_len].copy() for v in vs])
        for l in range(mc.n_layers):   # identical shared prefix rows (the merge dedups them)
            ks[l][:prefix_len] = shared[0][l]
            vs[l][:prefix_len] = shared[1][l]
        ids = prefix + rng.integers(0, vocab, n).tolist()
        out.append(ref.ChunkCache(ks, vs, ids, prefix_len, mc.tokenizer_id, model.fingerprint))
    return out


@dataclass
class RefShape:
    """What the estimate needs from a bench workload."""
    name: str
    primary: object      # config with n_layers, n_heads, ... (GQA fields ignored: MHA-expanded)
    aux: object
    prefix_len: int
    n_chunks: int
    chunk_len: int
    query_len: int


class RefRequestEstimator:
    """Stage-sampled timing of the stock reference's cacheclip_prefill."""

    def __init__(self, shape: RefShape, ratio: float, window_threshold: int, *, score_chunks: int = 2,
                 recompute_rows: tuple = (32, 128), seed: int = 0):
        ref = self.ref = load_reference()
        self.shape = shape
        self.L = shape.primary.n_layers
        self.n_tok = shape.n_chunks * shape.chunk_len
        self.config = ref.SelectionConfig(recomp_ratio=ratio, window_threshold=window_threshold)
        self.m = ref.selection_budget(ratio, self.n_tok)
        rng = np.random.default_rng(seed)
        vocab = min(shape.primary.vocab_size, shape.aux.vocab_size)
        self.prim1 = ref_model(ref, shape.primary, 1, seed)
        self.aux = ref_model(ref, shape.aux, shape.aux.n_layers, seed + 1)
        self.chunks1 = _chunk_caches(ref, rng, self.prim1, shape.prefix_len, [shape.chunk_len] * shape.n_chunks, vocab)
        self.s = min(score_chunks, shape.n_chunks)
        self.aux_chunks = _chunk_caches(ref, rng, self.aux, shape.prefix_len, [shape.chunk_len] * self.s, vocab)
        self.query = rng.integers(0, vocab, shape.query_len).tolist()
        self.scores = ref.ImportanceScores(scores=rng.random(self.n_tok, dtype=np.float32),
                                           chunk_lens=(shape.chunk_len,) * shape.n_chunks)
        self.spans = [ref.TokenSpan(0, i, i + 1) for i in range(self.n_tok)]
        self.r = tuple(sorted({max(1, min(r, self.m)) for r in recompute_rows}))
        # r rows spread over the chunk tokens like a top-k of random scores
        self.samples = [[shape.prefix_len + int(x) for x in np.linspace(0, self.n_tok - 1, r).round().astype(np.int64)]
                        for r in self.r]

    def step(self) -> dict:
        ref, t = self.ref, time.perf_counter
        t0 = t()
        merged = ref.merge_caches(self.chunks1, self.prim1.config.rope)
        t1 = t()
        ref.aux_score_tokens(self.aux, self.aux_chunks, self.query)
        t2 = t()
        sel = ref.select_tokens(self.scores, self.config)
        plan = ref.map_selection(sel, self.spans, self.spans, index_offset=merged.layout.sink_len)
        t3 = t()
        rec = []
        for idx in self.samples:
            a = t()
            ref.selective_forward(self.prim1, merged, idx)
            rec.append(t() - a)
        t4 = t()
        ref.extend_cache(self.prim1, merged, self.query)
        t5 = t()
        h = np.zeros((1, self.prim1.config.d_model), np.float32) + 1.0
        ref.model._final_logits(self.prim1, h, None, "decode")
        t6 = t()
        L, n = self.L, self.shape.n_chunks
        merge = (t1 - t0) * L
        score = (t2 - t1) * n / self.s
        select = t3 - t2
        head = t6 - t5
        if len(self.r) > 1:  # fixed + per-row cost of one selective_forward call
            b = max((rec[-1] - rec[0]) / (self.r[-1] - self.r[0]), 0.0)
            a = max(rec[0] - b * self.r[0], 0.0)
            if b == 0.0:
                a, b = 0.0, rec[-1] / self.r[-1]
        else:
            a, b = 0.0, rec[0] / self.r[0]
        recompute = (a + b * self.m) * L
        query = max(t5 - t4 - head, 0.0) * L + head
        ttft = max(merge, score + select) + recompute + query
        return {"ttft_s": ttft, "sample_s": t6 - t0, "rows": len(plan.indices),
                "stages_s": {"merge": merge, "score": score, "select": select, "recompute": recompute,
                             "query_and_head": query}}

    def describe(self) -> str:
        sh = self.shape
        return (f"stock reference (oracle/_ref) stages per step: merge_caches of {sh.n_chunks} chunks x 1/{self.L} "
                f"layers; aux_score_tokens of {self.s}/{sh.n_chunks} chunks at full scoring depth "
                f"({sh.aux.n_layers} layers); select_tokens + map_selection over {self.n_tok} tokens; "
                f"selective_forward of {' and '.join(map(str, self.r))} of {self.m} rows x 1/{self.L} layers (fixed + "
                f"per-row cost fitted); extend_cache of "
                f"{sh.query_len} query rows x 1/{self.L} layers + head; extrapolated per stage to the "
                f"{sh.name} request (merge || score as in pipeline.py:204-214; tokenisation excluded)")


def c1_check(ratio: float = 0.2, window_threshold: int = 1, reps: int = 3) -> dict:
    """At C1 (the reference's own CPU-runnable size) time the REAL stock
    ``cacheclip_prefill`` next to this module's stage extrapolation of it."""
    ref = load_reference()
    sys.path.insert(0, os.path.dirname(HERE))
    from oracle.synth import C1 as w
    from oracle import cacheclip_oracle as orc
    shape = RefShape("c1", w.primary, w.aux, w.prefix_len, w.n_chunks, w.chunk_len, w.query_len)
    est = RefRequestEstimator(shape, ratio, window_threshold, score_chunks=2)
    vocab = [chr(0x4E00 + i) for i in range(max(w.primary.vocab_size, w.aux.vocab_size))]
    tok = ref.GreedyTokenizer(vocab, "chars")
    mc = lambda c: ref.ModelConfig(n_layers=c.n_layers, n_heads=c.n_heads, d_model=c.d_model,  # noqa: E731
                                   d_head=c.d_head, d_ff=c.d_ff, vocab_size=c.vocab_size, rope_base=c.rope_base,
                                   norm_eps=c.norm_eps, activation=c.activation, mlp_gated=c.mlp_gated,
                                   attn_bias=c.attn_bias, mlp_bias=c.mlp_bias, tokenizer_id="chars")
    primary = ref.Model(mc(w.primary), orc.mha_expand(w.primary, orc.seeded_params(w.primary, 0)))
    aux = ref.Model(mc(w.aux), orc.mha_expand(w.aux, orc.seeded_params(w.aux, 1)))
    prefix, chunk_ids, query = w.token_ids(0)
    chunks = [ref.prefill_chunk(primary, prefix, c) for c in chunk_ids]
    aux_chunks = [ref.prefill_chunk(aux, prefix, c) for c in chunk_ids]
    cfg = ref.SelectionConfig(recomp_ratio=ratio, window_threshold=window_threshold)
    qt = tok.decode(query)
    real = []
    for _ in range(reps):
        t0 = time.perf_counter()
        ref.cacheclip_prefill(primary, aux, chunks, aux_chunks, qt, cfg, primary_tokenizer=tok, aux_tokenizer=tok)
        real.append(time.perf_counter() - t0)
    ests = [est.step()["ttft_s"] for _ in range(reps)]
    return {"request_ms": 1e3 * float(np.median(real)), "stage_estimate_ms": 1e3 * float(np.median(ests)),
            "note": "real stock cacheclip_prefill at C1 (tokenisation included) vs the stage extrapolation"}
