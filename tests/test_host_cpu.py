"""CPU-side checks: the C-ABI library loads and exports every symbol the
header declares, and the host logic (budget, tokenizers, alignment, MAC
accounting, weight layouts) matches the reference's contracts."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cacheclip_sm100.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|int64_t|void|const char\*)\s+(cc_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2510_10129_b200 import _lib
    lib = _lib.load()
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTED_SYMBOLS)
    assert lib.cc_abi_version() == 1


def test_struct_layouts_match_header():
    from paper_2510_10129_b200 import _lib
    assert ctypes.sizeof(_lib.KvSegment) == 56
    assert ctypes.sizeof(_lib.BankSeq) == 40


def test_budget_kats():
    from paper_2510_10129_b200 import selection_budget
    assert selection_budget(0.2, 125) == 25
    assert selection_budget(0.2, 16) == 4
    assert selection_budget(0.3, 10) == 3
    assert selection_budget(1.0, 7) == 7
    assert selection_budget(0.0, 7) == 0
    assert selection_budget(0.5, 0) == 0
    assert selection_budget(0.2, 32768) == 6554
    with pytest.raises(ValueError):
        selection_budget(0.5, -1)


def test_selection_config_validation():
    from paper_2510_10129_b200 import SelectionConfig
    with pytest.raises(ValueError):
        SelectionConfig(recomp_ratio=1.5)
    with pytest.raises(ValueError):
        SelectionConfig(recomp_ratio=0.5, window_len=0)
    with pytest.raises(ValueError):
        SelectionConfig(recomp_ratio=0.5, window_threshold=9)


def test_tokenizer_roundtrip_and_alignment():
    from paper_2510_10129_b200 import GreedyTokenizer, TokenSpan, align_spans, char_vocab
    from paper_2510_10129_b200.errors import SpanCoverageError, UnknownCharacterError
    tok = GreedyTokenizer(["a", "b", "ab", "abc", " "], "t")
    spans = tok.encode_with_offsets("abcab a")
    assert [s.token_id for s in spans] == [3, 2, 4, 0]
    assert tok.decode(tok.encode("abcab a")) == "abcab a"
    with pytest.raises(UnknownCharacterError):
        tok.encode("z")
    src = [TokenSpan(0, 0, 2), TokenSpan(1, 2, 3)]
    dst = [TokenSpan(0, 0, 1), TokenSpan(1, 1, 3)]
    assert align_spans(src, dst).images == ((0, 1), (1,))
    with pytest.raises(SpanCoverageError):
        align_spans(src, [TokenSpan(0, 0, 1)])
    v = char_vocab(152064)
    assert len(set(v)) == 152064
    ct = GreedyTokenizer(v, "chars")
    ids = list(np.random.default_rng(0).integers(0, 152064, 2000))
    assert ct.encode(ct.decode(ids)) == [int(i) for i in ids]


def test_mac_closed_forms_equal_reference_convention():
    """With n_kv_heads == n_heads the closed forms reproduce the reference's
    full_prefill_macs / extend_macs (flops.py:123-173) term by term."""
    from paper_2510_10129_b200 import ModelConfig, extend_macs, full_prefill_macs
    c = ModelConfig(n_layers=3, n_heads=4, d_model=48, d_head=12, d_ff=96, vocab_size=160, mlp_gated=True)
    L, dm, h, dh = 37, 48, 4, 12
    tri = L * (L + 1) // 2
    ref = 3 * (3 * L * dm * h * dh + L * h * dh * dm + 2 * L * h * 4 * (dh // 2) + 2 * h * tri * dh
               + 3 * L * dm * 96) + dm * 160
    assert full_prefill_macs(c, L) == ref
    n, p = 5, 20
    pairs = n * p + n * (n + 1) // 2
    ref_e = 3 * (3 * n * dm * h * dh + n * h * dh * dm + 2 * n * h * 4 * (dh // 2) + 2 * h * pairs * dh
                 + 3 * n * dm * 96) + dm * 160
    assert extend_macs(c, n, p) == ref_e


def test_glu_interleave_layout():
    import torch
    from paper_2510_10129_b200.weights import _interleave_bias, _interleave_glu
    g = torch.arange(300 * 2, dtype=torch.float32).view(300, 2)
    u = -g
    w = _interleave_glu(g, u)
    assert w.shape == (2 * 384, 2)
    assert torch.equal(w[0:128], g[0:128]) and torch.equal(w[128:256], u[0:128])
    assert torch.equal(w[512:512 + 44], g[256:300]) and torch.equal(w[640:640 + 44], u[256:300])
    assert torch.count_nonzero(w[512 + 44:640]) == 0
    b = _interleave_bias(torch.arange(300.), -torch.arange(300.))
    assert b.shape == (768,) and b[128] == 0 and b[129] == -1


def test_reference_init_matches_oracle_recipe():
    from oracle import cacheclip_oracle as orc
    from oracle.synth import C1_PRIMARY
    from paper_2510_10129_b200 import ModelConfig, reference_init_params
    c = ModelConfig(n_layers=4, n_heads=4, n_kv_heads=2, d_model=256, d_head=64, d_ff=1024, vocab_size=512,
                    rope_base=1e4, activation="silu", mlp_gated=True)
    a = reference_init_params(c, 0)
    b = orc.seeded_params(C1_PRIMARY, 0)
    assert a.keys() == b.keys()
    for k in a:
        np.testing.assert_array_equal(a[k], b[k])


def test_rope_inv_freq_matches_reference_formula():
    from paper_2510_10129_b200 import RopeParams
    r = RopeParams(128, 1e6)
    np.testing.assert_array_equal(r.inv_freq, 1e6 ** (-np.arange(0, 128, 2, dtype=np.float64) / 128))


def test_streamed_layer_groups_cover_every_layer_once():
    from paper_2510_10129_b200.kv_store import PRIMARY_GROUPS, SCORING_GROUPS, _layer_groups
    for n in (1, 2, 3, 5, 11, 24, 28, 48):
        for kw in (SCORING_GROUPS, PRIMARY_GROUPS):
            g = _layer_groups(n, **kw)
            assert g[0][0] == 0 and g[-1][1] == n
            assert all(a[1] == b[0] and a[0] < a[1] for a, b in zip(g, g[1:]))
    assert [l1 - l0 for l0, l1 in _layer_groups(24, **SCORING_GROUPS)] == [1, 2, 3, 6, 6, 4, 2]
    assert [l1 - l0 for l0, l1 in _layer_groups(28, **PRIMARY_GROUPS)] == [1, 3, 6, 8, 8, 2]


def test_uniform_runs_detects_pool_slots():
    """Chunks at a constant stride inside one allocation (HostCachePool slots)
    with the same rows copied and back-to-back destinations form one run;
    anything else breaks it (host logic only: tensors stand in for the pinned
    pool views, which need a GPU to allocate)."""
    from types import SimpleNamespace

    import torch
    from paper_2510_10129_b200.kv_store import _uniform_runs
    pool = torch.zeros(2, 5, 12, 2, 4)  # [L][slots][rows_max][H][D]

    def cc(slot, rows, t=pool):
        return SimpleNamespace(k=t[:, slot, :rows], v=t[:, slot, :rows])

    rb = 2 * 4 * 4
    c = [cc(s, 10) for s in range(5)]
    spec = [(c[0], 0, 0, 10)] + [(c[i], 2, 10 + 8 * (i - 1), 8) for i in range(1, 5)]
    assert _uniform_runs(spec, rb) == [(0, 1), (1, 5)]
    spec[3] = (c[3], 2, 10 + 8 * 2 + 1, 8)  # destination gap before and after chunk 3
    assert _uniform_runs(spec, rb) == [(0, 1), (1, 3), (3, 4), (4, 5)]
    class _Ptr:  # pointer/stride stand-in: slots 2^31 B apart, beyond the 2-D copy pitch limit
        def __init__(self, p):
            self.p = p

        def data_ptr(self):
            return self.p

        def stride(self):
            return (640, 32, 4, 1)

    far = [SimpleNamespace(k=_Ptr(i << 31), v=_Ptr((i << 31) + 4096)) for i in range(3)]
    assert _uniform_runs([(far[i], 2, 8 * i, 8) for i in range(3)], rb) == [(0, 1), (1, 2), (2, 3)]
    # separately allocated caches never form a run, even at a constant stride
    sep = [SimpleNamespace(k=torch.zeros(2, 10, 2, 4), v=torch.zeros(2, 10, 2, 4)) for _ in range(3)]
    assert _uniform_runs([(sep[i], 2, 8 * i, 8) for i in range(3)], rb) == [(0, 1), (1, 2), (2, 3)]
    rag = [(cc(0, 10), 0, 0, 10), (cc(1, 7), 2, 10, 5), (cc(2, 10), 2, 15, 8)]
    assert _uniform_runs(rag, rb) == [(0, 1), (1, 2), (2, 3)]


def test_request_validation_raises_before_any_device_work():
    """The reference's error conventions on the request path (every error a
    ValueError subclass, raised before any mutation: kv_store.py:193-235,
    pipeline.py:156-200, tokenizers.py): checked here on CPU tensors, so no
    kernel can have run when they fire."""
    import pytest
    import torch

    import paper_2510_10129_b200 as cc
    from paper_2510_10129_b200.config import RopeParams

    def chunk(prefix, body, fp="f", tok="t", dtype=torch.float32, heads=2):
        n = len(prefix) + len(body)
        k = torch.zeros(2, n, heads, 8, dtype=dtype)
        return cc.ChunkCache(k, k.clone(), list(prefix) + list(body), len(prefix), tok, fp)

    rope = RopeParams(8)
    a, b = chunk([1, 2], [3, 4, 5]), chunk([1, 2], [6, 7])
    with pytest.raises(cc.CacheConsistencyError):
        cc.merge_caches([], rope)
    with pytest.raises(cc.CacheConsistencyError):  # different prefix tokens
        cc.merge_caches([a, chunk([1, 9], [6])], rope)
    with pytest.raises(cc.CacheConsistencyError):  # different prefix length
        cc.merge_caches([a, chunk([1], [6])], rope)
    with pytest.raises(cc.CacheConsistencyError):  # different model
        cc.merge_caches([a, chunk([1, 2], [6], fp="g")], rope)
    with pytest.raises(cc.CacheConsistencyError):  # different tokenizer
        cc.merge_caches([a, chunk([1, 2], [6], tok="u")], rope)
    with pytest.raises(cc.CacheConsistencyError):  # different geometry
        cc.merge_caches([a, chunk([1, 2], [6], heads=1)], rope)
    with pytest.raises(cc.CacheConsistencyError):  # rows vs ids
        cc.ChunkCache(torch.zeros(2, 3, 2, 8), torch.zeros(2, 3, 2, 8), [1, 2], 1, "t", "f")
    with pytest.raises(cc.CacheConsistencyError):  # K / V shapes
        cc.ChunkCache(torch.zeros(2, 3, 2, 8), torch.zeros(2, 3, 1, 8), [1, 2, 3], 1, "t", "f")
    assert issubclass(cc.CacheConsistencyError, ValueError) and issubclass(cc.DimensionError, ValueError)
    model = object()  # never reached: the pipeline validates its inputs first
    cfg = cc.SelectionConfig(0.2)
    with pytest.raises(ValueError):
        cc.cacheclip_prefill(model, model, [a, b], [a], [1], cfg)      # chunk counts differ
    with pytest.raises(ValueError):
        cc.cacheclip_prefill(model, model, [], [], [1], cfg)          # no chunks
    with pytest.raises(ValueError):
        cc.cacheclip_prefill(model, model, [a], [b], [1], cfg)        # cached texts differ
    with pytest.raises(ValueError):
        cc.cacheclip_prefill(model, model, [a], [a], [], cfg)         # empty query
    with pytest.raises(ValueError):
        cc.cacheclip_prefill(model, model, [a], [a], "text", cfg)     # text query without tokenizers
    with pytest.raises(ValueError):
        cc.SelectionConfig(1.5)


def test_bench_reference_arm_json_contract():
    """`bench.py --impl reference` (the CPU reference path, no GPU needed)
    prints one JSON line with the contract's keys and the SAME metric string,
    unit and direction as our arm (so the driver can form the ratio). C1 keeps
    it fast; the stock reference from oracle/_ref when installed."""
    import json
    import subprocess
    import sys
    sys.path.insert(0, ROOT)
    import bench
    from paper_2510_10129_b200.workloads import WORKLOADS
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "config", "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["metric"] == bench.metric_name(WORKLOADS["c1"], 0.2)
    assert line["unit"] == "tok/s" and line["higher_is_better"] is True
    kind = "reference" if os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "cacheclip")) else "port"
    assert line["cpu_baseline"]["kind"] == kind and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    if kind == "reference":
        assert line["c1_check"]["request_ms"] > 0 and line["stages_ms"]["recompute"] > 0


def test_bench_metric_matches_baseline():
    import json
    import sys
    sys.path.insert(0, ROOT)
    import bench
    from paper_2510_10129_b200.workloads import WORKLOADS
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        assert bench.metric_name(WORKLOADS["c3"], 0.2) == json.load(f)["metric"]


def test_chunk_spans_identity_needs_equal_vocab_contents():
    """the identity-alignment shortcut keys on the vocabulary
    contents, not on tokenizer_id + vocab_size, and still applies the
    reference's re-encode check (pipeline.py:118-153)."""
    from types import SimpleNamespace

    from paper_2510_10129_b200 import GreedyTokenizer
    from paper_2510_10129_b200.pipeline import chunk_spans

    va = ["a", "b", "ab", "c"]
    vb = ["a", "b", "ba", "c"]  # same id, same size, different contents
    ta, tb = GreedyTokenizer(va, "tok"), GreedyTokenizer(vb, "tok")
    assert ta.vocab_digest != tb.vocab_digest
    assert GreedyTokenizer(list(va), "other").vocab_digest == ta.vocab_digest
    mk = lambda ids: SimpleNamespace(chunk_ids=list(ids), chunk_len=len(ids),  # noqa: E731
                                     chunk_key=lambda: np.asarray(ids, dtype=np.int64).tobytes())
    # equal contents: identity alignment
    spans, n = chunk_spans([mk([2, 3])], [mk([2, 3])], ta, GreedyTokenizer(list(va), "x"))
    assert spans is None and n == 2
    # non-canonical cached ids ("a","b" re-encodes to "ab") raise as in the reference
    with pytest.raises(ValueError, match="re-encode"):
        chunk_spans([mk([0, 1])], [mk([0, 1])], ta, ta)
    # colliding id/size but different vocabularies take the full alignment path:
    # "ab" under ta is [2]; under tb the text "ab" encodes to [0, 1]
    spans, n = chunk_spans([mk([2])], [mk([0, 1])], ta, tb)
    assert n is None
    p, a = spans
    assert [s.token_id for s in p] == [2] and [s.token_id for s in a] == [0, 1]


def test_gemm_argument_checks_before_any_device_work():
    """cc_gemm validates its arguments (status codes, no CUDA call) before it
    touches the device: the fused-RMSNorm partial-sum input is bf16-only,
    needs its part count and row pitch, and is refused on a RESIDUAL
    epilogue; shapes and alignment as before. Runs without a GPU."""
    import ctypes

    from paper_2510_10129_b200 import _lib as L
    lib = L.load()

    def args(**kw):
        a = L.GemmArgs()
        a.kind, a.epilogue = L.CC_GEMM_BF16, L.CC_EPI_STORE
        a.M, a.N, a.K = 4, 128, 64
        a.A = a.B = a.C = ctypes.c_void_p(1 << 20)   # aligned, never dereferenced
        a.lda = a.ldb = 64
        a.ldc = 128
        a.c_mode = L.CC_F32
        for k, v in kw.items():
            setattr(a, k, v)
        return a

    def rc(a):
        return lib.cc_gemm(ctypes.byref(a), None)

    ssq = ctypes.c_void_p(1 << 21)
    assert rc(args(M=-1)) == L.CC_ERR_DIMENSION
    assert rc(args(N=100)) == L.CC_ERR_UNSUPPORTED                      # N % 16
    assert rc(args(kind=L.CC_GEMM_TF32X3, lda=192, ldb=192, ssq_in=ssq, n_ssq=2, ld_ssq_in=4)) == \
        L.CC_ERR_UNSUPPORTED                                              # fused norm is bf16-only
    assert rc(args(ssq_in=ssq, n_ssq=0, ld_ssq_in=4)) == L.CC_ERR_DIMENSION
    assert rc(args(ssq_in=ssq, n_ssq=2, ld_ssq_in=2)) == L.CC_ERR_DIMENSION   # ld < M
    assert rc(args(epilogue=L.CC_EPI_RESIDUAL, ssq_in=ssq, n_ssq=2, ld_ssq_in=4)) == L.CC_ERR_UNSUPPORTED
    assert b"ssq" in lib.cc_last_error() or b"RMS" in lib.cc_last_error()
