"""Kernel-level checks of libcacheclip_sm100.so on a B200, each against a
plain torch / numpy reference of the same op (float64 where it matters)."""

import math

import numpy as np
import pytest
import torch

from oracle import cacheclip_oracle as orc

pytestmark = pytest.mark.gpu

DEV = "cuda"


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2510_10129_b200 import _lib as L
    L.load()
    L.require_device(0)
    return L


def _gemm(kind, epi, A, B, **kw):
    from paper_2510_10129_b200 import runtime
    M, N = A.shape[0], B.shape[0]
    K = B.shape[1] // (3 if kind == 1 else 1)
    runtime.gemm(kind, epi, M, N, K, A, B, **kw)
    torch.cuda.synchronize()


@pytest.mark.parametrize("M,N,K", [(1, 128, 64), (200, 256, 320), (1000, 4608, 512), (300, 1152, 896),
                                   (4096, 4096, 1024)])
def test_gemm_bf16_store(M, N, K):
    from paper_2510_10129_b200 import _lib as L
    g = torch.Generator(device=DEV).manual_seed(M + N + K)
    A = torch.randn(M, K, device=DEV, generator=g).to(torch.bfloat16)
    B = torch.randn(N, K, device=DEV, generator=g).to(torch.bfloat16)
    bias = torch.randn(N, device=DEV, generator=g)
    C = torch.empty(M, N, device=DEV, dtype=torch.float32)
    _gemm(L.CC_GEMM_BF16, L.CC_EPI_STORE, A, B, bias=bias, C=C, ldc=N, c_mode=L.CC_F32)
    ref = A.double() @ B.double().t() + bias.double()
    err = (C.double() - ref).abs().max().item()
    assert err < 1e-3 * math.sqrt(K), err


# (1100, 1152, 2080): CTA-pair tiles with a ragged last pair (rows 1024..1099 in
# one CTA, none in its peer) and a last phase of 1 K-block (65 = 8 x 8 + 1)
@pytest.mark.parametrize("M,N,K", [(64, 128, 128), (2048, 1152, 896), (33, 4864 * 2 // 2, 896), (1100, 1152, 2080)])
def test_gemm_tf32x3_is_fp32_faithful(M, N, K):
    from paper_2510_10129_b200 import _lib as L
    g = torch.Generator(device=DEV).manual_seed(7 + M)
    a = torch.randn(M, K, device=DEV, generator=g)
    b = torch.randn(N, K, device=DEV, generator=g)
    A = torch.empty(M, 3 * K, device=DEV)
    B = torch.empty(N, 3 * K, device=DEV)
    s = torch.cuda.current_stream().cuda_stream
    L.call("cc_convert_matrix", a.data_ptr(), M, K, A.data_ptr(), L.CC_F32_SPLIT3, 0, s)
    L.call("cc_convert_matrix", b.data_ptr(), N, K, B.data_ptr(), L.CC_F32_SPLIT3, 1, s)
    C = torch.empty(M, N, device=DEV)
    _gemm(L.CC_GEMM_TF32X3, L.CC_EPI_STORE, A, B, C=C, ldc=N, c_mode=L.CC_F32)
    ref = a.double() @ b.double().t()
    err = ((C.double() - ref).abs() / ref.abs().clamp_min(1.0)).max().item()
    fp32 = (a @ b.t()).double()
    err32 = ((fp32 - ref).abs() / ref.abs().clamp_min(1.0)).max().item()
    print(f"tf32x3 M={M} N={N} K={K}: max rel err {err:.2e} (fp32 sgemm {err32:.2e})")
    # tensor-core fp32 accumulation truncates once per MMA step (K=8 slice);
    # the phased accumulation folds every 256 K (8 K-blocks) into fp32
    # registers (round to nearest), so the truncation bias is bounded per
    # phase, not per K
    phase_k = min(K, 256)
    assert err < 5 * (3 * phase_k / 8) * 2.0 ** -23 + 4 * err32, (err, err32)


@pytest.mark.parametrize("epi", ["store", "glu", "residual"])
def test_gemm_tf32x3_row_blocks_bitwise_equal(epi):
    """Every output element of the phased 3xTF32 GEMM accumulates the same
    MMAs, phases and register sums whatever the tiling: an M=2048 GEMM (CTA
    pairs, 256-row tiles) equals its four 512-row blocks (single-CTA tiles,
    128- or 64-wide) bitwise, for store/residual and the GLU register
    epilogue."""
    from paper_2510_10129_b200 import _lib as L, runtime
    M, K = 2048, 896
    N = 2 * 1024 if epi == "glu" else 1152
    n_out = N // 2 if epi == "glu" else N
    g = torch.Generator(device=DEV).manual_seed(11)
    a = torch.randn(M, K, device=DEV, generator=g)
    b = torch.randn(N, K, device=DEV, generator=g) / math.sqrt(K)
    A = torch.empty(M, 3 * K, device=DEV)
    B = torch.empty(N, 3 * K, device=DEV)
    s = torch.cuda.current_stream().cuda_stream
    L.call("cc_convert_matrix", a.data_ptr(), M, K, A.data_ptr(), L.CC_F32_SPLIT3, 0, s)
    L.call("cc_convert_matrix", b.data_ptr(), N, K, B.data_ptr(), L.CC_F32_SPLIT3, 1, s)
    h0 = torch.randn(M, n_out, device=DEV, generator=g)

    def run(r0, r1):
        C = h0[r0:r1].clone()
        kw = dict(C=C, ldc=n_out, c_mode=L.CC_F32)
        e = {"store": L.CC_EPI_STORE, "residual": L.CC_EPI_RESIDUAL, "glu": L.CC_EPI_GLU}[epi]
        if epi == "glu":
            kw.update(act=L.CC_ACT_SILU, n_out=n_out)
        runtime.gemm(L.CC_GEMM_TF32X3, e, r1 - r0, N, K, A[r0:r1], B, **kw)
        return C

    whole = run(0, M)
    blocks = torch.cat([run(r, r + 512) for r in range(0, M, 512)])
    torch.cuda.synchronize()
    assert torch.equal(whole, blocks), epi
    if epi == "glu":   # and the GLU math against fp64
        ref = (a.double() @ b.double().t()).view(M, -1, 2, 128)
        gt, up = ref[:, :, 0].reshape(M, -1), ref[:, :, 1].reshape(M, -1)
        want = torch.nn.functional.silu(gt) * up
        err = ((whole.double() - want).abs() / want.abs().clamp_min(1.0)).max().item()
        assert err < 1e-5, err


def test_gemm_tf32x3_pair_ragged_rows_bitwise_equal():
    """A CTA-pair 3xTF32 GEMM whose last 256-row pair is ragged (M = 1100:
    rows 1024..1099 in one CTA, none in its peer) equals single-CTA GEMMs
    over the same rows bitwise (residual epilogue, QKV-width N)."""
    from paper_2510_10129_b200 import _lib as L
    M, N, K = 1100, 1152, 896
    g = torch.Generator(device=DEV).manual_seed(23)
    a = torch.randn(M, K, device=DEV, generator=g)
    b = torch.randn(N, K, device=DEV, generator=g) / math.sqrt(K)
    A = torch.empty(M, 3 * K, device=DEV)
    B = torch.empty(N, 3 * K, device=DEV)
    s = torch.cuda.current_stream().cuda_stream
    L.call("cc_convert_matrix", a.data_ptr(), M, K, A.data_ptr(), L.CC_F32_SPLIT3, 0, s)
    L.call("cc_convert_matrix", b.data_ptr(), N, K, B.data_ptr(), L.CC_F32_SPLIT3, 1, s)
    h0 = torch.randn(M, N, device=DEV, generator=g)
    whole = h0.clone()
    _gemm(L.CC_GEMM_TF32X3, L.CC_EPI_RESIDUAL, A, B, C=whole, ldc=N, c_mode=L.CC_F32)
    parts = []
    for r0, r1 in ((0, 600), (600, M)):   # M < 1024: single-CTA tiles
        c = h0[r0:r1].clone()
        _gemm(L.CC_GEMM_TF32X3, L.CC_EPI_RESIDUAL, A[r0:r1], B, C=c, ldc=N, c_mode=L.CC_F32)
        parts.append(c)
    torch.cuda.synchronize()
    assert torch.equal(whole, torch.cat(parts))


@pytest.mark.parametrize("epi", ["store", "residual"])
def test_gemm_tf32x3_narrow_tiles_bitwise_equal(epi):
    """Small-M 3xTF32 GEMMs (128-wide tiles would leave half the SMs idle) run
    64-wide tiles; per element the same MMAs accumulate in the same order, so
    rows of an M=512 GEMM (64-wide) equal the same rows of an M=2048 GEMM
    (128-wide) bitwise."""
    from paper_2510_10129_b200 import _lib as L
    M, N, K = 2048, 1152, 896
    g = torch.Generator(device=DEV).manual_seed(5)
    a = torch.randn(M, K, device=DEV, generator=g)
    b = torch.randn(N, K, device=DEV, generator=g) / math.sqrt(K)
    A = torch.empty(M, 3 * K, device=DEV)
    B = torch.empty(N, 3 * K, device=DEV)
    s = torch.cuda.current_stream().cuda_stream
    L.call("cc_convert_matrix", a.data_ptr(), M, K, A.data_ptr(), L.CC_F32_SPLIT3, 0, s)
    L.call("cc_convert_matrix", b.data_ptr(), N, K, B.data_ptr(), L.CC_F32_SPLIT3, 1, s)
    h0 = torch.randn(M, N, device=DEV, generator=g)
    e = L.CC_EPI_STORE if epi == "store" else L.CC_EPI_RESIDUAL
    wide = h0.clone()
    _gemm(L.CC_GEMM_TF32X3, e, A, B, C=wide, ldc=N, c_mode=L.CC_F32)
    narrow = h0[:512].clone()
    _gemm(L.CC_GEMM_TF32X3, e, A[:512], B, C=narrow, ldc=N, c_mode=L.CC_F32)
    assert torch.equal(wide[:512], narrow)


def test_gemm_residual_and_glu():
    from paper_2510_10129_b200 import _lib as L
    from paper_2510_10129_b200.weights import _interleave_glu, _interleave_bias
    g = torch.Generator(device=DEV).manual_seed(3)
    M, K, FF = 300, 256, 384
    x = torch.randn(M, K, device=DEV, generator=g).to(torch.bfloat16)
    wg = torch.randn(FF, K, device=DEV, generator=g) * 0.05
    wu = torch.randn(FF, K, device=DEV, generator=g) * 0.05
    bg = torch.randn(FF, device=DEV, generator=g) * 0.1
    bu = torch.randn(FF, device=DEV, generator=g) * 0.1
    W = _interleave_glu(wg, wu).to(torch.bfloat16)
    b = _interleave_bias(bg, bu)
    out = torch.empty(M, FF, device=DEV, dtype=torch.float32)
    _gemm(L.CC_GEMM_BF16, L.CC_EPI_GLU, x, W, bias=b, C=out, ldc=FF, c_mode=L.CC_F32, act=L.CC_ACT_SILU, n_out=FF)
    xd = x.double()
    gate = xd @ wg.to(torch.bfloat16).double().t() + bg.double()
    up = xd @ wu.to(torch.bfloat16).double().t() + bu.double()
    ref = gate / (1 + torch.exp(-gate)) * up
    assert (out.double() - ref).abs().max().item() < 2e-3
    # residual: h += x @ W^T
    Wr = (torch.randn(K, K, device=DEV, generator=g) * 0.05).to(torch.bfloat16)
    h = torch.randn(M, K, device=DEV, generator=g)
    h0 = h.clone()
    _gemm(L.CC_GEMM_BF16, L.CC_EPI_RESIDUAL, x, Wr, C=h, ldc=K, c_mode=L.CC_F32)
    ref = h0.double() + xd @ Wr.double().t()
    assert (h.double() - ref).abs().max().item() < 2e-3


@pytest.mark.parametrize("M,N,K", [(1, 3584, 3584), (43, 1024, 1024), (128, 3584, 18944), (43, 4608, 3584)])
def test_gemm_bf16_split_k(M, N, K):
    """Few-row bf16 GEMMs (decode, the default window rule) run split along K:
    slices' fp32 partials summed in slice order by the tile owner, then the
    fused epilogue. Against fp64; bitwise repeatable across launches (the
    per-tile counters re-arm); residual and GLU epilogues too."""
    from paper_2510_10129_b200 import _lib as L
    from paper_2510_10129_b200.weights import _interleave_bias, _interleave_glu
    g = torch.Generator(device=DEV).manual_seed(M + N + K)
    A = torch.randn(M, K, device=DEV, generator=g).to(torch.bfloat16)
    B = (torch.randn(N, K, device=DEV, generator=g) * 0.05).to(torch.bfloat16)
    bias = torch.randn(N, device=DEV, generator=g)
    ref = A.double() @ B.double().t() + bias.double()
    outs = []
    for _ in range(3):
        C = torch.empty(M, N, device=DEV, dtype=torch.float32)
        _gemm(L.CC_GEMM_BF16, L.CC_EPI_STORE, A, B, bias=bias, C=C, ldc=N, c_mode=L.CC_F32)
        outs.append(C)
    err = (outs[0].double() - ref).abs().max().item()
    assert err < 1e-4 * math.sqrt(K), err
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    h = torch.randn(M, N, device=DEV, generator=g) if K == N else None
    if h is not None:  # residual epilogue
        h0 = h.clone()
        _gemm(L.CC_GEMM_BF16, L.CC_EPI_RESIDUAL, A, B, C=h, ldc=N, c_mode=L.CC_F32)
        assert (h.double() - (h0.double() + A.double() @ B.double().t())).abs().max().item() < 1e-4 * math.sqrt(K)
    if N % 256 == 0:  # GLU (gate/up interleaved in 128-row blocks)
        FF = N // 2
        wg, wu = B[:FF].float(), B[FF:].float()
        W = _interleave_glu(wg, wu).to(torch.bfloat16)
        b = _interleave_bias(bias[:FF], bias[FF:])
        out = torch.empty(M, FF, device=DEV, dtype=torch.float32)
        _gemm(L.CC_GEMM_BF16, L.CC_EPI_GLU, A, W, bias=b, C=out, ldc=FF, c_mode=L.CC_F32, act=L.CC_ACT_SILU,
              n_out=FF)
        gate = A.double() @ wg.double().t() + bias[:FF].double()
        up = A.double() @ wu.double().t() + bias[FF:].double()
        glu = gate / (1 + torch.exp(-gate)) * up
        assert (out.double() - glu).abs().max().item() < 2e-4 * math.sqrt(K) * (1 + glu.abs().max().item())


@pytest.mark.parametrize("M,d,Hq,Hkv,dh", [(77, 256, 4, 2, 64), (43, 2048, 16, 2, 128),  # the second splits K
                                             (1, 3584, 28, 4, 128), (3, 256, 4, 2, 64)])  # GEMV (M <= 4)
def test_gemm_qkv_rope_scatter(M, d, Hq, Hkv, dh):
    from paper_2510_10129_b200 import _lib as L
    from paper_2510_10129_b200.config import RopeParams
    from paper_2510_10129_b200.runtime import gemm
    g = torch.Generator(device=DEV).manual_seed(5)
    N = (Hq + 2 * Hkv) * dh
    x = torch.randn(M, d, device=DEV, generator=g).to(torch.bfloat16)
    W = (torch.randn(N, d, device=DEV, generator=g) * 0.05).to(torch.bfloat16)
    bias = torch.randn(N, device=DEV, generator=g) * 0.1
    rows = np.sort(np.random.default_rng(0).choice(1000, M, replace=False)).astype(np.int64)
    pos = torch.from_numpy(rows).to(DEV)
    rope = RopeParams(dh, 1e6)
    cos, sin = rope.angles(rows)
    cos_t, sin_t = torch.from_numpy(cos).to(DEV), torch.from_numpy(sin).to(DEV)
    q = torch.empty(M, Hq * dh, device=DEV, dtype=torch.bfloat16)
    kc = torch.zeros(1000, Hkv, dh, device=DEV, dtype=torch.bfloat16)
    vc = torch.zeros_like(kc)
    kraw = torch.zeros(M, Hkv, dh, device=DEV, dtype=torch.bfloat16)
    gemm(L.CC_GEMM_BF16, L.CC_EPI_QKV_ROPE, M, N, d, x, W, bias=bias, rope=(cos_t, sin_t), q_out=q, ldq=Hq * dh,
         k_cache=kc, v_cache=vc, dst_rows=pos, k_raw=kraw, heads=(Hq, Hkv, dh))
    torch.cuda.synchronize()
    y = (x.float() @ W.float().t() + bias).cpu().numpy()
    qr = y[:, : Hq * dh].reshape(M, Hq, dh)
    kr = y[:, Hq * dh:(Hq + Hkv) * dh].reshape(M, Hkv, dh)
    vr = y[:, (Hq + Hkv) * dh:].reshape(M, Hkv, dh)
    q_ref = orc.rope_rotate(qr, rows, dh, 1e6)
    k_ref = orc.rope_rotate(kr, rows, dh, 1e6)
    tol = 3e-2
    np.testing.assert_allclose(q.float().cpu().numpy().reshape(M, Hq, dh), q_ref, atol=tol, rtol=1e-2)
    np.testing.assert_allclose(kc[pos].float().cpu().numpy(), k_ref, atol=tol, rtol=1e-2)
    np.testing.assert_allclose(vc[pos].float().cpu().numpy(), vr, atol=tol, rtol=1e-2)
    np.testing.assert_allclose(kraw.float().cpu().numpy(), kr, atol=tol, rtol=1e-2)
    untouched = np.setdiff1d(np.arange(1000), rows)
    assert kc[torch.from_numpy(untouched).to(DEV)].abs().max().item() == 0.0


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_assemble_bitwise_rope(dtype):
    """merge_caches rotation vs the oracle: bitwise in fp32 (tensor_core.py:83-84
    separately rounded products, float64 angles), bitwise after bf16 rounding."""
    from paper_2510_10129_b200 import ChunkCache, RopeParams, merge_caches
    rng = np.random.default_rng(11)
    L_, H, D, P = 3, 2, 128, 7
    prefix = list(range(P))
    base = 1e6
    chunks, o_chunks = [], []
    shared_k = rng.standard_normal((L_, P, H, D)).astype(np.float32)
    shared_v = rng.standard_normal((L_, P, H, D)).astype(np.float32)
    for i, n in enumerate((33, 1, 250, 64)):
        k = rng.standard_normal((L_, P + n, H, D)).astype(np.float32) * 3
        v = rng.standard_normal((L_, P + n, H, D)).astype(np.float32)
        k[:, :P], v[:, :P] = shared_k, shared_v
        if dtype == torch.bfloat16:
            k, v = orc.round_to_bf16(k), orc.round_to_bf16(v)
        ids = prefix + list(range(100 + 1000 * i, 100 + 1000 * i + n))
        chunks.append(ChunkCache(torch.from_numpy(k).to(DEV, dtype), torch.from_numpy(v).to(DEV, dtype), ids, P,
                                 "t", "m"))
        o_chunks.append(orc.Chunk([k[l] for l in range(L_)], [v[l] for l in range(L_)], ids, P))
    merged = merge_caches(chunks, RopeParams(D, base), capacity=500)
    ref = orc.merge(o_chunks, D, base)
    assert merged.token_ids == ref.token_ids and merged.source == ref.source
    assert merged.layout.sink_len == P and merged.layout.chunk_lens == ref.chunk_lens
    for l in range(L_):
        got_k = merged.keys[l].float().cpu().numpy()
        want_k = ref.keys[l] if dtype == torch.float32 else orc.round_to_bf16(ref.keys[l])
        np.testing.assert_array_equal(got_k, want_k)
        np.testing.assert_array_equal(merged.values[l].float().cpu().numpy(), ref.values[l])


def _attn_ref(q, k, v, limits, factor):
    """fp64 masked attention; q [m, Hq, D], k/v [n, Hkv, D]."""
    m, Hq, D = q.shape
    G = Hq // k.shape[1]
    kk = k.double().repeat_interleave(G, dim=1)
    vv = v.double().repeat_interleave(G, dim=1)
    s = torch.einsum("mhd,nhd->hmn", q.double(), kk) * factor
    n = k.shape[0]
    mask = torch.arange(n, device=q.device)[None, :] >= limits[:, None]
    s = s.masked_fill(mask[None], float("-inf"))
    w = torch.softmax(s, dim=-1)
    return torch.einsum("hmn,nhd->mhd", w, vv)


ATTN_ABS_TOL = 2e-2     # any element (about 2.5 bf16 ulps at |x| ~ 1)
ATTN_REL_L2 = 8e-3      # whole output: bf16 output rounding alone is ~1.1e-3
ATTN_ROW_REL_L2 = 3e-2  # every (row, head) vector, so one mis-scaled row cannot hide


def _check_attn(out, ref):
    """Absolute, global relative-L2 and per-(row, head) relative-L2 bounds
    against the fp64 reference (an absolute bound alone misses
    softmax-scale regressions on small outputs)."""
    got = out.double().view(ref.shape)
    diff = got - ref
    assert diff.abs().max().item() < ATTN_ABS_TOL, diff.abs().max().item()
    rel = (diff.norm() / ref.norm()).item()
    assert rel < ATTN_REL_L2, rel
    row = (diff.norm(dim=-1) / ref.norm(dim=-1).clamp_min(1e-30)).max().item()
    assert row < ATTN_ROW_REL_L2, row


@pytest.mark.parametrize("entry", ["cc_sparse_row_attention", "cc_sparse_row_attention_mma"])
@pytest.mark.parametrize("D,Hq,Hkv,m,n,spread", [(128, 28, 4, 300, 2000, "sorted"), (64, 4, 2, 100, 1040, "sorted"),
                                                 (128, 8, 8, 5, 70, "sorted"), (128, 28, 4, 1000, 1000, "dense"),
                                                 (64, 14, 2, 777, 5000, "tail")])
def test_sparse_row_attention(entry, D, Hq, Hkv, m, n, spread):
    from paper_2510_10129_b200 import _lib as L
    g = torch.Generator(device=DEV).manual_seed(D + m)
    q = torch.randn(m, Hq, D, device=DEV, generator=g).to(torch.bfloat16)
    k = (torch.randn(n, Hkv, D, device=DEV, generator=g) * 2).to(torch.bfloat16)
    v = torch.randn(n, Hkv, D, device=DEV, generator=g).to(torch.bfloat16)
    if spread == "dense":
        pos = torch.arange(n, device=DEV)
    elif spread == "tail":
        pos = torch.arange(n - m, n, device=DEV)
    else:
        pos = torch.sort(torch.randperm(n, generator=torch.Generator().manual_seed(1))[:m]).values.to(DEV)
    out = torch.zeros(m, Hq * D, device=DEV, dtype=torch.bfloat16)
    factor = 1.0 / math.sqrt(D)
    L.call(entry, q.data_ptr(), Hq * D, pos.data_ptr(), m, k.data_ptr(), v.data_ptr(), n, Hq,
           Hkv, D, factor, None, out.data_ptr(), Hq * D, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = _attn_ref(q, k, v, pos + 1, factor)
    _check_attn(out, ref)


@pytest.mark.parametrize("m,S", [(1, 32), (1, 7), (5, 16), (36, 4)])
def test_split_kv_attention_few_rows(m, S):
    """cc_sparse_row_attention_split (decode steps, the last layer's head row):
    each CTA's key tiles cut into S parts, fp32 partials merged by
    log-sum-exp — against the fp64 reference; and the split-count rule."""
    from paper_2510_10129_b200 import _lib as L
    D, Hq, Hkv, n = 128, 28, 4, 9000
    g = torch.Generator(device=DEV).manual_seed(m + S)
    q = torch.randn(m, Hq, D, device=DEV, generator=g).to(torch.bfloat16)
    k = (torch.randn(n, Hkv, D, device=DEV, generator=g) * 2).to(torch.bfloat16)
    v = torch.randn(n, Hkv, D, device=DEV, generator=g).to(torch.bfloat16)
    pos = torch.arange(n - m, n, device=DEV)  # the newest rows: every key visible
    pos[0] = min(int(pos[0]), 100)            # one row whose keys end in the first parts
    out = torch.zeros(m, Hq * D, device=DEV, dtype=torch.bfloat16)
    o_parts = torch.empty(S, m, Hq, D, device=DEV)
    lse = torch.empty(S, m, Hq, device=DEV)
    factor = 1.0 / math.sqrt(D)
    L.call("cc_sparse_row_attention_split", q.data_ptr(), Hq * D, pos.data_ptr(), None, m, k.data_ptr(),
           v.data_ptr(), n, Hq, Hkv, D, factor, None, S, o_parts.data_ptr(), lse.data_ptr(), out.data_ptr(),
           Hq * D, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = _attn_ref(q, k, v, pos + 1, factor)
    _check_attn(out, ref)
    lib = L.load()
    import os
    if os.environ.get("CC_ATTN_SPLIT", "1") != "0":
        assert lib.cc_attention_splits(1, Hq, Hkv, 32800) == 32
    assert lib.cc_attention_splits(1, Hq, Hkv, 2000) == 1       # short key ranges: never split
    assert lib.cc_attention_splits(6586, Hq, Hkv, 32800) == 1   # full grids: never split


@pytest.mark.parametrize("m,n,spread", [(43, 32800, "tail32"), (300, 9000, "sorted"), (557, 32800, "sorted"), (1000, 20000, "sorted")])
def test_split_kv_attention_small_grids(m, n, spread):
    """Low-ratio / default-rule launches (a few hundred rows over a long key
    bank) take the library's split count; the work-aware parts (long ranges
    cut, short ones whole, unused parts LSE = -inf) merge to the fp64 reference."""
    from paper_2510_10129_b200 import _lib as L
    D, Hq, Hkv = 128, 28, 4
    g = torch.Generator(device=DEV).manual_seed(m)
    q = torch.randn(m, Hq, D, device=DEV, generator=g).to(torch.bfloat16)
    k = (torch.randn(n, Hkv, D, device=DEV, generator=g) * 2).to(torch.bfloat16)
    v = torch.randn(n, Hkv, D, device=DEV, generator=g).to(torch.bfloat16)
    if spread == "tail32":  # selected rows spread out, then 32 query rows at the end
        sel = torch.sort(torch.randperm(n - 32, generator=torch.Generator().manual_seed(3))[:m - 32]).values
        pos = torch.cat([sel, torch.arange(n - 32, n)]).to(DEV)
    else:
        pos = torch.sort(torch.randperm(n, generator=torch.Generator().manual_seed(2))[:m]).values.to(DEV)
    S = L.load().cc_attention_splits(m, Hq, Hkv, n)
    assert S > 1
    out = torch.zeros(m, Hq * D, device=DEV, dtype=torch.bfloat16)
    o_parts = torch.full((S, m, Hq, D), float("nan"), device=DEV)  # unused parts must never be read
    lse = torch.empty(S, m, Hq, device=DEV)
    factor = 1.0 / math.sqrt(D)
    L.call("cc_sparse_row_attention_split", q.data_ptr(), Hq * D, pos.data_ptr(), None, m, k.data_ptr(),
           v.data_ptr(), n, Hq, Hkv, D, factor, None, S, o_parts.data_ptr(), lse.data_ptr(), out.data_ptr(),
           Hq * D, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    _check_attn(out, _attn_ref(q, k, v, pos + 1, factor))
    # rows whose keys end early leave their late parts empty
    assert torch.isinf(lse).any()


def test_sparse_row_attention_row_factor():
    from paper_2510_10129_b200 import _lib as L
    g = torch.Generator(device=DEV).manual_seed(9)
    m, n, Hq, Hkv, D = 40, 600, 8, 2, 128
    q = torch.randn(m, Hq, D, device=DEV, generator=g).to(torch.bfloat16)
    k = torch.randn(n, Hkv, D, device=DEV, generator=g).to(torch.bfloat16)
    v = torch.randn(n, Hkv, D, device=DEV, generator=g).to(torch.bfloat16)
    pos = torch.arange(n - m, n, device=DEV)
    rf = torch.full((m,), 0.9 / (math.sqrt(D) * 0.8), device=DEV)
    out = torch.empty(m, Hq * D, device=DEV, dtype=torch.bfloat16)
    L.call("cc_sparse_row_attention", q.data_ptr(), Hq * D, pos.data_ptr(), m, k.data_ptr(), v.data_ptr(), n, Hq,
           Hkv, D, 0.0, rf.data_ptr(), out.data_ptr(), Hq * D, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = _attn_ref(q, k, v, pos + 1, 0.9 / (math.sqrt(D) * 0.8))
    _check_attn(out, ref)


@pytest.mark.parametrize("fn", ["cc_banked_attention_f32", "cc_banked_attention_simt"])
@pytest.mark.parametrize("Hq,Hkv,D,Q,nbs", [
    (4, 2, 64, 8, (40, 3, 100)),
    (14, 2, 64, 32, (544, 0, 37, 300)),   # the 0.5B scoring model's heads, a C3 chunk bank
    (8, 8, 128, 20, (130, 1)),
    (14, 2, 64, 150, (0, 260)),           # chunk precompute shape: no bank, many new rows
])
def test_banked_attention_f32_matches_reference_math(fn, Hq, Hkv, D, Q, nbs):
    """cc_banked_attention_f32 (tcgen05 3xTF32) and the SIMT cross-check
    against the oracle's attend (tensor_core.py:109-170 order) in float64-free
    numpy fp32: context and last-layer weights at fp32-level tolerance."""
    from paper_2510_10129_b200 import _lib as L
    from paper_2510_10129_b200.runtime import bank_tables
    rng = np.random.default_rng(2 + Q)
    banks = [rng.standard_normal((1, nb, Hkv, D)).astype(np.float32) for nb in nbs]
    vbanks = [rng.standard_normal((1, nb, Hkv, D)).astype(np.float32) for nb in nbs]
    S = len(banks)
    q = rng.standard_normal((S * Q, Hq * D)).astype(np.float32)
    kn = rng.standard_normal((S * Q, Hkv * D)).astype(np.float32)
    vn = rng.standard_normal((S * Q, Hkv * D)).astype(np.float32)
    tk = [torch.from_numpy(b).to(DEV) for b in banks]
    tv = [torch.from_numpy(b).to(DEV) for b in vbanks]
    tables = bank_tables(1, [(tk[s], tv[s], banks[s].shape[1], s * Q, Q) for s in range(S)], DEV)
    qd, kd, vd = (torch.from_numpy(a).to(DEV) for a in (q, kn, vn))
    out = torch.empty(S * Q, Hq * D, device=DEV)
    factor = float(np.float32(1 / math.sqrt(D)))
    maxb = max(b.shape[1] for b in banks)
    st = torch.cuda.current_stream().cuda_stream
    L.call(fn, tables.data_ptr(), S, Q, maxb, qd.data_ptr(), kd.data_ptr(),
           vd.data_ptr(), Hq, Hkv, D, factor, out.data_ptr(), L.CC_F32, None, 0, 0, st)
    w = torch.zeros(S, Hq, Q, max(maxb, 1), device=DEV)
    L.call(fn, tables.data_ptr(), S, Q, maxb, qd.data_ptr(), kd.data_ptr(),
           vd.data_ptr(), Hq, Hkv, D, factor, out.data_ptr(), L.CC_F32, w.data_ptr(), 0, max(maxb, 1), st)
    split = torch.empty(S * Q, 3 * Hq * D, device=DEV)
    L.call(fn, tables.data_ptr(), S, Q, maxb, qd.data_ptr(), kd.data_ptr(),
           vd.data_ptr(), Hq, Hkv, D, factor, split.data_ptr(), L.CC_F32_SPLIT3, None, 0, 0, st)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    wg = w.cpu().numpy()
    sp = split.cpu().numpy()
    w_ = Hq * D
    # split layout [hi | . | lo] (the 3xTF32 GEMM reads hi and lo only; the
    # middle segment is not written): hi + lo reproduces the context to ~2^-22
    np.testing.assert_allclose(sp[:, :w_] + sp[:, 2 * w_:], got, rtol=1e-6, atol=1e-7)
    for s in range(S):
        nb = banks[s].shape[1]
        bank_k = np.concatenate([banks[s][0], kn[s * Q:(s + 1) * Q].reshape(Q, Hkv, D)])
        bank_v = np.concatenate([vbanks[s][0], vn[s * Q:(s + 1) * Q].reshape(Q, Hkv, D)])
        qq = q[s * Q:(s + 1) * Q].reshape(Q, Hq, D).transpose(1, 0, 2)
        ctx, wr = orc.attend(qq, bank_k.transpose(1, 0, 2), bank_v.transpose(1, 0, 2), nb + np.arange(Q) + 1)
        np.testing.assert_allclose(got[s * Q:(s + 1) * Q].reshape(Q, Hq, D), ctx.transpose(1, 0, 2),
                                   rtol=2e-5, atol=2e-6)
        np.testing.assert_allclose(wg[s, :, :, :nb], wr[:, :, :nb], rtol=2e-5, atol=1e-7)


def _sel_gpu(scores, lens, ratio, wl=8, thr=5, expand=False):
    from paper_2510_10129_b200 import ImportanceScores, SelectionConfig, select_tokens
    s = ImportanceScores(torch.from_numpy(np.asarray(scores, np.float32)).to(DEV), lens)
    return select_tokens(s, SelectionConfig(ratio, wl, thr, expand))


def test_select_kernel_matches_oracle_random_and_ties():
    rng = np.random.default_rng(9)
    for trial in range(30):
        n_chunks = int(rng.integers(1, 9))
        lens = [int(x) for x in rng.integers(1, 300, n_chunks)]
        n = sum(lens)
        if trial % 3 == 0:
            s = rng.integers(0, 4, n).astype(np.float32)  # massive ties
        elif trial % 3 == 1:
            s = rng.random(n, dtype=np.float32)
        else:
            s = (rng.random(n) * 1e-3).astype(np.float32)
            s[rng.integers(0, n, n // 4)] = 0.0
        ratio = float(rng.choice([0.0, 0.05, 0.1, 0.2, 0.25, 0.4, 0.5, 1.0]))
        thr = int(rng.integers(0, 9))
        expand = bool(rng.integers(0, 2))
        idx, wins = orc.select(s, lens, ratio, 8, thr, expand)
        got = _sel_gpu(s, lens, ratio, 8, thr, expand)
        assert got.indices == idx, (trial, ratio, thr)
        assert [(w.window_id, w.chunk, w.start, w.end, w.selected, w.kept, w.partial) for w in got.windows] == \
               [(w.window_id, w.chunk, w.start, w.end, w.selected, w.kept, w.partial) for w in wins]


def test_select_kats():
    got = _sel_gpu([10, 9, 8, 7, 6, 5, 0, 0, 4, 3, 0, 0, 0, 0, 0, 0], [16], 0.5)
    assert got.indices == (0, 1, 2, 3, 4, 5)
    from paper_2510_10129_b200 import top_candidates
    np.testing.assert_array_equal(top_candidates(np.array([1, 3, 3, .5], np.float32), 2), [1, 2])
    np.testing.assert_array_equal(top_candidates(np.ones(5, np.float32), 3), [0, 1, 2])
    big = np.random.default_rng(0).random(200_000, dtype=np.float32)
    np.testing.assert_array_equal(top_candidates(big, 40_000), orc.top_k_stable(big, 40_000))


def test_lm_head_argmax():
    from paper_2510_10129_b200 import _lib as L
    g = torch.Generator(device=DEV).manual_seed(4)
    d, V = 3584, 152064
    h = torch.randn(d, device=DEV, generator=g)
    gain = torch.rand(d, device=DEV, generator=g) + 0.5
    W = (torch.randn(V, d, device=DEV, generator=g) * d ** -0.5).to(torch.bfloat16)
    logits = torch.empty(V, device=DEV)
    am = torch.empty(1, dtype=torch.int64, device=DEV)
    ws = torch.empty(64, dtype=torch.uint8, device=DEV)
    L.call("cc_lm_head_argmax", h.data_ptr(), gain.data_ptr(), 1e-6, d, W.data_ptr(), L.CC_BF16, V,
           logits.data_ptr(), am.data_ptr(), ws.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    x = h.double() / torch.sqrt((h.double() ** 2).mean() + 1e-6) * gain.double()
    ref = W.double() @ x
    assert (logits.double() - ref).abs().max().item() < 1e-3
    assert int(am.item()) == int(torch.argmax(logits).item())


def test_streamed_merge_from_pinned_host_matches_device_merge():
    """Host-resident (pinned) chunk caches are merged straight from host memory
    by the copy engines layer group by layer group, keys rotated in place
    (per-layer events) — bitwise equal to the
    device-resident merge; the pipeline result is identical too."""
    import paper_2510_10129_b200 as cc
    from oracle.synth import C1_EXACT as w
    cfgp = cc.ModelConfig(n_layers=w.primary.n_layers, n_heads=w.primary.n_heads, d_model=w.primary.d_model,
                          d_head=w.primary.d_head, d_ff=w.primary.d_ff, vocab_size=w.primary.vocab_size,
                          rope_base=w.primary.rope_base, activation="silu", mlp_gated=True,
                          n_kv_heads=w.primary.kv_heads, dtype="bf16", tokenizer_id="chars")
    cfga = cc.ModelConfig(n_layers=w.aux.n_layers, n_heads=w.aux.n_heads, d_model=w.aux.d_model,
                          d_head=w.aux.d_head, d_ff=w.aux.d_ff, vocab_size=w.aux.vocab_size,
                          rope_base=w.aux.rope_base, activation="silu", mlp_gated=True,
                          n_kv_heads=w.aux.kv_heads, dtype="fp32", tokenizer_id="chars")
    primary = cc.from_params(cfgp, orc.seeded_params(w.primary, 0))
    aux = cc.from_params(cfga, orc.seeded_params(w.aux, 1))
    prefix, chunk_ids, query = w.token_ids(0)
    chunks = [cc.prefill_chunk(primary, prefix, c) for c in chunk_ids]
    aux_chunks = [cc.prefill_chunk(aux, prefix, c) for c in chunk_ids]
    host = [cc.ChunkCache(c.k.cpu().pin_memory(), c.v.cpu().pin_memory(), c.token_ids, c.prefix_len,
                          c.tokenizer_id, c.model_fingerprint) for c in chunks]
    host_aux = [cc.ChunkCache(c.k.cpu().pin_memory(), c.v.cpu().pin_memory(), c.token_ids, c.prefix_len,
                              c.tokenizer_id, c.model_fingerprint) for c in aux_chunks]
    a = cc.merge_caches(chunks, primary.config.rope, capacity=2000)
    b = cc.merge_caches(host, primary.config.rope, capacity=2000, device=DEV)
    assert b.layer_ready is not None and len(b.layer_ready) == primary.config.n_layers
    torch.cuda.synchronize()
    for l in range(primary.config.n_layers):
        assert torch.equal(a.keys[l], b.keys[l]) and torch.equal(a.values[l], b.values[l])
    cfg = cc.SelectionConfig(w.ratio, w.window_len, w.window_threshold)
    r1 = cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query, cfg)
    r2 = cc.cacheclip_prefill(primary, aux, host, host_aux, query, cfg)
    assert r1.plan.indices == r2.plan.indices
    np.testing.assert_array_equal(r1.logits, r2.logits)


def test_batched_silu_is_bitwise_the_ieee_formula():
    """The GLU epilogues' batched SiLU (div.rn fast path for the whole chunk,
    exact fallback outside its range) equals x / (1 + exp(-x)) with IEEE
    division bit for bit, over normal, tiny, huge, subnormal and special inputs."""
    from paper_2510_10129_b200 import _lib as L
    g = torch.Generator(device=DEV).manual_seed(7)
    parts = [torch.randn(1 << 20, device=DEV, generator=g) * s for s in (0.01, 1.0, 10.0, 60.0)]
    bits = torch.randint(0, 2 ** 31 - 1, (1 << 20,), device=DEV, generator=g, dtype=torch.int64).to(torch.int32)
    parts.append(bits.view(torch.float32))           # every exponent, both signs via the next line
    parts.append(-bits.view(torch.float32))
    parts.append(torch.tensor([0.0, -0.0, 1e-45, -1e-45, 1e-38, -1e-38, 88.0, -88.0, 89.0, -89.0, 104.0,
                               -104.0, 3e38, -3e38, float("inf"), float("-inf")], device=DEV))
    x = torch.cat(parts).contiguous()
    x = x[torch.isfinite(x) | torch.isinf(x)]   # NaN payloads excluded (NaN != NaN bitwise is not a defect)
    bad = torch.zeros(1, dtype=torch.int64, device=DEV)
    L.call("cc_check_silu", x.data_ptr(), x.numel(), bad.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert int(bad.item()) == 0


_BAND_SCRIPT = r"""
import sys, math
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
from paper_2510_10129_b200 import _lib as L, runtime
L.load()
DEV = "cuda:0"
g = torch.Generator(device=DEV).manual_seed(5)
# both operands > 60 MB: banded by default
M, N, K = 2600, 3584, 12288
A = torch.randn(M, K, device=DEV, generator=g).to(torch.bfloat16)
B = (torch.randn(N, K, device=DEV, generator=g) * 0.05).to(torch.bfloat16)
bias = torch.randn(N, device=DEV, generator=g)
C = torch.empty(M, N, device=DEV, dtype=torch.float32)
runtime.gemm(L.CC_GEMM_BF16, L.CC_EPI_STORE, M, N, K, A, B, bias=bias, C=C, ldc=N, c_mode=L.CC_F32)
h = torch.randn(M, N, device=DEV, generator=g)
runtime.gemm(L.CC_GEMM_BF16, L.CC_EPI_RESIDUAL, M, N, K, A, B, C=h, ldc=N, c_mode=L.CC_F32)
torch.cuda.synchronize()
ref = (A[:64].double() @ B.double().t() + bias.double())
err = (C[:64].double() - ref).abs().max().item()
assert err < 1e-4 * math.sqrt(K), err
# 3xTF32 on single-CTA tiles (split-plane operands, 12 bytes per element):
# A 80 MB, B 63 MB -> banded by 16 m tiles (21 m tiles: a ragged last band)
M2, N2, K2 = 2600, 2048, 2560
a = torch.randn(M2, K2, device=DEV, generator=g)
b = torch.randn(N2, K2, device=DEV, generator=g)
A2 = torch.empty(M2, 3 * K2, device=DEV)
B2 = torch.empty(N2, 3 * K2, device=DEV)
s = torch.cuda.current_stream().cuda_stream
L.call("cc_convert_matrix", a.data_ptr(), M2, K2, A2.data_ptr(), L.CC_F32_SPLIT3, 0, s)
L.call("cc_convert_matrix", b.data_ptr(), N2, K2, B2.data_ptr(), L.CC_F32_SPLIT3, 1, s)
C2 = torch.empty(M2, N2, device=DEV)
runtime.gemm(L.CC_GEMM_TF32X3, L.CC_EPI_STORE, M2, N2, K2, A2, B2, C=C2, ldc=N2, c_mode=L.CC_F32)
torch.cuda.synchronize()
np.savez(sys.argv[2], store=C.cpu().numpy(), residual=h.cpu().numpy(), tf32=C2.cpu().numpy())
"""


def test_gemm_banded_schedule_is_bitwise_the_same(tmp_path):
    """The CTA-pair GEMM bands its persistent tile schedule (m fastest inside
    bands of 8 m-pairs) unless A fits in L2 and B does not — e.g. the
    recompute's down projection, both operands > 60 MB; the single-CTA
    kernel (3xTF32 here) bands by 16 m tiles under the same rule. Every tile runs the same arithmetic whichever wave it
    lands in, so the banded run (default; and a band of 3 with a ragged last
    band) is bitwise the m-fastest run (CC_GEMM_GROUP=0)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for flag in ("", "0", "3"):
        f = tmp_path / f"band_{flag or 'default'}.npz"
        env = dict(os.environ)
        env.pop("CC_GEMM_GROUP", None)
        if flag:
            env["CC_GEMM_GROUP"] = flag
        r = subprocess.run([sys.executable, "-c", _BAND_SCRIPT, root, str(f)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[flag] = dict(np.load(f))
    for flag in ("", "3"):
        for key in ("store", "residual", "tf32"):
            assert np.array_equal(outs[flag][key], outs["0"][key]), (flag, key)


_GEMV_SCRIPT = r"""
import sys, math
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
from paper_2510_10129_b200 import _lib as L, runtime
from paper_2510_10129_b200.weights import _interleave_bias, _interleave_glu
L.load()
DEV = "cuda:0"
out = {}
for M in (1, 2, 3, 4):
    g = torch.Generator(device=DEV).manual_seed(40 + M)
    K, N = 3584, 4608
    A = torch.randn(M, K, device=DEV, generator=g).to(torch.bfloat16)
    B = (torch.randn(N, K, device=DEV, generator=g) * 0.05).to(torch.bfloat16)
    bias = torch.randn(N, device=DEV, generator=g)
    C = torch.empty(M, N, device=DEV)
    runtime.gemm(L.CC_GEMM_BF16, L.CC_EPI_STORE, M, N, K, A, B, bias=bias, C=C, ldc=N, c_mode=L.CC_F32)
    # residual + the next RMSNorm's fused outputs (bf16 h x gain, per-32-column partial sums)
    Wr = (torch.randn(K, K, device=DEV, generator=g) * 0.05).to(torch.bfloat16)
    h = torch.randn(M, K, device=DEV, generator=g)
    gain = torch.rand(K, device=DEV, generator=g) + 0.5
    xn = torch.empty(M, K, device=DEV, dtype=torch.bfloat16)
    ssq = torch.empty(K // 32, M, device=DEV)
    runtime.gemm(L.CC_GEMM_BF16, L.CC_EPI_RESIDUAL, M, K, K, A, Wr, C=h, ldc=K, c_mode=L.CC_F32,
                 xn_out=xn, ldxn=K, norm_gain=gain, ssq_out=ssq, ld_ssq=M)
    # GLU consuming the fused norm (1/rms from the partial sums)
    FF = 1024
    wg = torch.randn(FF, K, device=DEV, generator=g) * 0.05
    wu = torch.randn(FF, K, device=DEV, generator=g) * 0.05
    W = _interleave_glu(wg, wu).to(torch.bfloat16)
    b = _interleave_bias(bias[:FF], bias[FF:2 * FF])
    glu = torch.empty(M, FF, device=DEV)
    runtime.gemm(L.CC_GEMM_BF16, L.CC_EPI_GLU, M, 2 * FF, K, xn, W, bias=b, C=glu, ldc=FF, c_mode=L.CC_F32,
                 act=L.CC_ACT_SILU, n_out=FF, ssq_in=ssq, n_ssq=K // 32, ld_ssq_in=M, norm_eps=1e-6)
    torch.cuda.synchronize()
    for k, t in (("store", C), ("res", h), ("xn", xn.float()), ("ssq", ssq), ("glu", glu)):
        out[f"{k}{M}"] = t.cpu().numpy()
np.savez(sys.argv[2], **out)
"""


def test_gemv_matches_tensor_core_path(tmp_path):
    """GEMMs of at most 4 rows run as a weight-streaming GEMV on the CUDA cores
    with the tensor-core kernels' epilogue code. Against the tensor-core path
    (CC_GEMM_GEMV=0: split-K / whole-tile kernels) on the same inputs: STORE,
    RESIDUAL with the fused RMSNorm outputs (bf16 h x gain, partial sums) and a
    GLU consuming them agree to fp32 summation-order rounding, M = 1..4."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for flag in ("1", "0"):
        f = tmp_path / f"gemv_{flag}.npz"
        env = dict(os.environ, CC_GEMM_GEMV=flag)
        r = subprocess.run([sys.executable, "-c", _GEMV_SCRIPT, root, str(f)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[flag] = dict(np.load(f))
    for key in outs["0"]:
        a, b = outs["1"][key], outs["0"][key]
        scale = max(1.0, float(np.abs(b).max()))
        # xn is bf16 (one rounding step apart at most where h differs in its
        # last fp32 bit); the GLU consumes xn, so it inherits such a step
        tol = 1e-2 if key.startswith("xn") else (1e-3 if key.startswith("glu") else 1e-4)
        d = float(np.abs(a - b).max()) / scale
        print(f"{key}: max |gemv - tc| / max|tc| = {d:.2e}")
        assert d < tol, (key, d)
