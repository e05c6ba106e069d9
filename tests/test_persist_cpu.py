"""The .cclp format (kv_store.py:261-359): round trips, the reference's fault
injection cases (bad magic, version bump, flipped byte -> CRC, truncation),
and byte-level compatibility with files written by the reference itself
(tests/golden/ref_chunk.cclp, ref_merged.cclp from make_golden.py)."""

import os

import numpy as np
import pytest
import torch

from paper_2510_10129_b200 import (BadMagicError, CacheConsistencyError, CacheFormatError, ChecksumError, ChunkCache,
                                   MergedCache, MergeLayout, VersionMismatchError, load_cache, save_cache)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _chunk(rng, prefix, body, dtype=torch.float32, fp="m", tok="t"):
    n = len(prefix) + len(body)
    k = torch.from_numpy(rng.standard_normal((2, n, 2, 4), dtype=np.float32)).to(dtype)
    v = torch.from_numpy(rng.standard_normal((2, n, 2, 4), dtype=np.float32)).to(dtype)
    return ChunkCache(k, v, list(prefix) + list(body), len(prefix), tok, fp)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_chunk_round_trip(tmp_path, dtype):
    rng = np.random.default_rng(0)
    c = _chunk(rng, [5, 6], [7, 8, 9], dtype)
    p = tmp_path / "c.cclp"
    save_cache(c, p)
    d = load_cache(p, pin=False)
    assert isinstance(d, ChunkCache) and d.token_ids == c.token_ids and d.prefix_len == 2
    assert d.k.dtype == dtype and torch.equal(d.k, c.k) and torch.equal(d.v, c.v)
    assert int.from_bytes(p.read_bytes()[4:8], "little") == (1 if dtype == torch.float32 else 2)


def test_merged_round_trip(tmp_path):
    rng = np.random.default_rng(1)
    k = torch.from_numpy(rng.standard_normal((2, 5, 2, 4), dtype=np.float32))
    m = MergedCache(keys=list(k), values=list(k * 2), token_ids=[1, 2, 3, 4, 5], layout=MergeLayout(1, (2, 2)),
                    source=[(0, 0), (0, 1), (0, 2), (1, 1), (1, 2)], tokenizer_id="t", model_fingerprint="m",
                    recomputed_rows=(1, 4))
    p = tmp_path / "m.cclp"
    save_cache(m, p)
    d = load_cache(p, pin=False)
    assert isinstance(d, MergedCache) and d.layout == m.layout and d.source == m.source
    assert d.recomputed_rows == (1, 4) and d.token_ids == m.token_ids
    for a, b in zip(d.keys, m.keys):
        assert torch.equal(a, b)


def test_fault_injection(tmp_path):
    rng = np.random.default_rng(2)
    p = tmp_path / "junk.cclp"
    p.write_bytes(b"NOPE" + bytes(64))
    with pytest.raises(BadMagicError):
        load_cache(p)
    c = _chunk(rng, [1], [2, 3, 4])
    save_cache(c, p)
    data = bytearray(p.read_bytes())
    bumped = bytearray(data)
    bumped[4:8] = (999).to_bytes(4, "little")
    p.write_bytes(bytes(bumped))
    with pytest.raises(VersionMismatchError):
        load_cache(p)
    flipped = bytearray(data)
    flipped[-5] ^= 0xFF
    p.write_bytes(bytes(flipped))
    with pytest.raises(ChecksumError):
        load_cache(p)
    p.write_bytes(bytes(data[: len(data) // 2]))
    with pytest.raises(CacheFormatError):
        load_cache(p)


def test_reads_reference_written_files():
    """Files written by the unmodified reference load identically (v1 fp32)."""
    ref = dict(np.load(os.path.join(GOLDEN, "ref_files.npz")))
    c = load_cache(os.path.join(GOLDEN, "ref_chunk.cclp"), pin=False)
    assert c.token_ids == ref["chunk_token_ids"].tolist() and c.prefix_len == int(ref["chunk_prefix_len"])
    np.testing.assert_array_equal(c.k.numpy(), ref["chunk_k"])
    np.testing.assert_array_equal(c.v.numpy(), ref["chunk_v"])
    m = load_cache(os.path.join(GOLDEN, "ref_merged.cclp"), pin=False)
    assert m.layout.sink_len == int(ref["merged_sink"]) and list(m.layout.chunk_lens) == ref["merged_lens"].tolist()
    np.testing.assert_array_equal(np.stack([k.numpy() for k in m.keys]), ref["merged_k"])
    # and our v1 writer reproduces the reference's bytes exactly
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "x.cclp")
        save_cache(c, out)
        assert open(out, "rb").read() == open(os.path.join(GOLDEN, "ref_chunk.cclp"), "rb").read()


def test_cache_validation_errors():
    """kv_store.py:52-68 / test_kv_store.py:148-170."""
    rng = np.random.default_rng(3)
    keys = [torch.from_numpy(rng.standard_normal((3, 2, 4), dtype=np.float32))]
    values = [torch.from_numpy(rng.standard_normal((3, 2, 4), dtype=np.float32))]
    with pytest.raises(CacheConsistencyError):
        ChunkCache(keys, values, [1, 2], 0, "t", "m")
    with pytest.raises(CacheConsistencyError):
        ChunkCache(keys, values, [1, 2, 3], 4, "t", "m")
    with pytest.raises(CacheConsistencyError):
        ChunkCache(keys, [values[0][:2]], [1, 2, 3], 0, "t", "m")
    with pytest.raises(CacheConsistencyError):
        ChunkCache(keys, [values[0].double()], [1, 2, 3], 0, "t", "m")
    with pytest.raises(CacheConsistencyError):
        MergedCache(keys=keys, values=values, token_ids=[1, 2, 3], layout=MergeLayout(1, (2,)), source=[(0, 0)],
                    tokenizer_id="t", model_fingerprint="m")


def test_dtype_conversion_on_load_and_model_dtype_guard():
    """a reference v1 (fp32) file loads as fp32 and is
    rejected by a bf16 consumer's dtype guard; ``dtype=`` converts it on load
    (round-to-nearest-even, bitwise torch's .to(bfloat16))."""
    from paper_2510_10129_b200.kv_store import require_cache_dtype
    c = load_cache(os.path.join(GOLDEN, "ref_chunk.cclp"), pin=False)
    assert c.k.dtype == torch.float32
    with pytest.raises(CacheConsistencyError):
        require_cache_dtype([c], torch.bfloat16, "chunk")
    require_cache_dtype([c], torch.float32, "chunk")
    b = load_cache(os.path.join(GOLDEN, "ref_chunk.cclp"), pin=False, dtype=torch.bfloat16)
    assert b.k.dtype == torch.bfloat16 and torch.equal(b.k, c.k.to(torch.bfloat16))
    assert torch.equal(b.v, c.v.to(torch.bfloat16)) and b.token_ids == c.token_ids
    require_cache_dtype([b], torch.bfloat16, "chunk")
    with pytest.raises(CacheFormatError):
        load_cache(os.path.join(GOLDEN, "ref_chunk.cclp"), pin=False, dtype=torch.float16)
