""".cclp cache files (pkg/docs/cache_format.md, kv_store.py:261-359).

Layout (little endian):
    bytes 0..3   magic "CCLP"
    bytes 4..7   format version (u32)
    bytes 8..11  metadata length M (u32)
    bytes 12..   UTF-8 JSON metadata (M bytes)
    payload      per layer: key block then value block, row-major (rows, heads, head_dim)
    last 4 bytes CRC32 of everything before it (u32)

Version 1 is the reference's float32 format, written and read bit for bit
compatibly. bf16 caches (the primary model's device caches) are written as
version 2: identical framing, raw bfloat16 payload and ``"dtype": "bf16"`` in
the metadata, so a version-1 reader rejects them with VersionMismatchError
instead of misreading them.

load_cache returns caches in pinned host memory by default — the form the
streamed merge consumes (copy-engine DMA, merge_caches(..., device=...)), so loading
from disk overlaps with scoring on the request path — or directly on a device.
"""

from __future__ import annotations

import json
import zlib

import numpy as np
import torch

from .errors import BadMagicError, CacheFormatError, ChecksumError, VersionMismatchError
from .kv_store import ChunkCache, MergedCache, MergeLayout

CACHE_MAGIC = b"CCLP"
CACHE_VERSION = 1          # float32 payload (the reference's format)
CACHE_VERSION_BF16 = 2     # bfloat16 payload


def _u32(x: int) -> bytes:
    return int(x).to_bytes(4, "little")


def save_cache(cache, path) -> None:
    """Write a ChunkCache or MergedCache (device or host tensors)."""
    if isinstance(cache, ChunkCache):
        k, v = cache.k, cache.v
        meta_kind = {"kind": "chunk", "prefix_len": cache.prefix_len}
    elif isinstance(cache, MergedCache):
        k, v = cache.k_store[:, : cache.n_rows], cache.v_store[:, : cache.n_rows]
        meta_kind = {"kind": "merged", "sink_len": cache.layout.sink_len,
                     "chunk_lens": list(cache.layout.chunk_lens), "source": [list(s) for s in cache.source],
                     "recomputed_rows": list(cache.recomputed_rows)}
    else:
        raise TypeError(f"cannot persist {type(cache).__name__}")
    L, rows, heads, d_head = (int(x) for x in k.shape)
    bf16 = k.dtype == torch.bfloat16
    meta = {"n_layers": L, "rows": rows, "heads": heads, "d_head": d_head, "token_ids": list(cache.token_ids),
            "tokenizer_id": cache.tokenizer_id, "model_fingerprint": cache.model_fingerprint, **meta_kind}
    if bf16:
        meta["dtype"] = "bf16"
    kv = torch.stack([k, v], dim=1).contiguous().cpu()  # [L, 2, rows, heads, d_head]
    payload = (kv.view(torch.int16).numpy().astype("<i2") if bf16 else kv.numpy().astype("<f4")).tobytes()
    blob = bytearray(CACHE_MAGIC)
    blob += _u32(CACHE_VERSION_BF16 if bf16 else CACHE_VERSION)
    mb = json.dumps(meta, sort_keys=True).encode("utf-8")
    blob += _u32(len(mb))
    blob += mb
    blob += payload
    blob += _u32(zlib.crc32(bytes(blob)))
    with open(path, "wb") as f:
        f.write(bytes(blob))


def load_cache(path, *, device=None, pin: bool = True, dtype: torch.dtype | None = None):
    """Read a .cclp file (reference v1 fp32 or v2 bf16). Tensors land on
    ``device`` if given, else in (pinned) host memory. ``dtype`` converts the
    payload (round-to-nearest-even for fp32 -> bf16), e.g. a reference v1
    file for a bf16 primary; without it the cache keeps the file's dtype and
    a model of another dtype rejects it (CacheConsistencyError)."""
    with open(path, "rb") as f:
        blob = f.read()
    if len(blob) < 16:
        raise CacheFormatError(f"cache file truncated: {len(blob)} bytes")
    if blob[:4] != CACHE_MAGIC:
        raise BadMagicError(f"bad magic {blob[:4]!r}, expected {CACHE_MAGIC!r}")
    version = int.from_bytes(blob[4:8], "little")
    if version not in (CACHE_VERSION, CACHE_VERSION_BF16):
        raise VersionMismatchError(f"cache version {version}, expected {CACHE_VERSION} or {CACHE_VERSION_BF16}")
    if zlib.crc32(blob[:-4]) != int.from_bytes(blob[-4:], "little"):
        raise ChecksumError("cache checksum mismatch")
    meta_len = int.from_bytes(blob[8:12], "little")
    meta_end = 12 + meta_len
    if meta_end + 4 > len(blob):
        raise CacheFormatError("metadata length exceeds file size")
    try:
        meta = json.loads(blob[12:meta_end].decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise CacheFormatError(f"unreadable cache metadata: {exc}") from exc
    bf16 = version == CACHE_VERSION_BF16
    if bf16 != (meta.get("dtype") == "bf16"):
        raise CacheFormatError("payload dtype does not match the format version")
    L, rows, heads, d_head = meta["n_layers"], meta["rows"], meta["heads"], meta["d_head"]
    esize = 2 if bf16 else 4
    expected = meta_end + 2 * L * rows * heads * d_head * esize + 4
    if len(blob) != expected:
        raise CacheFormatError(f"payload size mismatch: file {len(blob)} bytes, expected {expected}")
    raw = np.frombuffer(blob, dtype="<i2" if bf16 else "<f4", count=2 * L * rows * heads * d_head, offset=meta_end)
    t = torch.from_numpy(raw.copy()).view(L, 2, rows, heads, d_head)
    if bf16:
        t = t.view(torch.bfloat16)
    k, v = t[:, 0].contiguous(), t[:, 1].contiguous()
    if dtype is not None and dtype != k.dtype:
        if dtype not in (torch.float32, torch.bfloat16):
            raise CacheFormatError(f"unsupported cache dtype {dtype}")
        k, v = k.to(dtype), v.to(dtype)
    if device is not None:
        k, v = k.to(device), v.to(device)
    elif pin and torch.cuda.is_available():
        k, v = k.pin_memory(), v.pin_memory()
    common = dict(token_ids=list(meta["token_ids"]), tokenizer_id=meta["tokenizer_id"],
                  model_fingerprint=meta["model_fingerprint"])
    if meta["kind"] == "chunk":
        return ChunkCache(k, v, prefix_len=meta["prefix_len"], **common)
    if meta["kind"] == "merged":
        return MergedCache(k, v, layout=MergeLayout(meta["sink_len"], tuple(meta["chunk_lens"])),
                           source=[tuple(s) for s in meta["source"]],
                           recomputed_rows=tuple(meta.get("recomputed_rows", ())), **common)
    raise CacheFormatError(f"unknown cache kind {meta['kind']!r}")
