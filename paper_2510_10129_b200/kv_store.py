"""Device-resident chunk and merged KV caches and the sink-deduplicating merge.

Same contract as pkg/src/cacheclip/kv_store.py: chunk caches hold keys
position-free; the merge keeps chunk 0's prefix (the shared attention sink),
concatenates every chunk's body and rotates each surviving key once, straight
into its global position; values pass through (kv_store.py:193-258).

HBM layout: one tensor per cache, [n_layers][rows][kv_heads][head_dim]
(bf16 for a bf16 model, fp32 for an fp32 model). A merged cache is allocated
with spare row capacity so the query rows of extend_cache append in place.
``.keys`` / ``.values`` return the reference's per-layer list view.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .config import RopeParams
from .errors import CacheConsistencyError
from .flops import PipelineTrace


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


class _PinnedRing:
    """Pinned host staging for small uploads, reused round-robin: a region is
    rewritten only after the upload that last read it has run (its event)."""

    SIZE = 16 << 20

    def __init__(self) -> None:
        self.buf = torch.empty(self.SIZE, dtype=torch.uint8, pin_memory=True)
        self.np = self.buf.numpy()
        self.ptr = self.buf.data_ptr()
        self.head = 0
        self.pending: list = []  # (start, end, event) in allocation order

    def alloc(self, n: int) -> int:
        n = (n + 255) & ~255
        if self.head + n > self.SIZE:
            self.head = 0
        start, end = self.head, self.head + n
        keep = []
        for a, b, ev in self.pending:
            if a < end and start < b:
                ev.synchronize()  # long done in practice: uploads run within microseconds
            else:
                keep.append((a, b, ev))
        self.pending = keep
        self.head = end
        return start

    def release(self, start: int, n: int) -> None:
        ev = torch.cuda.Event()
        ev.record()
        self.pending.append((start, start + n, ev))


_ring: _PinnedRing | None = None
_ring_lock = threading.Lock()


def host_to_device(data: np.ndarray, device) -> torch.Tensor:
    """Small host table -> device, stream-ordered. The bytes are staged in a
    pinned ring and read by the SMs (cc_upload), not the copy engines, so a
    table never waits behind streamed cache DMA (cc_h2d_segments)."""
    global _ring
    arr = np.ascontiguousarray(data)
    t = torch.from_numpy(arr)
    if torch.device(device).type != "cuda":
        return t.clone()
    if t.numel() == 0:
        return torch.empty(0, dtype=t.dtype, device=device)
    n = arr.nbytes
    if n > _PinnedRing.SIZE // 4:
        return t.pin_memory().to(device, non_blocking=True)
    out = torch.empty((n + 15) & ~15, dtype=torch.uint8, device=device)
    with _ring_lock:  # one ring per process, shared by host threads (e.g. thread-per-rank tests)
        if _ring is None:
            _ring = _PinnedRing()
        off = _ring.alloc(n)
        _ring.np[off:off + n] = arr.reshape(-1).view(np.uint8)
        with torch.cuda.device(out.device):
            _lib.call("cc_upload", out.data_ptr(), _ring.ptr + off, n, _stream())
            _ring.release(off, n)
    return out[:n].view(t.dtype).view(t.shape)


def _as_layers(x, device=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        if x.dim() != 4:
            raise CacheConsistencyError("cache tensor must be [layers, rows, heads, head_dim]")
        return x
    if isinstance(x, (list, tuple)) and x:
        parts = [p if isinstance(p, torch.Tensor) else torch.from_numpy(np.asarray(p)) for p in x]
        shape = tuple(parts[0].shape)
        for p in parts:
            if tuple(p.shape) != shape:
                raise CacheConsistencyError(f"layer shape {tuple(p.shape)} != {shape}")
        return torch.stack(parts).to(device if device is not None else parts[0].device)
    raise CacheConsistencyError("cache needs matching per-layer key/value lists")


def _rows_contiguous(t: torch.Tensor) -> bool:
    """[L, rows, H, D] with each layer's rows contiguous (any layer stride)."""
    L, R, H, D = t.shape
    return t.stride(3) == 1 and t.stride(2) == D and t.stride(1) == H * D and (L == 1 or t.stride(0) >= R * H * D)


def _layer_stride_rows(t: torch.Tensor) -> int:
    return t.stride(0) // (t.shape[2] * t.shape[3]) if t.shape[0] > 1 else t.shape[1]


def require_cache_dtype(caches, dtype: torch.dtype, what: str = "cache") -> None:
    """Every cache's K/V tensors must have the dtype the consuming model
    computes in (bf16 primary, fp32 scoring model): the kernels read the
    stores as that type. Raised before any device work (CacheConsistencyError,
    a ValueError). Reference v1 (.cclp) files are fp32: load them with
    ``load_cache(path, dtype=torch.bfloat16)`` for a bf16 primary."""
    for i, c in enumerate(caches):
        t = c.k_store if isinstance(c, MergedCache) else c.k
        if t.dtype != dtype:
            raise CacheConsistencyError(f"{what} {i} holds {t.dtype} K/V but the model computes in {dtype}")


class ChunkCache:
    """One chunk processed against the shared prefix, keys position-free."""

    KEYS_ROTATED = False

    def __init__(self, keys, values, token_ids, prefix_len: int, tokenizer_id: str,
                 model_fingerprint: str) -> None:
        k = _as_layers(keys)
        v = _as_layers(values, k.device)
        if k.shape != v.shape:
            raise CacheConsistencyError(f"layer shape {tuple(v.shape)} != {tuple(k.shape)}")
        if k.dtype not in (torch.float32, torch.bfloat16) or v.dtype != k.dtype:
            raise CacheConsistencyError(f"cache tensors must be float32 or bfloat16, got {k.dtype}")
        # pinned host views into a layer-major HostCachePool keep their layer
        # stride (the streaming copies read each layer through it); anything
        # else is stored contiguous
        pool_view = (not k.is_cuda and k.is_pinned() and v.is_pinned() and _rows_contiguous(k)
                     and v.stride() == k.stride())
        self.k, self.v = (k, v) if pool_view else (k.contiguous(), v.contiguous())
        self.token_ids = list(int(t) for t in token_ids)
        self.prefix_len = int(prefix_len)
        self.tokenizer_id = tokenizer_id
        self.model_fingerprint = model_fingerprint
        self._k_local = None
        if self.k.shape[1] != len(self.token_ids):
            raise CacheConsistencyError(f"{self.k.shape[1]} cache rows but {len(self.token_ids)} token ids")
        if not 0 <= self.prefix_len <= self.n_rows:
            raise CacheConsistencyError(f"prefix_len {self.prefix_len} outside 0..{self.n_rows}")

    @property
    def keys(self) -> list[torch.Tensor]:
        return list(self.k.unbind(0))

    @property
    def values(self) -> list[torch.Tensor]:
        return list(self.v.unbind(0))

    @property
    def n_layers(self) -> int:
        return self.k.shape[0]

    @property
    def n_rows(self) -> int:
        return self.k.shape[1]

    @property
    def chunk_ids(self) -> list[int]:
        return self.token_ids[self.prefix_len:]

    def token_ids_array(self) -> np.ndarray:
        """token_ids as int64, formed once (a chunk cache is immutable): the
        merge concatenates these instead of converting ~10^4 Python ints per
        request on the host's critical path."""
        arr = getattr(self, "_ids_np", None)
        if arr is None or arr.size != len(self.token_ids):
            arr = np.asarray(self.token_ids, dtype=np.int64)
            self._ids_np = arr
        return arr

    def chunk_key(self) -> bytes:
        """The chunk's token ids (after the prefix) as int64 bytes, formed
        once: equal chunk texts compare as one memcmp per request."""
        key = getattr(self, "_chunk_key", None)
        if key is None or len(key) != 8 * self.chunk_len:
            key = self.token_ids_array()[self.prefix_len:].tobytes()
            self._chunk_key = key
        return key

    @property
    def chunk_len(self) -> int:
        return self.n_rows - self.prefix_len

    def local_rotated_keys(self, rope: RopeParams) -> torch.Tensor:
        """Keys rotated at local positions 0..n-1 (attention_banks,
        kv_store.py:106-116), formed once and memoised: a chunk cache is
        immutable, so the per-call re-rotation of the reference is redundant."""
        if self._k_local is None:
            out = torch.empty_like(self.k)
            segs = host_to_device(_segments([(self, 0, 0, self.n_rows)]), self.k.device)
            inv = rope.inv_freq
            _lib.call("cc_assemble_kv", segs.data_ptr(), 1, self.n_rows, self.n_layers, self.k.shape[2],
                      self.k.shape[3], _dtype_code(self.k.dtype), inv.ctypes.data, 0,
                      out.data_ptr(), None, self.n_rows, _stream())
            self._k_local = out
        return self._k_local

    def attention_banks(self, rope: RopeParams, trace: PipelineTrace | None = None, stage: str = "decode"):
        k = self.local_rotated_keys(rope)
        return list(zip(k.unbind(0), self.v.unbind(0)))


def _dtype_code(dt: torch.dtype) -> int:
    return _lib.CC_BF16 if dt == torch.bfloat16 else _lib.CC_F32


def _segments(spec) -> np.ndarray:
    """[(chunk, src_row0, dst_row0, n_rows)] -> packed cc_kv_segment bytes
    (src_rows = the chunk tensors' layer stride in rows)."""
    arr = np.empty((len(spec), 7), dtype=np.int64)  # == cc_kv_segment (7 x 8 bytes)
    for i, item in enumerate(spec):
        c, s0, d0, n = item[:4]
        pos0 = item[4] if len(item) > 4 else d0  # RoPE position of the first row
        arr[i] = (c.k.data_ptr(), c.v.data_ptr(), _layer_stride_rows(c.k), s0, d0, n, pos0)
    return arr.view(np.uint8).reshape(-1)


@dataclass(frozen=True)
class MergeLayout:
    sink_len: int
    chunk_lens: tuple[int, ...]

    @property
    def total(self) -> int:
        return self.sink_len + sum(self.chunk_lens)

    def chunk_start(self, chunk: int) -> int:
        return self.sink_len + sum(self.chunk_lens[:chunk])


class MergedCache:
    """Concatenated chunk rows at contiguous positions, keys rotated.

    ``source`` is (chunk, row) per merged row, (-1, i) for appended rows;
    ``recomputed_rows`` is the selective-recompute provenance (kv_store.py:133-183).
    """

    KEYS_ROTATED = True

    def __init__(self, keys=None, values=None, token_ids=(), layout: MergeLayout | None = None, source=None,
                 tokenizer_id: str = "", model_fingerprint: str = "", recomputed_rows=(), *,
                 k_store: torch.Tensor | None = None, v_store: torch.Tensor | None = None,
                 n_rows: int | None = None) -> None:
        """Reference keyword form (keys/values per layer, kv_store.py:133-158), or
        the internal storage form (k_store/v_store [L, capacity, H, D] + n_rows)."""
        if k_store is None:
            k_store = _as_layers(keys)
            v_store = _as_layers(values, k_store.device)
            if tuple(v_store.shape) != tuple(k_store.shape):
                raise CacheConsistencyError(f"layer shape {tuple(v_store.shape)} != {tuple(k_store.shape)}")
            n_rows = k_store.shape[1]
        self.k_store, self.v_store = k_store, v_store
        self._n_rows = int(n_rows)
        self.token_ids = list(token_ids)
        self.layout = layout
        # source may be None: derived lazily from the layout (merge order)
        self._source = None if source is None else list(source)
        self.tokenizer_id = tokenizer_id
        self.model_fingerprint = model_fingerprint
        self.recomputed_rows = tuple(recomputed_rows)
        self._ids_dev = None
        self._ids_np = None  # int64 copy of token_ids when the merge formed one
        self.layer_ready = None  # per-layer events while a streamed merge is in flight
        if self._n_rows != len(self.token_ids) or (self._source is not None and self._n_rows != len(self._source)):
            raise CacheConsistencyError("rows, token ids, and source map disagree")

    @property
    def source(self) -> list[tuple[int, int]]:
        """(chunk, row) per merged row, (-1, i) for appended rows (kv_store.py:227-233)."""
        if self._source is None:
            lay = self.layout
            src = [(0, r) for r in range(lay.sink_len)]
            for ci, n in enumerate(lay.chunk_lens):
                src.extend((ci, lay.sink_len + j) for j in range(n))
            src.extend((-1, i) for i in range(lay.total, self._n_rows))
            self._source = src
        return self._source

    @source.setter
    def source(self, value) -> None:
        self._source = list(value)

    def token_ids_device(self) -> torch.Tensor:
        """Device copy of token_ids (uploaded once, extended in place on append)."""
        if self._ids_dev is None or self._ids_dev.numel() < self._n_rows:
            buf = torch.empty(max(self.capacity, self._n_rows), dtype=torch.int64, device=self.k_store.device)
            ids = self._ids_np if self._ids_np is not None and self._ids_np.size == self._n_rows \
                else np.asarray(self.token_ids, dtype=np.int64)
            buf[: self._n_rows].copy_(host_to_device(ids, buf.device))
            self._ids_dev = buf
        return self._ids_dev

    @property
    def n_rows(self) -> int:
        return self._n_rows

    @property
    def capacity(self) -> int:
        return self.k_store.shape[1]

    @property
    def keys(self) -> list[torch.Tensor]:
        return list(self.k_store[:, : self._n_rows].unbind(0))

    @property
    def values(self) -> list[torch.Tensor]:
        return list(self.v_store[:, : self._n_rows].unbind(0))

    @property
    def positions(self) -> np.ndarray:
        return np.arange(self._n_rows, dtype=np.int64)

    def attention_banks(self, rope=None, trace=None, stage="decode"):
        return list(zip(self.keys, self.values))

    def ensure_capacity(self, rows: int) -> None:
        """Grow the row capacity (copy) so `rows` rows fit in place."""
        if rows <= self.capacity:
            return
        L, _, H, D = self.k_store.shape
        cap = max(rows, int(self.capacity * 1.25) + 64)
        for name in ("k_store", "v_store"):
            old = getattr(self, name)
            new = torch.empty(L, cap, H, D, dtype=old.dtype, device=old.device)
            new[:, : self._n_rows].copy_(old[:, : self._n_rows])
            setattr(self, name, new)

    def _append_rows(self, token_ids, ids_dev: torch.Tensor | None = None) -> None:
        base = self._n_rows
        self.token_ids.extend(int(t) for t in token_ids)
        if self._source is not None:
            self._source.extend((-1, base + i) for i in range(len(token_ids)))
        self._n_rows += len(token_ids)
        if self._ids_dev is not None:
            if ids_dev is not None and self._ids_dev.numel() >= self._n_rows:
                self._ids_dev[base:self._n_rows].copy_(ids_dev)
            else:
                self._ids_dev = None

    def copy(self) -> "MergedCache":
        return MergedCache(token_ids=self.token_ids, layout=self.layout, source=self._source,
                           tokenizer_id=self.tokenizer_id, model_fingerprint=self.model_fingerprint,
                           recomputed_rows=self.recomputed_rows, k_store=self.k_store.clone(),
                           v_store=self.v_store.clone(), n_rows=self._n_rows)


def compute_positions(chunk_lens: Sequence[int], prefix_len: int) -> np.ndarray:
    if prefix_len < 0 or any(c < 0 for c in chunk_lens):
        raise ValueError("lengths must be non-negative")
    return np.arange(prefix_len + sum(chunk_lens), dtype=np.int64)


def _layer_groups(n_layers: int, ramp=(1, 2, 3), cap: int = 6, taper=(4, 2)) -> list[tuple[int, int]]:
    """[l0, l1) layer groups for streamed caches: ``ramp`` first (the consumer
    starts on layer 0 early), then groups of ``cap``, then ``taper`` (a
    transfer-bound consumer finishes soon after the last byte). Every group
    costs one 2-D copy per (chunk, K|V): tall groups keep the DMA efficient
    (~4 us fixed cost per copy) and the copy queue short (the driver blocks the
    host beyond ~1,000 queued copies)."""
    sizes, left = [], n_layers
    for s in ramp:
        if left <= 0:
            break
        sizes.append(min(s, left))
        left -= sizes[-1]
    tail = []
    for s in reversed(taper):
        if left <= 0:
            break
        tail.insert(0, min(s, left))
        left -= tail[0]
    while left > 0:
        sizes.append(min(cap, left))
        left -= sizes[-1]
    out, l0 = [], 0
    for s in sizes + tail:
        out.append((l0, l0 + s))
        l0 += s
    return out


# scoring caches gate the scoring pass layer by layer (transfer-bound): small
# first and last groups; primary caches are needed only after the selection
SCORING_GROUPS = dict(ramp=(1, 2, 3), cap=6, taper=(4, 2))
PRIMARY_GROUPS = dict(ramp=(1, 3, 6), cap=8, taper=())


_copy_streams: dict = {}


def _copy_stream(dev: torch.device) -> torch.cuda.Stream:
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    if key not in _copy_streams:
        _copy_streams[key] = torch.cuda.Stream(device=dev)
    return _copy_streams[key]


_MAX_PITCH = 1 << 30  # cudaMemcpy2DAsync rejects larger row pitches


def _same_storage(a, b) -> bool:
    """One 2-D copy must stay inside one host allocation (a pool tensor)."""
    try:
        return a.untyped_storage().data_ptr() == b.untyped_storage().data_ptr()
    except AttributeError:  # pointer stand-ins in host-logic tests
        return True


def _uniform_runs(spec, row_bytes: int) -> list[tuple[int, int]]:
    """Split spec into runs [i, j) whose chunks sit at a constant host stride
    inside one allocation (HostCachePool slots), copy the same rows (s0, n)
    and land back to back: a run moves as one 2-D copy per (layer, K|V)."""
    runs, i = [], 0
    while i < len(spec):
        j = i + 1
        c0, s0, d0, n = spec[i][:4]
        if j < len(spec):
            step = spec[j][0].k.data_ptr() - c0.k.data_ptr()
            while j < len(spec):
                c, s, d, m = spec[j][:4]
                prev = spec[j - 1][0]
                if (s != s0 or m != n or d != d0 + (j - i) * n or c.k.stride() != c0.k.stride()
                        or not (_same_storage(c.k, c0.k) and _same_storage(c.v, c0.v))
                        or c.k.data_ptr() - prev.k.data_ptr() != step
                        or c.v.data_ptr() - prev.v.data_ptr() != step or not n * row_bytes <= step <= _MAX_PITCH):
                    break
                j += 1
        runs.append((i, j))
        i = j
    return runs


def _stream_in(spec, rot: np.ndarray, n_rows: int, k_store: torch.Tensor, v_store: torch.Tensor,
               rope: RopeParams, groups: dict, v_layers: int | None = None) -> list:
    """Host-resident (pinned) chunk caches -> k_store / v_store
    ([L][cap][H][D]): per layer group, the copy engines DMA every segment's
    rows on a dedicated copy stream (no SM is spent on the transfer) — runs of
    chunks stored at a constant stride (HostCachePool slots) as one 2-D copy
    per (layer, K|V) (cc_h2d_uniform), other chunks one 2-D copy per
    (chunk, K|V) over the group's layers (cc_h2d_segments) — then the current
    stream rotates the group's keys in place (cc_rope_rows_inplace, segments
    ``rot`` give each row's position). Returns one event per layer, recorded
    on the current stream after its rotation. ``v_layers``: values are
    copied for layers < v_layers only (the scoring layer reads no values)."""
    for i, item in enumerate(spec):
        c = item[0]
        if not (c.k.is_pinned() and c.v.is_pinned()):
            raise CacheConsistencyError(f"chunk {i}: host caches must be in pinned memory")
    L, cap, H, D = k_store.shape
    dt = _dtype_code(k_store.dtype)
    row_bytes = H * D * k_store.element_size()
    runs = _uniform_runs(spec, row_bytes)
    singles = [spec[i] for i, j in runs if j - i == 1]
    host_segs = np.ascontiguousarray(_segments(singles)) if singles else None
    rot_dev = host_to_device(rot, k_store.device)
    cur = torch.cuda.current_stream()
    cp = _copy_stream(k_store.device)
    cp.wait_stream(cur)  # destination allocated / previous users done
    k_store.record_stream(cp)
    v_store.record_stream(cp)
    inv = rope.inv_freq
    ready = []
    v_end = L if v_layers is None else v_layers
    for l0, l1 in _layer_groups(L, **groups):
        # [l0, lv) with values, [lv, l1) keys only
        for a, b, with_v in ((l0, min(l1, v_end), True), (max(l0, v_end), l1, False)):
            if a >= b:
                continue
            vdst = v_store.data_ptr() if with_v else None
            if singles:
                _lib.call("cc_h2d_segments", host_segs.ctypes.data, len(singles), a, b - a, H, D, dt,
                          k_store.data_ptr(), vdst, cap, cp.cuda_stream)
            for i, j in runs:
                if j - i == 1:
                    continue
                c, s0, d0, n = spec[i][:4]
                step = spec[i + 1][0].k.data_ptr() - c.k.data_ptr()
                lstride = c.k.stride(0) * c.k.element_size()
                _lib.call("cc_h2d_uniform", c.k.data_ptr() + s0 * row_bytes, c.v.data_ptr() + s0 * row_bytes,
                          step, lstride, k_store.data_ptr() + d0 * row_bytes,
                          v_store.data_ptr() + d0 * row_bytes if with_v else None, n * row_bytes,
                          cap * row_bytes, n * row_bytes, j - i, a, b - a, cp.cuda_stream)
        copied = torch.cuda.Event()
        copied.record(cp)
        cur.wait_event(copied)
        _lib.call("cc_rope_rows_inplace", rot_dev.data_ptr(), len(rot) // (7 * 8), n_rows, l1 - l0, H, D, dt,
                  inv.ctypes.data, k_store.data_ptr() + l0 * cap * row_bytes, cap, _stream())
        ev = torch.cuda.Event()
        ev.record(cur)
        ready.extend([ev] * (l1 - l0))
    return ready


class HostCachePool:
    """Pinned host storage for chunk caches, LAYER-MAJOR across slots:
    ``k``, ``v`` = [layers][slots][rows_max][kv_heads][head_dim]. A chunk
    stored in slot s is the view k[:, s, :rows] (a ChunkCache like any other).
    The caches of chunks in consecutive slots form one pitched region per
    layer, so streaming a request's caches to the GPU (merge_caches /
    aux_score_tokens with host caches) costs one 2-D DMA per (layer, K|V)
    instead of one copy per chunk: fewer, larger copies keep PCIe at full
    rate (each copy has a fixed ~4 us cost on the DMA engine)."""

    def __init__(self, n_slots: int, rows_max: int, n_layers: int, kv_heads: int, head_dim: int,
                 dtype: torch.dtype = torch.bfloat16) -> None:
        if min(n_slots, rows_max, n_layers, kv_heads, head_dim) <= 0:
            raise ValueError("pool dimensions must be positive")
        shape = (n_layers, n_slots, rows_max, kv_heads, head_dim)
        self.k = torch.empty(shape, dtype=dtype, pin_memory=True)
        self.v = torch.empty(shape, dtype=dtype, pin_memory=True)
        self.n_slots, self.rows_max = n_slots, rows_max
        self._next = 0

    def store(self, cache: ChunkCache, slot: int | None = None) -> ChunkCache:
        """Copy `cache` into `slot` (default: the next free one); returns the
        pool-resident ChunkCache (same ids, prefix, tokenizer, fingerprint)."""
        slot = self._next if slot is None else int(slot)
        if not 0 <= slot < self.n_slots:
            raise ValueError(f"slot {slot} outside 0..{self.n_slots - 1}")
        L, R, H, D = cache.k.shape
        if (L, H, D) != (self.k.shape[0], self.k.shape[3], self.k.shape[4]) or cache.k.dtype != self.k.dtype:
            raise CacheConsistencyError("chunk cache geometry does not match the pool")
        if R > self.rows_max:
            raise CacheConsistencyError(f"{R} rows exceed the pool's {self.rows_max} rows per slot")
        k, v = self.k[:, slot, :R], self.v[:, slot, :R]
        k.copy_(cache.k)
        v.copy_(cache.v)
        self._next = max(self._next, slot + 1)
        return ChunkCache(k, v, cache.token_ids, cache.prefix_len, cache.tokenizer_id, cache.model_fingerprint)


def stream_local_banks(chunks: Sequence[ChunkCache], rope: RopeParams, device):
    """Host-resident (pinned) chunk caches -> one device bank per layer
    holding every chunk's keys rotated at its LOCAL positions and its values
    (what ChunkCache.local_rotated_keys + .v give per chunk). The copy engines
    bring the caches in layer group by layer group (_stream_in); each layer
    has an event so the scoring pass starts on layer l while later layers are
    still in flight. Returns (K [L,R,H,D], V, row offsets per chunk, events)."""
    first = chunks[0]
    for i, c in enumerate(chunks):
        if not (c.k.is_pinned() and c.v.is_pinned()):
            raise CacheConsistencyError(f"chunk {i}: host caches must be in pinned memory")
        if c.n_layers != first.n_layers or c.k.shape[2:] != first.k.shape[2:] or c.k.dtype != first.k.dtype:
            raise CacheConsistencyError(f"chunk {i} has mismatched tensor geometry")
    L, H, D = first.n_layers, first.k.shape[2], first.k.shape[3]
    offs = np.concatenate([[0], np.cumsum([c.n_rows for c in chunks])]).astype(np.int64)
    total = int(offs[-1])
    dev = torch.device(device)
    K = torch.empty(L, total, H, D, dtype=first.k.dtype, device=dev)
    V = torch.empty_like(K)
    spec = [(c, 0, int(o), c.n_rows, 0) for c, o in zip(chunks, offs[:-1])]  # pos0 = 0: local positions
    # the scoring layer (the last) reads no values: its V never crosses PCIe
    ready = _stream_in(spec, _segments(spec), total, K, V, rope, SCORING_GROUPS, v_layers=L - 1)
    return K, V, offs[:-1], ready


def merge_caches(chunks: Sequence[ChunkCache], rope: RopeParams, trace: PipelineTrace | None = None,
                 *, capacity: int | None = None, device=None) -> MergedCache:
    """Concatenate chunk caches keeping only the first copy of the prefix and
    rotate keys to global positions in one HBM pass (kv_store.py:193-258).
    ``capacity`` reserves rows for in-place appends (query rows). Chunk caches
    may also be host-resident (pinned): they are then streamed in layer by
    layer onto ``device`` and ``MergedCache.layer_ready`` holds one event per
    layer for consumers that overlap with the transfer."""
    if not chunks:
        raise CacheConsistencyError("nothing to merge")
    first = chunks[0]
    sink = first.prefix_len
    prefix_ids = first.token_ids[:sink]
    geom = tuple(first.k.shape[2:])
    for i, c in enumerate(chunks):
        if c.prefix_len != sink:
            raise CacheConsistencyError(f"chunk {i} prefix_len {c.prefix_len} != {sink}")
        if c.token_ids[:sink] != prefix_ids:
            raise CacheConsistencyError(f"chunk {i} has different prefix tokens")
        if c.model_fingerprint != first.model_fingerprint:
            raise CacheConsistencyError(f"chunk {i} built with a different model")
        if c.tokenizer_id != first.tokenizer_id:
            raise CacheConsistencyError(f"chunk {i} built with a different tokenizer")
        if c.n_layers != first.n_layers or tuple(c.k.shape[2:]) != geom or c.k.dtype != first.k.dtype \
                or c.k.device != first.k.device:
            raise CacheConsistencyError(f"chunk {i} has mismatched tensor geometry")
    lens = tuple(c.chunk_len for c in chunks)
    total = sink + sum(lens)
    cap = max(total, capacity or 0)
    token_ids = list(prefix_ids)
    spec = []
    dst = 0
    for ci, c in enumerate(chunks):
        token_ids.extend(c.token_ids[sink:])
        s0 = 0 if ci == 0 else sink
        n = c.n_rows - s0
        if n:
            spec.append((c, s0, dst, n))
        dst += n
    L, H, D = first.n_layers, geom[0], geom[1]
    streamed = not first.k.is_cuda
    if streamed and device is None:
        raise CacheConsistencyError("host-resident chunk caches need a target device")
    dev = torch.device(device) if streamed else first.k.device
    k_store = torch.empty(L, cap, H, D, dtype=first.k.dtype, device=dev)
    v_store = torch.empty_like(k_store)
    layer_ready = None
    if total and not streamed:
        segs = host_to_device(_segments(spec), dev)
        inv = rope.inv_freq
        _lib.call("cc_assemble_kv", segs.data_ptr(), len(spec), total, L, H, D, _dtype_code(first.k.dtype),
                  inv.ctypes.data, 0, k_store.data_ptr(), v_store.data_ptr(), cap, _stream())
    elif total:
        # Host-resident (pinned) chunk caches: copy-engine DMA straight into
        # the merged stores, keys rotated in place per layer group; each layer
        # records an event so a consumer can start on layer l while later
        # layers are still streaming in.
        rot = _segments([(first, 0, 0, total, 0)])  # merged row r sits at position r
        layer_ready = _stream_in(spec, rot, total, k_store, v_store, rope, PRIMARY_GROUPS)
    if trace is not None:  # one rotation per merged row per layer (kv_store.py:245-248), folded
        trace.rope("merge_overhead", L * total * H, D)
    # source map is derived lazily from the layout (MergedCache.source)
    merged = MergedCache(token_ids=token_ids, layout=MergeLayout(sink, lens), source=None,
                         tokenizer_id=first.tokenizer_id, model_fingerprint=first.model_fingerprint,
                         k_store=k_store, v_store=v_store, n_rows=total)
    merged.layer_ready = layer_ready
    merged._ids_np = np.concatenate([first.token_ids_array()[:sink]] +
                                    [c.token_ids_array()[sink:] for c in chunks])
    return merged
