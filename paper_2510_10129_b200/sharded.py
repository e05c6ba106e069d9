"""Sequence-sharded CacheClip prefill with split-KV attention.

Very long contexts (C4: 400 chunks, 200K tokens, 14B primary) are sharded by
CHUNK: chunk c lives on rank c % W (round-robin balances the causal attention
work), the shared prefix (the attention sink) on chunk 0's owner, which also
owns the query rows. Every rank assembles its chunks at their GLOBAL RoPE
positions (no communication) and scores them with the scoring model. Then:

  exchange 1   all_gather of the fp32 importance scores; every rank runs the
               identical deterministic top-k + window selection (H9);
  per layer    owners compute Q/K/V of their selected rows and scatter K/V into
               their shard; Q of all rows is all_gathered (bf16); every rank
               runs split-KV partial attention of all rows against its shard
               (keys visible iff global position <= row position) emitting
               (O, log-sum-exp); an all_to_all returns each row's partials to
               its owner, which merges them (LSE merge) and runs o-proj + MLP.

The reference has no distributed path; the math is
causal_attention over the merged cache (tensor_core.py:109-170,
model.py:715-720), partitioned along keys and recombined exactly:
softmax(s) V = sum_w 2^{lse_w - M} O_w / sum_w 2^{lse_w - M}.

Compute and communication are separated: ``ShardCompute`` is the per-rank math
(``DeviceShardCompute`` = the sm_100a kernels) and ``Exchange`` the collectives
(torch.distributed: NCCL over NVLink on B200s, gloo in the CPU tests).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Protocol, Sequence

import numpy as np
import torch

from . import _lib
from .flops import PipelineTrace
from .kv_store import ChunkCache, host_to_device
from .selector import ImportanceScores, SelectionConfig, aux_score_tokens, selection_budget


# ---------------------------------------------------------------------------
# plan: who owns which chunk / row
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class ShardPlan:
    world: int
    rank: int
    prefix_len: int
    chunk_lens: tuple[int, ...]
    query_len: int

    @property
    def n_chunks(self) -> int:
        return len(self.chunk_lens)

    @property
    def owner(self) -> np.ndarray:
        return np.arange(self.n_chunks) % self.world

    @property
    def chunk_start(self) -> np.ndarray:
        """Global merged row of each chunk's first body row."""
        return self.prefix_len + np.concatenate([[0], np.cumsum(self.chunk_lens)[:-1]]).astype(np.int64)

    @property
    def total(self) -> int:
        return self.prefix_len + int(sum(self.chunk_lens))

    @property
    def head_rank(self) -> int:
        """Owner of chunk 0: holds the sink (prefix) and the query rows."""
        return 0

    def local_chunks(self, r: int | None = None) -> list[int]:
        r = self.rank if r is None else r
        return [c for c in range(self.n_chunks) if c % self.world == r]

    def local_positions(self, r: int | None = None, with_query: bool = True) -> np.ndarray:
        """Sorted global positions of rank r's shard rows."""
        r = self.rank if r is None else r
        parts = []
        if r == self.head_rank:
            parts.append(np.arange(self.prefix_len, dtype=np.int64))
        starts = self.chunk_start
        for c in self.local_chunks(r):
            parts.append(np.arange(starts[c], starts[c] + self.chunk_lens[c], dtype=np.int64))
        if with_query and r == self.head_rank:
            parts.append(np.arange(self.total, self.total + self.query_len, dtype=np.int64))
        return np.concatenate(parts) if parts else np.zeros(0, np.int64)

    def owner_of_positions(self, pos: np.ndarray) -> np.ndarray:
        pos = np.asarray(pos, dtype=np.int64)
        out = np.full(pos.shape, self.head_rank, dtype=np.int64)
        body = (pos >= self.prefix_len) & (pos < self.total)
        chunk = np.searchsorted(self.chunk_start, pos[body], side="right") - 1
        out[body] = self.owner[chunk]
        return out

    def local_row_of(self, pos: np.ndarray, r: int | None = None) -> np.ndarray:
        """Row of each global position inside rank r's shard (positions must be owned by r)."""
        lp = self.local_positions(r)
        idx = np.searchsorted(lp, pos)
        if np.any(idx >= lp.size) or np.any(lp[np.minimum(idx, lp.size - 1)] != pos):
            raise ValueError("position not held by this shard")
        return idx.astype(np.int64)


def plan_shards(chunk_lens: Sequence[int], prefix_len: int, query_len: int, world: int, rank: int) -> ShardPlan:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return ShardPlan(world, rank, int(prefix_len), tuple(int(c) for c in chunk_lens), int(query_len))


@dataclass
class RowPlan:
    """The rows of the recompute+query pass and their owners (same on every rank)."""
    pos: np.ndarray          # [R] global positions (selected rows ascending, then query rows)
    owner: np.ndarray        # [R]
    r_max: int               # rows per owner slot in the rank-major exchange layout
    packed_pos: np.ndarray   # [W * r_max] positions in exchange order (-1 = padding)
    own: list[np.ndarray]    # per rank: indices into pos of its rows (ascending)

    @classmethod
    def build(cls, plan: ShardPlan, selected: np.ndarray, parts: int = 1) -> "RowPlan":
        q = np.arange(plan.total, plan.total + plan.query_len, dtype=np.int64)
        pos = np.concatenate([np.asarray(selected, dtype=np.int64), q])
        owner = plan.owner_of_positions(pos)
        own = [np.flatnonzero(owner == r) for r in range(plan.world)]
        r_max = max(1, max(len(o) for o in own))
        r_max = -(-r_max // parts) * parts   # slots split evenly into the pipeline's parts
        packed = np.full(plan.world * r_max, -1, dtype=np.int64)
        for r, o in enumerate(own):
            packed[r * r_max:r * r_max + len(o)] = pos[o]
        return cls(pos, owner, r_max, packed, own)


# ---------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------
def _wire(t: torch.Tensor) -> torch.Tensor:
    """bf16 payloads travel as raw bytes (uint8 view, last dim doubled) over
    backends without bf16 (gloo rejects both bf16 and int16)."""
    return t.view(torch.uint8) if t.dtype == torch.bfloat16 else t


class _Done:
    """Handle of a collective that already completed (world 1, host-staged)."""

    def __init__(self, t: torch.Tensor) -> None:
        self.t = t

    def wait(self) -> torch.Tensor:
        return self.t


class _Pending:
    """Handle of an in-flight NCCL collective: ``wait()`` orders the current
    stream after it (no host block) and returns the output tensor."""

    def __init__(self, work, t: torch.Tensor) -> None:
        self.work, self.t = work, t

    def wait(self) -> torch.Tensor:
        self.work.wait()
        return self.t


class Exchange:
    """The collectives of the sharded path over torch.distributed (world 1:
    local copies). NCCL moves device tensors directly and can run
    asynchronously (``async_op=True``: the collective runs on NCCL's stream
    while the caller launches more work; ``wait()`` on the handle orders the
    compute stream after it). A gloo group (the CPU tests, or several ranks
    sharing one GPU) stages device tensors through host memory."""

    def __init__(self, world: int, group=None) -> None:
        self.world = world
        self.group = group
        self._gloo = None

    def _host_staged(self, t: torch.Tensor) -> bool:
        """gloo: payloads move as host tensors in a dtype gloo carries."""
        if self._gloo is None:
            import torch.distributed as dist
            self._gloo = dist.get_backend(self.group) == "gloo"
        return self._gloo

    def all_gather(self, t: torch.Tensor, async_op: bool = False):
        """[n, ...] on every rank -> [W * n, ...] in rank order."""
        if self.world == 1:
            return _Done(t) if async_op else t
        import torch.distributed as dist
        if self._host_staged(t):
            src = _wire(t.detach().cpu().contiguous())
            out = torch.empty((self.world * src.shape[0],) + tuple(src.shape[1:]), dtype=src.dtype)
            dist.all_gather_into_tensor(out, src, group=self.group)
            res = out.view(t.dtype).to(t.device)
            return _Done(res) if async_op else res
        out = torch.empty((self.world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        work = dist.all_gather_into_tensor(out, t.contiguous(), group=self.group, async_op=async_op)
        return _Pending(work, out) if async_op else out

    def all_to_all(self, t: torch.Tensor, async_op: bool = False):
        """[W * n, ...]: slot s goes to rank s; returns [W * n, ...] with slot w from rank w."""
        if self.world == 1:
            return _Done(t) if async_op else t
        import torch.distributed as dist
        if self._host_staged(t):
            src = _wire(t.detach().cpu().contiguous())
            out = torch.empty_like(src)
            dist.all_to_all_single(out, src, group=self.group)
            res = out.view(t.dtype).to(t.device)
            return _Done(res) if async_op else res
        out = torch.empty_like(t)
        work = dist.all_to_all_single(out, t.contiguous(), group=self.group, async_op=async_op)
        return _Pending(work, out) if async_op else out


# ---------------------------------------------------------------------------
# per-rank compute
# ---------------------------------------------------------------------------
class ShardCompute(Protocol):
    def assemble(self, chunks: list, plan: ShardPlan): ...
    def local_scores(self, aux_chunks: list, query_ids) -> torch.Tensor: ...
    def select(self, scores: torch.Tensor, chunk_lens, config: SelectionConfig, offset: int) -> np.ndarray: ...
    def begin(self, rows: RowPlan, plan: ShardPlan, own_ids: np.ndarray, knobs) -> None: ...
    def pre_attention(self, layer: int) -> torch.Tensor: ...
    def partial_attention(self, layer: int, q_all: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]: ...
    def post_attention(self, layer: int, o_recv: torch.Tensor, lse_recv: torch.Tensor) -> None: ...
    def logits(self) -> torch.Tensor: ...


@dataclass
class ShardedOutcome:
    indices: tuple[int, ...]           # selected merged rows (identical on every rank)
    logits: np.ndarray | None          # first-token logits (head rank only)
    first_token: int | None
    scores: torch.Tensor | None = field(default=None, repr=False)


def cacheclip_prefill_sharded(compute: ShardCompute, exchange: Exchange, plan: ShardPlan, chunks_local: list,
                              aux_chunks_local: list, chunk_token_ids: dict, query_ids: Sequence[int],
                              config: SelectionConfig, *, n_layers: int, knobs=None,
                              pipeline: int = 2) -> ShardedOutcome:
    """One sequence-sharded CacheClip request. chunks_local / aux_chunks_local
    are this rank's chunk caches (plan.local_chunks() order); chunk_token_ids
    maps each local chunk to its body token ids (for the recompute rows).

    ``pipeline=2`` (computes with ``supports_parts``): each rank's exchange
    slots are split in two halves that flow through the layer independently,
    so the Q all_gather of half 1 overlaps the partial attention of half 0,
    the partial all_to_all of half 0 overlaps the partial attention of half
    1, and that of half 1 overlaps the LSE merge + o-proj + MLP of half 0
    (async NCCL collectives; the compute stream waits per half)."""
    W, r = plan.world, plan.rank
    # 1. shard assembly at global positions (no communication)
    compute.assemble(chunks_local, plan)
    # 2. local scores -> exchange 1 (all_gather) -> identical global selection everywhere
    local = compute.local_scores(aux_chunks_local, query_ids)
    lens = np.asarray(plan.chunk_lens, dtype=np.int64)
    counts = [int(lens[plan.local_chunks(w)].sum()) for w in range(W)]
    l_max = max(1, max(counts))
    buf = torch.zeros(l_max, dtype=torch.float32, device=local.device)
    buf[: local.numel()] = local
    gathered = exchange.all_gather(buf)
    order = []
    offs = {w: 0 for w in range(W)}
    for c in range(plan.n_chunks):
        w = c % W
        order.append(np.arange(w * l_max + offs[w], w * l_max + offs[w] + lens[c]))
        offs[w] += int(lens[c])
    perm = host_to_device(np.concatenate(order).astype(np.int64), gathered.device)
    scores = gathered.index_select(0, perm)
    selected = compute.select(scores, plan.chunk_lens, config, plan.prefix_len)
    # 3. row plan (same on every rank) and the recompute + query pass
    parts = 2 if pipeline >= 2 and getattr(compute, "supports_parts", False) else 1
    rows = RowPlan.build(plan, selected, parts)
    own_pos = rows.pos[rows.own[r]]
    starts = plan.chunk_start
    own_ids = np.empty(own_pos.size, dtype=np.int64)
    for k, p in enumerate(own_pos):
        if p >= plan.total:
            own_ids[k] = int(query_ids[p - plan.total])
        else:
            c = int(np.searchsorted(starts, p, side="right") - 1)
            own_ids[k] = chunk_token_ids[c][p - starts[c]]
    compute.begin(rows, plan, own_ids, knobs)
    H = rows.r_max // parts
    for layer in range(n_layers):
        q_local = compute.pre_attention(layer)                  # [r_max, Hq*D], own rows first
        if parts == 1:
            q_all = exchange.all_gather(q_local)                     # [W * r_max, Hq*D]
            o_part, lse = compute.partial_attention(layer, q_all)    # vs this shard's keys
            o_recv = exchange.all_to_all(o_part)                     # slot w: partials of my rows from rank w
            lse_recv = exchange.all_to_all(lse)
            compute.post_attention(layer, o_recv, lse_recv)          # LSE merge, o-proj, MLP
            continue
        gathers = [exchange.all_gather(q_local[p * H:(p + 1) * H], async_op=True) for p in range(parts)]
        sends = []
        for p in range(parts):
            o_part, lse = compute.partial_attention(layer, gathers[p].wait(), part=p)
            sends.append((exchange.all_to_all(o_part, async_op=True), exchange.all_to_all(lse, async_op=True)))
        for p, (o_h, l_h) in enumerate(sends):
            compute.post_attention(layer, o_h.wait(), l_h.wait(), part=p)
    logits = first = None
    if r == plan.head_rank:
        lg = compute.logits()
        logits = lg.detach().float().cpu().numpy()
        first = int(np.argmax(logits))
    return ShardedOutcome(tuple(int(i) for i in selected), logits, first, scores)


class DeviceShardCompute:
    """The sm_100a kernels behind the sharded orchestration (bf16 primary,
    fp32 scoring model)."""

    supports_parts = True   # pipelined halves (cacheclip_prefill_sharded pipeline=2)

    def __init__(self, primary, aux) -> None:
        self.p = primary
        self.aux = aux
        self.dev = primary.device

    # -- shard assembly ----------------------------------------------------
    def assemble(self, chunks: list, plan: ShardPlan) -> None:
        from .kv_store import _dtype_code, _segments
        c = self.p.config
        lp = plan.local_positions(with_query=False)
        self.local_pos_np = plan.local_positions(with_query=True)
        n = lp.size
        cap = self.local_pos_np.size
        L, H, D = c.n_layers, c.kv_heads, c.d_head
        self.k = torch.empty(L, max(cap, 1), H, D, dtype=torch.bfloat16, device=self.dev)
        self.v = torch.empty_like(self.k)
        spec = []
        dst = 0
        starts = plan.chunk_start
        for ci, ch in zip(plan.local_chunks(), chunks):
            if ci == 0 and plan.rank == plan.head_rank:
                spec.append((ch, 0, dst, ch.n_rows, 0))  # sink + body of chunk 0
                dst += ch.n_rows
            else:
                spec.append((ch, ch.prefix_len, dst, ch.chunk_len, int(starts[ci])))
                dst += ch.chunk_len
        if dst != n:
            raise ValueError("chunk caches do not match the shard plan")
        if spec:
            segs = host_to_device(_segments(spec), self.dev)
            inv = c.rope.inv_freq
            _lib.call("cc_assemble_kv", segs.data_ptr(), len(spec), n, L, H, D, _dtype_code(torch.bfloat16),
                      inv.ctypes.data, 0, self.k.data_ptr(), self.v.data_ptr(), self.k.shape[1],
                      torch.cuda.current_stream().cuda_stream)
        self.n_local = n
        self.local_pos = host_to_device(self.local_pos_np, self.dev)

    # -- scoring / selection ----------------------------------------------
    def local_scores(self, aux_chunks: list, query_ids) -> torch.Tensor:
        if not aux_chunks:
            return torch.zeros(0, dtype=torch.float32, device=self.dev)
        return aux_score_tokens(self.aux, aux_chunks, list(query_ids)).device_scores

    def select(self, scores: torch.Tensor, chunk_lens, config: SelectionConfig, offset: int) -> np.ndarray:
        from .selector import select_tokens_device
        sel = select_tokens_device(ImportanceScores(scores, chunk_lens), config, index_offset=offset)
        return sel.idx_host

    # -- recompute + query pass -------------------------------------------
    def begin(self, rows: RowPlan, plan: ShardPlan, own_ids: np.ndarray, knobs) -> None:
        c = self.p.config
        r = plan.rank
        self.rows, self.plan = rows, plan
        own = rows.own[r]
        self.n_own = len(own)
        own_pos = rows.pos[own]
        dst_local = np.searchsorted(self.local_pos_np, own_pos).astype(np.int64)
        R = rows.r_max
        pad = lambda a: np.concatenate([a, np.zeros(R - a.size, dtype=np.int64)])  # noqa: E731
        host = np.concatenate([pad(own_ids), pad(own_pos), pad(dst_local), rows.packed_pos])
        buf = host_to_device(host, self.dev)
        self.ids, self.pos, self.dst = buf[:R], buf[R:2 * R], buf[2 * R:3 * R]
        packed_pos = buf[3 * R:]
        W = plan.world
        # causal limits of every exchanged row against this shard's keys
        self.limits = torch.empty(W * R, dtype=torch.int64, device=self.dev)
        _lib.call("cc_local_limits", packed_pos.data_ptr(), W * R, self.local_pos.data_ptr(), self.local_pos.numel(),
                  self.limits.data_ptr(), torch.cuda.current_stream().cuda_stream)
        self.row_factor = None
        if knobs is not None:
            t, s = knobs
            f = np.full(W * R, np.float32(1.0 / math.sqrt(c.d_head)), dtype=np.float32)
            f[rows.packed_pos >= plan.total] = np.float32(s / (math.sqrt(c.d_head) * t))
            self.row_factor = host_to_device(f, self.dev)
        from .runtime import rope_table
        self.cos_sin = rope_table(self.p, self.pos)
        d, qw = c.d_model, c.attn_width
        self.h = torch.zeros(R, d, dtype=torch.float32, device=self.dev)
        self.x = torch.empty(R, d, dtype=torch.bfloat16, device=self.dev)
        self.q = torch.zeros(R, qw, dtype=torch.bfloat16, device=self.dev)
        self.ctx = torch.zeros(R, qw, dtype=torch.bfloat16, device=self.dev)
        self.act = torch.empty(R, c.d_ff, dtype=torch.bfloat16, device=self.dev)
        # bf16 partials: half the all_to_all and merge bytes (merged in fp32)
        self.o_part = torch.empty(W * R, c.n_heads, c.d_head, dtype=torch.bfloat16, device=self.dev)
        self.lse = torch.empty(W * R, c.n_heads, dtype=torch.float32, device=self.dev)
        # pipelined halves: per-part limits / factors in [W][R/2] order and
        # separate partial buffers (half 0 is in flight while half 1 computes)
        self.part_rows = R // 2 if R % 2 == 0 else 0
        if self.part_rows:
            Hh = self.part_rows
            lim = self.limits.view(W, R)
            self.part_limits = [lim[:, p * Hh:(p + 1) * Hh].reshape(-1).contiguous() for p in range(2)]
            self.part_factor = None
            if self.row_factor is not None:
                rf = self.row_factor.view(W, R)
                self.part_factor = [rf[:, p * Hh:(p + 1) * Hh].reshape(-1).contiguous() for p in range(2)]
            self.part_o = [torch.empty(W * Hh, c.n_heads, c.d_head, dtype=torch.bfloat16, device=self.dev)
                           for _ in range(2)]
            self.part_lse = [torch.empty(W * Hh, c.n_heads, dtype=torch.float32, device=self.dev) for _ in range(2)]

    def _s(self) -> int:
        return torch.cuda.current_stream().cuda_stream

    def pre_attention(self, layer: int) -> torch.Tensor:
        from .runtime import gemm
        c = self.p.config
        lw = self.p.layers[layer]
        n, d, qw = self.n_own, c.d_model, c.attn_width
        if n:
            if layer == 0:
                _lib.call("cc_embed_rmsnorm", self.ids.data_ptr(), n, self.p.embed.data_ptr(), _lib.CC_BF16,
                          c.vocab_size, d, self.h.data_ptr(), lw.attn_norm.data_ptr(), c.norm_eps, self.x.data_ptr(),
                          _lib.CC_BF16, self._s())
            else:
                _lib.call("cc_rmsnorm", self.h.data_ptr(), n, d, d, lw.attn_norm.data_ptr(), c.norm_eps,
                          self.x.data_ptr(), _lib.CC_BF16, self._s())
            gemm(_lib.CC_GEMM_BF16, _lib.CC_EPI_QKV_ROPE, n, lw.w_qkv.shape[0], d, self.x, lw.w_qkv, bias=lw.b_qkv,
                 rope=self.cos_sin, q_out=self.q, ldq=qw, q_mode=_lib.CC_BF16, k_cache=self.k[layer],
                 v_cache=self.v[layer], cache_dtype=_lib.CC_BF16, dst_rows=self.dst,
                 heads=(c.n_heads, c.kv_heads, c.d_head))
        return self.q

    def partial_attention(self, layer: int, q_all: torch.Tensor, part: int | None = None):
        c = self.p.config
        qw = c.attn_width
        factor = float(np.float32(1.0 / math.sqrt(c.d_head)))
        if part is None:
            lim, rf, o, lse = self.limits, self.row_factor, self.o_part, self.lse
        else:
            lim, o, lse = self.part_limits[part], self.part_o[part], self.part_lse[part]
            rf = self.part_factor[part] if self.part_factor is not None else None
        _lib.call("cc_sparse_row_attention_partial", q_all.data_ptr(), qw, lim.data_ptr(), q_all.shape[0],
                  self.k[layer].data_ptr(), self.v[layer].data_ptr(), self.local_pos.numel(), c.n_heads, c.kv_heads,
                  c.d_head, factor, rf.data_ptr() if rf is not None else None,
                  o.data_ptr(), _lib.CC_BF16, lse.data_ptr(), self._s())
        return o, lse

    def post_attention(self, layer: int, o_recv: torch.Tensor, lse_recv: torch.Tensor,
                       part: int | None = None) -> None:
        from .runtime import _mlp, gemm
        c = self.p.config
        lw = self.p.layers[layer]
        d, qw = c.d_model, c.attn_width
        W = self.plan.world
        if part is None:
            a, b, stride = 0, self.n_own, self.rows.r_max
        else:
            stride = self.part_rows
            a, b = part * stride, min(self.n_own, (part + 1) * stride)
        n = b - a
        if n <= 0:
            return
        ctx = self.ctx[a:b]
        _lib.call("cc_lse_merge", o_recv.data_ptr(), _lib.CC_BF16, lse_recv.data_ptr(), W, stride, n, c.n_heads,
                  c.d_head, ctx.data_ptr(), qw, _lib.CC_BF16, self._s())
        h = self.h[a:b]
        gemm(_lib.CC_GEMM_BF16, _lib.CC_EPI_RESIDUAL, n, d, qw, ctx, lw.w_o, bias=lw.b_o, C=h, ldc=d,
             c_mode=_lib.CC_F32)
        _mlp(self.p, lw, h, self.x[a:b], self.act[a:b], _lib.CC_GEMM_BF16, _lib.CC_BF16)

    def logits(self) -> torch.Tensor:
        from .runtime import final_logits
        lg, _ = final_logits(self.p, self.h[self.n_own - 1])
        return lg
