"""Sequence-sharded path on CPU: the shard plan logic, and the full
multi-rank orchestration over a real torch.distributed gloo group
(world size 2 and 3) with a numpy per-rank compute built from the oracle
(test-only). The sharded result must reproduce the oracle's unsharded
cacheclip: identical selection, first-token logits within fp32 rounding."""

import math
import os
import socket

import numpy as np
import pytest
import torch

from oracle import cacheclip_oracle as orc
from oracle.synth import B1, C1_EXACT

LOG2E = 1.4426950408889634


def test_shard_plan_layout():
    from paper_2510_10129_b200.sharded import RowPlan, plan_shards
    lens = [5, 7, 3, 9, 4]
    P, Q = 3, 2
    plans = [plan_shards(lens, P, Q, 2, r) for r in range(2)]
    assert plans[0].local_chunks() == [0, 2, 4] and plans[1].local_chunks() == [1, 3]
    allpos = np.concatenate([p.local_positions() for p in plans])
    total = P + sum(lens)
    assert sorted(allpos.tolist()) == list(range(total + Q))            # every row exactly once
    for p in plans:
        lp = p.local_positions()
        assert np.all(np.diff(lp) > 0)                                  # sorted -> causal limits are prefixes
    assert plans[0].local_positions()[:P].tolist() == [0, 1, 2]         # sink on the head rank
    sel = np.array([3, 4, 9, 10, 20, 30])
    rp = RowPlan.build(plans[0], sel)
    assert rp.pos.tolist() == [3, 4, 9, 10, 20, 30, total, total + 1]
    assert rp.owner.tolist() == [0, 0, 1, 1, 1, 0, 0, 0]
    assert rp.r_max == 5 and rp.packed_pos.tolist() == [3, 4, 30, total, total + 1, 9, 10, 20, -1, -1]
    for r, p in enumerate(plans):
        own = rp.pos[rp.own[r]]
        assert np.array_equal(p.local_positions()[p.local_row_of(own)], own)


class OracleShardCompute:
    """numpy (oracle) implementation of the ShardCompute contract — test only."""

    def __init__(self, primary, aux):
        self.p, self.aux = primary, aux

    def assemble(self, chunks, plan):
        c = self.p.cfg
        self.lp = plan.local_positions()
        L, H, D = c.n_layers, c.kv_heads, c.d_head
        self.K = np.zeros((L, self.lp.size, H, D), np.float32)
        self.V = np.zeros_like(self.K)
        dst = 0
        starts = plan.chunk_start
        for ci, ch in zip(plan.local_chunks(), chunks):
            if ci == 0 and plan.rank == plan.head_rank:
                rows, pos0 = slice(0, ch.n_rows), 0
            else:
                rows, pos0 = slice(ch.prefix_len, ch.n_rows), int(starts[ci])
            n = rows.stop - rows.start
            pos = np.arange(pos0, pos0 + n)
            for layer in range(L):
                self.K[layer, dst:dst + n] = orc.rope_rotate(ch.keys[layer][rows], pos, D, c.rope_base)
                self.V[layer, dst:dst + n] = ch.values[layer][rows]
            dst += n

    def local_scores(self, aux_chunks, query):
        if not aux_chunks:
            return torch.zeros(0)
        return torch.from_numpy(orc.aux_scores(self.aux, aux_chunks, query))

    def select(self, scores, chunk_lens, config, offset):
        idx, _ = orc.select(scores.numpy(), chunk_lens, config.recomp_ratio, config.window_len,
                            config.window_threshold, config.expand_full_window)
        return np.asarray(idx, dtype=np.int64) + offset

    def begin(self, rows, plan, own_ids, knobs):
        self.rows, self.plan = rows, plan
        own = rows.own[plan.rank]
        self.n = len(own)
        self.pos = rows.pos[own]
        self.dst = np.searchsorted(self.lp, self.pos)
        self.h = orc.embed(self.p, own_ids) if self.n else np.zeros((0, self.p.cfg.d_model), np.float32)

    def pre_attention(self, layer):
        c = self.p.cfg
        out = np.zeros((self.rows.r_max, c.q_width), np.float32)
        if self.n:
            q, k, v = orc.qkv_project(self.p, layer, self.h)
            self.K[layer, self.dst] = orc.rope_rotate(k, self.pos, c.d_head, c.rope_base)
            self.V[layer, self.dst] = v
            out[:self.n] = orc.rope_rotate(q, self.pos, c.d_head, c.rope_base).reshape(self.n, -1)
        return torch.from_numpy(out)

    def _part_pos(self, part):
        ppos = self.rows.packed_pos
        if part is None:
            return ppos
        W, R = self.plan.world, self.rows.r_max
        H = R // 2
        return ppos.reshape(W, R)[:, part * H:(part + 1) * H].reshape(-1)

    def partial_attention(self, layer, q_all, part=None):
        c = self.p.cfg
        q = q_all.numpy().reshape(-1, c.n_heads, c.d_head)
        ppos = self._part_pos(part)
        lim = np.searchsorted(self.lp, ppos, side="right")        # visible local keys per row
        o = np.zeros(q.shape, np.float32)
        lse = np.full(q.shape[:2], -np.inf, np.float32)
        factor = np.float32(1.0 / math.sqrt(c.d_head))
        g = c.group
        for i in range(q.shape[0]):
            if ppos[i] < 0 or lim[i] == 0:
                continue
            for h in range(c.n_heads):
                k = self.K[layer, :lim[i], h // g]
                s = (k @ q[i, h]) * factor
                mx = s.max()
                e = np.exp(s - mx)
                l = e.sum()
                o[i, h] = (e @ self.V[layer, :lim[i], h // g]) / l
                lse[i, h] = (mx + np.log(l)) * LOG2E
        return torch.from_numpy(o), torch.from_numpy(lse)

    def post_attention(self, layer, o_recv, lse_recv, part=None):
        W, R = self.plan.world, self.rows.r_max
        if part is None:
            lo, hi, S = 0, self.n, R
        else:
            S = R // 2
            lo, hi = part * S, min(self.n, (part + 1) * S)
        if hi <= lo:
            return
        o = o_recv.numpy().reshape(W, S, *o_recv.shape[1:])[:, :hi - lo]
        lse = lse_recv.numpy().reshape(W, S, -1)[:, :hi - lo]
        m = lse.max(axis=0)
        a = np.where(np.isinf(lse), 0.0, np.exp2(lse - m))
        ctx = (a[..., None] * o).sum(0) / a.sum(0)[..., None]
        h = self.h[lo:hi] + orc.out_project(self.p, layer, ctx.astype(np.float32))
        self.h[lo:hi] = h + orc.mlp(self.p, layer, h)

    def logits(self):
        return torch.from_numpy(orc.final_logits(self.p, self.h[:self.n]))


class OracleShardComputeParts(OracleShardCompute):
    """The same math through the pipelined two-half exchange."""
    supports_parts = True


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, wname, outdir, pipeline=1):
    import torch.distributed as dist

    from oracle.synth import WORKLOADS
    from paper_2510_10129_b200 import SelectionConfig
    from paper_2510_10129_b200.sharded import Exchange, cacheclip_prefill_sharded, plan_shards
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = WORKLOADS[wname]
        prim = orc.OracleModel(w.primary, orc.seeded_params(w.primary, w.primary_seed, w.bias_std))
        aux = orc.OracleModel(w.aux, orc.seeded_params(w.aux, w.aux_seed, w.bias_std))
        prefix, chunk_ids, query = w.token_ids(0)
        plan = plan_shards([len(c) for c in chunk_ids], len(prefix), len(query), world, rank)
        mine = plan.local_chunks()   # each rank precomputes only its own chunks
        chunks = [orc.prefill_chunk(prim, prefix, chunk_ids[c]) for c in mine]
        aux_chunks = [orc.prefill_chunk(aux, prefix, chunk_ids[c]) for c in mine]
        compute = (OracleShardComputeParts if pipeline == 2 else OracleShardCompute)(prim, aux)
        res = cacheclip_prefill_sharded(compute, Exchange(world), plan, chunks, aux_chunks,
                                        {c: chunk_ids[c] for c in mine}, query,
                                        SelectionConfig(w.ratio, w.window_len, w.window_threshold),
                                        n_layers=w.primary.n_layers, pipeline=pipeline)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), indices=np.asarray(res.indices),
                 logits=res.logits if res.logits is not None else np.zeros(0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,wname,pipeline", [(2, "c1_exact", 1), (3, "b1", 1), (2, "c1_exact", 2),
                                                  (3, "b1", 2)])
def test_gloo_sharded_matches_oracle(tmp_path, world, wname, pipeline):
    """pipeline=2: each rank's exchange slots flow through the layer as two
    halves with async collectives (overlap); results identical to pipeline=1."""
    import torch.multiprocessing as mp

    from oracle.synth import WORKLOADS
    mp.spawn(_worker, args=(world, _free_port(), wname, str(tmp_path), pipeline), nprocs=world, join=True)
    w = WORKLOADS[wname]
    prim = orc.OracleModel(w.primary, orc.seeded_params(w.primary, w.primary_seed, w.bias_std))
    aux = orc.OracleModel(w.aux, orc.seeded_params(w.aux, w.aux_seed, w.bias_std))
    prefix, chunk_ids, query = w.token_ids(0)
    chunks = [orc.prefill_chunk(prim, prefix, c) for c in chunk_ids]
    aux_chunks = [orc.prefill_chunk(aux, prefix, c) for c in chunk_ids]
    ref = orc.cacheclip(prim, aux, chunks, aux_chunks, query, w.ratio, window_len=w.window_len,
                        threshold=w.window_threshold)
    outs = [dict(np.load(os.path.join(tmp_path, f"r{r}.npz"))) for r in range(world)]
    for o in outs:
        assert tuple(o["indices"].tolist()) == ref.indices
    np.testing.assert_allclose(outs[0]["logits"], ref.logits, rtol=0, atol=5e-5)


def _bf16_worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist

    from paper_2510_10129_b200.sharded import Exchange
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(rank)
        x = torch.randn(4, 3, 8, generator=g).to(torch.bfloat16)
        ex = Exchange(world)
        gathered = ex.all_gather(x, async_op=True).wait()
        swapped = ex.all_to_all(torch.cat([x] * world), async_op=False)
        np.savez(os.path.join(outdir, f"b{rank}.npz"), g=gathered.view(torch.int16).numpy(),
                 s=swapped.view(torch.int16).numpy(), dt=str(gathered.dtype) + str(swapped.dtype))
    finally:
        dist.destroy_process_group()


def test_gloo_exchange_carries_bf16_bytewise(tmp_path):
    """gloo has neither bf16 nor int16: the Exchange moves bf16 payloads as
    raw bytes and hands back bf16 tensors bit-identical to what was sent."""
    import torch
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_bf16_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    sent = [torch.randn(4, 3, 8, generator=torch.Generator().manual_seed(r)).to(torch.bfloat16).view(torch.int16)
            .numpy() for r in range(world)]
    for r in range(world):
        o = np.load(os.path.join(tmp_path, f"b{r}.npz"))
        assert str(o["dt"]) == "torch.bfloat16torch.bfloat16"
        np.testing.assert_array_equal(o["g"], np.concatenate(sent))
        np.testing.assert_array_equal(o["s"], np.concatenate(sent))
