"""Sequence-sharded CacheClip on the device.

* kernel level: split-KV partial attention over interleaved key shards +
  LSE merge equals full attention;
* world 1: the sharded orchestration equals the unsharded pipeline;
* world 2 and 3 on ONE GPU: ranks run as threads with an in-process exchange
  (same collectives contract as torch.distributed), so the whole multi-rank
  data path — shard assembly at global positions, score all_gather, identical
  selection, Q all_gather, partial attention, all_to_all, LSE merge — is
  checked against the single-GPU result.
"""

import math
import threading

import numpy as np
import pytest
import torch

from oracle import cacheclip_oracle as orc
from oracle.synth import C1_EXACT

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _attn_ref(q, k, v, limits, factor):
    m, Hq, D = q.shape
    G = Hq // k.shape[1]
    kk = k.double().repeat_interleave(G, dim=1)
    vv = v.double().repeat_interleave(G, dim=1)
    s = torch.einsum("mhd,nhd->hmn", q.double(), kk) * factor
    mask = torch.arange(k.shape[0], device=q.device)[None, :] >= limits[:, None]
    s = s.masked_fill(mask[None], float("-inf"))
    return torch.einsum("hmn,nhd->mhd", torch.softmax(s, -1), vv)


@pytest.mark.parametrize("part", ["f32", "bf16"])
@pytest.mark.parametrize("D,Hq,Hkv", [(128, 28, 4), (64, 4, 2)])
def test_partial_attention_and_lse_merge(D, Hq, Hkv, part):
    from paper_2510_10129_b200 import _lib as L
    pdt = L.CC_BF16 if part == "bf16" else L.CC_F32
    g = torch.Generator(device=DEV).manual_seed(D)
    n, m, W = 1500, 300, 3
    q = torch.randn(m, Hq, D, device=DEV, generator=g).to(torch.bfloat16)
    k = torch.randn(n, Hkv, D, device=DEV, generator=g).to(torch.bfloat16)
    v = torch.randn(n, Hkv, D, device=DEV, generator=g).to(torch.bfloat16)
    pos = torch.sort(torch.randperm(n, generator=torch.Generator().manual_seed(5))[:m]).values.to(DEV)
    # interleaved 100-key "chunks" over W shards (round-robin, like the shard plan)
    owner = (torch.arange(n, device=DEV) // 100) % W
    factor = 1.0 / math.sqrt(D)
    s = torch.cuda.current_stream().cuda_stream
    o_parts = torch.empty(W, m, Hq, D, device=DEV, dtype=torch.bfloat16 if part == "bf16" else torch.float32)
    lse_parts = torch.empty(W, m, Hq, device=DEV)
    for w in range(W):
        local_pos = torch.nonzero(owner == w).flatten().contiguous()
        lk, lv = k[local_pos].contiguous(), v[local_pos].contiguous()
        lim = torch.empty(m, dtype=torch.int64, device=DEV)
        L.call("cc_local_limits", pos.data_ptr(), m, local_pos.data_ptr(), local_pos.numel(), lim.data_ptr(), s)
        ref_lim = torch.searchsorted(local_pos, pos, right=True) - 1
        assert torch.equal(lim, ref_lim)
        L.call("cc_sparse_row_attention_partial", q.data_ptr(), Hq * D, lim.data_ptr(), m, lk.data_ptr(),
               lv.data_ptr(), lk.shape[0], Hq, Hkv, D, factor, None, o_parts[w].data_ptr(), pdt,
               lse_parts[w].data_ptr(), s)
    out = torch.empty(m, Hq * D, device=DEV, dtype=torch.bfloat16)
    L.call("cc_lse_merge", o_parts.data_ptr(), pdt, lse_parts.data_ptr(), W, m, m, Hq, D, out.data_ptr(), Hq * D,
           L.CC_BF16, s)
    torch.cuda.synchronize()
    ref = _attn_ref(q, k, v, pos + 1, factor)
    err = (out.double().view(m, Hq, D) - ref).abs().max().item()
    assert err < 2e-2, err


def _cfg(oc, dtype):
    from paper_2510_10129_b200 import ModelConfig
    return ModelConfig(n_layers=oc.n_layers, n_heads=oc.n_heads, d_model=oc.d_model, d_head=oc.d_head,
                       d_ff=oc.d_ff, vocab_size=oc.vocab_size, rope_base=oc.rope_base, norm_eps=oc.norm_eps,
                       activation=oc.activation, mlp_gated=oc.mlp_gated, attn_bias=oc.attn_bias,
                       mlp_bias=oc.mlp_bias, tokenizer_id="chars", n_kv_heads=oc.kv_heads, dtype=dtype)


class _Done:
    def __init__(self, t):
        self.t = t

    def wait(self):
        return self.t


class ThreadExchange:
    """In-process stand-in for torch.distributed collectives between rank threads."""

    def __init__(self, world):
        self.world = world
        self.slots = [None] * world
        self.bar = threading.Barrier(world)

    def for_rank(self, r):
        ex = self

        class _E:
            world = ex.world

            def all_gather(self, t, async_op=False):
                if async_op:
                    return _Done(self.all_gather(t))
                torch.cuda.current_stream().synchronize()
                ex.slots[r] = t
                ex.bar.wait()
                out = torch.cat([s.to(t.device) for s in ex.slots])
                torch.cuda.current_stream().synchronize()
                ex.bar.wait()
                return out

            def all_to_all(self, t, async_op=False):
                if async_op:
                    return _Done(self.all_to_all(t))
                torch.cuda.current_stream().synchronize()
                ex.slots[r] = t
                ex.bar.wait()
                n = t.shape[0] // ex.world
                out = torch.cat([ex.slots[w][r * n:(r + 1) * n] for w in range(ex.world)])
                torch.cuda.current_stream().synchronize()
                ex.bar.wait()
                return out
        return _E()


@pytest.fixture(scope="module")
def setup():
    import paper_2510_10129_b200 as cc
    w = C1_EXACT
    primary = cc.from_params(_cfg(w.primary, "bf16"), orc.seeded_params(w.primary, 0))
    aux = cc.from_params(_cfg(w.aux, "fp32"), orc.seeded_params(w.aux, 1))
    prefix, chunk_ids, query = w.token_ids(0)
    chunks = [cc.prefill_chunk(primary, prefix, c) for c in chunk_ids]
    aux_chunks = [cc.prefill_chunk(aux, prefix, c) for c in chunk_ids]
    config = cc.SelectionConfig(w.ratio, w.window_len, w.window_threshold)
    ref = cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query, config)
    return w, primary, aux, prefix, chunk_ids, query, chunks, aux_chunks, config, ref


def _run_rank(setup, W, r, exchange, out):
    from paper_2510_10129_b200.sharded import DeviceShardCompute, cacheclip_prefill_sharded, plan_shards
    w, primary, aux, prefix, chunk_ids, query, chunks, aux_chunks, config, ref = setup
    with torch.cuda.stream(torch.cuda.Stream()):
        plan = plan_shards([len(c) for c in chunk_ids], len(prefix), len(query), W, r)
        mine = plan.local_chunks()
        res = cacheclip_prefill_sharded(DeviceShardCompute(primary, aux), exchange, plan, [chunks[c] for c in mine],
                                        [aux_chunks[c] for c in mine], {c: chunk_ids[c] for c in mine}, query,
                                        config, n_layers=primary.config.n_layers)
        torch.cuda.current_stream().synchronize()
    out[r] = res


@pytest.mark.parametrize("W", [1, 2, 3])
def test_sharded_matches_single_gpu(setup, W):
    from paper_2510_10129_b200.sharded import Exchange
    ref = setup[-1]
    out = [None] * W
    if W == 1:
        _run_rank(setup, 1, 0, Exchange(1), out)
    else:
        tx = ThreadExchange(W)
        errs = []

        def body(r):
            try:
                _run_rank(setup, W, r, tx.for_rank(r), out)
            except Exception as e:  # pragma: no cover
                errs.append(e)
                tx.bar.abort()
        th = [threading.Thread(target=body, args=(r,)) for r in range(W)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=300)
        assert not errs, errs
    for r in range(W):
        assert out[r].indices == ref.plan.indices           # identical selection on every rank
    head = out[0]
    std = ref.logits.std()
    err = np.abs(head.logits - ref.logits).max()
    print(f"W={W}: |dlogits| vs unsharded {err:.3e} (std {std:.3f})")
    assert err < 3e-2 * std
    assert head.first_token == ref.first_token


def _dist_worker(rank, world, port, outdir, pipeline):
    import os as _os

    import torch.distributed as dist

    import paper_2510_10129_b200 as cc
    from paper_2510_10129_b200.sharded import DeviceShardCompute, Exchange, cacheclip_prefill_sharded, plan_shards
    _os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = C1_EXACT
        primary = cc.from_params(_cfg(w.primary, "bf16"), orc.seeded_params(w.primary, 0))
        aux = cc.from_params(_cfg(w.aux, "fp32"), orc.seeded_params(w.aux, 1))
        prefix, chunk_ids, query = w.token_ids(0)
        plan = plan_shards([len(c) for c in chunk_ids], len(prefix), len(query), world, rank)
        mine = plan.local_chunks()   # each rank precomputes only its own chunks
        chunks = [cc.prefill_chunk(primary, prefix, chunk_ids[c]) for c in mine]
        aux_chunks = [cc.prefill_chunk(aux, prefix, chunk_ids[c]) for c in mine]
        res = cacheclip_prefill_sharded(DeviceShardCompute(primary, aux), Exchange(world), plan, chunks, aux_chunks,
                                        {c: chunk_ids[c] for c in mine}, query,
                                        cc.SelectionConfig(w.ratio, w.window_len, w.window_threshold),
                                        n_layers=primary.config.n_layers, pipeline=pipeline)
        torch.cuda.synchronize()
        np.savez(_os.path.join(outdir, f"r{rank}.npz"), indices=np.asarray(res.indices),
                 logits=res.logits if res.logits is not None else np.zeros(0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,pipeline", [(2, 2), (2, 1), (3, 2)])
def test_multiprocess_sharded_over_torch_distributed(setup, tmp_path, world, pipeline):
    """W processes (gloo, sharing cuda:0) run DeviceShardCompute
    and the real torch.distributed Exchange on CUDA tensors: score all_gather,
    identical selection, per-layer Q all_gather, partial attention, all_to_all,
    LSE merge — pipelined in two halves (async collectives) or not. Every rank
    selects the unsharded plan; the head rank's logits match the single-GPU
    pipeline."""
    import os
    import socket

    import torch.multiprocessing as mp
    ref = setup[-1]
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mp.spawn(_dist_worker, args=(world, port, str(tmp_path), pipeline), nprocs=world, join=True)
    outs = [dict(np.load(os.path.join(tmp_path, f"r{r}.npz"))) for r in range(world)]
    for o in outs:
        assert tuple(o["indices"].tolist()) == ref.plan.indices
    std = ref.logits.std()
    err = np.abs(outs[0]["logits"] - ref.logits).max()
    print(f"W={world} pipeline={pipeline}: |dlogits| vs unsharded {err:.3e} (std {std:.3f})")
    assert err < 3e-2 * std
    assert int(np.argmax(outs[0]["logits"])) == ref.first_token
