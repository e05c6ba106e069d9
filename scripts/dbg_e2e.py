"""Where does the e2e (host-pinned chunk caches) step lose time against the
device-resident step?  Wall-clock per step for: device caches, pinned caches
with the copy-engine streamed merge, and a bare H2D copy."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2510_10129_b200 as cc
from paper_2510_10129_b200 import kv_store
from paper_2510_10129_b200.workloads import WORKLOADS

w = WORKLOADS["c3"]
dev = torch.device("cuda")
primary = cc.init_model(w.primary, 0, device=dev, source="torch")
aux = cc.init_model(w.aux, 1, device=dev, source="torch")
prefix, chunk_ids, query = w.token_ids(1000)
chunks = cc.prefill_chunks(primary, prefix, chunk_ids)
aux_chunks = cc.prefill_chunks(aux, prefix, chunk_ids)
config = cc.SelectionConfig(0.2, 8, 1)


def host(cs, m):
    return [cc.ChunkCache(c.k.cpu().pin_memory(), c.v.cpu().pin_memory(), c.token_ids, c.prefix_len,
                          m.config.tokenizer_id, m.fingerprint) for c in cs]


pc, ac = host(chunks, primary), host(aux_chunks, aux)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def wall(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    return float(np.median(ts)), float(np.min(ts))


def ev(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


print("device caches  events %.1f ms  wall med/min %.1f / %.1f ms" % (
    ev(lambda: cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query, config)),
    *wall(lambda: cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query, config))))
print("pinned caches wall med/min %.1f / %.1f ms" % (
    wall(lambda: cc.cacheclip_prefill(primary, aux, pc, ac, query, config))), flush=True)
t0 = time.perf_counter()
for _ in range(5):
    kv_store.merge_caches(pc, primary.config.rope, device=dev)
    kv_store.stream_local_banks(ac, aux.config.rope, dev)
print("host issue cost of both streamed transfers %.2f ms" % ((time.perf_counter() - t0) / 5 * 1e3))
torch.cuda.synchronize()

# bare H2D: every chunk cache with copy engines, and the streamed merges alone
dst = [torch.empty_like(c.k, device=dev) for c in pc] + [torch.empty_like(c.k, device=dev) for c in ac]
srcs = [c.k for c in pc] + [c.k for c in ac]
nbytes = 2 * sum(s.numel() * s.element_size() for s in srcs)


def h2d():
    for d, s in zip(dst, srcs):
        d.copy_(s, non_blocking=True)
        d.copy_(s, non_blocking=True)


t = ev(h2d)
print("bare H2D copy-engine %.2f GB in %.1f ms = %.1f GB/s" % (nbytes / 1e9, t, nbytes / t / 1e6))
t = ev(lambda: kv_store.merge_caches(pc, primary.config.rope, device=dev))
print("copy-engine merge alone (primary) %.1f ms" % t)
t = ev(lambda: kv_store.stream_local_banks(ac, aux.config.rope, dev))
print("copy-engine scoring banks alone %.1f ms" % t)
