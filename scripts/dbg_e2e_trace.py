"""CUPTI timeline (torch.profiler) of one C3 e2e step from host-pinned chunk
caches: per stream, what runs when; idle gaps on the compute stream."""
import os
import sys
import time
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2510_10129_b200 as cc
from paper_2510_10129_b200.workloads import WORKLOADS

w = WORKLOADS["c3"]
dev = torch.device("cuda")
primary = cc.init_model(w.primary, 0, device=dev, source="torch")
aux = cc.init_model(w.aux, 1, device=dev, source="torch")
prefix, chunk_ids, query = w.token_ids(1000)
chunks = cc.prefill_chunks(primary, prefix, chunk_ids)
aux_chunks = cc.prefill_chunks(aux, prefix, chunk_ids)
config = cc.SelectionConfig(0.2, 8, 1)
pc = [cc.ChunkCache(c.k.cpu().pin_memory(), c.v.cpu().pin_memory(), c.token_ids, c.prefix_len,
                    primary.config.tokenizer_id, primary.fingerprint) for c in chunks]
ac = [cc.ChunkCache(c.k.cpu().pin_memory(), c.v.cpu().pin_memory(), c.token_ids, c.prefix_len,
                    aux.config.tokenizer_id, aux.fingerprint) for c in aux_chunks]
mode = sys.argv[1] if len(sys.argv) > 1 else "host"


def to_pool(caches):
    L, _, H, D = caches[0].k.shape
    pool = cc.HostCachePool(len(caches), max(c.n_rows for c in caches), L, H, D, caches[0].k.dtype)
    return [pool.store(c) for c in caches]


args = {"host": (pc, ac), "device": (chunks, aux_chunks)}.get(mode) or (to_pool(chunks), to_pool(aux_chunks))
for _ in range(3):
    cc.cacheclip_prefill(primary, aux, *args, query, config)
torch.cuda.synchronize()
t = time.perf_counter()
cc.cacheclip_prefill(primary, aux, *args, query, config)
torch.cuda.synchronize()
print(f"{mode}: wall {1e3 * (time.perf_counter() - t):.1f} ms")
from paper_2510_10129_b200 import _lib
_orig_call = _lib.call
host_log = []


def _timed_call(name, *a, **k):
    t1 = time.perf_counter()
    _orig_call(name, *a, **k)
    host_log.append((name, t1, time.perf_counter()))


_lib.call = _timed_call
torch.cuda.synchronize()
tw = time.perf_counter()
cc.cacheclip_prefill(primary, aux, *args, query, config)
agg = defaultdict(lambda: [0, 0.0, 1e9, 0.0])
for name, a, b in host_log:
    g = agg[name]
    g[0] += 1; g[1] += (b - a) * 1e3; g[2] = min(g[2], (a - tw) * 1e3); g[3] = max(g[3], (b - tw) * 1e3)
print("host calls: name, count, total ms, first start, last end (ms from step start)")
for name, (n, tot, a, b) in sorted(agg.items(), key=lambda kv: kv[1][2]):
    print(f"   {name:34s} {n:5d} {tot:8.2f} {a:8.2f} {b:8.2f}")
_lib.call = _orig_call
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    cc.cacheclip_prefill(primary, aux, *args, query, config)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in evs)
by_stream = defaultdict(list)
for e in evs:
    by_stream[getattr(e, "device_resource_id", 0)].append(e)


def cat(name):
    n = name.lower()
    for key in ("gemm2", "gemm_kernel", "fa_sparse", "banked", "rmsnorm", "rope_inplace", "assemble", "memcpy",
                "select", "lm_head", "reduce", "embed"):
        if key in n:
            return key
    return name[:40]


for sid, lst in sorted(by_stream.items()):
    lst.sort(key=lambda e: e.time_range.start)
    spans = defaultdict(lambda: [1e18, 0.0, 0.0, 0])
    for e in lst:
        s = spans[cat(e.name)]
        a, b = (e.time_range.start - t0) / 1e3, (e.time_range.end - t0) / 1e3
        s[0] = min(s[0], a); s[1] = max(s[1], b); s[2] += b - a; s[3] += 1
    print(f"stream {sid}: {len(lst)} ops, {(lst[0].time_range.start - t0) / 1e3:.1f} .. "
          f"{(lst[-1].time_range.end - t0) / 1e3:.1f} ms")
    for k, (a, b, busy, n) in sorted(spans.items(), key=lambda kv: kv[1][0]):
        print(f"   {k:28s} x{n:5d}  {a:7.2f} .. {b:7.2f} ms  busy {busy:7.2f} ms")
    gaps = []
    for x, y in zip(lst, lst[1:]):
        g = (y.time_range.start - x.time_range.end) / 1e3
        if g > 0.2:
            gaps.append((g, (x.time_range.end - t0) / 1e3, cat(x.name), cat(y.name)))
    gaps.sort(reverse=True)
    for g in gaps[:8]:
        print(f"   gap {g[0]:.2f} ms at {g[1]:.2f} after {g[2]} before {g[3]}")
