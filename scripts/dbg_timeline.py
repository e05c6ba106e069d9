"""Launch timeline of one C3 request (in-library profiler events): GPU idle
time between launches, the largest gaps and what surrounds them.

    python scripts/dbg_timeline.py [c3|c2] [ratio] [window_threshold]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_10129_b200 as cc  # noqa: E402
from paper_2510_10129_b200 import _lib  # noqa: E402
from paper_2510_10129_b200.workloads import WORKLOADS  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
ratio = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2
thr = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w = WORKLOADS[wl]
dev = torch.device("cuda")
primary = cc.init_model(w.primary, 0, device=dev, source="torch")
aux = cc.init_model(w.aux, 1, device=dev, source="torch")
prefix, chunk_ids, query = w.token_ids(1000)
chunks = cc.prefill_chunks(primary, prefix, chunk_ids)
aux_chunks = cc.prefill_chunks(aux, prefix, chunk_ids)
cfg = cc.SelectionConfig(ratio, 8, thr)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query, cfg)
torch.cuda.synchronize()
for rep in range(2):
    _lib.profile_collect()
    flush.fill_(1)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _lib.profile_enable(True)
    a.record()
    cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query, cfg)
    b.record()
    torch.cuda.synchronize()
    _lib.profile_enable(False)
    tl = _lib.profile_timeline()
    _lib.profile_collect()
    wall = a.elapsed_time(b)
    ev = sorted(tl, key=lambda r: r[1])
    busy, cur_end, gaps = 0.0, None, []
    prev = None
    for op, t0, t1 in ev:
        if cur_end is None:
            busy += t1 - t0
            cur_end = t1
        elif t0 > cur_end:
            gaps.append((t0 - cur_end, prev, op, cur_end))
            busy += t1 - t0
            cur_end = t1
        elif t1 > cur_end:
            busy += t1 - cur_end
            cur_end = t1
        prev = op
    span = ev[-1][2] - ev[0][1]
    print(f"== {wl} ratio {ratio} thr {thr}: wall {wall:.2f} ms, first..last launch {span:.2f} ms, "
          f"covered {busy:.2f} ms, idle {span - busy:.2f} ms in {len(gaps)} gaps, {len(ev)} launches")
    gaps.sort(reverse=True)
    for g, p, n, t in gaps[:15]:
        print(f"   gap {g * 1e3:8.1f} us at {t:8.2f} ms: {p} -> {n}")
    hist = {}
    for g, p, n, t in gaps:
        k = f"{p} -> {n}"
        c, s = hist.get(k, (0, 0.0))
        hist[k] = (c + 1, s + g)
    for k, (c, s) in sorted(hist.items(), key=lambda kv: -kv[1][1])[:10]:
        print(f"   {k:40s} {c:4d} gaps {s * 1e3:8.1f} us total")
