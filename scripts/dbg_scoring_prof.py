"""Per-launch times of the scoring pass (3xTF32 GEMMs, banked attention,
RMSNorm) inside the C3 request vs the scoring pass alone, with the in-library
launch profiler: does the side-stream merge (or anything else in the request)
slow the scoring GEMMs down?"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_10129_b200 as cc  # noqa: E402
from paper_2510_10129_b200 import _lib  # noqa: E402
from paper_2510_10129_b200.workloads import WORKLOADS  # noqa: E402

w = WORKLOADS["c3"]
dev = torch.device("cuda")
primary = cc.init_model(w.primary, 0, device=dev, source="torch")
aux = cc.init_model(w.aux, 1, device=dev, source="torch")
prefix, chunk_ids, query = w.token_ids(1000)
chunks = cc.prefill_chunks(primary, prefix, chunk_ids)
aux_chunks = cc.prefill_chunks(aux, prefix, chunk_ids)
cfg = cc.SelectionConfig(0.2, 8, 1)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def prof(fn, label):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    _lib.profile_collect()
    flush.fill_(1)
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    _lib.profile_enable(False)
    recs = _lib.profile_collect()
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for op, _, ms in recs:
        tot[op] += ms
        cnt[op] += 1
    print(f"== {label}: {a.elapsed_time(b):.2f} ms wall")
    for op in sorted(tot, key=lambda k: -tot[k]):
        print(f"   {op:24s} {cnt[op]:4d} launches {tot[op]:8.3f} ms")
    g = [ms for op, _, ms in recs if op == "gemm_3xtf32"]
    print("   3xTF32 per launch (first 12):", " ".join(f"{x * 1e3:.0f}" for x in g[:12]), "us")
    print("   3xTF32 per launch (last 12):", " ".join(f"{x * 1e3:.0f}" for x in g[-12:]), "us")
    return recs


prof(lambda: cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query, cfg), "C3 request")
prof(lambda: cc.aux_score_tokens(aux, aux_chunks, query), "scoring pass alone")
prof(lambda: cc.cacheclip_prefill(primary, aux, chunks, aux_chunks, query, cfg), "C3 request again")
