"""PCIe paths for host-resident chunk caches at C3: copy-engine streamed
assembly (scoring banks, primary merge) vs a plain pinned cudaMemcpy."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_10129_b200 as cc  # noqa: E402
from paper_2510_10129_b200.kv_store import stream_local_banks  # noqa: E402
from paper_2510_10129_b200.workloads import WORKLOADS  # noqa: E402

w = WORKLOADS["c3"]
dev = torch.device("cuda", 0)
primary = cc.init_model(w.primary, 0, device=dev, source="torch")
aux = cc.init_model(w.aux, 1, device=dev, source="torch")
prefix, chunk_ids, query = w.token_ids(1000)
pc = cc.prefill_chunks(primary, prefix, chunk_ids)
ac = cc.prefill_chunks(aux, prefix, chunk_ids)


def host(c, m):
    return cc.ChunkCache(c.k.cpu().pin_memory(), c.v.cpu().pin_memory(), c.token_ids, c.prefix_len,
                         m.config.tokenizer_id, m.fingerprint)


hp = [host(c, primary) for c in pc]
ha = [host(c, aux) for c in ac]
del pc, ac
torch.cuda.empty_cache()


def timed(fn, label, nbytes):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    fn()
    b.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"{label:40s} {ms:8.2f} ms  {nbytes / ms / 1e6:7.1f} GB/s  (host issue {1e3 * (t1 - t0):.2f} ms)", flush=True)


abytes = sum(c.k.numel() * 4 * 2 for c in ha)
pbytes = sum(c.k.numel() * 2 * 2 for c in hp)
timed(lambda: stream_local_banks(ha, aux.config.rope, dev), "scoring banks, copy-engine stream", abytes)
timed(lambda: cc.merge_caches(hp, primary.config.rope, device=dev), "primary merge, copy-engine stream", pbytes)
big = torch.empty(abytes // 4, dtype=torch.float32).pin_memory()
dst = torch.empty_like(big, device=dev)
timed(lambda: dst.copy_(big, non_blocking=True), "one pinned cudaMemcpy (copy engine)", abytes)
