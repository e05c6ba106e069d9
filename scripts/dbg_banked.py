import math, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2510_10129_b200 import _lib as L
from paper_2510_10129_b200.runtime import bank_tables
from oracle import cacheclip_oracle as orc
DEV = torch.device("cuda", 0)
Hq, Hkv, D, Q, nbs = 4, 2, 64, 8, (40, 3, 100)
import os; print(os.environ.get("CACHECLIP_SM100_LIB"))
rng = np.random.default_rng(3)
banks = [rng.standard_normal((1, nb, Hkv, D)).astype(np.float32) for nb in nbs]
vbanks = [rng.standard_normal((1, nb, Hkv, D)).astype(np.float32) for nb in nbs]
S = len(banks)
q = rng.standard_normal((S * Q, Hq * D)).astype(np.float32)
kn = rng.standard_normal((S * Q, Hkv * D)).astype(np.float32)
vn = rng.standard_normal((S * Q, Hkv * D)).astype(np.float32)
tk = [torch.from_numpy(b).to(DEV) for b in banks]
tv = [torch.from_numpy(b).to(DEV) for b in vbanks]
tables = bank_tables(1, [(tk[s], tv[s], banks[s].shape[1], s * Q, Q) for s in range(S)], DEV)
qd, kd, vd = (torch.from_numpy(a).to(DEV) for a in (q, kn, vn))
factor = float(np.float32(1 / math.sqrt(D)))
maxb = max(nbs)
st = torch.cuda.current_stream().cuda_stream
for fn in ("cc_banked_attention_f32", "cc_banked_attention_simt"):
    out = torch.zeros(S * Q, Hq * D, device=DEV)
    w = torch.zeros(S, Hq, Q, maxb, device=DEV)
    L.call(fn, tables.data_ptr(), S, Q, maxb, qd.data_ptr(), kd.data_ptr(), vd.data_ptr(), Hq, Hkv, D, factor,
           out.data_ptr(), L.CC_F32, None, 0, 0, st)
    L.call(fn, tables.data_ptr(), S, Q, maxb, qd.data_ptr(), kd.data_ptr(), vd.data_ptr(), Hq, Hkv, D, factor,
           out.data_ptr(), L.CC_F32, w.data_ptr(), 0, maxb, st)
    torch.cuda.synchronize()
    got, wg = out.cpu().numpy(), w.cpu().numpy()
    for s in range(S):
        nb = nbs[s]
        bank_k = np.concatenate([banks[s][0], kn[s * Q:(s + 1) * Q].reshape(Q, Hkv, D)])
        bank_v = np.concatenate([vbanks[s][0], vn[s * Q:(s + 1) * Q].reshape(Q, Hkv, D)])
        qq = q[s * Q:(s + 1) * Q].reshape(Q, Hq, D).transpose(1, 0, 2)
        ctx, wr = orc.attend(qq, bank_k.transpose(1, 0, 2), bank_v.transpose(1, 0, 2), nb + np.arange(Q) + 1)
        g = got[s * Q:(s + 1) * Q].reshape(Q, Hq, D)
        print(fn, s, "ctx maxerr", np.abs(g - ctx.transpose(1, 0, 2)).max(), "ctx absmax", np.abs(g).max(),
              "w maxerr", np.abs(wg[s, :, :, :nb] - wr[:, :, :nb]).max() if nb else 0)
        if s == 0 and fn.endswith("f32"):
            print(" got[0,0,:8]", g[0, 0, :8]); print(" ref[0,0,:8]", ctx.transpose(1, 0, 2)[0, 0, :8])
