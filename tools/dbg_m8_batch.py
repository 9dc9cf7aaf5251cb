"""Debug: multi-job M-token GemvBatch parity (cfg4 / cfg2 layer shapes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_16144_b200 as tb
from paper_2410_16144_b200 import _lib as L
from paper_2410_16144_b200.kernels import ActRecords, GemvBatch, GemvPlan
from oracle import c_oracle as CO, ternpack_oracle as O
CO.build()
h, kv, i = (4096, 1024, 14336) if os.environ.get("SMALL") else (10240, 1280, 32768)
shapes = [(h, h, 0), (kv, h, 0), (kv, h, 0), (h, h, 0), (i, h, 0), (i, h, 0), (h, i, 1)]
g = torch.Generator(device="cuda").manual_seed(5)
mats = []
for n, k, src in shapes:
    w = torch.randn(n, k, generator=g, device="cuda") * 0.02
    mats.append((tb.encode_i2s(tb.ternarize_weights(w, n, k)), src)); del w
for M in [int(v) for v in os.environ.get("MS", "8,4,2,1").split(",")]:
  for sel in (list(range(7)), [0, 4], [4, 5], [5, 6], [4, 5, 6]):
    plans = [(GemvPlan(p, max_tokens=M, out_dtype=torch.float32), src) for p, src in (mats[j] for j in sel)]
    recs = [ActRecords(L.I2S, M, h), ActRecords(L.I2S, M, i)]
    xs = [torch.randn(M, h, generator=g, device="cuda"), torch.randn(M, i, generator=g, device="cuda")]
    for r, x in zip(recs, xs): r.quantize(x)
    GemvBatch([(pl, recs[s]) for pl, s in plans]).run()
    torch.cuda.synchronize()
    xh = [x.cpu().numpy() for x in xs]
    res = []
    for j, (pl, s) in zip(sel, plans):
        got = pl.out32.cpu().numpy(); pk = pl.p.data.cpu().numpy()
        for t in range(M):
            q, sc = CO.quantize(xh[s][t], 4)
            want = O.make_output(CO.gemv_i2s(pk, q, 0), pl.p.scale, sc).astype(np.float32)
            d = np.nonzero(got[t] != want)[0]
            if d.size: res.append((j, t, d.size, int(d[0]), int(d[-1])))
    print("M", M, "jobs", sel, "OK" if not res else res[:6], flush=True)
