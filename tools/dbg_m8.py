"""Debug: M=8 records-path GEMV parity at cfg4 shapes (mismatch statistics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_16144_b200 as tb
from paper_2410_16144_b200 import _lib as L
from paper_2410_16144_b200.kernels import ActRecords, GemvBatch, GemvPlan, StepGlue
from oracle import c_oracle as CO, ternpack_oracle as O
CO.build()
M = int(os.environ.get("M", 8))
def check(plan, x, tag):
    got = plan.out32.cpu().numpy()
    pl = plan.p.data.cpu().numpy()
    bad = []
    for t in range(M):
        q, s = CO.quantize(x[t], 4)
        want = O.make_output(CO.gemv_i2s(pl, q, 0), plan.p.scale, s).astype(np.float32)
        d = np.nonzero(got[t] != want)[0]
        if d.size: bad.append((t, d.size, int(d[0]), int(d[-1])))
    print(tag, "OK" if not bad else bad, flush=True)
g = torch.Generator(device="cuda").manual_seed(5)
for n, k in ((1280, 10240), (10240, 10240), (32768, 10240), (10240, 32768), (14336, 4096)):
    w = torch.randn(n, k, generator=g, device="cuda") * 0.02
    p = tb.encode_i2s(tb.ternarize_weights(w, n, k)); del w
    plan = GemvPlan(p, max_tokens=M, out_dtype=torch.float32)
    rec = ActRecords(L.I2S, M, k)
    x = torch.randn(M, k, generator=g, device="cuda")
    rec.quantize(x)
    GemvBatch([(plan, rec)]).run()
    torch.cuda.synchronize()
    check(plan, x.cpu().numpy(), f"single {n}x{k}")
    # glue form
    b = GemvBatch([(plan, rec)])
    x2 = torch.randn(M, k, generator=g, device="cuda")
    StepGlue([(x2, rec)]).run(); b.run(finalize=False); StepGlue([]).retarget(b).run()
    torch.cuda.synchronize()
    check(plan, x2.cpu().numpy(), f"glue   {n}x{k}")
