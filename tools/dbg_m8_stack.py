"""Debug: M=8 LayerStack parity (cfg4 shapes, few layers), chained vs synced."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2410_16144_b200.stack import LayerStack
from oracle import c_oracle as CO, ternpack_oracle as O
CO.build()
M = 8
LAY = int(os.environ.get("LAY", 3))
cfg = dict(hidden=10240, kv=1280, inter=32768, layers=LAY)
if os.environ.get("SMALL"):
    cfg = dict(hidden=4096, kv=1024, inter=14336, layers=LAY)
st = LayerStack(cfg, fmt="i2s", seed=11, tokens=M)
g = torch.Generator(device="cuda").manual_seed(99)
h, i = cfg["hidden"], cfg["inter"]
XH = torch.randn(LAY, M, h, generator=g, device="cuda")
XI = torch.randn(LAY, M, i, generator=g, device="cuda")
glues = st.make_glues(XH, XI)
def check(tag):
    for li in range(LAY):
        xs = [XH[li].cpu().numpy(), XI[li].cpu().numpy()]
        for plan, (pname, rows, cols, src) in zip(st.layers[li], st.shapes):
            got = plan.out32.cpu().numpy(); pl = plan.p.data.cpu().numpy()
            bad = []
            for t in range(M):
                q, s = CO.quantize(xs[src][t], 4)
                want = O.make_output(CO.gemv_i2s(pl, q, 0), plan.p.scale, s).astype(np.float32)
                d = np.nonzero(got[t] != want)[0]
                if d.size: bad.append((t, d.size, int(d[0]), int(d[-1])))
            if bad: print(tag, li, pname, bad[:4], flush=True)
    print(tag, "checked", flush=True)
mode = os.environ.get("MODE", "chain")
if mode == "chain":
    st.token_pass(None, None, glues)
else:  # synchronize between every launch
    prev = None
    for li, b in enumerate(st.batches):
        glues[li].retarget(prev).run(); torch.cuda.synchronize()
        b.run(finalize=False); torch.cuda.synchronize()
        prev = b
    st.tail.retarget(prev).run()
torch.cuda.synchronize()
check(mode)
