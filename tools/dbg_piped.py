"""Debug: pipelined vs serial M>1 stack; which layers mismatch, and whose scales were used."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_16144_b200 import _lib as L
from paper_2410_16144_b200.stack import LayerStack

M = int(os.environ.get("M", 2))
NL = int(os.environ.get("NL", 6))
PASSES = int(os.environ.get("PASSES", 1))
cfg = {"hidden": 1024, "kv": 256, "inter": 3072, "layers": NL}
g = torch.Generator(device="cuda").manual_seed(7)
XH = torch.randn(NL, M, 1024, generator=g, device="cuda")
XI = torch.randn(NL, M, 3072, generator=g, device="cuda")
serial = LayerStack(cfg, seed=5, tokens=M, pipelined=False)
piped = LayerStack(cfg, seed=5, tokens=M, pipelined=True)
serial.token_pass(None, None, serial.make_glues(XH, XI))
glues = piped.make_glues(XH, XI)
torch.cuda.synchronize()
for p in range(PASSES):
    piped.token_pass(None, None, glues)
    if os.environ.get("SYNC_EACH"):
        torch.cuda.synchronize()
torch.cuda.synchronize()
print("timeouts", L.load().tb_sync_timeouts(), "sync", piped.sync.flatten().tolist())
scales = [[piped.rec[li % 3][s].scales.clone() for s in range(2)] for li in range(NL)]
for li in range(NL):
    for j, (a, b) in enumerate(zip(serial.layers[li], piped.layers[li])):
        if not torch.equal(a.out32, b.out32):
            r = (b.out32[:, :4] / a.out32[:, :4]).tolist()
            print("layer", li, "job", j, "mismatch; ratio", [[round(v, 4) for v in row] for row in r])
ss = [[serial.rec[li % 2][s].scales.tolist() for s in range(2)] for li in range(NL)]
print("serial-set scales now (2 sets):", [[round(v, 5) for v in x[0]] for x in ss[:2]])
print("piped-set scales now (3 sets):", [[round(v, 5) for v in piped.rec[k][0].scales.tolist()] for k in range(3)])
