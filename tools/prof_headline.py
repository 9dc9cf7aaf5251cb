"""cfg4 token pass: eager chain vs CUDA graph, same stack and inputs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_16144_b200 import _lib as L
if os.environ.get("TB_LIB"):
    L.load(os.environ["TB_LIB"])
from paper_2410_16144_b200.stack import STACKS, LayerStack
LAY = int(os.environ.get("LAY", 80)); P = int(os.environ.get("P", 5))
st = LayerStack(STACKS["cfg4"], "i2s", seed=11, tokens=1, layers=LAY)
g = torch.Generator(device="cuda").manual_seed(99)
XH = torch.randn(LAY, 10240, generator=g, device="cuda"); XI = torch.randn(LAY, 32768, generator=g, device="cuda")
xh, xi = list(XH), list(XI)
def run(n):
    for _ in range(n): st.token_pass(xh, xi)
def t_eager(n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); run(n); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n / LAY * 1e3
run(3); torch.cuda.synchronize()
print(f"eager: {t_eager(P):.2f} us/layer", flush=True)
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
gr = torch.cuda.CUDAGraph()
with torch.cuda.stream(s), torch.cuda.graph(gr, stream=s):
    run(P)
with torch.cuda.stream(s):
    gr.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record(); gr.replay(); e1.record()
torch.cuda.synchronize()
print(f"graph: {e0.elapsed_time(e1) / P / LAY * 1e3:.2f} us/layer", flush=True)
print(f"eager again: {t_eager(P):.2f} us/layer", flush=True)
