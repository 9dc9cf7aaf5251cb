"""Time the prefill activation path pieces (graph of R replays each)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_16144_b200 import _lib as L
from paper_2410_16144_b200.core import quantize_into
lib = L.load()
M = int(os.environ.get("M", 512)); R = 20
def gtime(fn):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(R): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / R
for K in (4096, 14336):
    x = torch.randn(M, K, device="cuda")
    q = torch.empty((M, K), dtype=torch.int8, device="cuda")
    sc = torch.empty(M, dtype=torch.float64, device="cuda")
    til = torch.empty(lib.tb_gemm_act_bytes(M, K), dtype=torch.uint8, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    f_q = lambda: quantize_into(x, q, sc)
    f_t = lambda: L.check(lib.tb_gemm_tile_act(q.data_ptr(), M, K, K, til.data_ptr(), L.stream_ptr()))
    f_f = lambda: L.check(lib.tb_gemm_quantize_act(x.data_ptr(), M, K, K, sc.data_ptr(), flag.data_ptr(), til.data_ptr(), L.stream_ptr()))
    f_c = lambda: torch.add(x, 1.0, out=x) if False else None
    y = torch.empty_like(x)
    f_copy = lambda: y.copy_(x)
    print(f"K={K} M={M}: quantize {gtime(f_q):.1f} us, tile {gtime(f_t):.1f} us, fused {gtime(f_f):.1f} us, "
          f"f32 copy {gtime(f_copy):.1f} us ({M*K*4/1e6:.1f} MB)", flush=True)
