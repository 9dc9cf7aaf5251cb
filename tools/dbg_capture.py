"""Which cfg3 piece breaks CUDA-graph capture (debug helper)."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_16144_b200 as tb
from paper_2410_16144_b200 import _lib as L
from paper_2410_16144_b200.core import quantize_into
lib = L.load()
M, K = 512, 4096
x = torch.randn(M, K, device="cuda")
q = torch.empty((M, K), dtype=torch.int8, device="cuda")
sc = torch.empty(M, dtype=torch.float64, device="cuda")
til = torch.empty(lib.tb_gemm_act_bytes(M, K), dtype=torch.uint8, device="cuda")
w = torch.randn(K, K, device="cuda") * 0.02
p = tb.encode_i2s(tb.ternarize_weights(w, K, K))
main, _ = p.tiled()
out = torch.empty((M, K), dtype=torch.float32, device="cuda")
d = (L.GemmDesc * 1)()
d[0].tiled, d[0].rows, d[0].cols, d[0].act_tiled = main.data_ptr(), K, K, til.data_ptr()
d[0].a_scale, d[0].w_scale, d[0].out32 = sc.data_ptr(), float(p.scale), out.data_ptr()
pieces = {
    "quant": lambda: quantize_into(x, q, sc),
    "tile": lambda: L.check(lib.tb_gemm_tile_act(q.data_ptr(), M, K, K, til.data_ptr(), L.stream_ptr()), "t"),
    "gemm": lambda: L.check(lib.tb_gemm_batch(L.I2S, 1, C.cast(d, C.c_void_p), M, L.stream_ptr()), "g"),
}
a = torch.randint(-127, 127, (1024, 1024), dtype=torch.int8, device="cuda")
bt = torch.randint(-127, 127, (1024, 1024), dtype=torch.int8, device="cuda").t()
pieces["int_mm"] = lambda: torch._int_mm(a, bt)
for n, f in pieces.items():
    f(); torch.cuda.synchronize()
for n, f in pieces.items():
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                f()
        torch.cuda.synchronize()
        print(n, "capture ok", flush=True)
    except Exception as e:
        print(n, "capture FAILED", type(e).__name__, str(e)[:300], flush=True)
        torch.cuda.synchronize()
