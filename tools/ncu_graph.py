"""One CUDA-graph replay of a bench workload inside an NVTX range "prof", for
ncu --graph-profiling graph --nvtx --nvtx-include "prof/" (the chained,
in-graph behaviour: DRAM bytes and throughput over the whole chain).

    python tools/ncu_graph.py cfg4|cfg2i2s|cfg2tl2|cfg1|cfg4m8 [layers]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_16144_b200 as tb  # noqa: E402
from paper_2410_16144_b200.stack import STACKS, LayerStack  # noqa: E402


def workload(name, layers):
    g = torch.Generator(device="cuda").manual_seed(99)
    if name in ("cfg4", "cfg2i2s", "cfg2tl2", "cfg4m8"):
        cfg = STACKS["cfg4" if name.startswith("cfg4") else "cfg2"]
        fmt = "tl2" if name == "cfg2tl2" else "i2s"
        M = 8 if name == "cfg4m8" else 1
        st = LayerStack(cfg, fmt, seed=11, tokens=M, layers=layers)
        h, i = cfg["hidden"], cfg["inter"]
        if M == 1:
            xh = list(torch.randn(layers, h, generator=g, device="cuda"))
            xi = list(torch.randn(layers, i, generator=g, device="cuda"))
            return st, lambda: st.token_pass(xh, xi)
        XH = torch.randn(layers, M, h, generator=g, device="cuda")
        XI = torch.randn(layers, M, i, generator=g, device="cuda")
        glues = st.make_glues(XH, XI)
        return st, lambda: st.token_pass(None, None, glues)
    if name == "cfg1":
        H, I = 4096, 14336
        plans = []
        for c in range(6):
            gen = torch.Generator(device="cuda").manual_seed(1000 + c)
            mats = {}
            for nm, r, k in (("gate", I, H), ("up", I, H), ("down", H, I)):
                w = torch.randn(r, k, generator=gen, device="cuda") * 0.02
                mats[nm] = tb.GemvPlan(tb.encode_tl1(tb.ternarize_weights(w, r, k)))
            plans.append(tb.GemvStep([(mats["gate"], 0), (mats["up"], 0), (mats["down"], 1)],
                                     [H, I]))
            plans[-1]._mats = mats
        XH = torch.randn(64, H, generator=g, device="cuda")
        XI = torch.randn(64, I, generator=g, device="cuda")

        def run():
            prev = None
            for j in range(layers):
                st = plans[j % 6]
                st.run([XH[j % 64], XI[j % 64]], prev=prev)
                prev = st
            prev.finalize()
        return plans, run
    raise SystemExit(f"unknown workload {name}")


def main():
    name = sys.argv[1]
    layers = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    keep, fn = workload(name, layers)
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s), torch.cuda.graph(gr, stream=s):
        fn()
    with torch.cuda.stream(s):
        gr.replay()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("prof")
    with torch.cuda.stream(s):
        gr.replay()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    print("done", name, layers)


if __name__ == "__main__":
    main()
