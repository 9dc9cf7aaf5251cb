"""BASELINE configs[0] (one I2_S GEMV, M=1, 4096 x 4096) as a chain of fused
launches over rotating weight copies; TB_LIB selects a variant build.

    python tools/prof_cfg0.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_16144_b200 import _lib as L  # noqa: E402

if os.environ.get("TB_LIB"):
    L.load(os.environ["TB_LIB"])
import paper_2410_16144_b200 as tb  # noqa: E402


IND = os.environ.get("CHAINED", "0") != "1"


def main(copies=32, steps=400):
    n = k = int(os.environ.get("N", 4096))
    g = torch.Generator(device="cuda").manual_seed(3)
    objs = []
    for _ in range(copies):
        w = torch.randn(n, k, generator=g, device="cuda") * 0.02
        plan = tb.GemvPlan(tb.encode_i2s(tb.ternarize_weights(w, n, k)), out_dtype=torch.float32)
        objs.append(tb.GemvStep([(plan, 0)], [k], independent=IND))
    X = torch.randn(16, k, generator=g, device="cuda")

    def run(cnt):
        if IND:  # independent self-finalising launches (the bench form)
            for i in range(cnt):
                objs[i % copies].run([X[i % 16]])
            return
        for i in range(cnt):
            objs[i % copies].run([X[i % 16]], prev=objs[(i - 1) % copies])
        objs[(cnt - 1) % copies].finalize()

    run(copies)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            run(steps)
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    graph.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / steps
    algo = n * k // 4 + k + 4 * n
    print(f"{n}x{k} I2_S GEMV chain: {us:.2f} us per launch, {algo / us / 1e3:.0f} GB/s")


if __name__ == "__main__":
    main()
