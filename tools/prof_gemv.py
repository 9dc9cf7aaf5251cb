"""Profiling driver: one decode-GEMV shape over rotating weight copies.

    python tools/prof_gemv.py --fmt tl1 --rows 14336 --cols 4096 --iters 48

Times the GEMV kernel alone (activation records prepared once) inside a CUDA
graph, and prints GB/s of packed bytes.
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2410_16144_b200 import _lib as _L  # noqa: E402

if os.environ.get("TB_LIB"):
    _L.load(os.environ["TB_LIB"])  # a variant build (tools/build_variant.sh)

import paper_2410_16144_b200 as tb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fmt", default="tl1", choices=["i2s", "tl1", "tl2"])
    ap.add_argument("--rows", type=int, default=14336)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--m", type=int, default=1)
    ap.add_argument("--iters", type=int, default=48)
    ap.add_argument("--copies", type=int, default=8)
    ap.add_argument("--eager", action="store_true", help="no graph (for ncu)")
    ap.add_argument("--with-finalize", action="store_true",
                    help="time GEMV + finalize pass (default: the GEMV kernel alone)")
    a = ap.parse_args()
    enc = {"i2s": tb.encode_i2s, "tl1": tb.encode_tl1, "tl2": tb.encode_tl2}[a.fmt]
    g = torch.Generator(device="cuda").manual_seed(0)
    plans = []
    for c in range(a.copies):
        w = torch.randn(a.rows, a.cols, generator=g, device="cuda") * 0.02
        plans.append(tb.GemvPlan(enc(tb.ternarize_weights(w, a.rows, a.cols)), max_tokens=a.m))
        del w
    x = torch.randn(a.m, a.cols, generator=g, device="cuda")
    rec = tb.ActRecords(plans[0].p.FMT, a.m, a.cols).quantize(x)
    batches = [tb.GemvBatch([(p, rec)]) for p in plans]
    fin = a.with_finalize

    def launch(i):
        batches[i % a.copies].run(finalize=fin)

    for i in range(3):
        launch(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if a.eager:
        for i in range(a.iters):
            launch(i)
        torch.cuda.synchronize()
        return
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(gr, stream=s):
            for i in range(a.iters):
                launch(i)
    gr.replay()
    torch.cuda.synchronize()
    e0.record()
    gr.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.iters
    p = plans[0].p
    if a.fmt == "tl2":
        packed = p.index_data.numel() + p.sign_data.numel()
    else:
        packed = p.data.numel()
    print(f"{a.fmt} {a.rows}x{a.cols} M={a.m}{' +fin' if fin else ''}: graph {us:.2f} us/launch = "
          f"{packed / us / 1e3:.1f} GB/s of reference packed bytes")


if __name__ == "__main__":
    main()
