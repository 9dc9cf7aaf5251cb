"""Break down the host-driven decode step (HostStep) of bench.py's e2e."""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_16144_b200 as tb  # noqa: E402

H, I = 4096, 14336


def wall(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    plans = []
    for rows, cols in ((I, H), (I, H), (H, I)):
        w = torch.randn(rows, cols, generator=g, device="cuda") * 0.02
        plans.append(tb.GemvPlan(tb.encode_tl1(tb.ternarize_weights(w, rows, cols))))
    step = tb.GemvStep([(plans[0], 0), (plans[1], 0), (plans[2], 1)], [H, I])
    hs = tb.HostStep([(plans[0], 0), (plans[1], 0), (plans[2], 1)], [H, I])
    xh = torch.randn(H).pin_memory()
    xi = torch.randn(I).pin_memory()
    s = torch.cuda.current_stream()
    print(f"HostStep call          {wall(lambda: hs([xh, xi])):8.2f} us")
    print(f"graph replay + sync    {wall(lambda: (hs._record.replay(), s.synchronize())):8.2f} us")
    print(f"host staging copies    {wall(lambda: (hs.x_host[0].copy_(xh), hs.x_host[1].copy_(xi))):8.2f} us")
    print(f"flags max              {wall(lambda: int(hs.flags_host.max())):8.2f} us")
    print(f"stream sync (idle)     {wall(lambda: s.synchronize()):8.2f} us")
    print(f"step+finalize eager    {wall(lambda: (step.run(hs.x_dev), step.finalize(), s.synchronize())):8.2f} us")
    d = torch.empty(I, device="cuda")
    print(f"H2D 57KB + sync        {wall(lambda: (d.copy_(xi, non_blocking=True), s.synchronize())):8.2f} us")
    o = torch.empty(I).pin_memory()
    print(f"D2H 57KB + sync        {wall(lambda: (o.copy_(d, non_blocking=True), s.synchronize())):8.2f} us")


if __name__ == "__main__":
    main()
