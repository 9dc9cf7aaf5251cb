"""Eager fused decode steps of the bench workload, for one ncu capture.

    ncu --set full -k regex:tgemv_kernel --launch-skip 6 --launch-count 1 \
        python tools/ncu_step.py
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_16144_b200 as tb  # noqa: E402

H, I, NCOPY = 4096, 14336, 6


def main():
    steps = []
    for c in range(NCOPY):
        gen = torch.Generator(device="cuda").manual_seed(1000 + c)
        plans = []
        for rows, cols in ((I, H), (I, H), (H, I)):
            w = torch.randn(rows, cols, generator=gen, device="cuda") * 0.02
            plans.append(tb.GemvPlan(tb.encode_tl1(tb.ternarize_weights(w, rows, cols))))
            del w
        steps.append(tb.GemvStep([(plans[0], 0), (plans[1], 0), (plans[2], 1)], [H, I]))
    gen = torch.Generator(device="cuda").manual_seed(77)
    xh = torch.randn(H, generator=gen, device="cuda")
    xi = torch.randn(I, generator=gen, device="cuda")
    for i in range(12):
        steps[i % NCOPY].run([xh, xi], prev=steps[(i - 1) % NCOPY])
    steps[11 % NCOPY].finalize()
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
