"""Eager fused decode steps of the bench workload, for one ncu capture.

    ncu --set full -k regex:tgemv_kernel --launch-skip 6 --launch-count 1 \
        python tools/ncu_step.py
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2410_16144_b200 import _lib as L  # noqa: E402

if os.environ.get("TB_LIB"):
    L.load(os.environ["TB_LIB"])  # a variant build (tools/build_variant.sh)

import paper_2410_16144_b200 as tb  # noqa: E402

H, I, NCOPY = 4096, 14336, 6
if len(sys.argv) > 2:  # e.g. 10240 32768: the cfg4 FFN shapes (one 16-warp CTA per SM)
    H, I, NCOPY = int(sys.argv[1]), int(sys.argv[2]), 2


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
    for i in range(6 * NCOPY if NCOPY < 6 else 12):
        steps[i % NCOPY].run([xh, xi], prev=steps[(i - 1) % NCOPY])
    steps[(6 * NCOPY - 1 if NCOPY < 6 else 11) % NCOPY].finalize()
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
