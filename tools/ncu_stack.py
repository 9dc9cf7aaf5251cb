"""A few token passes of a small layer stack, for one ncu capture of its kernels.

    ncu --set full -k regex:tgemv_kernel --launch-skip 4 --launch-count 1 \
        python tools/ncu_stack.py cfg4 i2s 8 2
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2410_16144_b200 import _lib as L  # noqa: E402

if os.environ.get("TB_LIB"):
    L.load(os.environ["TB_LIB"])

from paper_2410_16144_b200.stack import STACKS, LayerStack  # noqa: E402
from paper_2410_16144_b200 import kernels as tb_kernels  # noqa: E402


def main():
    name, fmt, M, layers = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    st = LayerStack(STACKS[name], fmt, tokens=M, layers=layers)
    h, i = STACKS[name]["hidden"], STACKS[name]["inter"]
    g = torch.Generator(device="cuda").manual_seed(5)
    if M == 1:
        xh = [torch.randn(h, generator=g, device="cuda") for _ in range(layers)]
        xi = [torch.randn(i, generator=g, device="cuda") for _ in range(layers)]
        pool = None
    else:
        xh = [torch.randn(M, h, generator=g, device="cuda") for _ in range(layers)]
        xi = [torch.randn(M, i, generator=g, device="cuda") for _ in range(layers)]
        pool = st.make_glues(xh, xi)
    if os.environ.get("ONLY") == "gemv" and M > 1:  # timing only: the GEMVs without the glue
        def gemv_only(*_):
            for b in st.batches:
                b.run(finalize=False)
        st.token_pass = gemv_only
    elif os.environ.get("ONLY") == "glue" and M > 1:  # timing only: the glues alone
        def glue_only(xh_, xi_, pool_):
            prev = None
            for li, b in enumerate(st.batches):
                pool_[li].retarget(prev).run()
                prev = b
        st.token_pass = glue_only
    elif os.environ.get("ONLY") == "gq" and M > 1:  # timing only: the glues' quantisation
        def gq(xh_, xi_, pool_):
            for li in range(len(st.batches)):
                pool_[li].retarget(None).run()
        st.token_pass = gq
    elif os.environ.get("ONLY") == "gf" and M > 1:  # timing only: the glues' finalize
        fin = tb_kernels.StepGlue([])

        def gf(xh_, xi_, pool_):
            for b in st.batches:
                fin.retarget(b).run()
        st.token_pass = gf
    elif os.environ.get("ONLY") == "gemvq" and M > 1:  # timing only: quantise + GEMV (no finalize)
        def gemvq(xh_, xi_, pool_):
            for li, b in enumerate(st.batches):
                pool_[li].retarget(None).run()
                b.run(finalize=False)
        st.token_pass = gemvq
    elif os.environ.get("ONLY") == "gemvf" and M > 1:  # timing only: finalize + GEMV (no quantise)
        fin2 = tb_kernels.StepGlue([])

        def gemvf(xh_, xi_, pool_):
            prev = None
            for b in st.batches:
                fin2.retarget(prev).run() if prev is not None else None
                b.run(finalize=False)
                prev = b
        st.token_pass = gemvf
    if os.environ.get("ONLY") == "gemvp" and M > 1:  # timing only: GEMV + tail finalize (no glue)
        def gemvp(xh_, xi_, pool_):
            prev = None
            for b in st.batches:
                b.run(finalize=False, prev=prev)
                prev = b
        st.token_pass = gemvp
    if os.environ.get("GRAPH"):
        run1 = st.token_pass
        run1(xh, xi, pool)
        torch.cuda.synchronize()
        s_ = torch.cuda.Stream()
        s_.wait_stream(torch.cuda.current_stream())
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s_), torch.cuda.graph(gr, stream=s_):
            run1(xh, xi, pool)
        st.token_pass = lambda *a: gr.replay()
    for _ in range(4):
        st.token_pass(xh, xi, pool)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        st.token_pass(xh, xi, pool)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} {fmt} M={M} layers={layers}: {e0.elapsed_time(e1) / 5 / layers * 1e3:.1f} us/layer "
          f"({st.algo_bytes / layers / 1e6:.1f} MB/layer)")


if __name__ == "__main__":
    main()
