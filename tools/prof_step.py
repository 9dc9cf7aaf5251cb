"""Attribute the decode-step time of bench.py (cfg1 TL1 FFN, M=1).

    python tools/prof_step.py

Times CUDA graphs of step variants over the same rotating weight copies:
GEMV alone, glue alone, glue(quantise only)+GEMV, the full bench step, and
the public per-call API pieces with host inputs (wall clock).
"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2410_16144_b200 import _lib as L  # noqa: E402

if os.environ.get("TB_LIB"):
    L.load(os.environ["TB_LIB"])  # a variant build (tools/build_variant.sh)

import paper_2410_16144_b200 as tb  # noqa: E402

ONLY = sys.argv[1:]  # e.g. fused_step api -- subsets of the variants below

H, I, NCOPY, NX, R = 4096, 14336, 6, 16, 48


def graph_us(fn, reps=R):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(reps):
                fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


def main():
    plans = []
    for c in range(NCOPY):
        gen = torch.Generator(device="cuda").manual_seed(1000 + c)
        mats = {}
        for name, rows, cols in (("gate", I, H), ("up", I, H), ("down", H, I)):
            w = torch.randn(rows, cols, generator=gen, device="cuda") * 0.02
            mats[name] = tb.encode_tl1(tb.ternarize_weights(w, rows, cols))
            del w
        plans.append({k: tb.GemvPlan(v, out_dtype=torch.float32) for k, v in mats.items()})
        plans[-1]["mats"] = mats
    gen = torch.Generator(device="cuda").manual_seed(77)
    XH = torch.randn(NX, H, generator=gen, device="cuda")
    XI = torch.randn(NX, I, generator=gen, device="cuda")
    # two record sets: a glue never quantises into the records of the batch it
    # finalises (copies alternate sets; NCOPY and NX are even)
    recs = [(tb.ActRecords(L.TL1, 1, H), tb.ActRecords(L.TL1, 1, I)) for _ in range(2)]
    for c, pl in enumerate(plans):
        rec_h, rec_i = recs[c % 2]
        pl["batch"] = tb.GemvBatch([(pl["gate"], rec_h), (pl["up"], rec_h), (pl["down"], rec_i)])
    for pl in plans:
        pl["step"] = tb.GemvStep([(pl["gate"], 0), (pl["up"], 0), (pl["down"], 1)], [H, I])
    glues = [tb.StepGlue([(XH[j:j + 1], recs[j % 2][0]), (XI[j:j + 1], recs[j % 2][1])])
             for j in range(NX)]
    fin_only = tb.StepGlue([])

    def gemv_nofin(i):
        plans[i % NCOPY]["batch"].run(finalize=False)

    def gemv_fin(i):
        plans[i % NCOPY]["batch"].run(finalize=True)

    def quant_only(i):
        glues[i % NX].retarget(None).run()

    def fin_glue(i):
        fin_only.retarget(plans[i % NCOPY]["batch"]).run()

    def glue_full(i):
        glues[i % NX].retarget(plans[(i - 1) % NCOPY]["batch"]).run()

    def quant_gemv(i):
        quant_only(i)
        gemv_nofin(i)

    def step(i):
        glues[i % NX].retarget(plans[(i - 1) % NCOPY]["batch"] if i else None).run()
        gemv_nofin(i)

    def step_sep(i):  # quantise glue, GEMV, separate finalize glue
        quant_only(i)
        gemv_nofin(i)
        fin_glue(i)

    def fused(i):
        plans[i % NCOPY]["step"].run([XH[i % NX], XI[i % NX]], prev=plans[(i - 1) % NCOPY]["step"])

    def fused_noprev(i):
        plans[i % NCOPY]["step"].run([XH[i % NX], XI[i % NX]])

    res = {}
    for name, fn in (("gemv_nofin", gemv_nofin), ("gemv_fin", gemv_fin),
                     ("quant_only", quant_only), ("fin_glue", fin_glue),
                     ("glue_full", glue_full), ("quant+gemv", quant_gemv),
                     ("bench_step", step), ("quant+gemv+fin", step_sep),
                     ("fused_step", fused), ("fused_noprev", fused_noprev)):
        if ONLY and name not in ONLY:
            continue
        res[name] = graph_us(fn)
        for pl in plans:  # leave the workspaces clean
            fin_only.retarget(pl["batch"]).run()
            pl["step"].finalize()
        torch.cuda.synchronize()
        print(f"{name:16s} {res[name]:8.2f} us", flush=True)

    if ONLY and "api" not in ONLY:
        return
    # public per-call API pieces, host inputs (wall clock)
    xh = torch.randn(NX, H).pin_memory()
    mats = plans[0]["mats"]
    K = tb.KernelKind

    def wall(fn, n=200):
        for i in range(5):
            fn(i)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(n):
            fn(i)
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / n * 1e6

    qa = tb.quantize_activations(xh[0], pad_to=2)
    print(f"{'api quantize':16s} {wall(lambda i: tb.quantize_activations(xh[i % NX], pad_to=2)):8.2f} us")
    print(f"{'api quant nochk':16s} "
          f"{wall(lambda i: tb.quantize_activations(xh[i % NX], pad_to=2, check_finite=False)):8.2f} us")
    print(f"{'api gemv(dev)':16s} {wall(lambda i: tb.gemv_parallel(K.TL1, mats['gate'], qa)):8.2f} us")
    print(f"{'api gemv+cpu':16s} "
          f"{wall(lambda i: tb.gemv_parallel(K.TL1, mats['gate'], qa).output.cpu()):8.2f} us")
    out = torch.empty(I, dtype=torch.float64, device="cuda")
    print(f"{'d2h 115KB':16s} {wall(lambda i: out.cpu()):8.2f} us")
    print(f"{'empty sync':16s} {wall(lambda i: torch.cuda.synchronize()):8.2f} us")


if __name__ == "__main__":
    main()
