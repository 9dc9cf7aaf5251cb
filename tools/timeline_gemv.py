"""Per-warp timeline of one decode-GEMV launch (debug library built with
-DTB_TIMELINE into tools/libternary_b200_timeline.so).

Marks: 0 entry, 1 prologue done (fused step: inputs quantised), 2 first
stage landed, 3 compute done, 4 flush done.  --step: one fused decode step of
the bench workload (gate/up/down, two inputs).  Prints quantiles of each mark relative to the earliest entry.
"""

import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2410_16144_b200 import _lib as L  # noqa: E402

lib = L.load(os.environ.get("TB_LIB", os.path.join(ROOT, "tools", "libternary_b200_timeline.so")))
lib.tb_timeline_fetch.argtypes = [C.c_void_p, C.c_int64]
lib.tb_timeline_clear.argtypes = []

import torch  # noqa: E402

import paper_2410_16144_b200 as tb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fmt", default="tl1")
    ap.add_argument("--rows", type=int, default=14336)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--step", action="store_true")
    ap.add_argument("--chain", type=int, default=0, help="--step: marks of the last of N chained steps")
    ap.add_argument("--isolated", action="store_true", help="--step: HostStep's isolated launches")
    ap.add_argument("--hoststep", action="store_true", help="HostStep's copy-in + self-finalising step")
    a = ap.parse_args()
    if a.hoststep:
        return hoststep_timeline()
    if a.step:
        return step_timeline(a.chain, a.isolated)
    enc = {"i2s": tb.encode_i2s, "tl1": tb.encode_tl1, "tl2": tb.encode_tl2}[a.fmt]
    g = torch.Generator(device="cuda").manual_seed(0)
    plans = []
    for c in range(4):
        w = torch.randn(a.rows, a.cols, generator=g, device="cuda") * 0.02
        plans.append(tb.GemvPlan(enc(tb.ternarize_weights(w, a.rows, a.cols))))
    x = torch.randn(1, a.cols, generator=g, device="cuda")
    rec = tb.ActRecords(plans[0].p.FMT, 1, a.cols).quantize(x)
    for i in range(6):
        plans[i % 4].run_records(rec)
    torch.cuda.synchronize()
    for trial in range(3):
        lib.tb_timeline_clear()
        torch.cuda.synchronize()
        plans[trial % 4].run_records(rec)
        torch.cuda.synchronize()
        buf = np.zeros((148 * 32, 5), dtype=np.uint64)
        lib.tb_timeline_fetch(buf.ctypes.data_as(C.c_void_p), buf.nbytes)
        used = buf[:, 0] > 0
        t = buf[used].astype(np.int64)
        t0 = t[:, 0].min()
        rel = (t - t0) / 1000.0
        print(f"trial {trial}: {used.sum()} warps; us since first entry  (min / p50 / p90 / max)")
        for k, name in enumerate(["entry", "bar init", "first data", "compute done", "flushed"]):
            col = rel[:, k]
            print(f"  {name:13s} {col.min():7.2f} {np.median(col):7.2f} "
                  f"{np.quantile(col, 0.9):7.2f} {col.max():7.2f}")


def report(name):
    buf = np.zeros((148 * 32, 5), dtype=np.uint64)
    lib.tb_timeline_fetch(buf.ctypes.data_as(C.c_void_p), buf.nbytes)
    cp = buf[-1].astype(np.int64).copy()  # copy-in kernel (HostStep): entry, exit
    buf[-1] = 0
    used = buf[:, 0] > 0
    t = buf[used].astype(np.int64)
    if cp[0] > 0 and not os.environ.get("TL_CLOCK"):
        t0 = t[:, 0].min()
        print(f"  copy-in kernel: entry {(cp[0] - t0) / 1000:7.2f}  block 0 exit {(cp[1] - t0) / 1000:7.2f}")
    if os.environ.get("TL_CLOCK"):  # per-warp clock64 deltas since its own entry, in k-cycles
        rel = (t - t[:, :1]) / 1000.0
    else:
        rel = (t - t[:, 0].min()) / 1000.0
    print(f"{name}: {used.sum()} warps; us since first entry  (min / p50 / p90 / max)")
    for k, nm in enumerate(["entry", "prologue", "first data", "compute done", "flushed"]):
        col = rel[:, k]
        print(f"  {nm:13s} {col.min():7.2f} {np.median(col):7.2f} "
              f"{np.quantile(col, 0.9):7.2f} {col.max():7.2f}")


def step_timeline(chain=0, isolated=False):
    H, I = 4096, 14336
    g = torch.Generator(device="cuda").manual_seed(0)
    steps = []
    for c in range(4):
        plans = []
        for rows, cols in ((I, H), (I, H), (H, I)):
            w = torch.randn(rows, cols, generator=g, device="cuda") * 0.02
            plans.append(tb.GemvPlan(tb.encode_tl1(tb.ternarize_weights(w, rows, cols))))
            del w
        steps.append(tb.GemvStep([(plans[0], 0), (plans[1], 0), (plans[2], 1)], [H, I],
                                 isolated=isolated))
    xh = torch.randn(H, generator=g, device="cuda")
    xi = torch.randn(I, generator=g, device="cuda")
    for i in range(8):
        steps[i % 4].run([xh, xi], prev=steps[(i - 1) % 4])
    torch.cuda.synchronize()
    if chain:
        for trial in range(3):
            lib.tb_timeline_clear()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(chain):
                steps[i % 4].run([xh, xi], prev=steps[(i - 1) % 4])
            e1.record()
            torch.cuda.synchronize()
            print(f"chain of {chain}: {e0.elapsed_time(e1) * 1e3 / chain:.2f} us/step (eager launches)")
            report(f"last step of the chain, trial {trial}")
        return
    for trial in range(3):
        lib.tb_timeline_clear()
        torch.cuda.synchronize()
        torch.cuda._sleep(200000)  # the launch is queued behind a busy GPU
        if isolated:
            steps[trial % 4].run([xh, xi])
            steps[trial % 4].finalize()
        else:
            steps[trial % 4].run([xh, xi], prev=steps[(trial - 1) % 4])
        torch.cuda.synchronize()
        report(f"isolated step {trial}")


def hoststep_timeline():
    H, I = 4096, 14336
    g = torch.Generator(device="cuda").manual_seed(0)
    pairs = []
    for (rows, cols), src in (((I, H), 0), ((I, H), 0), ((H, I), 1)):
        w = torch.randn(rows, cols, generator=g, device="cuda") * 0.02
        pairs.append((tb.GemvPlan(tb.encode_tl1(tb.ternarize_weights(w, rows, cols)),
                                  out_dtype=torch.float32), src))
        del w
    hs = tb.HostStep(pairs, [H, I])
    xs = [np.random.default_rng(0).standard_normal(k).astype(np.float32) for k in (H, I)]
    for _ in range(3):
        hs(xs)
    for trial in range(3):
        lib.tb_timeline_clear()
        torch.cuda.synchronize()
        with torch.cuda.stream(hs._stream):
            torch.cuda._sleep(200000)
            hs._issue()
        torch.cuda.synchronize()
        report(f"HostStep step {trial}")


if __name__ == "__main__":
    main()
