"""Prefill GEMM throughput on BASELINE configs[3] (one Llama-3-8B-shaped
layer, M=512, I2_S): one grouped tb_gemm_batch launch over q/k/v/o/gate/up
(x_h) and down (x_i); int8 TOPS = 2*M*sum(N*K) / time.  Also measures the
cuBLASLt int8 peak (torch._int_mm, 8192^3) as the roofline denominator.

    python tools/prof_gemm.py [--fmt i2s|tl1] [--m 512]
"""

import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2410_16144_b200 import _lib as L  # noqa: E402

if os.environ.get("TB_LIB"):
    L.load(os.environ["TB_LIB"])  # a variant build (tools/build_variant.sh)

import paper_2410_16144_b200 as tb  # noqa: E402

H, I, KV = 4096, 14336, 1024


def events_us(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


def int8_peak_tops():
    a = torch.randint(-127, 127, (8192, 8192), dtype=torch.int8, device="cuda")
    bt = torch.randint(-127, 127, (8192, 8192), dtype=torch.int8, device="cuda").t()
    us = events_us(lambda: torch._int_mm(a, bt), 10)
    return 2 * 8192 ** 3 / (us * 1e-6) / 1e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fmt", default="i2s", choices=["i2s", "tl1"])
    ap.add_argument("--m", type=int, default=512)
    ap.add_argument("--copies", type=int, default=3)
    ap.add_argument("--only", default="", help="comma list of projections (default: all 7)")
    a = ap.parse_args()
    enc = tb.encode_i2s if a.fmt == "i2s" else tb.encode_tl1
    M = a.m
    g = torch.Generator(device="cuda").manual_seed(0)
    xh = tb.quantize_tokens(torch.randn(M, H, generator=g, device="cuda"))
    xi = tb.quantize_tokens(torch.randn(M, I, generator=g, device="cuda"))
    shapes = [("q", H, H, xh), ("k", KV, H, xh), ("v", KV, H, xh), ("o", H, H, xh),
              ("gate", I, H, xh), ("up", I, H, xh), ("down", H, I, xi)]
    if a.only:
        shapes = [t for t in shapes if t[0] in a.only.split(",")]
    ops = 2 * M * sum(n * k for _, n, k, _ in shapes)
    lib = L.load()
    tiled_in = {}
    for qa, k in ((xh, H), (xi, I)):
        t = torch.empty(lib.tb_gemm_act_bytes(M, k), dtype=torch.uint8, device="cuda")
        L.check(lib.tb_gemm_tile_act(qa.data.data_ptr(), M, qa.data.stride(0), k, t.data_ptr(),
                                     L.stream_ptr()))
        tiled_in[id(qa)] = t
    layers = []
    for c in range(a.copies):
        descs = (L.GemmDesc * len(shapes))()
        keep = []
        for d, (_, n, k, qa) in zip(descs, shapes):
            w = torch.randn(n, k, generator=g, device="cuda") * 0.02
            p = enc(tb.ternarize_weights(w, n, k))
            del w
            main, _ = p.tiled()
            out = torch.empty((M, n), dtype=torch.float32, device="cuda")
            d.tiled, d.rows, d.cols = main.data_ptr(), n, k
            d.act_tiled = tiled_in[id(qa)].data_ptr()
            d.a_scale, d.w_scale, d.out32 = qa.scales.data_ptr(), float(p.scale), out.data_ptr()
            keep.append((p, main, out))
        layers.append((descs, keep))
    s = L.stream_ptr()
    it = [0]

    def run():
        descs, _ = layers[it[0] % len(layers)]
        it[0] += 1
        L.check(lib.tb_gemm_batch(L.TL1 if a.fmt == "tl1" else L.I2S, len(shapes),
                                  C.cast(descs, C.c_void_p), M, s))

    us = events_us(run, 12)
    if os.environ.get("TRACE_EPI"):
        import numpy as np
        lib.tb_gemm_epi_trace_fetch.argtypes = [C.c_void_p, C.c_int64]
        run()
        torch.cuda.synchronize()
        buf = np.zeros((16, 3), dtype=np.int64)
        lib.tb_gemm_epi_trace_fetch(buf.ctypes.data_as(C.c_void_p), buf.nbytes)
        t0 = buf[0, 0]
        print("tile: decoders_done  tfull_ok  epilogue_done (clk since tile0 decode end)")
        for t in range(16):
            if buf[t, 0]:
                print(t, *(int(v - t0) for v in buf[t]))
    if os.environ.get("TRACE"):
        import numpy as np
        lib.tb_gemm_trace_fetch.argtypes = [C.c_void_p, C.c_int64]
        run()
        torch.cuda.synchronize()
        buf = np.zeros((64, 6), dtype=np.int64)
        lib.tb_gemm_trace_fetch(buf.ctypes.data_as(C.c_void_p), buf.nbytes)
        t0 = buf[0, 0]
        print("stage: p_empty_ok p_issued d_full d_ready m_start m_done (clk since stage0 issue)"
              if not os.environ.get("TRACE_DEC") else
              "stage: d_top d_full d_bempty d_ready m_start d_stored")
        for p in range(0, 64, 1):
            print(p, *(int(v - t0) for v in buf[p]))
    tops = ops / (us * 1e-6) / 1e12
    peak = int8_peak_tops() if not os.environ.get("NO_PEAK") else float("nan")
    print(f"prefill {a.fmt} M={M} [{','.join(t[0] for t in shapes)}]: {us:.1f} us per layer, {tops:.1f} int8 TOPS "
          f"({ops / 1e9:.1f} GOP); cuBLASLt int8 8192^3 peak {peak:.1f} TOPS -> {tops / peak:.3f}")


if __name__ == "__main__":
    main()
