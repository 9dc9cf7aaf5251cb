"""Out-of-bounds write checks with guard bands (compute-sanitizer is closed on
this GPU pool, so the kernels' global writes are checked directly): every
output / workspace / operand buffer a kernel writes is carved out of a larger
allocation whose guard bands before and after are filled with a pattern, and
the bands must be intact after the launches -- over ragged shapes (rows not
a multiple of the 32-row tile, K not a multiple of a chunk), every format,
M = 1 .. 16 decode, the fused step chain and the prefill GEMM."""

import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GUARD = 4096  # bytes each side
PAT = 0x5A


class Guarded:
    def __init__(self, n, dtype):
        es = torch.tensor([], dtype=dtype).element_size()
        self.raw = torch.full((2 * GUARD + n * es + 16,), PAT, dtype=torch.uint8, device="cuda")
        self.t = self.raw[GUARD:GUARD + n * es].view(dtype)
        assert self.t.data_ptr() % 16 == 0

    def intact(self):
        lo, hi = self.raw[:GUARD], self.raw[GUARD + self.t.numel() * self.t.element_size():]
        return bool((lo == PAT).all()) and bool((hi == PAT).all())


@pytest.fixture(scope="module")
def tb():
    import paper_2410_16144_b200 as tb
    return tb


def test_gemv_guards(tb):
    from paper_2410_16144_b200 import _lib as L
    lib = L.load()
    rng = np.random.default_rng(9)
    enc = {1: tb.encode_i2s, 2: tb.encode_tl1, 3: tb.encode_tl2}
    for fmt in (1, 2, 3):
        for rows, cols in ((33, 70), (100, 4100), (1, 1), (257, 193)):
            p = enc[fmt](tb.TernaryMatrix(rows, cols, rng.integers(-1, 2, (rows, cols),
                                                                     dtype=np.int8), 0.5))
            main, sign = p.tiled()
            for M in (1, 4, 16):
                pad = {1: 4, 2: 2, 3: 3}[fmt]
                qa = tb.quantize_tokens(rng.standard_normal((M, cols)).astype(np.float32), pad)
                acts = qa.data.reshape(M, -1)
                ws = Guarded(lib.tb_gemv_workspace_bytes(fmt, rows, cols) // 4, torch.int32)
                ws.t.zero_()
                acc = Guarded(M * rows, torch.int32)
                o64 = Guarded(M * rows, torch.float64)
                o32 = Guarded(M * rows, torch.float32)
                L.check(lib.tb_gemv(fmt, L.ptr(main), L.ptr(sign), rows, cols, L.ptr(acts), M,
                                    acts.stride(0), acts.shape[1], L.ptr(qa.scales), 0.5,
                                    L.ptr(ws.t), L.ptr(acc.t), L.ptr(o64.t), L.ptr(o32.t),
                                    L.stream_ptr()), "gemv")
                torch.cuda.synchronize()
                for g in (ws, acc, o64, o32):
                    assert g.intact(), (fmt, rows, cols, M)


def test_fused_step_chain_guards(tb):
    rng = np.random.default_rng(10)
    shapes = [((70, 1000), 0), ((33, 1000), 0), ((300, 97), 1), ((1, 97), 1)]
    for fmt, enc in ((1, tb.encode_i2s), (3, tb.encode_tl2)):
        steps, guards = [], []
        for _ in range(2):
            pairs = []
            for (rows, cols), src in shapes:
                v = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
                plan = tb.GemvPlan(enc(tb.TernaryMatrix(rows, cols, v, 1.0)),
                                   out_dtype=torch.float32)
                g = Guarded(rows, torch.float32)
                plan.out32 = g.t.view(1, rows)
                wsg = Guarded(plan.ws.numel(), torch.int32)
                wsg.t.zero_()
                plan.ws = wsg.t
                guards += [g, wsg]
                pairs.append((plan, src))
            steps.append(tb.GemvStep(pairs, [1000, 97]))
        xs = [torch.randn(1000, device="cuda"), torch.randn(97, device="cuda")]
        prev = None
        for j in range(5):
            steps[j % 2].run(xs, prev=prev)
            prev = steps[j % 2]
        prev.finalize()
        torch.cuda.synchronize()
        assert all(g.intact() for g in guards), fmt


def test_gemm_and_quantize_act_guards(tb):
    from paper_2410_16144_b200 import _lib as L
    lib = L.load()
    rng = np.random.default_rng(11)
    for M, rows, cols in ((130, 300, 4100), (512, 256, 1000), (1, 33, 64)):
        x = torch.from_numpy(rng.standard_normal((M, cols)).astype(np.float32)).cuda()
        til = Guarded(lib.tb_gemm_act_bytes(M, cols), torch.uint8)
        sc = Guarded(M, torch.float64)
        L.check(lib.tb_gemm_quantize_act(x.data_ptr(), M, cols, cols, L.ptr(sc.t), None,
                                         L.ptr(til.t), L.stream_ptr()), "quantize_act")
        v = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
        p = tb.encode_i2s(tb.TernaryMatrix(rows, cols, v, 1.0))
        main, _ = p.tiled()
        d = (L.GemmDesc * 1)()
        o32 = Guarded(M * rows, torch.float32)
        acc = Guarded(M * rows, torch.int32)
        d[0].tiled, d[0].rows, d[0].cols, d[0].act_tiled = main.data_ptr(), rows, cols, til.t.data_ptr()
        d[0].a_scale, d[0].w_scale = sc.t.data_ptr(), 1.0
        d[0].out32, d[0].acc_out = o32.t.data_ptr(), acc.t.data_ptr()
        L.check(lib.tb_gemm_batch(L.I2S, 1, C.cast(d, C.c_void_p), M, L.stream_ptr()), "gemm")
        torch.cuda.synchronize()
        for g in (til, sc, o32, acc):
            assert g.intact(), (M, rows, cols)
