"""Parity of every path bench.py times, at the shape it is timed at.

* cfg3: the whole prefill layer (q/k/v/o/gate/up/down, M=512, K up to 14336)
  through ONE grouped tb_gemm_batch launch -- once with int32 accumulators
  (SHA-pinned to the reference, tests/golden/large.json) and once with the
  bench's descriptor (fp32 outputs only, the 128-bit-store epilogue), within
  the north star's 1e-5 relative of the oracle's float64 make_result.
* cfg1: the TL1 FFN block exactly as the bench builds it (6 weight copies,
  one fused GemvStep per token, chained with programmatic dependent launch
  and captured in a CUDA graph); copy 0 holds the reference-pinned
  matrices, every step's outputs are checked.
* cfg2 (I2_S, TL2) and cfg4 (I2_S, M=1 and M=8): the full-size LayerStack the
  bench builds (seed, shapes, layer count), layers 0 and L-1 checked after a
  whole token pass against the C port of the reference kernels
  (oracle/c, pinned by tests/test_c_oracle.py).
"""

import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import c_oracle as CO
from oracle import ternpack_oracle as O
from workloads import LARGE_CASES, activations, latent_weights, sha

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).parent / "golden"
LARGE = json.loads((GOLD / "large.json").read_text())
STACK_SEED = 11  # bench.py


def host(t):
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module")
def tb():
    import paper_2410_16144_b200 as tb
    CO.build()
    return tb


# --------------------------------------------------------------------- cfg3

def test_cfg3_layer_gemm_batch(tb):
    from paper_2410_16144_b200 import _lib as L
    lib = L.load()
    case, gold = LARGE_CASES["cfg3"], LARGE["cfg3"]
    M = 512
    acts = {}
    for name, mm, k, seed in case["acts"]:
        qa = tb.quantize_tokens(torch.from_numpy(activations(seed, mm, k)).cuda(), pad_to=4)
        assert sha(host(qa.data)) == gold["acts"][name]["data_p4"]
        assert [float(s).hex() for s in host(qa.scales)] == gold["acts"][name]["scales"]
        til = torch.empty(lib.tb_gemm_act_bytes(M, k), dtype=torch.uint8, device="cuda")
        L.check(lib.tb_gemm_tile_act(qa.data.data_ptr(), M, qa.data.stride(0), k,
                                     til.data_ptr(), L.stream_ptr()), "tile")
        acts[name] = (qa, til)
    src = dict(case["gemv"])
    jobs = []
    for name, n, k, seed in case["matrices"]:
        m = tb.ternarize_weights(torch.from_numpy(latent_weights(seed, n, k)).cuda(), n, k)
        assert m.scale.hex() == gold["matrices"][name]["scale"]
        p = tb.encode_i2s(m)
        assert sha(host(p.data)) == gold["matrices"][name]["i2s"]
        main, _ = p.tiled()
        jobs.append((name, p, main, acts[src[name]]))

    def launch(kind):
        descs = (L.GemmDesc * len(jobs))()
        outs = []
        for d, (name, p, main, (qa, til)) in zip(descs, jobs):
            d.tiled, d.rows, d.cols, d.act_tiled = main.data_ptr(), p.rows, p.cols, til.data_ptr()
            d.a_scale, d.w_scale = qa.scales.data_ptr(), float(p.scale)
            dt = {"acc": torch.int32, "out32": torch.float32, "out64": torch.float64}[kind]
            o = torch.empty((M, p.rows), dtype=dt, device="cuda")
            setattr(d, {"acc": "acc_out"}.get(kind, kind), o.data_ptr())
            outs.append(o)
        L.check(lib.tb_gemm_batch(L.I2S, len(jobs), C.cast(descs, C.c_void_p), M,
                                  L.stream_ptr()), "gemm_batch")
        torch.cuda.synchronize()
        return [host(o) for o in outs]

    accs = launch("acc")
    for (name, *_), acc in zip(jobs, accs):
        assert sha(acc) == gold["gemv"][f"{name}:{src[name]}"]["acc"], name
    # the exact float64 chain (core.py:99-101); repeated: its slow epilogue is
    # where the staging rows (in the B slots) once raced the next tile's unpack
    for rep in range(4):
        out64 = launch("out64")
        for (name, *_), o in zip(jobs, out64):
            assert sha(o) == gold["gemv"][f"{name}:{src[name]}"]["out"], (name, rep)
    out32 = launch("out32")  # the bench's descriptor: fp32 outputs only
    for (name, p, main, (qa, til)), acc, o in zip(jobs, accs, out32):
        want = acc.astype(np.float64) * float(p.scale) * host(qa.scales)[:, None]
        np.testing.assert_allclose(o, want, rtol=1e-5, atol=0, err_msg=name)


def test_cfg3_fused_quantize_tile(tb):
    """The bench's per-layer activation path (quantise straight into the GEMM
    operand layout, one launch per input) writes the same bytes, scales and
    row sums as quantize_tokens + tb_gemm_tile_act."""
    from paper_2410_16144_b200 import _lib as L
    lib = L.load()
    if not hasattr(lib, "tb_gemm_quantize_act"):
        pytest.skip("no fused quantise-tile entry point")
    rng = np.random.default_rng(3)
    for M, K in ((512, 4096), (512, 14336), (200, 1000), (1, 64), (130, 4100), (40, 20000)):
        x = torch.from_numpy(rng.standard_normal((M, K)).astype(np.float32)).cuda()
        x[0, 5] = 0.0
        if M > 3:
            x[3] = 0.0
        qa = tb.quantize_tokens(x, pad_to=4)
        want = torch.empty(lib.tb_gemm_act_bytes(M, K), dtype=torch.uint8, device="cuda")
        L.check(lib.tb_gemm_tile_act(qa.data.data_ptr(), M, qa.data.stride(0), K,
                                     want.data_ptr(), L.stream_ptr()), "tile")
        got = torch.full_like(want, 0xAB)
        sc = torch.empty(M, dtype=torch.float64, device="cuda")
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        L.check(lib.tb_gemm_quantize_act(x.data_ptr(), M, K, K, sc.data_ptr(), flag.data_ptr(),
                                         got.data_ptr(), L.stream_ptr()), "quantize_act")
        torch.cuda.synchronize()
        # (the buffer's tail holds the quantiser's per-token reciprocal scales:
        # scratch that tb_gemm_tile_act does not write)
        mpad = 128 if M <= 128 else -(-M // 256) * 256
        n = want.numel() - 12 * mpad
        assert torch.equal(got[:n], want[:n]), (M, K)
        assert torch.equal(sc, qa.scales) and int(flag.item()) == 0
    x[1, 2] = float("inf")
    L.check(lib.tb_gemm_quantize_act(x.data_ptr(), M, K, K, sc.data_ptr(), flag.data_ptr(),
                                     got.data_ptr(), L.stream_ptr()), "quantize_act")
    torch.cuda.synchronize()
    assert int(flag.item()) == 1


def test_cfg3_grouped_quantize(tb):
    """tb_gemm_quantize_act_multi (a layer's two inputs in one launch pair, the
    bench's form) writes exactly what one call per input writes, including
    ragged shapes and the per-input non-finite flags."""
    from paper_2410_16144_b200 import _lib as L
    lib = L.load()
    rng = np.random.default_rng(8)
    for M, Ks in ((512, (4096, 14336)), (130, (1000, 64, 4100)), (1, (64,)), (9, (300, 17000))):
        xs = [torch.from_numpy(rng.standard_normal((M, K)).astype(np.float32)).cuda() for K in Ks]
        xs[-1][0, 1] = float("nan")
        want, got, scw, scg, fw, fg = [], [], [], [], [], []
        descs = (L.QactDesc * len(Ks))()
        for d, x, K in zip(descs, xs, Ks):
            nb = lib.tb_gemm_act_bytes(M, K)
            want.append(torch.full((nb,), 0xAB, dtype=torch.uint8, device="cuda"))
            got.append(torch.full((nb,), 0xAB, dtype=torch.uint8, device="cuda"))
            scw.append(torch.empty(M, dtype=torch.float64, device="cuda"))
            scg.append(torch.empty(M, dtype=torch.float64, device="cuda"))
            fw.append(torch.zeros(1, dtype=torch.int32, device="cuda"))
            fg.append(torch.zeros(1, dtype=torch.int32, device="cuda"))
            L.check(lib.tb_gemm_quantize_act(x.data_ptr(), M, K, K, scw[-1].data_ptr(),
                                             fw[-1].data_ptr(), want[-1].data_ptr(),
                                             L.stream_ptr()), "quantize_act")
            d.x, d.cols, d.ldx = x.data_ptr(), K, K
            d.scale, d.nonfinite_flag, d.act_tiled = (scg[-1].data_ptr(), fg[-1].data_ptr(),
                                                      got[-1].data_ptr())
        L.check(lib.tb_gemm_quantize_act_multi(len(Ks), C.cast(descs, C.c_void_p), M,
                                               L.stream_ptr()), "quantize_act_multi")
        torch.cuda.synchronize()
        mpad = 128 if M <= 128 else -(-M // 256) * 256
        for i in range(len(Ks)):
            n = want[i].numel() - 12 * mpad  # (the tail is the two-launch form's scratch)
            assert torch.equal(got[i][:n], want[i][:n]), (M, Ks[i])
            assert torch.equal(scg[i].view(torch.int64), scw[i].view(torch.int64))
            assert int(fg[i].item()) == int(fw[i].item()) == (1 if i == len(Ks) - 1 else 0)


# --------------------------------------------------------------------- cfg1

def test_cfg1_step_chain(tb):
    H, I = 4096, 14336
    gold = LARGE["cfg1"]
    ncopy, nx = 6, 8
    copies = []
    for c in range(ncopy):
        mats = {}
        for name, rows, cols, seed in LARGE_CASES["cfg1"]["matrices"]:
            if c == 0:  # the reference-pinned matrices
                w = torch.from_numpy(latent_weights(seed, rows, cols)).cuda()
            else:       # the bench's generator
                g = torch.Generator(device="cuda").manual_seed(1000 + c * 7 + len(mats))
                w = torch.randn(rows, cols, generator=g, device="cuda") * 0.02
            m = tb.ternarize_weights(w, rows, cols)
            del w
            mats[name] = tb.encode_tl1(m)
            if c == 0:
                assert sha(host(mats[name].data)) == gold["matrices"][name]["tl1"]
        pl = {k: tb.GemvPlan(v, out_dtype=torch.float32) for k, v in mats.items()}
        step = tb.GemvStep([(pl["gate"], 0), (pl["up"], 0), (pl["down"], 1)], [H, I])
        copies.append((mats, pl, step))
    xs = [torch.from_numpy(activations(13, 1, H)[0]).cuda(),
          torch.from_numpy(activations(14, 1, I)[0]).cuda()]
    g = torch.Generator(device="cuda").manual_seed(77)
    XH = torch.randn(nx, H, generator=g, device="cuda")
    XI = torch.randn(nx, I, generator=g, device="cuda")
    XH[0], XI[0] = xs  # step 0 sees the reference-pinned activations

    def run(j0, n):
        prev = None
        for j in range(j0, j0 + n):
            st = copies[j % ncopy][2]
            st.run([XH[j % nx], XI[j % nx]], prev=prev)
            prev = st
        prev.finalize()

    # eager, then the bench's form: a CUDA graph of the chain
    for form in ("eager", "graph"):
        if form == "eager":
            run(0, ncopy)
        else:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s), torch.cuda.graph(graph, stream=s):
                run(ncopy, ncopy)
            graph.replay()
        torch.cuda.synchronize()
        j0 = 0 if form == "eager" else ncopy
        for j in range(j0, j0 + ncopy):
            mats, pl, _ = copies[j % ncopy]
            xh, xi = host(XH[j % nx]), host(XI[j % nx])
            qh, sh = CO.quantize(xh, 2)
            qi, si = CO.quantize(xi, 2)
            for name, q, s_ in (("gate", qh, sh), ("up", qh, sh), ("down", qi, si)):
                acc = CO.gemv_tl1(host(mats[name].data), CO.lut_tl1(q, q.size // 2), 0)
                if j == 0:
                    src = "xh" if name != "down" else "xi"
                    assert sha(acc[None]) == gold["gemv"][f"{name}:{src}"]["acc"]
                want = O.make_output(acc, mats[name].scale, s_).astype(np.float32)
                assert np.array_equal(host(pl[name].out32[0]), want), (form, j, name)


# ---------------------------------------------------------- cfg2 / cfg4 stacks

def _planes(p, fmt):
    if fmt == "tl2":
        return host(p.index_data), host(p.sign_data)
    return (host(p.data),)


def _c_acc(fmt, planes, x, cols):
    if fmt == "i2s":
        q, s = CO.quantize(x, 4)
        return CO.gemv_i2s(planes[0], q, 0), s
    q, s = CO.quantize(x, 3)
    return CO.gemv_tl2(planes[0], planes[1], CO.lut_tl2(q, -(-cols // 6) * 2), 0), s


@pytest.mark.parametrize("name,fmt,tokens", [("cfg2", "i2s", 1), ("cfg2", "tl2", 1),
                                             ("cfg4", "i2s", 1), ("cfg4", "i2s", 8)])
def test_full_stack_layers(tb, name, fmt, tokens):
    from paper_2410_16144_b200.stack import STACKS, LayerStack
    cfg = STACKS[name]
    st = LayerStack(cfg, fmt=fmt, seed=STACK_SEED, tokens=tokens)
    L, h, i = st.nlayers, cfg["hidden"], cfg["inter"]
    g = torch.Generator(device="cuda").manual_seed(99)
    if tokens == 1:
        XH = torch.randn(L, h, generator=g, device="cuda")
        XI = torch.randn(L, i, generator=g, device="cuda")
        st.token_pass(list(XH), list(XI))
    else:
        XH = torch.randn(L, tokens, h, generator=g, device="cuda")
        XI = torch.randn(L, tokens, i, generator=g, device="cuda")
        st.token_pass(None, None, st.make_glues(XH, XI))
    torch.cuda.synchronize()
    for li in (0, L - 1):
        xs = [host(XH[li]).reshape(tokens, h), host(XI[li]).reshape(tokens, i)]
        for plan, (pname, rows, cols, src) in zip(st.layers[li], st.shapes):
            planes = _planes(plan.p, fmt)
            got = host(plan.out32)
            for t in range(tokens):
                acc, s = _c_acc(fmt, planes, xs[src][t], cols)
                want = O.make_output(acc, plan.p.scale, s).astype(np.float32)
                assert np.array_equal(got[t], want), (name, fmt, tokens, li, pname, t)
    del st
    torch.cuda.empty_cache()


def test_glue_refuses_scale_hazard(tb):
    """A glue that finalises a batch may not quantise into that batch's
    records: its finalize rows read the per-token scales the quantise rows
    overwrite (the M>1 stack alternates two record sets)."""
    from paper_2410_16144_b200 import _lib as L
    v = np.ones((64, 128), np.int8)
    plan = tb.GemvPlan(tb.encode_i2s(tb.TernaryMatrix(64, 128, v, 1.0)), max_tokens=2)
    rec, rec2 = tb.ActRecords(L.I2S, 2, 128), tb.ActRecords(L.I2S, 2, 128)
    batch = tb.GemvBatch([(plan, rec)])
    x = torch.ones(2, 128, device="cuda")
    with pytest.raises(ValueError, match="alternate two ActRecords sets"):
        tb.StepGlue([(x, rec)], finalize=batch)
    tb.StepGlue([(x, rec2)], finalize=batch)  # a different set is fine


def test_small_step_after_large(tb):
    """A small fused step (its grid sized down by the chunks-per-warp rule)
    finalises a LARGE previous step: the grid must still cover the previous
    outputs (the launch keeps enough threads), and both steps'
    outputs are exact."""
    rng = np.random.default_rng(12)
    H, I = 4096, 14336
    big = []
    for rows, cols in ((I, H), (H, I)):
        v = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
        big.append((tb.GemvPlan(tb.encode_i2s(tb.TernaryMatrix(rows, cols, v, 0.5)),
                                out_dtype=torch.float32), v))
    vs = rng.integers(-1, 2, size=(40, 256), dtype=np.int8)
    small = tb.GemvPlan(tb.encode_i2s(tb.TernaryMatrix(40, 256, vs, 0.25)), out_dtype=torch.float32)
    s_big = tb.GemvStep([(big[0][0], 0), (big[1][0], 1)], [H, I])
    s_small = tb.GemvStep([(small, 0)], [256])
    xh = rng.standard_normal(H).astype(np.float32)
    xi = rng.standard_normal(I).astype(np.float32)
    xs = rng.standard_normal(256).astype(np.float32)
    s_big.run([torch.from_numpy(xh).cuda(), torch.from_numpy(xi).cuda()])
    s_small.run([torch.from_numpy(xs).cuda()], prev=s_big)  # finalises the big step
    s_small.finalize()
    torch.cuda.synchronize()
    for (plan, v), x in zip(big, (xh, xi)):
        q, s = CO.quantize(x, 4)
        want = O.make_output(CO.gemv_i2s(O.encode_i2s(v), q, 0), 0.5, s).astype(np.float32)
        assert np.array_equal(host(plan.out32[0]), want)
    q, s = CO.quantize(xs, 4)
    want = O.make_output(CO.gemv_i2s(O.encode_i2s(vs), q, 0), 0.25, s).astype(np.float32)
    assert np.array_equal(host(small.out32[0]), want)


@pytest.mark.parametrize("fmt,M", [("i2s", 2), ("i2s", 3), ("tl1", 5), ("i2s", 8)])
def test_records_table_mode_windows(tb, fmt, M):
    """The M > 1 records-table GEMV (tb_gemv_batch_launch_inline): jobs on two
    record buffers, one matrix contracted as three ragged K-windows sharing a
    workspace (outputs on the first), ragged rows and K, and the previous
    batch finalised in the next launch's tail -- against the oracle."""
    from paper_2410_16144_b200 import _lib as L
    from paper_2410_16144_b200.stack import _windowed
    rng = np.random.default_rng(40 + M)
    enc = tb.encode_i2s if fmt == "i2s" else tb.encode_tl1
    K0, K1 = 1000, 2900  # ragged: neither a multiple of 256
    recs = [tb.ActRecords(L.I2S, M, K0), tb.ActRecords(L.I2S, M, K1)]
    batches, truth = [], []
    for b in range(2):
        jobs, tr = [], []
        for rows, src in ((70, 0), (33, 0), (300, 1)):
            v = rng.integers(-1, 2, size=(rows, (K0, K1)[src]), dtype=np.int8)
            p = enc(tb.TernaryMatrix(rows, v.shape[1], v, 0.5 + b))
            if src == 1:  # three K-windows (~16 chunks each), one workspace
                view, wj = _windowed(p, fmt, M, src, 16)
                jobs += [(pl, recs[src], c0) for pl, _, c0 in wj]
                tr.append((view, v, src))
            else:
                pl = tb.GemvPlan(p, max_tokens=M, out_dtype=torch.float32)
                jobs.append((pl, recs[src], 0))
                tr.append((pl, v, src))
        batches.append(tb.GemvBatch(jobs))
        truth.append(tr)
    assert len(batches[0].pairs) == 5
    xs = [torch.from_numpy(rng.standard_normal((M, k)).astype(np.float32)).cuda() for k in (K0, K1)]
    for r, x in zip(recs, xs):
        r.quantize(x)
    n0 = L.load().tb_gemv_table_launches()
    batches[0].run(finalize=False)
    batches[1].run(finalize=False, prev=batches[0])  # finalises batch 0 in its tail
    assert L.load().tb_gemv_table_launches() == n0 + 2  # the records-table kernel ran
    tb.StepGlue([]).retarget(batches[1]).run()       # and batch 1
    torch.cuda.synchronize()
    xh = [host(x) for x in xs]
    for b in range(2):
        for plan, v, src in truth[b]:
            got = host(plan.out32)
            for t in range(M):
                q, s, _ = O.quantize(xh[src][t], 1)
                want = O.make_output(O.gemv_ref_int32(v, q), plan.p.scale, s).astype(np.float32)
                assert np.array_equal(got[t], want), (fmt, M, b, v.shape, t)


@pytest.mark.parametrize("M", [2, 8])
def test_pipelined_layers(tb, M):
    """Pipelined M > 1 layers (tb_step_glue_sync / tb_gemv_batch_launch_sync:
    a layer's GEMV waits for its glue's records through counters, not for the
    previous GEMV) against the oracle and the serial chain: EVERY layer of a
    small stack (grids of a few CTAs, so many layers are resident at once),
    back-to-back token passes eagerly and as replays of one CUDA graph with
    fresh inputs; the counters are back at zero and no wait timed out."""
    from paper_2410_16144_b200 import _lib as L
    from paper_2410_16144_b200.stack import LayerStack
    cfg = {"hidden": 1024, "kv": 256, "inter": 3072, "layers": 6}
    nl, h, i = 6, 1024, 3072
    g = torch.Generator(device="cuda").manual_seed(7)
    XH = torch.randn(nl, M, h, generator=g, device="cuda")
    XI = torch.randn(nl, M, i, generator=g, device="cuda")
    serial = LayerStack(cfg, seed=5, tokens=M, pipelined=False)
    piped = LayerStack(cfg, seed=5, tokens=M, pipelined=True)
    assert piped.piped and not serial.piped
    sglues = serial.make_glues(XH, XI)
    glues = piped.make_glues(XH, XI)

    def oracle_check(st):
        for li in range(nl):
            xs = [host(XH[li]), host(XI[li])]
            for plan, (pname, rows, cols, src) in zip(st.layers[li], st.shapes):
                got = host(plan.out32)
                planes = _planes(plan.p, "i2s")
                for t in range(M):
                    acc, sc = _c_acc("i2s", planes, xs[src][t], cols)
                    want = O.make_output(acc, plan.p.scale, sc).astype(np.float32)
                    assert np.array_equal(got[t], want), (M, li, pname, t)

    serial.token_pass(None, None, sglues)
    for _ in range(3):
        piped.token_pass(None, None, glues)
    torch.cuda.synchronize()
    oracle_check(piped)
    oracle_check(serial)
    assert int(piped.sync.abs().sum().item()) == 0
    assert L.load().tb_sync_timeouts() == 0
    # graph replays (fresh inputs in the fixed buffers each time)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(gr, stream=s):
            piped.token_pass(None, None, glues)
            piped.token_pass(None, None, glues)
    for rep in range(3):
        XH.copy_(torch.randn(nl, M, h, generator=g, device="cuda"))
        XI.copy_(torch.randn(nl, M, i, generator=g, device="cuda"))
        for plans in piped.layers:
            for pl in plans:
                pl.out32.zero_()
        gr.replay()
        serial.token_pass(None, None, sglues)
        torch.cuda.synchronize()
        for li in range(nl):
            for a, b in zip(serial.layers[li], piped.layers[li]):
                assert torch.equal(a.out32, b.out32), (M, rep, li)
        assert int(piped.sync.abs().sum().item()) == 0
        assert L.load().tb_sync_timeouts() == 0
    oracle_check(piped)


def test_independent_steps(tb):
    """TB_STEP_INDEPENDENT: self-finalising launches that never wait for their
    predecessor (the cfg0 bench form), 60 launches over 20 ragged plans
    back to back, every output against the oracle."""
    rng = np.random.default_rng(77)
    plans, vals, steps = [], [], []
    for c in range(20):
        rows, cols = 100 + 37 * c, 1024 + 64 * (c % 5)
        v = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
        p = tb.GemvPlan(tb.encode_i2s(tb.TernaryMatrix(rows, cols, v, 0.25 + c)),
                        out_dtype=torch.float32)
        plans.append(p)
        vals.append(v)
        steps.append(tb.GemvStep([(p, 0)], [cols], independent=True))
    xs = [[torch.from_numpy(rng.standard_normal(v.shape[1]).astype(np.float32)).cuda()
           for v in vals] for _ in range(3)]
    for rep in range(3):
        for c in range(20):
            steps[c].run([xs[rep][c]])
        torch.cuda.synchronize()
        for c in range(20):
            q, sc, _ = O.quantize(host(xs[rep][c]), 1)
            want = O.make_output(O.gemv_ref_int32(vals[c], q), 0.25 + c, sc).astype(np.float32)
            assert np.array_equal(host(plans[c].out32[0]), want), (rep, c)
    with pytest.raises(ValueError):
        tb.GemvStep([(plans[0], 0)], [vals[0].shape[1]], independent=True, x_after_wait=True)
