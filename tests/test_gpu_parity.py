"""GPU parity: the CUDA path against the reference's golden fixtures and the oracle.

Bit-exact for int8 activations, float64 scales, packed bytes, int32
accumulators and float64 outputs; the fp32 output of the fused path is
checked against the float64 reference with rel. tolerance 1e-5 (north star).
"""

import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import ternpack_oracle as O  # noqa: E402
from workloads import LARGE_CASES, activations, latent_weights, sha  # noqa: E402

GOLD = Path(__file__).parent / "golden"
SMALL = np.load(GOLD / "small.npz")
LARGE = json.loads((GOLD / "large.json").read_text())


@pytest.fixture(scope="module")
def tb():
    import paper_2410_16144_b200 as tb
    return tb


def split(flat, offs):
    return [flat[offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]


def host(t):
    return t.detach().cpu().numpy()


# ----------------------------------------------------------------- core

def test_quantize_golden(tb):
    xs = split(SMALL["q_x"], SMALL["q_xoff"])
    for pad in (1, 2, 3, 4):
        want = split(SMALL[f"q_data_p{pad}"], SMALL[f"q_doff_p{pad}"])
        for x, d, s in zip(xs, want, SMALL[f"q_scale_p{pad}"]):
            qa = tb.quantize_activations(x, pad_to=pad)
            assert np.array_equal(host(qa.data), d)
            assert qa.scale == s
            assert len(qa) == d.size and qa.original_len == x.size


def test_quantize_batch_and_errors(tb):
    x = np.random.default_rng(5).standard_normal((7, 333)).astype(np.float32)
    qa = tb.quantize_tokens(x, pad_to=3)
    for i in range(7):
        d, s, _ = O.quantize(x[i], 3)
        assert np.array_equal(host(qa.data[i]), d) and host(qa.scales)[i] == s
    with pytest.raises(ValueError, match=r"pad_to must be in \{1, 2, 3, 4\}"):
        tb.quantize_activations([1.0], pad_to=5)
    with pytest.raises(ValueError, match="activations must be finite"):
        tb.quantize_activations([1.0, np.nan])
    with pytest.raises(ValueError, match="empty activation vector"):
        tb.quantize_activations(np.zeros(0))


def test_quantize_reference_shape_semantics(tb):
    """core.py:123 flattens ANY input to one vector with one scale: a (1, K)
    row and a (K, 1) column are one token, not K tokens."""
    x = np.random.default_rng(6).standard_normal(50).astype(np.float32)
    d, s, _ = O.quantize(x, 2)
    for shaped in (x.reshape(1, -1), x.reshape(-1, 1), x.reshape(5, 10)):
        qa = tb.quantize_activations(shaped, pad_to=2)
        assert qa.data.dim() == 1 and qa.tokens == 1
        assert np.array_equal(host(qa.data), d) and qa.scale == s


def test_quantize_scale_matches_device_for_every_dtype(tb):
    """The host fast path's scale (reference attribute) equals the device
    scales[0] for every accepted input dtype, incl. bf16, requires_grad and
    an int8 -128 (whose |x| must not wrap)."""
    rng = np.random.default_rng(9)
    base = rng.standard_normal(300)
    cases = [base.astype(np.float32), base, base.astype(np.float16),
             np.array([-128, 5, 3], dtype=np.int8), np.array([7, -3], dtype=np.int64),
             torch.from_numpy(base.astype(np.float32)).to(torch.bfloat16),
             torch.from_numpy(base.astype(np.float32)).requires_grad_(True)]
    for x in cases:
        qa = tb.quantize_activations(x, pad_to=4)
        ref = x.detach().to(torch.float64).numpy() if isinstance(x, torch.Tensor) else x
        d, s, _ = O.quantize(np.asarray(ref, dtype=np.float64), 4)
        assert qa.scale == float(host(qa.scales)[0]) == s, type(x)
        assert np.array_equal(host(qa.data), d)
    # check_finite=False: no sync at quantisation, the scale is read lazily
    qa = tb.quantize_activations(base, pad_to=1, check_finite=False)
    assert qa.scale == float(host(qa.scales)[0]) == O.quantize(base, 1)[1]


def test_records_quantizer_golden(tb):
    """The fused quantise->records kernel (the GEMV's hot input path) produces
    the reference's int8 codes and scales, and the same records as building
    them from the natural codes."""
    xs = split(SMALL["q_x"], SMALL["q_xoff"])
    want = split(SMALL["q_data_p4"], SMALL["q_doff_p4"])
    for fmt in (1, 2, 3):
        for x, d, s in zip(xs, want, SMALL["q_scale_p4"]):
            r = tb.ActRecords(fmt, 1, x.size, keep_natural_pad=4)
            r.quantize(torch.from_numpy(np.ascontiguousarray(x)).cuda().reshape(1, -1))
            assert np.array_equal(host(r.natural)[0], d)
            assert host(r.scales)[0] == s
            r2 = tb.ActRecords(fmt, 1, x.size).prep(r.natural)
            assert torch.equal(r.buf, r2.buf)


def test_ternarize_golden(tb):
    offs = np.cumsum([0] + [r * c for r, c in SMALL["t_shape"]])
    ws, qs = split(SMALL["t_w"], offs), split(SMALL["t_q"], offs)
    for w, q, (r, c), s in zip(ws, qs, SMALL["t_shape"], SMALL["t_scale"]):
        m = tb.ternarize_weights(w, int(r), int(c))
        assert m.scale == s and np.array_equal(host(m.values).ravel(), q)
    with pytest.raises(ValueError, match="degenerate weight matrix"):
        tb.ternarize_weights([0.0] * 4, 2, 2)
    with pytest.raises(ValueError, match="weights must be finite"):
        tb.ternarize_weights([1.0, np.inf], 1, 2)


def test_round_half_away(tb):
    got = host(tb.round_half_away(np.array([0.5, -0.5, 1.5, -1.5, 0.49, 2.5, -2.5])))
    assert got.tolist() == [1, -1, 2, -2, 0, 3, -3]


# -------------------------------------------------------------- packing

def _packing_cases():
    shapes = SMALL["p_shape"]
    vals = split(SMALL["p_vals"], np.cumsum([0] + [r * c for r, c in shapes]))
    return (shapes, vals, split(SMALL["p_i2s"], SMALL["p_i2s_off"]),
            split(SMALL["p_tl1"], SMALL["p_tl1_off"]), split(SMALL["p_tl2i"], SMALL["p_tl2i_off"]),
            split(SMALL["p_tl2s"], SMALL["p_tl2s_off"]))


def test_encode_decode_golden(tb):
    shapes, vals, i2s, tl1, tl2i, tl2s = _packing_cases()
    for k, (r, c) in enumerate(shapes):
        v = vals[k].reshape(r, c)
        m = tb.TernaryMatrix(int(r), int(c), v, 1.0)
        pi, p1, p2 = tb.encode_i2s(m), tb.encode_tl1(m), tb.encode_tl2(m)
        assert np.array_equal(host(pi.data).ravel(), i2s[k])
        assert np.array_equal(host(p1.data).ravel(), tl1[k])
        assert np.array_equal(host(p2.index_data).ravel(), tl2i[k])
        assert np.array_equal(host(p2.sign_data).ravel(), tl2s[k])
        for dec, p in ((tb.decode_i2s, pi), (tb.decode_tl1, p1), (tb.decode_tl2, p2)):
            assert np.array_equal(host(dec(p).values), v)


def test_tiled_repack_roundtrip(tb):
    from paper_2410_16144_b200 import _lib as L
    lib = L.load()
    shapes, vals, *_ = _packing_cases()
    for k, (r, c) in enumerate(shapes):
        m = tb.TernaryMatrix(int(r), int(c), vals[k].reshape(r, c), 1.0)
        for p in (tb.encode_i2s(m), tb.encode_tl1(m), tb.encode_tl2(m)):
            main, sign = p.tiled()
            ref = p._main_ref()
            back = torch.empty_like(ref)
            sref = p._sign_ref()
            sback = torch.empty_like(sref) if sref is not None else None
            L.check(lib.tb_unrepack(p.FMT, L.ptr(main), L.ptr(sign), p.rows, p.cols,
                                    L.ptr(back), L.ptr(sback), L.stream_ptr()))
            assert torch.equal(back, ref)
            if sref is not None:
                assert torch.equal(sback, sref)


def test_invalid_codes(tb):
    bad = tb.PackedI2S(rows=1, cols=4, padded_cols=4, data=np.array([[0xFF]], np.uint8), scale=1.0)
    with pytest.raises(ValueError, match="invalid I2_S code"):
        tb.decode_i2s(bad)
    with pytest.raises(ValueError, match="invalid I2_S code at row 0"):
        bad.validate()
    data = np.full((3, 1), 0x55, np.uint8)
    data[2, 0] = 0xC5
    with pytest.raises(ValueError, match="invalid I2_S code at row 2"):
        tb.PackedI2S(rows=3, cols=4, padded_cols=4, data=data, scale=1.0).validate()
    bad1 = tb.PackedTL1(rows=1, cols=4, padded_cols=4, data=np.array([[0xF5]], np.uint8), scale=1.0)
    with pytest.raises(ValueError, match="invalid TL1 index"):
        tb.decode_tl1(bad1)
    good2 = tb.encode_tl2(tb.TernaryMatrix(1, 6, np.array([[1, 1, 1, -1, -1, 0]]), 1.0))
    bad2 = tb.PackedTL2(rows=1, cols=6, padded_cols=6, index_data=np.array([[0xED]], np.uint8),
                        sign_data=host(good2.sign_data), scale=1.0)
    with pytest.raises(ValueError, match="invalid TL2 index"):
        tb.decode_tl2(bad2)
    nc = tb.PackedTL2(rows=1, cols=6, padded_cols=6, index_data=np.array([[0x00]], np.uint8),
                      sign_data=np.array([[0b01]], np.uint8), scale=1.0)
    with pytest.raises(ValueError, match="non-canonical zero"):
        tb.decode_tl2(nc)
    with pytest.raises(ValueError, match="non-canonical zero at row 0"):
        nc.validate()
    # untrusted containers are validated by the kernels (test_kernels.py:146-161)
    qa = tb.QuantizedActivations(data=np.array([1, 2, 3, 4], np.int8), scale=1.0, original_len=4)
    lut = tb.build_lut_tl1(qa)
    badk = tb.PackedTL1(rows=1, cols=4, padded_cols=4, data=np.array([[0xF0]], np.uint8), scale=1.0)
    with pytest.raises(ValueError, match="invalid TL1 index"):
        tb.gemv_tl1(badk, lut, qa.scale)
    with pytest.raises(ValueError, match="group-count mismatch"):
        p = tb.encode_tl1(tb.TernaryMatrix(1, 4, np.array([[1, -1, 0, 0]]), 1.0))
        qa2 = tb.QuantizedActivations(data=np.array([1, 2], np.int8), scale=1.0, original_len=2)
        tb.gemv_tl1(p, tb.build_lut_tl1(qa2), 1.0)


# ------------------------------------------------------------------ lut

def test_lut_golden(tb):
    xs = split(SMALL["l_x"], SMALL["l_xoff"])
    for x, extra, e1, e2 in zip(xs, SMALL["l_extra"], split(SMALL["l_tl1"], SMALL["l_tl1_off"]),
                                split(SMALL["l_tl2"], SMALL["l_tl2_off"])):
        q2 = tb_q(x, 2)
        q3 = tb_q(x, 3)
        l1 = TB.build_lut_tl1(q2, groups=len(q2) // 2 + int(extra))
        l2 = TB.build_lut_tl2(q3, groups=len(q3) // 3 + int(extra))
        assert np.array_equal(host(l1.entries).ravel(), e1)
        assert np.array_equal(host(l2.entries).ravel(), e2)


import paper_2410_16144_b200 as TB  # noqa: E402


def tb_q(x, pad):
    return TB.quantize_activations(x, pad_to=pad)


# -------------------------------------------------------------- kernels

def _cross_instances(n):
    shapes = SMALL["g_shape"]
    vals = split(SMALL["g_vals"], np.cumsum([0] + [r * c for r, c in shapes]))
    xs = split(SMALL["g_x"], SMALL["g_xoff"])
    accs = split(SMALL["g_acc"], SMALL["g_accoff"])
    outs = split(SMALL["g_out"], SMALL["g_accoff"])
    for k in range(n):
        r, c = shapes[k]
        yield (vals[k].reshape(r, c), float(SMALL["g_wscale"][k]), xs[k], accs[k], outs[k])


@pytest.mark.parametrize("lo,hi", [(0, 500), (500, 1000), (1000, 2000)])
def test_cross_kernel_golden(tb, lo, hi):
    K = tb.KernelKind
    for k, (v, ws, x, acc, out) in enumerate(_cross_instances(hi)):
        if k < lo:
            continue
        m = tb.TernaryMatrix(v.shape[0], v.shape[1], v, ws)
        packs = {K.I2_S: tb.encode_i2s(m), K.TL1: tb.encode_tl1(m), K.TL2: tb.encode_tl2(m)}
        for kind, p in packs.items():
            qa = tb.quantize_activations(x, pad_to=tb.KERNEL_PAD[kind])
            r = tb.gemv_parallel(kind, p, qa)
            assert np.array_equal(host(r.accumulators), acc), (k, kind)
            assert np.array_equal(host(r.output), out), (k, kind)
        r = tb.gemv_ref_int32(m, tb.quantize_activations(x, pad_to=1))
        assert np.array_equal(host(r.accumulators), acc)
        if k % 4 == 0:  # explicit-LUT kernels (verify.py:17-33 path)
            q2, q3 = tb.quantize_activations(x, pad_to=2), tb.quantize_activations(x, pad_to=3)
            r1 = tb.gemv_tl1(packs[K.TL1], tb.build_lut_tl1(q2, groups=packs[K.TL1].groups), q2.scale)
            r2 = tb.gemv_tl2(packs[K.TL2], tb.build_lut_tl2(q3, groups=packs[K.TL2].groups), q3.scale)
            assert np.array_equal(host(r1.accumulators), acc)
            assert np.array_equal(host(r2.accumulators), acc)
            assert np.array_equal(host(r1.output), out)


def test_kernel_kats(tb):
    K = tb.KernelKind
    m = tb.TernaryMatrix(1, 4, np.array([[1, -1, 0, 1]]), 1.0)
    qa = tb.QuantizedActivations(data=np.array([2, 3, -1, 4], np.int8), scale=1.0, original_len=4)
    assert host(tb.gemv_ref_int32(m, qa).accumulators).tolist() == [3]
    assert host(tb.gemv_parallel(K.I2_S, tb.encode_i2s(m), qa, thread_count=8).accumulators).tolist() == [3]
    with pytest.raises(ValueError, match="thread_count must be >= 1"):
        tb.gemv_parallel(K.I2_S, tb.encode_i2s(m), qa, thread_count=0)
    with pytest.raises(ValueError, match="dimension mismatch"):
        tb.gemv_ref_int32(tb.TernaryMatrix(1, 3, np.array([[1, -1, 0]]), 1.0),
                          tb.QuantizedActivations(data=np.array([1, 2], np.int8), scale=1.0,
                                                  original_len=2))
    with pytest.raises(ValueError, match="dimension mismatch"):
        tb.gemv_ref_int32(tb.TernaryMatrix(1, 1, np.array([[1]]), 1.0),
                          tb.QuantizedActivations(data=np.array([1, 2], np.int8), scale=1.0,
                                                  original_len=2))
    r = tb.gemv_ref_int32(tb.TernaryMatrix(1, 2, np.array([[1, 1]]), 0.5),
                          tb.QuantizedActivations(data=np.array([10, 20], np.int8), scale=0.25,
                                                  original_len=2))
    assert host(r.output)[0] == 30 * 0.5 * 0.25
    p = tb.encode_tl2(tb.TernaryMatrix(1, 3, np.array([[-1, -1, -1]]), 1.0))
    qa3 = tb.QuantizedActivations(data=np.array([1, 2, 3], np.int8), scale=1.0, original_len=3)
    assert host(tb.gemv_tl2(p, tb.build_lut_tl2(qa3, groups=p.groups), 1.0).accumulators).tolist() == [-6]
    out = host(tb.gemv_f32_ref(tb.TernaryMatrix(1, 3, np.array([[1, 0, -1]]), 1.0),
                               [0.5, 9.9, 0.25]).output)
    assert out[0] == pytest.approx(0.25)


def test_checked_paths_and_overflow(tb):
    for cols in (4092, 16384):
        v, a, acc = SMALL[f"ov_v{cols}"], SMALL[f"ov_a{cols}"], SMALL[f"ov_acc{cols}"]
        m = tb.TernaryMatrix(6, cols, v, 1.0)
        qa = tb.QuantizedActivations(data=a, scale=1.0, original_len=cols)
        assert np.array_equal(host(tb.gemv_i2s(tb.encode_i2s(m), qa).accumulators), acc)
        p1, p2 = tb.encode_tl1(m), tb.encode_tl2(m)
        l1 = tb.build_lut_tl1(qa, groups=p1.groups)
        l2 = tb.build_lut_tl2(qa, groups=p2.groups)
        for chk in (False, True):
            assert np.array_equal(host(tb.gemv_tl1(p1, l1, 1.0, checked=chk).accumulators), acc)
            assert np.array_equal(host(tb.gemv_tl2(p2, l2, 1.0, checked=chk).accumulators), acc)
        for kind, p in ((tb.KernelKind.TL1, p1), (tb.KernelKind.TL2, p2)):
            assert np.array_equal(host(tb.gemv_parallel(kind, p, qa).accumulators), acc)


def test_batched_tokens_match_single(tb):
    rng = np.random.default_rng(3)
    for rows, cols in ((70, 1000), (33, 4096), (5, 97)):
        v = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
        m = tb.TernaryMatrix(rows, cols, v, 0.7)
        x = rng.standard_normal((13, cols)).astype(np.float32)
        for kind, enc in ((tb.KernelKind.I2_S, tb.encode_i2s), (tb.KernelKind.TL1, tb.encode_tl1),
                          (tb.KernelKind.TL2, tb.encode_tl2)):
            p = enc(m)
            for M in (1, 2, 3, 5, 8, 13):
                qa = tb.quantize_tokens(x[:M], pad_to=tb.KERNEL_PAD[kind])
                r = tb.gemv_parallel(kind, p, qa)
                want = np.stack([O.gemv_ref_int32(v, O.quantize(x[i], 1)[0]) for i in range(M)])
                assert np.array_equal(host(r.accumulators), want), (kind, M)


def test_workspace_self_cleans(tb):
    rng = np.random.default_rng(4)
    v = rng.integers(-1, 2, size=(300, 2000), dtype=np.int8)
    p = tb.encode_tl2(tb.TernaryMatrix(300, 2000, v, 1.0))
    qa = tb.quantize_activations(rng.standard_normal(2000), pad_to=3)
    a1 = host(tb.gemv_parallel(tb.KernelKind.TL2, p, qa).accumulators)
    a2 = host(tb.gemv_parallel(tb.KernelKind.TL2, p, qa).accumulators)
    assert np.array_equal(a1, a2)
    T = -(-300 // 32)
    # accumulator + counter region is zero again (the record scratch after it is not)
    assert int(p.workspace()[: 16 * T * 32 + T].abs().sum()) == 0


def test_gemv_plan_fp32_output(tb):
    rng = np.random.default_rng(8)
    v = rng.integers(-1, 2, size=(1000, 4096), dtype=np.int8)
    m = tb.TernaryMatrix(1000, 4096, v, 0.0123)
    x = rng.standard_normal((4, 4096)).astype(np.float32)
    for enc, pad in ((tb.encode_i2s, 4), (tb.encode_tl1, 2), (tb.encode_tl2, 3)):
        plan = tb.GemvPlan(enc(m), max_tokens=4, out_dtype=torch.float32, want_acc=True)
        qa = tb.quantize_tokens(x, pad_to=pad)
        out = host(plan.run(qa.data, qa.scales)).astype(np.float64)
        for i in range(4):
            d, s, _ = O.quantize(x[i], 1)
            ref = O.make_output(O.gemv_ref_int32(v, d), 0.0123, s)
            np.testing.assert_allclose(out[i], ref, rtol=1e-5, atol=0)


def test_grouped_gemv_batch(tb):
    """Several GEMVs (different shapes, shared and separate inputs, M up to 5)
    in one launch -- including tiny matrices whose tiles straddle warp ranges."""
    rng = np.random.default_rng(12)
    for fmt, enc, pad in ((1, tb.encode_i2s, 4), (2, tb.encode_tl1, 2), (3, tb.encode_tl2, 3)):
        shapes = [(70, 1000), (33, 1000), (5, 97), (4096, 1000), (1, 1000), (300, 97)]
        M = 5 if fmt == 2 else 1
        xs = {k: rng.standard_normal((M, k)).astype(np.float32) for k in (1000, 97)}
        recs = {k: tb.ActRecords(fmt, M, k).quantize(torch.from_numpy(xs[k]).cuda()) for k in xs}
        pairs, want = [], []
        for rows, cols in shapes:
            v = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
            plan = tb.GemvPlan(enc(tb.TernaryMatrix(rows, cols, v, 0.3)), max_tokens=M,
                               out_dtype=torch.float64, want_acc=True)
            pairs.append((plan, recs[cols]))
            want.append(np.stack([O.gemv_ref_int32(v, O.quantize(xs[cols][i], 1)[0])
                                  for i in range(M)]))
        batch = tb.GemvBatch(pairs)
        for _ in range(2):  # twice: the workspaces must self-clean
            batch.run()
            for (plan, rec), w in zip(pairs, want):
                assert np.array_equal(host(plan.acc)[:M], w)
                s = host(rec.scales)
                np.testing.assert_array_equal(host(plan.out64)[:M], w * 0.3 * s[:, None])


def _tie_vector(rng, k):
    """Random f32 vector with amax 127 (scale 1) and exact / near rounding ties."""
    x = rng.standard_normal(k).astype(np.float32) * 20
    x[0] = 127.0
    ties = np.array([0.5, -0.5, 1.5, -2.5, 126.5, -126.5, np.nextafter(np.float32(0.5), 1),
                     np.nextafter(np.float32(0.5), 0), np.nextafter(np.float32(-2.5), 0)],
                    dtype=np.float32)
    x[1:1 + len(ties)] = ties[: max(0, min(len(ties), k - 1))]
    return x


def test_fused_step_sequence(tb):
    """One-launch decode steps (quantise + grouped GEMV + previous finalize),
    chained A -> B -> A with the last one finalised explicitly."""
    rng = np.random.default_rng(21)
    for fmt, enc in ((1, tb.encode_i2s), (2, tb.encode_tl1), (3, tb.encode_tl2)):
        k0, k1 = (1000, 97) if fmt != 1 else (1000, 100)
        shapes = [((70, k0), 0), ((33, k0), 0), ((300, k1), 1), ((4096, k0), 0), ((1, k1), 1)]
        steps, truth = [], []
        for sidx in range(2):
            pairs, vals = [], []
            for (rows, cols), src in shapes:
                v = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
                ws = 0.3 + 0.1 * sidx
                plan = tb.GemvPlan(enc(tb.TernaryMatrix(rows, cols, v, ws)),
                                   out_dtype=torch.float64, want_acc=True)
                pairs.append((plan, src))
                vals.append((v, ws))
            steps.append(tb.GemvStep(pairs, [k0, k1]))
            truth.append(vals)
        xs_host = [[_tie_vector(rng, k0), rng.standard_normal(k1).astype(np.float32)]
                   for _ in range(3)]
        xs_dev = [[torch.from_numpy(x).cuda() for x in xs] for xs in xs_host]

        def check(si, xi):
            st = steps[si]
            q = [O.quantize(x, 1) for x in xs_host[xi]]
            np.testing.assert_array_equal(host(st.scales), [q[0][1], q[1][1]])
            for (plan, src, _), (v, ws) in zip(st.pairs, truth[si]):
                want = O.gemv_ref_int32(v, q[src][0])
                assert np.array_equal(host(plan.acc)[0], want), (fmt, si, v.shape)
                np.testing.assert_array_equal(host(plan.out64)[0],
                                              want.astype(np.float64) * ws * q[src][1])

        steps[0].run(xs_dev[0])
        steps[1].run(xs_dev[1], prev=steps[0])
        torch.cuda.synchronize()
        check(0, 0)
        steps[0].run(xs_dev[2], prev=steps[1])
        torch.cuda.synchronize()
        check(1, 1)
        steps[0].finalize()
        torch.cuda.synchronize()
        check(0, 2)
        assert int(host(steps[0].flags).sum()) == 0
        with pytest.raises(ValueError):
            steps[0].run(xs_dev[0], prev=steps[0])


def test_fused_step_segments_and_clusters(tb):
    """Fused steps over the full grid (CTA pairs sharing the quantisation
    through DSMEM) with per-input warp segments, and with more input runs
    than segments (one segment: CTAs quantise several inputs), chained."""
    rng = np.random.default_rng(29)
    k0, k1 = 1024, 2048
    for fmt, enc in ((1, tb.encode_i2s), (2, tb.encode_tl1)):
        for srcs in ((0, 1), (0, 1, 0, 1, 0)):
            steps, truth = [], []
            for sidx in range(2):
                pairs, vals = [], []
                for j, src in enumerate(srcs):
                    rows, cols = (4096 if len(srcs) == 2 else 1536), (k0, k1)[src]
                    v = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
                    ws = 0.25 + 0.05 * j + 0.1 * sidx
                    plan = tb.GemvPlan(enc(tb.TernaryMatrix(rows, cols, v, ws)),
                                       out_dtype=torch.float64, want_acc=True)
                    pairs.append((plan, src))
                    vals.append((v, ws))
                steps.append(tb.GemvStep(pairs, [k0, k1]))
                truth.append(vals)
            xs_host = [[_tie_vector(rng, k0), rng.standard_normal(k1).astype(np.float32)]
                       for _ in range(3)]
            xs_dev = [[torch.from_numpy(x).cuda() for x in xs] for xs in xs_host]

            def check(si, xi):
                q = [O.quantize(x, 1) for x in xs_host[xi]]
                for (plan, src, _), (v, ws) in zip(steps[si].pairs, truth[si]):
                    want = O.gemv_ref_int32(v, q[src][0])
                    assert np.array_equal(host(plan.acc)[0], want), (fmt, srcs, si)
                    np.testing.assert_array_equal(host(plan.out64)[0],
                                                  want.astype(np.float64) * ws * q[src][1])

            steps[0].run(xs_dev[0])
            steps[1].run(xs_dev[1], prev=steps[0])
            steps[0].run(xs_dev[2], prev=steps[1])
            torch.cuda.synchronize()
            check(1, 1)
            steps[0].finalize()
            torch.cuda.synchronize()
            check(0, 2)


def test_host_pipeline_block_ramps(tb):
    """HostPipeline over step counts that exercise the copy-block ramps
    (1 step, a partial ramp, ramp + full blocks + ramp down)."""
    rng = np.random.default_rng(41)
    v0 = rng.integers(-1, 2, size=(256, 512), dtype=np.int8)
    v1 = rng.integers(-1, 2, size=(64, 768), dtype=np.int8)
    plans = [tb.GemvPlan(tb.encode_i2s(tb.TernaryMatrix(256, 512, v0, 0.5))),
             tb.GemvPlan(tb.encode_i2s(tb.TernaryMatrix(64, 768, v1, 0.25)))]
    pairs = [(plans[0], 0), (plans[1], 1)]
    for T in (1, 5, 70):
        pipe = tb.HostPipeline([pairs, pairs], [512, 768], steps=T, block=8)
        xs0 = rng.standard_normal((T, 512)).astype(np.float32)
        xs1 = rng.standard_normal((T, 768)).astype(np.float32)
        pipe.inputs[0].copy_(torch.from_numpy(xs0))
        pipe.inputs[1].copy_(torch.from_numpy(xs1))
        for _ in range(2):  # the ready flags re-arm between runs
            outs = pipe.run()
            for i in range(T):
                (q0, s0, _), (q1, s1, _) = O.quantize(xs0[i], 1), O.quantize(xs1[i], 1)
                w0 = (O.gemv_ref_int32(v0, q0).astype(np.float64) * 0.5 * s0).astype(np.float32)
                w1 = (O.gemv_ref_int32(v1, q1).astype(np.float64) * 0.25 * s1).astype(np.float32)
                np.testing.assert_array_equal(outs[0][i].numpy(), w0, err_msg=f"T={T} i={i}")
                np.testing.assert_array_equal(outs[1][i].numpy(), w1, err_msg=f"T={T} i={i}")


def test_fused_step_large_input(tb):
    """Inputs too large for the register-held quantiser take the looped path."""
    rng = np.random.default_rng(5)
    for enc in (tb.encode_i2s, tb.encode_tl1, tb.encode_tl2):
        k = 30001
        v = rng.integers(-1, 2, size=(45, k), dtype=np.int8)
        plan = tb.GemvPlan(enc(tb.TernaryMatrix(45, k, v, 0.5)), out_dtype=torch.float64,
                           want_acc=True)
        st = tb.GemvStep([(plan, 0)], [k])
        x = _tie_vector(rng, k)
        x[17] = 3e-3  # a tiny magnitude as well
        st.run([torch.from_numpy(x).cuda()])
        st.finalize()
        torch.cuda.synchronize()
        q, s, _ = O.quantize(x, 1)
        want = O.gemv_ref_int32(v, q)
        assert host(st.scales)[0] == s
        assert np.array_equal(host(plan.acc)[0], want)
        np.testing.assert_array_equal(host(plan.out64)[0], want.astype(np.float64) * 0.5 * s)


def test_tp_shards_through_kernels(tb):
    """Row-parallel K-slices (byte slices of the reference planes) through the
    CUDA GEMV: the int32 partials sum to the unsharded result (what the NCCL
    all-reduce computes across ranks); column shards concatenate to it."""
    from paper_2410_16144_b200 import tp
    rng = np.random.default_rng(8)
    rows, cols = 300, 2000
    v = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    x = rng.standard_normal(cols).astype(np.float32)
    q, s, _ = O.quantize(x, 1)
    want = O.gemv_ref_int32(v, q)
    K = tb.KernelKind
    for name, enc, kind in (("i2s", tb.encode_i2s, K.I2_S), ("tl1", tb.encode_tl1, K.TL1),
                            ("tl2", tb.encode_tl2, K.TL2)):
        full = enc(tb.TernaryMatrix(rows, cols, v, 1.0))
        planes = (full.index_data, full.sign_data) if name == "tl2" else (full.data,)
        cls = type(full)
        for world in (2, 4):
            total = np.zeros(rows, dtype=np.int64)
            for r in range(world):
                k0, k1 = tp.shard_range(cols, world, r, tp.K_ALIGN[full.FMT])
                sp, sc = tp.row_shard(name, planes, cols, k0, k1)
                pc = -(-sc // {1: 4, 2: 2, 3: 6}[full.FMT]) * {1: 4, 2: 2, 3: 6}[full.FMT]
                if name == "tl2":
                    shard = cls(rows=rows, cols=sc, padded_cols=pc, index_data=sp[0].contiguous(),
                                sign_data=sp[1].contiguous(), scale=1.0)
                else:
                    shard = cls(rows=rows, cols=sc, padded_cols=pc, data=sp[0].contiguous(),
                                scale=1.0)
                # the shard's activations are the full vector's codes (one scale)
                qa = tb.QuantizedActivations(data=torch.from_numpy(q[k0:k1]).cuda(), scale=s,
                                             original_len=k1 - k0)
                total += host(tb.gemv_parallel(kind, shard, qa).accumulators).astype(np.int64)
            assert np.array_equal(total, want), (name, world)
            r0, r1 = tp.shard_range(rows, world, 1)
            cs = tp.column_shard(planes, r0, r1)
            if name == "tl2":
                shard = cls(rows=r1 - r0, cols=cols, padded_cols=full.padded_cols,
                            index_data=cs[0].contiguous(), sign_data=cs[1].contiguous(), scale=1.0)
            else:
                shard = cls(rows=r1 - r0, cols=cols, padded_cols=full.padded_cols,
                            data=cs[0].contiguous(), scale=1.0)
            qa = tb.QuantizedActivations(data=torch.from_numpy(q).cuda(), scale=s,
                                         original_len=cols)
            assert np.array_equal(host(tb.gemv_parallel(kind, shard, qa).accumulators),
                                  want[r0:r1])


@pytest.mark.parametrize("M,rows,cols", [(1, 130, 256), (64, 128, 128), (128, 256, 512),
                                         (200, 300, 1000), (512, 129, 4096), (700, 64, 192)])
def test_prefill_gemm_tensor_cores(tb, M, rows, cols):
    """tcgen05 kind::i8 GEMM: every token's row equals the reference GEMV of
    that token (exact int32, f64 outputs), I2_S and TL1, ragged M/N/K."""
    rng = np.random.default_rng(M * 7 + rows)
    v = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    x = rng.standard_normal((M, cols)).astype(np.float32)
    x[0, : min(cols, 4)] = [127.0, -0.5, 0.5, 2.5][: min(cols, 4)]
    qa = tb.quantize_tokens(torch.from_numpy(x).cuda())
    q = host(qa.data.reshape(M, -1))
    scales = host(qa.scales)
    want = np.stack([O.gemv_ref_int32(v, q[m]) for m in range(M)])
    for enc in (tb.encode_i2s, tb.encode_tl1):
        p = enc(tb.TernaryMatrix(rows, cols, v, 0.75))
        r = tb.gemm_prefill(p, qa)
        acc = host(r.accumulators).reshape(M, rows)
        assert np.array_equal(acc, want), (enc.__name__, M, rows, cols)
        np.testing.assert_array_equal(host(r.output).reshape(M, rows),
                                      want.astype(np.float64) * 0.75 * scales[:, None])


def test_prefill_gemm_batch_grouped(tb):
    """One launch over several projections with two inputs (a layer's q/k/v/o/
    gate/up on x_h, down on x_i), through the C ABI."""
    from paper_2410_16144_b200 import _lib as L
    import ctypes as C
    lib = L.load()
    rng = np.random.default_rng(3)
    M, H, I = 256, 512, 1024
    xh = tb.quantize_tokens(torch.from_numpy(rng.standard_normal((M, H)).astype(np.float32)).cuda())
    xi = tb.quantize_tokens(torch.from_numpy(rng.standard_normal((M, I)).astype(np.float32)).cuda())
    shapes = [(H, H, xh), (128, H, xh), (128, H, xh), (H, H, xh), (I, H, xh), (I, H, xh), (H, I, xi)]
    descs = (L.GemmDesc * len(shapes))()
    keep, wants = [], []
    tiled_in = {}
    for qa, k in ((xh, H), (xi, I)):
        t = torch.empty(lib.tb_gemm_act_bytes(M, k), dtype=torch.uint8, device="cuda")
        L.check(lib.tb_gemm_tile_act(qa.data.data_ptr(), M, qa.data.stride(0), k, t.data_ptr(),
                                     L.stream_ptr()))
        tiled_in[id(qa)] = t
    for d, (n, k, qa) in zip(descs, shapes):
        v = rng.integers(-1, 2, size=(n, k), dtype=np.int8)
        p = tb.encode_i2s(tb.TernaryMatrix(n, k, v, 1.0))
        main, _ = p.tiled()
        acc = torch.empty((M, n), dtype=torch.int32, device="cuda")
        o32 = torch.empty((M, n), dtype=torch.float32, device="cuda")
        d.out32 = o32.data_ptr()  # fp32 outputs: within 1e-5 relative (north star)
        d.tiled, d.rows, d.cols = main.data_ptr(), n, k
        d.act_tiled = tiled_in[id(qa)].data_ptr()
        d.a_scale, d.w_scale, d.acc_out = qa.scales.data_ptr(), 1.0, acc.data_ptr()
        keep.append((p, main, acc, qa, o32))
        q = host(qa.data)
        wants.append(np.stack([O.gemv_ref_int32(v, q[m]) for m in range(M)]))
    L.check(lib.tb_gemm_batch(1, len(shapes), C.cast(descs, C.c_void_p), M, L.stream_ptr()))
    torch.cuda.synchronize()
    for (p, main, acc, qa, o32), want in zip(keep, wants):
        assert np.array_equal(host(acc), want)
        ref = want.astype(np.float64) * 1.0 * host(qa.scales)[:, None]
        np.testing.assert_allclose(host(o32), ref, rtol=1e-5, atol=0)


def test_host_step(tb):
    """Host-memory decode step (one graph: H2D, step, finalize, D2H)."""
    rng = np.random.default_rng(31)
    v0 = rng.integers(-1, 2, size=(200, 640), dtype=np.int8)
    v1 = rng.integers(-1, 2, size=(64, 300), dtype=np.int8)
    p0 = tb.GemvPlan(tb.encode_tl1(tb.TernaryMatrix(200, 640, v0, 0.25)), out_dtype=torch.float32)
    p1 = tb.GemvPlan(tb.encode_tl1(tb.TernaryMatrix(64, 300, v1, 0.5)), out_dtype=torch.float64)
    hs = tb.HostStep([(p0, 0), (p1, 1)], [640, 300])
    for _ in range(3):
        x0 = rng.standard_normal(640).astype(np.float32)
        x1 = rng.standard_normal(300).astype(np.float32)
        o0, o1 = hs([x0, x1])
        (q0, s0, _), (q1, s1, _) = O.quantize(x0, 1), O.quantize(x1, 1)
        w0 = O.gemv_ref_int32(v0, q0).astype(np.float64) * 0.25 * s0
        w1 = O.gemv_ref_int32(v1, q1).astype(np.float64) * 0.5 * s1
        np.testing.assert_array_equal(o0.numpy(), w0.astype(np.float32))
        np.testing.assert_array_equal(o1.numpy(), w1.astype(np.float32))
    bad = np.ones(640, np.float32)
    bad[3] = np.inf
    with pytest.raises(ValueError, match="activations must be finite"):
        hs([bad, x1])


def test_host_step_self_finalize(tb):
    """HostStep = copy-in kernel + a self-finalising step (the warp completing
    a row tile writes its outputs): every format, ragged rows, the cfg1 FFN
    shapes, consecutive tokens (the per-tile counters reset), a non-finite
    token in between."""
    rng = np.random.default_rng(41)
    enc = {"i2s": tb.encode_i2s, "tl1": tb.encode_tl1, "tl2": tb.encode_tl2}
    cases = [("i2s", [((300, 1000), 0), ((70, 200), 1)], [1000, 200]),
             ("tl2", [((33, 960), 0), ((257, 97), 1)], [960, 97]),
             ("tl1", [((14336, 4096), 0), ((14336, 4096), 0), ((4096, 14336), 1)], [4096, 14336])]
    for fmt, shapes, ks in cases:
        e = enc[fmt]
        vals, pairs = [], []
        for (rows, cols), src in shapes:
            v = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
            vals.append(v)
            pairs.append((tb.GemvPlan(e(tb.TernaryMatrix(rows, cols, v, 0.375)),
                                      out_dtype=torch.float32), src))
        hs = tb.HostStep(pairs, ks)
        for tok in range(4):
            xs = [rng.standard_normal(k).astype(np.float32) for k in ks]
            if tok == 2:
                bad = xs[0].copy()
                bad[5] = np.nan
                with pytest.raises(ValueError, match="activations must be finite"):
                    hs([bad, xs[1]])
            if tok == 3:  # the graph replays on the caller's current stream
                with torch.cuda.stream(torch.cuda.Stream()):
                    outs = hs(xs)
            else:
                outs = hs(xs)
            qs = [O.quantize(x, 1) for x in xs]
            for o, v, (_, src) in zip(outs, vals, shapes):
                q, sc, _ = qs[src]
                want = (O.gemv_ref_int32(v, q).astype(np.float64) * 0.375 * sc).astype(np.float32)
                np.testing.assert_array_equal(o.numpy(), want, err_msg=f"{fmt} token {tok}")


def test_host_pipeline(tb):
    """Independent steps streamed host -> device -> host on three streams."""
    rng = np.random.default_rng(37)
    v0 = rng.integers(-1, 2, size=(200, 640), dtype=np.int8)
    v1 = rng.integers(-1, 2, size=(64, 300), dtype=np.int8)
    v2 = rng.integers(-1, 2, size=(96, 640), dtype=np.int8)
    mats = [tb.TernaryMatrix(200, 640, v0, 0.25), tb.TernaryMatrix(64, 300, v1, 0.5),
            tb.TernaryMatrix(96, 640, v2, 0.125)]
    plans = [tb.GemvPlan(tb.encode_tl1(m)) for m in mats]
    pairs = [(plans[0], 0), (plans[1], 1), (plans[2], 0)]
    T = 7
    pipe = tb.HostPipeline([pairs, pairs, pairs], [640, 300], steps=T)
    for trial in range(2):
        xs0 = rng.standard_normal((T, 640)).astype(np.float32)
        xs1 = rng.standard_normal((T, 300)).astype(np.float32)
        pipe.inputs[0].copy_(torch.from_numpy(xs0))
        pipe.inputs[1].copy_(torch.from_numpy(xs1))
        outs = pipe.run()
        for i in range(T):
            (q0, s0, _), (q1, s1, _) = O.quantize(xs0[i], 1), O.quantize(xs1[i], 1)
            for j, (vals, ws, q, s_) in enumerate(((v0, 0.25, q0, s0), (v1, 0.5, q1, s1),
                                                   (v2, 0.125, q0, s0))):
                want = (O.gemv_ref_int32(vals, q).astype(np.float64) * ws * s_).astype(np.float32)
                np.testing.assert_array_equal(outs[j][i].numpy(), want, err_msg=f"{trial} {i} {j}")
    pipe.inputs[1][4, 7] = float("nan")
    with pytest.raises(ValueError, match="activations must be finite"):
        pipe.run()
    pipe.inputs[1][4, 7] = 0.0
    pipe.run()  # the verdict is per run


def test_fused_step_nonfinite_flag(tb):
    v = np.ones((40, 64), dtype=np.int8)
    plan = tb.GemvPlan(tb.encode_tl1(tb.TernaryMatrix(40, 64, v, 1.0)), out_dtype=torch.float64)
    st = tb.GemvStep([(plan, 0)], [64])
    x = torch.ones(64, device="cuda")
    x[5] = float("nan")
    st.run([x])
    st.finalize()
    torch.cuda.synchronize()
    assert int(host(st.flags)[0]) == 1


# ------------------------------------------------------- config-sized pins

def _run_large(tb, cname, formats=("i2s", "tl1", "tl2")):
    case, gold = LARGE_CASES[cname], LARGE[cname]
    K = tb.KernelKind
    kinds = {"i2s": (K.I2_S, tb.encode_i2s, 4), "tl1": (K.TL1, tb.encode_tl1, 2),
             "tl2": (K.TL2, tb.encode_tl2, 3)}
    mats = {}
    for name, n, k, seed in case["matrices"]:
        m = tb.ternarize_weights(torch.from_numpy(latent_weights(seed, n, k)), n, k)
        g = gold["matrices"][name]
        assert m.scale.hex() == g["scale"], (cname, name)
        packs = {}
        for f in formats:
            kind, enc, _ = kinds[f]
            p = enc(m)
            if f == "tl2":
                assert sha(host(p.index_data)) == g["tl2_index"]
                assert sha(host(p.sign_data)) == g["tl2_sign"]
            else:
                assert sha(host(p.data)) == g[f], (cname, name, f)
            packs[f] = p
        mats[name] = (m, packs)
    for name, mm, k, seed in case["acts"]:
        x = torch.from_numpy(activations(seed, mm, k))
        for pad in (1, 2, 3, 4):
            qa = tb.quantize_tokens(x, pad_to=pad)
            assert sha(host(qa.data)) == gold["acts"][name][f"data_p{pad}"]
            assert [float(s).hex() for s in host(qa.scales)] == gold["acts"][name]["scales"]
    for wname, aname in case["gemv"]:
        m, packs = mats[wname]
        mm, k, seed = [(a[1], a[2], a[3]) for a in case["acts"] if a[0] == aname][0]
        x = torch.from_numpy(activations(seed, mm, k))
        g = gold["gemv"][f"{wname}:{aname}"]
        for f, p in packs.items():
            kind, _, pad = kinds[f]
            qa = tb.quantize_tokens(x, pad_to=pad)
            r = tb.gemv_parallel(kind, p, qa)
            acc = host(r.accumulators).reshape(mm, -1)
            out = host(r.output).reshape(mm, -1)
            assert sha(acc) == g["acc"], (cname, wname, f)
            assert sha(out) == g["out"], (cname, wname, f)


def test_large_cfg0(tb):
    _run_large(tb, "cfg0")


def test_large_cfg1(tb):
    _run_large(tb, "cfg1")


def test_large_cfg2(tb):
    _run_large(tb, "cfg2", formats=("i2s", "tl2"))


def test_large_cfg3(tb):
    _run_large(tb, "cfg3", formats=("i2s",))


def test_large_cfg4(tb):
    _run_large(tb, "cfg4", formats=("i2s",))


# ----------------------------------------------- toy decoder

def test_toy_decoder_lossless_golden(tb):
    """runtime.ToyDecoder / decode_tokens on the GPU kernels reproduce the
    reference's token sequences (tests/golden, runtime.lossless_report
    protocol, seed 13) -- and, with the corrupted LUT, the reference's
    fault-injected sequences token for token."""
    from paper_2410_16144_b200 import runtime as R
    K = tb.KernelKind
    for i in range(3):
        d = R.ToyDecoder.build(seed=int(SMALL["d_seed"][i]))
        prompt = int(SMALL["d_prompt"][i])
        want = SMALL["d_tokens"][i].tolist()
        for k in (K.REF_INT32, K.I2_S, K.TL1, K.TL2):
            assert R.decode_tokens(d, k, prompt, 24) == want, k
        assert R.decode_tokens(d, K.TL1, prompt, 24, _lut_hook=R._corrupting_hook) == \
            SMALL["d_fault_tl1"][i].tolist()
        assert R.decode_tokens(d, K.TL2, prompt, 24, _lut_hook=R._corrupting_hook) == \
            SMALL["d_fault_tl2"][i].tolist()
    with pytest.raises(ValueError, match="steps must be >= 1"):
        R.decode_tokens(d, K.I2_S, 0, 0)
    with pytest.raises(ValueError, match="prompt token out of range"):
        R.decode_tokens(d, K.I2_S, 999, 1)


def test_lossless_report(tb):
    from paper_2410_16144_b200 import runtime as R
    acc = R.lossless_report(trials=2, max_steps=6, seed=3)
    assert all(v == 1.0 for v in acc.values())
    table = R.format_lossless_table(acc)
    assert "I2_S" in table and "100.0%" in table
    with pytest.raises(ValueError, match="trials must be >= 1"):
        R.lossless_report(trials=0, max_steps=1)


# ----------------------------------------------------- TPK1

def test_tpk_load_to_device_and_write(tb, tmp_path):
    """Reference-written TPK1 files load straight into validated, tiled device
    matrices whose GEMV equals the oracle, and write back byte-identically."""
    from paper_2410_16144_b200 import container as Ct
    gold = json.loads((GOLD / "tpk_golden.json").read_text())
    rng = np.random.default_rng(4)
    for fmt, blob in gold["files"].items():
        path = tmp_path / f"m_{fmt}.tpk"
        path.write_bytes(bytes.fromhex(blob))
        got_fmt, mats = Ct.load_model(path)
        assert got_fmt == fmt
        for (name, p), m in zip(mats, gold["matrices"]):
            v = np.array(m["values"], dtype=np.int8).reshape(m["rows"], m["cols"])
            x = rng.standard_normal(m["cols"]).astype(np.float32)
            q, s, _ = O.quantize(x, 1)
            kind = {"i2s": tb.KernelKind.I2_S, "tl1": tb.KernelKind.TL1,
                    "tl2": tb.KernelKind.TL2}[fmt]
            pad = {"i2s": 4, "tl1": 2, "tl2": 3}[fmt]
            r = tb.gemv_parallel(kind, p, tb.quantize_activations(x, pad_to=pad))
            assert np.array_equal(host(r.accumulators), O.gemv_ref_int32(v, q)), (fmt, name)
        out = tmp_path / f"w_{fmt}.tpk"
        Ct.write_model(out, mats)
        assert out.read_bytes() == bytes.fromhex(blob)
    # content validation happens on the device with the reference's message
    bad = bytearray(bytes.fromhex(gold["files"]["i2s"]))
    bad[-1] = 0xFF  # last payload byte of the last matrix: code 0b11
    path = tmp_path / "bad.tpk"
    path.write_bytes(bytes(bad))
    with pytest.raises(ValueError, match=r"invalid I2_S code at row 6"):
        Ct.load_model(path)


def test_layer_stack_small(tb):
    """Stack runner on a small config: every layer's projections equal the
    oracle for that layer's inputs (M=1 fused steps and the M=3 glue path)."""
    from paper_2410_16144_b200.stack import LayerStack
    cfg = {"hidden": 192, "kv": 64, "inter": 320, "layers": 3}
    for fmt, tokens in (("i2s", 1), ("tl2", 1), ("i2s", 3)):
        st = LayerStack(cfg, fmt=fmt, seed=2, tokens=tokens)
        g = torch.Generator(device="cuda").manual_seed(8)
        if tokens == 1:
            XH = torch.randn(3, 192, generator=g, device="cuda")
            XI = torch.randn(3, 320, generator=g, device="cuda")
            # run layer by layer so every layer's outputs can be checked
            for li, step in enumerate(st.steps):
                step.run([XH[li], XI[li]])
                step.finalize()
                torch.cuda.synchronize()
                xs = [host(XH[li]), host(XI[li])]
                for plan, (_, rows, cols, src) in zip(st.layers[li], st.shapes):
                    v = host(tb.decode_i2s(plan.p).values) if fmt == "i2s" else \
                        host(tb.decode_tl2(plan.p).values)
                    q, s, _ = O.quantize(xs[src], 1)
                    want = O.gemv_ref_int32(v, q).astype(np.float64) * plan.p.scale * s
                    np.testing.assert_array_equal(host(plan.out32[0]), want.astype(np.float32))
        else:
            XH = torch.randn(3, tokens, 192, generator=g, device="cuda")
            XI = torch.randn(3, tokens, 320, generator=g, device="cuda")
            glues = st.make_glues(XH, XI)
            st.token_pass(None, None, glues)
            torch.cuda.synchronize()
            li = 2  # outputs of the last layer are finalised at the end of the pass
            for plan, (_, rows, cols, src) in zip(st.layers[li], st.shapes):
                v = host(tb.decode_i2s(plan.p).values)
                x = host(XH[li] if src == 0 else XI[li])
                for m in range(tokens):
                    q, s, _ = O.quantize(x[m], 1)
                    want = O.gemv_ref_int32(v, q).astype(np.float64) * plan.p.scale * s
                    np.testing.assert_array_equal(host(plan.out32[m]), want.astype(np.float32))


# ----------------------------------------- verify / bench / CLI (8(f) 3-4)

def test_cli_gpu_commands(tb, tmp_path, capsys):
    from paper_2410_16144_b200 import cli
    rng = np.random.default_rng(0)
    raw = tmp_path / "w.bin"
    raw.write_bytes(rng.standard_normal(24 * 40).astype("<f4").tobytes())
    for fmt in ("i2s", "tl1", "tl2"):
        out = tmp_path / f"{fmt}.tpk"
        assert cli.main(["pack", str(raw), str(out), "--rows", "24", "--cols", "40",
                         "--format", fmt]) == 0
        assert cli.main(["verify", str(out), "--vectors", "3", "--decoder-trials", "1",
                         "--steps", "4"]) == 0
        assert "100% exact (3/3 GEMVs)" in capsys.readouterr().out
    gold = json.loads((GOLD / "tpk_golden.json").read_text())
    bad = bytearray(bytes.fromhex(gold["files"]["i2s"]))
    bad[-1] = 0xFF
    (tmp_path / "bad.tpk").write_bytes(bytes(bad))
    assert cli.main(["verify", str(tmp_path / "bad.tpk"), "--decoder-trials", "1"]) == 1
    assert "invalid I2_S code at matrix 2 row 6" in capsys.readouterr().err
    assert cli.main(["verify", "--random", "24", "--decoder-trials", "1", "--steps", "3"]) == 0
    assert "cross-kernel exactness (24 instances): I2S 100% TL1 100% TL2 100%" in \
        capsys.readouterr().out
    assert cli.main(["verify", "--random", "8", "--decoder-trials", "4", "--steps", "8",
                     "--fault-inject"]) == 1  # the harness detects the corrupted LUT
    jl = tmp_path / "b.jsonl"
    assert cli.main(["bench", "--config", "125M", "--tokens", "2", "--reps", "1",
                     "--out", str(jl)]) == 0
    out = capsys.readouterr().out
    assert "GEMV-only token proxy" in out and "i2s" in out and "(" in out
    recs = [json.loads(l) for l in jl.read_text().splitlines()]
    assert {r["kernel"] for r in recs} == {"ref_f32", "i2s", "tl1", "tl2"}
    assert all(r["tokens_per_sec"] > 0 for r in recs)
