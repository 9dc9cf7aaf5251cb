"""Pin the CPU oracle to the reference: known-answer tests + golden fixtures.

The known answers are the ones the reference's own suite asserts
(pkg/tests/test_core.py, test_packing.py, test_lut.py, test_kernels.py,
test_acceptance.py); the fixtures in tests/golden/ were produced by running
the reference itself (tests/golden/make_golden.py).
"""

import itertools
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import ternpack_oracle as O
from workloads import LARGE_CASES, activations, latent_weights, sha

GOLD = Path(__file__).parent / "golden"
SMALL = np.load(GOLD / "small.npz")
LARGE = json.loads((GOLD / "large.json").read_text())


def split(flat, offs):
    return [flat[offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]


# ---------------------------------------------------------------- KATs (core)

def test_round_half_away_kat():                     # test_core.py:15-21
    assert O.round_half_away(0.5) == 1 and O.round_half_away(-0.5) == -1
    assert O.round_half_away(1.5) == 2 and O.round_half_away(-1.5) == -2
    assert O.round_half_away(0.49) == 0
    assert O.round_half_away(np.array([2.5, -2.5])).tolist() == [3, -3]


def test_ternarize_kat():                            # test_core.py:25-49
    with pytest.raises(ValueError, match="degenerate weight matrix"):
        O.ternarize([0, 0, 0, 0], 2, 2)
    q, s = O.ternarize([1.0, -1.0, 1.0, -1.0], 2, 2)
    assert s == 1.0 and q.ravel().tolist() == [1, -1, 1, -1]
    q, s = O.ternarize([0.9, -0.1, 0.05, -0.85], 2, 2)
    assert s == pytest.approx(0.475) and q.ravel().tolist() == [1, 0, 0, -1]
    with pytest.raises(ValueError):
        O.ternarize([1.0, np.inf], 1, 2)


def test_quantize_kat():                             # test_core.py:53-71
    d, s, n = O.quantize([0, 0, 0], 2)
    assert d.tolist() == [0, 0, 0, 0] and s == 1.0 and n == 3
    d, s, _ = O.quantize([0.5, -1.0, 0.25], 3)
    assert s == pytest.approx(1 / 127) and d.tolist() == [64, -127, 32]
    d, s, _ = O.quantize([127.0], 4)
    assert d.tolist() == [127, 0, 0, 0] and s == 1.0
    with pytest.raises(ValueError, match=r"pad_to must be in \{1, 2, 3, 4\}"):
        O.quantize([1.0], 5)


# ------------------------------------------------------------ KATs (packing)

def test_code_tables_kat():                          # test_packing.py:39-84
    expected = {(-1, -1): 0, (-1, 0): 1, (-1, 1): 2, (0, -1): 3, (0, 0): 4,
                (0, 1): 5, (1, -1): 6, (1, 0): 7, (1, 1): 8}
    for pair, idx in expected.items():
        assert O.tl1_index(*pair) == idx
    assert O.tl2_code(-1, -1, -1) == (1, 0b1101)
    assert O.tl2_code(-1, 0, -1) == (1, 0b1010)
    assert O.tl2_code(0, 0, 0) == (0, 0)
    assert O.tl2_code(1, 1, -1) == (0, 0b1011)
    codes = {O.tl2_code(*t) for t in itertools.product((-1, 0, 1), repeat=3)}
    assert codes == {(0, 0)} | {(s, i) for s in (0, 1) for i in range(1, 14)}


def test_byte_layout_kat():                          # test_packing.py:93-150
    assert O.encode_i2s([[-1, 0, 1, 0]])[0, 0] == 0x64
    assert O.encode_i2s([[1]])[0, 0] == 0x56
    assert O.decode_i2s(np.array([[0x64]], np.uint8), 4).ravel().tolist() == [-1, 0, 1, 0]
    with pytest.raises(ValueError, match="invalid I2_S code at row 0"):
        O.validate_i2s(np.array([[0xFF]], np.uint8))
    assert O.encode_tl1([[0, 1, 1, -1]])[0, 0] == 0x65
    with pytest.raises(ValueError, match="invalid TL1 index"):
        O.decode_tl1(np.array([[0xF5]], np.uint8), 4)
    assert O.decode_tl1(O.encode_tl1([[1, -1, 0]]), 3).ravel().tolist() == [1, -1, 0]
    ip, sp = O.encode_tl2([[1, 1, 1, -1, -1, 0]])
    assert ip[0, 0] == 0xCD and sp[0, 0] == 0b10
    with pytest.raises(ValueError, match="invalid TL2 index"):
        O.decode_tl2(np.array([[0xED]], np.uint8), sp, 6)
    with pytest.raises(ValueError, match="non-canonical zero"):
        O.decode_tl2(np.array([[0x00]], np.uint8), np.array([[1]], np.uint8), 6)


def test_payload_sizes_kat():                        # test_packing.py:193-201
    assert O.i2s_bytes(768, 768) == 147456
    assert O.tl1_bytes(768, 768) == 147456
    assert O.tl2_bytes(768, 768) == (98304, 24576)


# ---------------------------------------------------------------- KATs (lut)

def test_lut_kat():                                  # test_lut.py:31-104
    e = O.lut_tl1(np.array([3, -2], np.int8), 2)
    assert e.shape == (1, 9) and e[0, 8] == 1 and e[0, 0] == -1 and e[0, 4] == 0
    e = O.lut_tl2(np.array([1, 2, 3], np.int8), 3)
    assert e[0, 10] == 4 and e[0, 13] == 6 and e[0, 0] == 0
    assert np.abs(O.lut_tl1(np.array([127, -127], np.int8), 2)).max() == 254
    assert np.abs(O.lut_tl2(np.array([127, -127, 127], np.int8), 3)).max() == 381
    d, _, n = O.quantize([1.0, -0.5, 0.25], 3)
    e = O.lut_tl2(d, n, groups=4)
    assert e.shape == (4, 14) and np.all(e[1:] == 0)
    d, _, n = O.quantize([1.0] * 9, 3)
    with pytest.raises(ValueError):
        O.lut_tl2(d, n, groups=2)


# ------------------------------------------------------------ KATs (kernels)

def test_kernel_kat():                               # test_kernels.py:34-119
    acc = O.gemv_ref_int32([[1, -1, 0, 1]], np.array([2, 3, -1, 4], np.int8))
    assert acc.tolist() == [3]
    assert O.make_output(np.array([30]), 0.5, 0.25)[0] == 30 * 0.5 * 0.25
    with pytest.raises(ValueError, match="dimension mismatch"):
        O.gemv_ref_int32([[1, -1, 0]], np.array([1, 2], np.int8))
    with pytest.raises(ValueError, match="dimension mismatch"):
        O.gemv_ref_int32([[1]], np.array([1, 2], np.int8))
    a = np.array([3, -2], np.int8)
    assert O.gemv_tl1(O.encode_tl1([[0, 1]]), 2, O.lut_tl1(a, 2)).tolist() == [-2]
    a = np.array([1, 2, 3], np.int8)
    ip, sp = O.encode_tl2([[-1, -1, -1]])
    assert O.gemv_tl2(ip, sp, 3, O.lut_tl2(a, 3, groups=2)).tolist() == [-6]
    # all-ones x 127 at 8192 cols -> 1,040,384 on every path (test_kernels.py:107-119)
    v = np.ones((2, 8192), np.int8)
    a = np.full(8192, 127, np.int8)
    ref = O.gemv_ref_int32(v, a)
    assert ref[0] == 1_040_384
    ip, sp = O.encode_tl2(v)
    assert np.array_equal(O.gemv_tl1(O.encode_tl1(v), 8192, O.lut_tl1(a, 8192), checked=True), ref)
    assert np.array_equal(O.gemv_tl2(ip, sp, 8192, O.lut_tl2(a, 8192, groups=2731 + 1),
                                     checked=True), ref)


def test_row_bounds():                               # kernels.py:181-186
    assert O.row_bounds(1, 8) == [(0, 1)]
    b = O.row_bounds(611, 4)
    assert b[0][0] == 0 and b[-1][1] == 611 and all(lo % 64 == 0 for lo, _ in b)


# --------------------------------------------------------- golden: small.npz

def test_golden_quantize():
    xs = split(SMALL["q_x"], SMALL["q_xoff"])
    for pad in (1, 2, 3, 4):
        want = split(SMALL[f"q_data_p{pad}"], SMALL[f"q_doff_p{pad}"])
        scales = SMALL[f"q_scale_p{pad}"]
        for x, d, s in zip(xs, want, scales):
            got, gs, _ = O.quantize(x, pad)
            assert np.array_equal(got, d)
            assert gs == s  # bit exact


def test_golden_ternarize():
    ws = split(SMALL["t_w"], np.cumsum([0] + [r * c for r, c in SMALL["t_shape"]]))
    qs = split(SMALL["t_q"], np.cumsum([0] + [r * c for r, c in SMALL["t_shape"]]))
    for w, q, (r, c), s in zip(ws, qs, SMALL["t_shape"], SMALL["t_scale"]):
        gq, gs = O.ternarize(w, int(r), int(c))
        assert gs == s and np.array_equal(gq.ravel(), q)


def test_golden_packing_roundtrip():
    shapes = SMALL["p_shape"]
    vals = split(SMALL["p_vals"], np.cumsum([0] + [r * c for r, c in shapes]))
    i2s = split(SMALL["p_i2s"], SMALL["p_i2s_off"])
    tl1 = split(SMALL["p_tl1"], SMALL["p_tl1_off"])
    tl2i = split(SMALL["p_tl2i"], SMALL["p_tl2i_off"])
    tl2s = split(SMALL["p_tl2s"], SMALL["p_tl2s_off"])
    for k, (r, c) in enumerate(shapes):
        v = vals[k].reshape(r, c)
        assert np.array_equal(O.encode_i2s(v).ravel(), i2s[k])
        assert np.array_equal(O.encode_tl1(v).ravel(), tl1[k])
        ip, sp = O.encode_tl2(v)
        assert np.array_equal(ip.ravel(), tl2i[k]) and np.array_equal(sp.ravel(), tl2s[k])
        assert np.array_equal(O.decode_i2s(O.encode_i2s(v), c), v)
        assert np.array_equal(O.decode_tl1(O.encode_tl1(v), c), v)
        assert np.array_equal(O.decode_tl2(ip, sp, c), v)


def test_golden_lut():
    xs = split(SMALL["l_x"], SMALL["l_xoff"])
    l1 = split(SMALL["l_tl1"], SMALL["l_tl1_off"])
    l2 = split(SMALL["l_tl2"], SMALL["l_tl2_off"])
    for x, extra, e1, e2 in zip(xs, SMALL["l_extra"], l1, l2):
        d2, _, n2 = O.quantize(x, 2)
        d3, _, n3 = O.quantize(x, 3)
        assert np.array_equal(O.lut_tl1(d2, n2, d2.size // 2 + int(extra)).ravel(), e1)
        assert np.array_equal(O.lut_tl2(d3, n3, d3.size // 3 + int(extra)).ravel(), e2)


def test_golden_cross_kernel():
    shapes = SMALL["g_shape"]
    vals = split(SMALL["g_vals"], np.cumsum([0] + [r * c for r, c in shapes]))
    xs = split(SMALL["g_x"], SMALL["g_xoff"])
    accs = split(SMALL["g_acc"], SMALL["g_accoff"])
    outs = split(SMALL["g_out"], SMALL["g_accoff"])
    for k, (r, c) in enumerate(shapes[:600]):
        v = vals[k].reshape(r, c)
        got = O.check_instance(v, xs[k])
        for name in ("ref", "i2s", "tl1", "tl2"):
            assert np.array_equal(got[name], accs[k]), (k, name)
        _, s, _ = O.quantize(xs[k], 1)
        assert np.array_equal(O.make_output(accs[k], SMALL["g_wscale"][k], s), outs[k])


def test_golden_overflow():
    for cols in (4092, 16384):
        v, a, acc = SMALL[f"ov_v{cols}"], SMALL[f"ov_a{cols}"], SMALL[f"ov_acc{cols}"]
        assert np.array_equal(O.gemv_ref_int32(v, a), acc)
        assert np.array_equal(O.gemv_i2s(O.encode_i2s(v), cols, a), acc)
        g1 = O.pad_len(cols, 2) // 2
        g2 = O.pad_len(cols, 6) // 3
        ip, sp = O.encode_tl2(v)
        for chk in (False, True):
            assert np.array_equal(O.gemv_tl1(O.encode_tl1(v), cols, O.lut_tl1(a, cols, g1),
                                             checked=chk), acc)
            assert np.array_equal(O.gemv_tl2(ip, sp, cols, O.lut_tl2(a, cols, g2),
                                             checked=chk), acc)


def test_golden_toy_decoder():
    for dseed, prompt, toks in zip(SMALL["d_seed"][:4], SMALL["d_prompt"][:4],
                                   SMALL["d_tokens"][:4]):
        emb, layers, head = O.toy_decoder(seed=int(dseed))
        assert O.toy_decode(emb, layers, head, int(prompt), 24) == toks.tolist()


# --------------------------------------------------------- golden: large.json

@pytest.mark.parametrize("cname", ["cfg0", "cfg1"])
def test_golden_large_config(cname):
    case, gold = LARGE_CASES[cname], LARGE[cname]
    mats = {}
    for name, n, k, seed in case["matrices"]:
        q, s = O.ternarize(latent_weights(seed, n, k), n, k)
        g = gold["matrices"][name]
        assert s.hex() == g["scale"] and sha(q) == g["values"]
        assert sha(O.encode_i2s(q)) == g["i2s"]
        assert sha(O.encode_tl1(q)) == g["tl1"]
        mats[name] = (q, s)
    acts = {}
    for name, m, k, seed in case["acts"]:
        x = activations(seed, m, k)
        for pad in (1, 2, 3, 4):
            d, s = O.quantize_rows(x, pad)
            assert sha(d) == gold["acts"][name][f"data_p{pad}"]
            assert [v.hex() for v in s] == gold["acts"][name]["scales"]
        acts[name] = O.quantize_rows(x, 1)
    for wname, aname in case["gemv"]:
        q, ws = mats[wname]
        d, s = acts[aname]
        acc = np.stack([O.gemv_ref_int32(q, d[i]) for i in range(d.shape[0])])
        out = np.stack([O.make_output(acc[i], ws, s[i]) for i in range(d.shape[0])])
        g = gold["gemv"][f"{wname}:{aname}"]
        assert sha(acc) == g["acc"] and sha(out) == g["out"]
