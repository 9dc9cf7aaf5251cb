"""Pin the C port of the reference's byte-table CPU kernels (oracle/c).

oracle/c/tern_oracle.c is the CPU baseline beside the reference arm and the
fast checker the full-size GPU stack tests use (tests/test_bench_shapes_gpu.py),
so it is pinned here against the reference's own outputs: the golden fixtures
that tests/golden/make_golden.py wrote by running /root/reference
(small.npz: 2,000 cross-kernel instances, LUTs, the overflow rows;
large.json: config-shaped packed bytes / activations / accumulators).
CPU only: no GPU needed.
"""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import c_oracle as CO
from oracle import ternpack_oracle as O
from workloads import LARGE_CASES, activations, latent_weights, sha

GOLD = Path(__file__).parent / "golden"
SMALL = np.load(GOLD / "small.npz")
LARGE = json.loads((GOLD / "large.json").read_text())


def split(flat, offs):
    return [flat[offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]


@pytest.fixture(scope="module", autouse=True)
def _built():
    CO.build()


def _c_gemvs(v, x, threads):
    """Accumulators of the three packed C kernels on ternary values v and
    real activations x (quantised by the pinned Python oracle, per-kernel pad)."""
    rows, cols = v.shape
    q4, _, _ = O.quantize(x, 4)
    q2, _, _ = O.quantize(x, 2)
    q3, _, _ = O.quantize(x, 3)
    i2s = CO.gemv_i2s(O.encode_i2s(v), q4, threads)
    tl1 = CO.gemv_tl1(O.encode_tl1(v), CO.lut_tl1(q2, q2.size // 2), threads)
    ip, sp = O.encode_tl2(v)
    tl2 = CO.gemv_tl2(ip, sp, CO.lut_tl2(q3, O.pad_len(cols, 6) // 3), threads)  # weights.groups
    return {"i2s": i2s, "tl1": tl1, "tl2": tl2}


def test_c_cross_kernel_golden():
    """The 2,000 reference cross-kernel instances (verify.py schedule, seed 11),
    every packed C kernel, 1 and 4 threads (results independent of threads,
    kernels.py:181-186)."""
    shapes = SMALL["g_shape"]
    vals = split(SMALL["g_vals"], np.cumsum([0] + [r * c for r, c in shapes]))
    xs = split(SMALL["g_x"], SMALL["g_xoff"])
    accs = split(SMALL["g_acc"], SMALL["g_accoff"])
    for k, (r, c) in enumerate(shapes):
        v = vals[k].reshape(r, c)
        for name, got in _c_gemvs(v, xs[k], 1 if k % 2 else 4).items():
            assert np.array_equal(got, accs[k]), (k, name)


def test_c_lut_golden():
    xs = split(SMALL["l_x"], SMALL["l_xoff"])
    l1 = split(SMALL["l_tl1"], SMALL["l_tl1_off"])
    l2 = split(SMALL["l_tl2"], SMALL["l_tl2_off"])
    for x, extra, e1, e2 in zip(xs, SMALL["l_extra"], l1, l2):
        d2, _, _ = O.quantize(x, 2)
        d3, _, _ = O.quantize(x, 3)
        assert np.array_equal(CO.lut_tl1(d2, d2.size // 2 + int(extra)).ravel(), e1)
        assert np.array_equal(CO.lut_tl2(d3, d3.size // 3 + int(extra)).ravel(), e2)


def test_c_overflow_golden():
    """Acceptance criterion 5's adversarial rows (test_acceptance.py:159-185)."""
    for cols in (4092, 16384):
        v, a, acc = SMALL[f"ov_v{cols}"], SMALL[f"ov_a{cols}"], SMALL[f"ov_acc{cols}"]
        assert np.array_equal(CO.gemv_i2s(O.encode_i2s(v), a, 2), acc)
        a2 = np.zeros(O.pad_len(cols, 2), np.int8)
        a2[:cols] = a
        assert np.array_equal(CO.gemv_tl1(O.encode_tl1(v), CO.lut_tl1(a2, a2.size // 2), 2), acc)
        a3 = np.zeros(O.pad_len(cols, 6), np.int8)
        a3[:cols] = a
        ip, sp = O.encode_tl2(v)
        assert np.array_equal(CO.gemv_tl2(ip, sp, CO.lut_tl2(a3, a3.size // 3), 2), acc)


def test_c_quantize_float32():
    """The C quantiser on float32 input (the bench's activations) against the
    pinned oracle: random scales, exact ties, zeros, a single element."""
    rng = np.random.default_rng(5)
    cases = [rng.standard_normal(int(n)).astype(np.float32) * np.float32(10.0 ** e)
             for n, e in zip(rng.integers(1, 5000, 40), rng.uniform(-30, 30, 40))]
    s = np.float32(3.7) / np.float32(127.0)
    cases.append((np.arange(-126, 127, dtype=np.float32) + np.float32(0.5)) * s)
    cases += [np.zeros(7, np.float32), np.array([127.0], np.float32),
              np.array([-1e-38, 2e-38], np.float32)]
    for x in cases:
        for pad in (1, 2, 3, 4):
            q, sc = CO.quantize(x, pad)
            d, so, _ = O.quantize(x, pad)
            assert np.array_equal(q, d) and sc == so, (x.size, pad)
    with pytest.raises(ValueError):
        CO.quantize(np.array([1.0, np.nan], np.float32), 1)


@pytest.mark.parametrize("cname", ["cfg0", "cfg1"])
def test_c_large_golden(cname):
    """Config-shaped pins (large.json, written by the reference): the C
    quantiser's codes and scales on the float32 activations, and the three C
    kernels' accumulators, on the full BASELINE shapes (cfg1: the TL1 FFN
    block the bench times)."""
    case, gold = LARGE_CASES[cname], LARGE[cname]
    acts = {}
    for name, mm, k, seed in case["acts"]:
        x = activations(seed, mm, k)
        for pad in (2, 3, 4):
            qs = [CO.quantize(x[i], pad) for i in range(mm)]
            assert sha(np.stack([q for q, _ in qs])) == gold["acts"][name][f"data_p{pad}"]
            assert [s.hex() for _, s in qs] == gold["acts"][name]["scales"]
            acts[(name, pad)] = [q for q, _ in qs]
    mats = {}
    for name, n, k, seed in case["matrices"]:
        q, s = O.ternarize(latent_weights(seed, n, k), n, k)
        assert s.hex() == gold["matrices"][name]["scale"]
        mats[name] = q

    def k_of(aname):
        return [a[2] for a in case["acts"] if a[0] == aname][0]

    for wname, aname in case["gemv"]:
        v = mats[wname]
        g = gold["gemv"][f"{wname}:{aname}"]
        i2s = np.stack([CO.gemv_i2s(O.encode_i2s(v), a, 0) for a in acts[(aname, 4)]])
        assert sha(i2s) == g["acc"], (cname, wname, "i2s")
        tl1 = np.stack([CO.gemv_tl1(O.encode_tl1(v), CO.lut_tl1(a, a.size // 2), 0)
                        for a in acts[(aname, 2)]])
        assert sha(tl1) == g["acc"], (cname, wname, "tl1")
        ip, sp = O.encode_tl2(v)
        tl2 = np.stack([CO.gemv_tl2(ip, sp, CO.lut_tl2(a, O.pad_len(k_of(aname), 6) // 3), 0)
                        for a in acts[(aname, 3)]])
        assert sha(tl2) == g["acc"], (cname, wname, "tl2")
