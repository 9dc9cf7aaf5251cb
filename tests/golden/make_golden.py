"""Generate the golden fixtures by running the REAL reference package.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``ternpack`` from /root/reference/pkg/src (read-only; numba falls
back to the user cache dir) and writes

  * tests/golden/small.npz  -- small inputs with the reference's outputs
  * tests/golden/large.json -- sha256 pins of config-shaped cases (BASELINE
                               configs 0..4): packed bytes, int8 activations,
                               float64 scales, int32 accumulators, f64 outputs

Nothing here is imported at test time; tests read only the written files and
regenerate the large inputs from the seeds in ``workloads.py``.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE))

import ternpack as tp  # noqa: E402  (the reference itself)
from ternpack import kernels as tk  # noqa: E402
from ternpack import runtime as trt  # noqa: E402

from workloads import LARGE_CASES, activations, latent_weights, sha  # noqa: E402


def _cat(arrs, dtype):
    arrs = [np.asarray(a, dtype=dtype).reshape(-1) for a in arrs]
    offs = np.cumsum([0] + [a.size for a in arrs]).astype(np.int64)
    return (np.concatenate(arrs) if arrs else np.zeros(0, dtype)), offs


def small_fixtures():
    out = {}
    rng = np.random.default_rng(2024)

    # -- quantize_activations: random, scaled, special and rounding-adversarial
    xs = []
    for _ in range(60):
        n = int(rng.integers(1, 300))
        xs.append(rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 3))
    xs.append(np.zeros(3))
    xs.append(np.array([127.0]))
    xs.append(np.array([0.5, -1.0, 0.25]))
    for amax in (1.0, 3.7, 1e-3, 12345.678):
        s = amax / 127.0
        k = np.arange(-126, 127, dtype=np.float64) + 0.5
        base = k * s
        xs.append(np.concatenate([[amax], base, np.nextafter(base, np.inf),
                                  np.nextafter(base, -np.inf)]))
    # float32-valued activations as in the BASELINE configs
    for _ in range(20):
        xs.append(rng.standard_normal(int(rng.integers(1, 2000)), dtype=np.float32)
                  .astype(np.float64))
    xcat, xoff = _cat(xs, np.float64)
    out["q_x"], out["q_xoff"] = xcat, xoff
    for pad in (1, 2, 3, 4):
        datas, scales = [], []
        for x in xs:
            qa = tp.quantize_activations(x, pad_to=pad)
            datas.append(qa.data)
            scales.append(qa.scale)
        out[f"q_data_p{pad}"], out[f"q_doff_p{pad}"] = _cat(datas, np.int8)
        out[f"q_scale_p{pad}"] = np.array(scales, dtype=np.float64)

    # -- ternarize_weights
    ws, shapes, qs, scales = [], [], [], []
    for i in range(30):
        r, c = int(rng.integers(1, 17)), int(rng.integers(1, 41))
        w = rng.standard_normal(r * c) * 10.0 ** rng.uniform(-2, 2)
        if i % 3 == 0:
            w = w.astype(np.float32).astype(np.float64)
        m = tp.ternarize_weights(w, r, c)
        ws.append(w); shapes.append((r, c)); qs.append(m.values); scales.append(m.scale)
    m = tp.ternarize_weights([0.9, -0.1, 0.05, -0.85], 2, 2)
    ws.append(np.array([0.9, -0.1, 0.05, -0.85])); shapes.append((2, 2))
    qs.append(m.values); scales.append(m.scale)
    out["t_w"], _ = _cat(ws, np.float64)
    out["t_shape"] = np.array(shapes, dtype=np.int64)
    out["t_q"], _ = _cat(qs, np.int8)
    out["t_scale"] = np.array(scales, dtype=np.float64)

    # -- packing codecs over every cols-mod-12 residue and a few larger shapes
    shapes, vals, i2s, tl1, tl2i, tl2s = [], [], [], [], [], []
    dims = [(int(rng.integers(1, 13)), c) for c in range(1, 49)]
    dims += [(3, 768), (5, 1000), (2, 4092), (33, 100), (64, 512)]
    for r, c in dims:
        v = rng.integers(-1, 2, size=(r, c), dtype=np.int8)
        m = tp.TernaryMatrix(r, c, v, 1.0)
        pi, p1, p2 = tp.encode_i2s(m), tp.encode_tl1(m), tp.encode_tl2(m)
        shapes.append((r, c)); vals.append(v); i2s.append(pi.data); tl1.append(p1.data)
        tl2i.append(p2.index_data); tl2s.append(p2.sign_data)
    out["p_shape"] = np.array(shapes, dtype=np.int64)
    out["p_vals"], _ = _cat(vals, np.int8)
    out["p_i2s"], out["p_i2s_off"] = _cat(i2s, np.uint8)
    out["p_tl1"], out["p_tl1_off"] = _cat(tl1, np.uint8)
    out["p_tl2i"], out["p_tl2i_off"] = _cat(tl2i, np.uint8)
    out["p_tl2s"], out["p_tl2s_off"] = _cat(tl2s, np.uint8)

    # -- activation LUTs (groups=None and an explicit larger group count)
    l1, l2, lx, lextra = [], [], [], []
    for _ in range(40):
        n = int(rng.integers(1, 200))
        x = rng.standard_normal(n) * 40
        extra = int(rng.integers(0, 3))
        qa2 = tp.quantize_activations(x, pad_to=2)
        qa3 = tp.quantize_activations(x, pad_to=3)
        l1.append(tp.build_lut_tl1(qa2, groups=len(qa2) // 2 + extra).entries)
        l2.append(tp.build_lut_tl2(qa3, groups=len(qa3) // 3 + extra).entries)
        lx.append(x); lextra.append(extra)
    out["l_x"], out["l_xoff"] = _cat(lx, np.float64)
    out["l_extra"] = np.array(lextra, dtype=np.int64)
    out["l_tl1"], out["l_tl1_off"] = _cat(l1, np.int16)
    out["l_tl2"], out["l_tl2_off"] = _cat(l2, np.int16)

    # -- cross-kernel instances (verify.cross_kernel_suite schedule, seed 11)
    from ternpack.verify import _instance_shape, check_instance  # reference's own
    r2 = np.random.default_rng(11)
    shapes, vals, xs, accs, outs, wsc = [], [], [], [], [], []
    for i in range(2000):
        rows, cols = _instance_shape(i, r2)
        v = r2.integers(-1, 2, size=(rows, cols), dtype=np.int8)
        scale = float(r2.uniform(0.1, 2.0))
        x = r2.standard_normal(cols) * float(r2.uniform(0.01, 10.0))
        m = tp.TernaryMatrix(rows, cols, v, scale)
        ok = check_instance(m, x)
        assert all(ok.values()), i
        ref = tp.gemv_ref_int32(m, tp.quantize_activations(x, pad_to=1))
        shapes.append((rows, cols)); vals.append(v); xs.append(x)
        accs.append(ref.accumulators); outs.append(ref.output); wsc.append(scale)
    out["g_shape"] = np.array(shapes, dtype=np.int64)
    out["g_vals"], _ = _cat(vals, np.int8)
    out["g_x"], out["g_xoff"] = _cat(xs, np.float64)
    out["g_wscale"] = np.array(wsc, dtype=np.float64)
    out["g_acc"], out["g_accoff"] = _cat(accs, np.int32)
    out["g_out"], _ = _cat(outs, np.float64)

    # -- acceptance criterion 5: adversarial overflow rows (test_acceptance.py:159-185)
    r3 = np.random.default_rng(31)
    ov_vals, ov_act, ov_acc = [], [], []
    for cols in (4092, 16384):
        v = np.ones((6, cols), dtype=np.int8)
        v[1] = -1
        v[2, ::2] = -1
        v[3:] = r3.integers(-1, 2, size=(3, cols), dtype=np.int8)
        sign = np.where(r3.random(cols) < 0.5, -1, 1)
        a = (127 * sign).astype(np.int8)
        m = tp.TernaryMatrix(6, cols, v, 1.0)
        qa = tp.QuantizedActivations(data=a, scale=1.0, original_len=cols)
        ref = tp.gemv_ref_int32(m, qa).accumulators
        assert np.array_equal(tp.gemv_i2s(tp.encode_i2s(m), qa).accumulators, ref)
        ov_vals.append(v); ov_act.append(a); ov_acc.append(ref)
    out["ov_v4092"], out["ov_v16384"] = ov_vals
    out["ov_a4092"], out["ov_a16384"] = ov_act
    out["ov_acc4092"], out["ov_acc16384"] = ov_acc

    # -- toy decoder token sequences (runtime.lossless_report protocol, seed 13)
    root = np.random.SeedSequence(13)
    dseeds, prompts, toks, ftl1, ftl2 = [], [], [], [], []
    for child in root.spawn(12):
        r4 = np.random.default_rng(child)
        dseed = int(r4.integers(0, 2**63))
        prompt = int(r4.integers(0, 256))
        d = trt.ToyDecoder.build(seed=dseed)
        ref = trt.decode_tokens(d, tk.KernelKind.REF_INT32, prompt, 24)
        for k in (tk.KernelKind.I2_S, tk.KernelKind.TL1, tk.KernelKind.TL2):
            assert trt.decode_tokens(d, k, prompt, 24) == ref
        f1 = trt.decode_tokens(d, tk.KernelKind.TL1, prompt, 24, _lut_hook=trt._corrupting_hook)
        f2 = trt.decode_tokens(d, tk.KernelKind.TL2, prompt, 24, _lut_hook=trt._corrupting_hook)
        dseeds.append(dseed); prompts.append(prompt); toks.append(ref)
        ftl1.append(f1); ftl2.append(f2)
    out["d_seed"] = np.array(dseeds, dtype=np.uint64)
    out["d_prompt"] = np.array(prompts, dtype=np.int64)
    out["d_tokens"] = np.array(toks, dtype=np.int64)
    out["d_fault_tl1"] = np.array(ftl1, dtype=np.int64)
    out["d_fault_tl2"] = np.array(ftl2, dtype=np.int64)
    return out


def large_fixtures(only=None):
    res = {}
    for cname, case in LARGE_CASES.items():
        if only is not None and cname not in only:
            continue
        t0 = time.time()
        mats, acts, entry = {}, {}, {"matrices": {}, "acts": {}, "gemv": {}}
        for name, n, k, seed in case["matrices"]:
            m = tp.ternarize_weights(latent_weights(seed, n, k), n, k)
            mats[name] = m
            pi, p1, p2 = tp.encode_i2s(m), tp.encode_tl1(m), tp.encode_tl2(m)
            entry["matrices"][name] = {
                "rows": n, "cols": k, "seed": seed, "scale": m.scale.hex(),
                "values": sha(m.values), "i2s": sha(pi.data), "tl1": sha(p1.data),
                "tl2_index": sha(p2.index_data), "tl2_sign": sha(p2.sign_data),
            }
            mats[name] = (m, pi, p1, p2)
        for name, mm, k, seed in case["acts"]:
            x = activations(seed, mm, k)
            per = {"m": mm, "k": k, "seed": seed}
            for pad in (1, 2, 3, 4):
                qs = [tp.quantize_activations(x[i], pad_to=pad) for i in range(mm)]
                per[f"data_p{pad}"] = sha(np.stack([q.data for q in qs]))
                per["scales"] = [q.scale.hex() for q in qs]
                acts[(name, pad)] = qs
            entry["acts"][name] = per
        for wname, aname in case["gemv"]:
            m, pi, p1, p2 = mats[wname]
            qs1 = acts[(aname, 1)]
            acc = np.stack([tp.gemv_ref_int32(m, q).accumulators for q in qs1])
            outv = np.stack([tp.gemv_ref_int32(m, q).output for q in qs1])
            # the reference's own packed kernels agree (checked on token 0)
            q4, q2, q3 = acts[(aname, 4)][0], acts[(aname, 2)][0], acts[(aname, 3)][0]
            assert np.array_equal(tk.gemv_parallel(tk.KernelKind.I2_S, pi, q4).accumulators, acc[0])
            assert np.array_equal(tk.gemv_parallel(tk.KernelKind.TL1, p1, q2).accumulators, acc[0])
            assert np.array_equal(tk.gemv_parallel(tk.KernelKind.TL2, p2, q3).accumulators, acc[0])
            entry["gemv"][f"{wname}:{aname}"] = {"acc": sha(acc), "out": sha(outv),
                                                 "acc_sum": int(acc.astype(np.int64).sum())}
        res[cname] = entry
        print(f"{cname}: {time.time() - t0:.1f}s", flush=True)
    return res


def main():
    """No arguments: every fixture.  ``--large cfgN ...``: regenerate only
    those large cases and merge them into the existing large.json."""
    t0 = time.time()
    only = sys.argv[sys.argv.index("--large") + 1:] if "--large" in sys.argv else None
    if only is None:
        small = small_fixtures()
        np.savez_compressed(HERE / "small.npz", **small)
        print(f"small.npz written ({time.time() - t0:.1f}s)", flush=True)
        large = large_fixtures()
    else:
        large = json.loads((HERE / "large.json").read_text())
        large.update(large_fixtures(only))
    (HERE / "large.json").write_text(json.dumps(large, indent=1, sort_keys=True) + "\n")
    print(f"large.json written ({time.time() - t0:.1f}s)")


if __name__ == "__main__":
    main()
