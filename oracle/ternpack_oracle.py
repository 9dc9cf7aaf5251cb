"""CPU oracle for the ternary BitLinear hot path -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference package ``ternpack``
(/root/reference/pkg/src/ternpack, read-only, not shipped).  Every function
cites the reference file:line whose behaviour it restates.  It exists so that
the CUDA path in ``paper_2410_16144_b200`` can be checked bit-for-bit:

  * packed weight bytes (I2_S / TL1 / TL2)        -> bit exact
  * int8 activations + float64 activation scale  -> bit exact
  * int32 accumulators                           -> bit exact
  * float64 outputs (acc * w_scale * a_scale)    -> bit exact

Parity of this oracle with the real reference is PINNED by
``tests/golden/`` (fixtures produced by importing the reference itself in the
build container, see ``tests/golden/make_golden.py``) and checked by
``tests/test_oracle_golden.py``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module.  The product package never
does: its GEMV path is CUDA-only and fails loudly without the extension.
"""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# core: rounding, ternarisation, activation quantisation   (core.py)
# ---------------------------------------------------------------------------


def round_half_away(x):
    """Nearest integer, ties away from zero, evaluated in float64.

    Restates core.py:24-27: trunc(x + copysign(0.5, x)).  NB: this is *not*
    C ``round()``: for x just below k+0.5 the float64 add can round up.
    """
    v = np.asarray(x, dtype=np.float64)
    return np.trunc(v + np.copysign(0.5, v))


def ternarize(weights, rows: int, cols: int):
    """Absmean ternarisation -> (int8 values [rows, cols], float scale).

    Restates core.py:104-113.  The scale is ``np.mean(np.abs(w))`` of the
    float64 copy (NumPy pairwise summation), q = clip(rha(w / scale), -1, 1).
    """
    w = np.asarray(weights, dtype=np.float64).reshape(rows, cols)
    if not np.isfinite(w).all():
        raise ValueError("weights must be finite")
    scale = float(np.mean(np.abs(w)))
    if scale == 0.0:
        raise ValueError("degenerate weight matrix")
    q = np.clip(round_half_away(w / scale), -1, 1).astype(np.int8)
    return q, scale


def pad_len(n: int, multiple: int) -> int:
    return -(-n // multiple) * multiple


def quantize(x, pad_to: int = 1):
    """Per-token absmax int8 quantisation -> (data int8 [K_pad], scale, K).

    Restates core.py:116-134: float64 absmax, scale = amax/127 (1.0 for an
    all-zero vector), q = clip(rha(x / scale), -127, 127), zero padding to a
    multiple of ``pad_to`` in {1, 2, 3, 4}.
    """
    if pad_to not in (1, 2, 3, 4):
        raise ValueError("pad_to must be in {1, 2, 3, 4}")
    v = np.asarray(x, dtype=np.float64).reshape(-1)
    if v.size == 0:
        raise ValueError("empty activation vector")
    if not np.isfinite(v).all():
        raise ValueError("activations must be finite")
    amax = float(np.abs(v).max())
    scale = amax / 127.0 if amax > 0.0 else 1.0
    q = np.clip(round_half_away(v / scale), -127, 127).astype(np.int8)
    out = np.zeros(pad_len(v.size, pad_to), dtype=np.int8)
    out[: v.size] = q
    return out, scale, v.size


def quantize_rows(x2d, pad_to: int = 1):
    """Prefill helper: one independent per-token quantisation per row.

    The reference has no multi-token type (QuantizedActivations is 1-D,
    core.py:71); M tokens are M calls of core.py:116-134.
    """
    x2d = np.atleast_2d(np.asarray(x2d))
    datas, scales = [], []
    for row in x2d:
        d, s, _ = quantize(row, pad_to)
        datas.append(d)
        scales.append(s)
    return np.stack(datas), np.array(scales, dtype=np.float64)


def make_output(acc, w_scale: float, a_scale: float):
    """float64 output = float64(acc) * w_scale * a_scale, left to right.

    Restates core.py:99-101.
    """
    return np.asarray(acc).astype(np.float64) * float(w_scale) * float(a_scale)


# ---------------------------------------------------------------------------
# packing codecs   (packing.py)
# ---------------------------------------------------------------------------

TL1_ZERO_NIBBLE = 4  # packing.py:35 -- filler for an odd trailing pair


def i2s_bytes(rows: int, cols: int) -> int:          # packing.py:42-43
    return rows * (pad_len(cols, 4) // 4)


def tl1_bytes(rows: int, cols: int) -> int:          # packing.py:46-47
    groups = pad_len(cols, 2) // 2
    return rows * (-(-groups // 2))


def tl2_bytes(rows: int, cols: int):                 # packing.py:50-53
    pc = pad_len(cols, 6)
    return rows * (pc // 6), rows * (-(-(pc // 3) // 8))


def tl1_index(w0: int, w1: int) -> int:              # packing.py:56-60
    if w0 not in (-1, 0, 1) or w1 not in (-1, 0, 1):
        raise ValueError("weights must be ternary")
    return 3 * (w0 + 1) + (w1 + 1)


def tl2_code(w0: int, w1: int, w2: int):             # packing.py:63-74
    if any(w not in (-1, 0, 1) for w in (w0, w1, w2)):
        raise ValueError("weights must be ternary")
    d = 9 * (w0 + 1) + 3 * (w1 + 1) + (w2 + 1) - 13
    return (1 if d < 0 else 0), abs(d)


def _padded_values(values, multiple: int):
    v = np.asarray(values, dtype=np.int16)
    rows, cols = v.shape
    out = np.zeros((rows, pad_len(cols, multiple)), dtype=np.int16)
    out[:, :cols] = v
    return out


def encode_i2s(values):
    """I2_S bytes [rows, pc/4]: code = w+1, weight 4j+s at bits 2s..2s+1.

    Restates packing.py:200-206 (padding weights are 0 -> code 01).
    """
    codes = (_padded_values(values, 4) + 1).astype(np.uint8)
    rows, pc = codes.shape
    c = codes.reshape(rows, pc // 4, 4)
    return (c[..., 0] | (c[..., 1] << 2) | (c[..., 2] << 4) | (c[..., 3] << 6)).astype(np.uint8)


def i2s_codes(data, padded_cols: int):
    b = np.asarray(data, dtype=np.uint8)
    shifts = np.array([0, 2, 4, 6], dtype=np.uint8)
    c = (b[..., None] >> shifts) & 3
    return c.reshape(b.shape[0], -1)[:, :padded_cols]


def validate_i2s(data):
    """First row holding reserved code 0b11 -> ValueError (packing.py:98-107)."""
    bad = (i2s_codes(data, 4 * np.asarray(data).shape[1]) == 3).any(axis=1)
    if bad.any():
        raise ValueError(f"invalid I2_S code at row {int(np.flatnonzero(bad)[0])}")


def decode_i2s(data, cols: int):                      # packing.py:209-219
    codes = i2s_codes(data, pad_len(cols, 4))
    if (codes == 3).any():
        raise ValueError("invalid I2_S code")
    return (codes[:, :cols].astype(np.int8) - 1).astype(np.int8)


def encode_tl1(values):
    """TL1 bytes: pair g -> 3(w0+1)+(w1+1); pair 2j low nibble, 2j+1 high.

    Restates packing.py:222-233 (odd pair count -> filler nibble 4).
    """
    w = _padded_values(values, 2)
    idx = (3 * (w[:, 0::2] + 1) + (w[:, 1::2] + 1)).astype(np.uint8)
    if idx.shape[1] % 2:
        idx = np.concatenate(
            [idx, np.full((idx.shape[0], 1), TL1_ZERO_NIBBLE, np.uint8)], axis=1)
    return (idx[:, 0::2] | (idx[:, 1::2] << 4)).astype(np.uint8)


def tl1_nibbles(data):
    b = np.asarray(data, dtype=np.uint8)
    out = np.empty((b.shape[0], 2 * b.shape[1]), dtype=np.uint8)
    out[:, 0::2] = b & 15
    out[:, 1::2] = b >> 4
    return out


def validate_tl1(data):                               # packing.py:135-141
    bad = (tl1_nibbles(data) > 8).any(axis=1)
    if bad.any():
        raise ValueError(f"invalid TL1 index at row {int(np.flatnonzero(bad)[0])}")


def decode_tl1(data, cols: int):                      # packing.py:236-247
    nib = tl1_nibbles(data)
    if (nib > 8).any():
        raise ValueError("invalid TL1 index")
    groups = pad_len(cols, 2) // 2
    nib = nib[:, :groups].astype(np.int8)
    vals = np.empty((nib.shape[0], 2 * groups), dtype=np.int8)
    vals[:, 0::2] = nib // 3 - 1
    vals[:, 1::2] = nib % 3 - 1
    return vals[:, :cols]


def encode_tl2(values):
    """TL2 planes: per triple d = base3(w+1) - 13, sign = d<0, index = |d|.

    Restates packing.py:250-262: index nibbles two per byte (triple 2j low),
    sign bits eight per byte, bit j = triple 8k+j (little bit order).
    """
    w = _padded_values(values, 6)
    d = 9 * (w[:, 0::3] + 1) + 3 * (w[:, 1::3] + 1) + (w[:, 2::3] + 1) - 13
    idx = np.abs(d).astype(np.uint8)
    sign = (d < 0).astype(np.uint8)
    index_plane = (idx[:, 0::2] | (idx[:, 1::2] << 4)).astype(np.uint8)
    sign_plane = np.packbits(sign, axis=1, bitorder="little")
    return index_plane, sign_plane


def tl2_fields(index_plane, sign_plane, groups: int):
    ib = np.asarray(index_plane, dtype=np.uint8)
    nib = np.empty((ib.shape[0], 2 * ib.shape[1]), dtype=np.uint8)
    nib[:, 0::2] = ib & 15
    nib[:, 1::2] = ib >> 4
    sgn = np.unpackbits(np.asarray(sign_plane, dtype=np.uint8), axis=1,
                        bitorder="little")[:, :groups]
    return nib[:, :groups], sgn


def validate_tl2(index_plane, sign_plane, groups: int):   # packing.py:176-186
    nib, sgn = tl2_fields(index_plane, sign_plane, groups)
    bad = (nib > 13).any(axis=1)
    if bad.any():
        raise ValueError(f"invalid TL2 index at row {int(np.flatnonzero(bad)[0])}")
    nc = ((sgn == 1) & (nib == 0)).any(axis=1)
    if nc.any():
        raise ValueError(f"non-canonical zero at row {int(np.flatnonzero(nc)[0])}")


def decode_tl2(index_plane, sign_plane, cols: int):   # packing.py:265-277
    pc = pad_len(cols, 6)
    nib, sgn = tl2_fields(index_plane, sign_plane, pc // 3)
    if (nib > 13).any():
        raise ValueError("invalid TL2 index")
    if ((sgn == 1) & (nib == 0)).any():
        raise ValueError("non-canonical zero")
    d = nib.astype(np.int16) * (1 - 2 * sgn.astype(np.int16)) + 13
    vals = np.empty((nib.shape[0], pc), dtype=np.int8)
    vals[:, 0::3] = d // 9 - 1
    vals[:, 1::3] = (d // 3) % 3 - 1
    vals[:, 2::3] = d % 3 - 1
    return vals[:, :cols]


# ---------------------------------------------------------------------------
# activation LUTs   (lut.py)
# ---------------------------------------------------------------------------

# lut.py:20 -- pattern i is the pair (i//3 - 1, i%3 - 1)
TL1_PATTERNS = np.array([[i // 3 - 1, i % 3 - 1] for i in range(9)], dtype=np.int64)
# lut.py:23-26 -- pattern i is the sign-0 triple whose base-3 value is i+13
TL2_PATTERNS = np.array([[(i + 13) // 9 - 1, (i + 13) // 3 % 3 - 1, (i + 13) % 3 - 1]
                         for i in range(14)], dtype=np.int64)


def _groups_of(data, original_len: int, width: int, groups):
    """Zero-extended activation groups (lut.py:52-62)."""
    d = np.asarray(data, dtype=np.int64).reshape(-1)
    n = d.size
    if groups is None:
        groups = -(-max(n, width) // width)
    total = groups * width
    if original_len > total:
        raise ValueError("activation vector longer than the requested table")
    g = np.zeros(total, dtype=np.int64)
    g[: min(n, total)] = d[: min(n, total)]
    return g.reshape(groups, width)


def lut_tl1(data, original_len: int, groups=None):
    """int16 [groups, 9]: entry[g, i] = w0*a[2g] + w1*a[2g+1] (lut.py:72-75)."""
    g = _groups_of(data, original_len, 2, groups)
    return (g @ TL1_PATTERNS.T).astype(np.int16)


def lut_tl2(data, original_len: int, groups=None):
    """int16 [groups, 14] canonical triple dots, sign applied at lookup (lut.py:78-84)."""
    g = _groups_of(data, original_len, 3, groups)
    return (g @ TL2_PATTERNS.T).astype(np.int16)


# ---------------------------------------------------------------------------
# GEMV kernels   (kernels.py, _fast.py)
# ---------------------------------------------------------------------------


def check_cover(data, cols: int):
    """kernels.py:45-49 -- activation length / padding checks."""
    d = np.asarray(data)
    if d.size < cols:
        raise ValueError("dimension mismatch: activations shorter than matrix cols")
    if (d[cols:] != 0).any():
        raise ValueError("dimension mismatch: nonzero activations beyond matrix cols")


def gemv_ref_int32(values, data):
    """Ground truth: int32 multiply-then-add on ternary values (kernels.py:59-63)."""
    v = np.asarray(values)
    check_cover(data, v.shape[1])
    return v.astype(np.int32) @ np.asarray(data)[: v.shape[1]].astype(np.int32)


def gemv_f32_ref(values, scale: float, x):
    """Dequantised fp32 sgemv baseline (kernels.py:66-72)."""
    v = np.asarray(values)
    x = np.asarray(x, dtype=np.float32).reshape(-1)
    if x.size != v.shape[1]:
        raise ValueError("dimension mismatch")
    deq = v.astype(np.float32) * np.float32(scale)
    return (deq @ x).astype(np.float64)


def i2s_byte_table(data, padded_cols: int):
    """int32 [pc/4, 256]: t[j, b] = sum_s (code_s(b) - 1) * a[4j+s].

    Restates kernels.py:75-83 + _fast.py:98-129 (nibble tables combined into
    one 256-entry table per byte column).
    """
    a = np.zeros(padded_cols, dtype=np.int64)
    d = np.asarray(data, dtype=np.int64)
    n = min(d.size, padded_cols)
    a[:n] = d[:n]
    b = np.arange(256)
    codes = np.stack([(b >> (2 * s)) & 3 for s in range(4)], axis=1) - 1  # [256, 4]
    return (a.reshape(-1, 4) @ codes.T).astype(np.int32)


def tl1_byte_table(lut, bytes_per_row: int):
    """int32 [bc, 256]: t[j, b] = lut[2j, b & 15] + lut[2j+1, b >> 4].

    Restates kernels.py:97-106 + _fast.py:115-129 (nibbles > 8 and groups
    past the LUT read 0).
    """
    lut = np.asarray(lut, dtype=np.int64)
    planes = np.zeros((2 * bytes_per_row, 16), dtype=np.int64)
    planes[: lut.shape[0], :9] = lut
    b = np.arange(256)
    return (planes[0::2][:, b & 15] + planes[1::2][:, b >> 4]).astype(np.int32)


def tl2_signed_table(lut):
    """int32 [groups/2, 1024]: index = (sign pair << 8) | nibble byte.

    Restates kernels.py:129-137 + _fast.py:132-147.
    """
    lut = np.asarray(lut, dtype=np.int64)
    planes = np.zeros((lut.shape[0], 16), dtype=np.int64)
    planes[:, :14] = lut
    lo, hi = planes[0::2], planes[1::2]
    i = np.arange(1024)
    s, byte = i >> 8, i & 255
    fl = 1 - 2 * (s & 1)
    fh = 1 - 2 * (s >> 1)
    return (fh * hi[:, byte >> 4] + fl * lo[:, byte & 15]).astype(np.int32)


def byte_gemv(packed, table):
    """out[i] = sum_j table[j, packed[i, j]] with int32 wrap (_fast.py:25-51)."""
    p = np.asarray(packed, dtype=np.intp)
    t = np.asarray(table)
    cols = np.arange(p.shape[1])
    return t[cols[None, :], p].sum(axis=1, dtype=np.int64).astype(np.int32)


def tl2_byte_gemv(index_plane, sign_plane, table):
    """TL2 gather with both triple signs folded into the index (_fast.py:54-95)."""
    ib = np.asarray(index_plane, dtype=np.intp)
    sb = np.asarray(sign_plane, dtype=np.intp)
    bc = ib.shape[1]
    j = np.arange(bc)
    s = (sb[:, j >> 2] >> ((j & 3) * 2)) & 3
    t = np.asarray(table)
    return t[j[None, :], (s << 8) | ib].sum(axis=1, dtype=np.int64).astype(np.int32)


def gemv_i2s(data_packed, cols: int, act):
    """kernels.py:86-94: validate -> cover check -> byte table -> gather."""
    validate_i2s(data_packed)
    check_cover(act, cols)
    return byte_gemv(data_packed, i2s_byte_table(act, pad_len(cols, 4)))


def gemv_tl1(data_packed, cols: int, lut, checked: bool = False):
    """kernels.py:109-126 (fast byte table, or the checked int16 path)."""
    validate_tl1(data_packed)
    groups = pad_len(cols, 2) // 2
    if np.asarray(lut).shape[0] != groups:
        raise ValueError("group-count mismatch")
    if checked:
        nib = tl1_nibbles(data_packed)[:, :groups].astype(np.intp)
        vals = np.asarray(lut)[np.arange(groups)[None, :], nib]
        return widened_sum(vals)
    return byte_gemv(data_packed, tl1_byte_table(lut, np.asarray(data_packed).shape[1]))


def gemv_tl2(index_plane, sign_plane, cols: int, lut, checked: bool = False):
    """kernels.py:140-157."""
    groups = pad_len(cols, 6) // 3
    validate_tl2(index_plane, sign_plane, groups)
    if np.asarray(lut).shape[0] != groups:
        raise ValueError("group-count mismatch")
    if checked:
        nib, sgn = tl2_fields(index_plane, sign_plane, groups)
        vals = np.asarray(lut)[np.arange(groups)[None, :], nib.astype(np.intp)].astype(np.int16)
        vals = np.where(sgn.astype(bool), -vals, vals).astype(np.int16)
        return widened_sum(vals)
    return tl2_byte_gemv(index_plane, sign_plane, tl2_signed_table(lut))


WIDEN_GROUPS = 64  # kernels.py:34


def widened_sum(vals):
    """int16 partial sums folded every 64 groups, asserting |partial| <= 32767.

    Restates kernels.py:160-173.
    """
    vals = np.asarray(vals, dtype=np.int64)
    rows, groups = vals.shape
    blocks = -(-groups // WIDEN_GROUPS)
    padded = np.zeros((rows, blocks * WIDEN_GROUPS), dtype=np.int64)
    padded[:, :groups] = vals
    running = np.cumsum(padded.reshape(rows, blocks, WIDEN_GROUPS), axis=2)
    peak = int(np.abs(running).max()) if running.size else 0
    if peak > 32767:
        raise AssertionError(f"16-bit partial sum overflow: |{peak}| > 32767")
    return running[:, :, -1].sum(axis=1).astype(np.int32)


_ROW_BLOCK = 64  # kernels.py:178


def row_bounds(rows: int, thread_count: int):
    """Contiguous row chunks snapped to 64-row edges (kernels.py:181-186)."""
    n = max(1, min(thread_count, rows))
    edges = np.linspace(0, rows, n + 1, dtype=int)
    snapped = [0] + [min(rows, int(e) // _ROW_BLOCK * _ROW_BLOCK)
                     for e in edges[1:-1]] + [rows]
    return [(lo, hi) for lo, hi in zip(snapped[:-1], snapped[1:]) if hi > lo]


# ---------------------------------------------------------------------------
# cross-kernel harness   (verify.py)
# ---------------------------------------------------------------------------

KERNEL_PAD = {"ref_int32": 1, "i2s": 4, "tl1": 2, "tl2": 3}  # runtime.py:32-37


def check_instance(values, x):
    """Accumulators of every packed kernel on one instance (verify.py:17-33)."""
    values = np.asarray(values, dtype=np.int8)
    cols = values.shape[1]
    ref = gemv_ref_int32(values, quantize(x, 1)[0])
    q4 = quantize(x, 4)[0]
    q2, _, n2 = quantize(x, 2)
    q3, _, n3 = quantize(x, 3)
    r_i2s = gemv_i2s(encode_i2s(values), cols, q4)
    g1 = pad_len(cols, 2) // 2
    r_tl1 = gemv_tl1(encode_tl1(values), cols, lut_tl1(q2, n2, g1))
    ip, sp = encode_tl2(values)
    g2 = pad_len(cols, 6) // 3
    r_tl2 = gemv_tl2(ip, sp, cols, lut_tl2(q3, n3, g2))
    return {"ref": ref, "i2s": r_i2s, "tl1": r_tl1, "tl2": r_tl2}


def instance_shape(i: int, rng):
    """verify.py:36-42 shape schedule."""
    if i % 8 == 7:
        return int(rng.integers(1, 65)), int(rng.integers(1, 513))
    j = i % 128
    return j // 16 + 1, j % 16 + 1


def cross_kernel_instances(instances: int, seed: int = 0):
    """Yield the (values, scale, x) instances of verify.py:45-64, in order."""
    rng = np.random.default_rng(seed)
    for i in range(instances):
        rows, cols = instance_shape(i, rng)
        vals = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
        scale = float(rng.uniform(0.1, 2.0))
        x = rng.standard_normal(cols) * float(rng.uniform(0.01, 10.0))
        yield vals, scale, x


# ---------------------------------------------------------------------------
# workloads + toy decoder   (runtime.py) -- for the lossless protocol
# ---------------------------------------------------------------------------

APPENDIX_A = [  # runtime.py:54-67 (name, hidden, intermediate, layers, heads)
    ("125M", 768, 3072, 11, 12), ("350M", 1024, 3072, 24, 16),
    ("700M", 1536, 4096, 24, 16), ("1B", 2048, 3584, 24, 32),
    ("1.5B", 1536, 9216, 28, 32), ("2.5B", 2560, 6912, 30, 20),
    ("3.8B", 3840, 8192, 24, 32), ("7B", 4096, 12032, 32, 32),
    ("13B", 5120, 13824, 40, 40), ("30B", 6656, 16384, 60, 52),
    ("70B", 8192, 24576, 80, 64), ("100B", 8192, 45568, 72, 64),
]


def toy_decoder(vocab_size=256, depth=4, hidden=64, seed=0):
    """Weights of runtime.ToyDecoder.build (runtime.py:117-128)."""
    rng = np.random.default_rng(seed)
    emb = rng.standard_normal((vocab_size, hidden))
    layers = [ternarize(rng.standard_normal(hidden * hidden), hidden, hidden)
              for _ in range(depth)]
    head = ternarize(rng.standard_normal(vocab_size * hidden), vocab_size, hidden)
    return emb, layers, head


def toy_decode(emb, layers, head, prompt: int, steps: int):
    """Greedy decode with the int32 oracle (runtime.py:163-188)."""
    token = prompt
    out = []
    for _ in range(steps):
        x = emb[token].astype(np.float64)
        for vals, ws in layers:
            d, s, _ = quantize(x, 1)
            x = np.maximum(make_output(gemv_ref_int32(vals, d), ws, s), 0.0)
        d, s, _ = quantize(x, 1)
        logits = make_output(gemv_ref_int32(head[0], d), head[1], s)
        token = int(np.argmax(logits))
        out.append(token)
    return out
