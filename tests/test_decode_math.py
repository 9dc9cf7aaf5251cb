"""CPU emulation of the GEMV kernel's SIMD-within-a-register decode.

gemv.cu decodes packed bytes with 32-bit word arithmetic (no per-byte
branches).  These tests replay exactly that arithmetic in NumPy uint32 over
every possible input byte/nibble/sign combination and compare the recovered
weights with the oracle's decoders, so a wrong constant is caught before any
GPU time is spent.
"""

import itertools

import numpy as np

from oracle import ternpack_oracle as O

U = np.uint32


def prmt_sign_replicate(x):
    """prmt(x, 0, 0xBA98): byte b = 0xFF if bit 7 of byte b of x else 0x00."""
    out = U(0)
    for b in range(4):
        if (int(x) >> (8 * b + 7)) & 1:
            out |= U(0xFF << (8 * b))
    return out


def bytes_of(w):
    return [(int(w) >> (8 * b)) & 0xFF for b in range(4)]


def test_i2s_slot_masks():
    # byte b of (W & (3 << 2s)) / 4^s = code of weight 4b+s of this word
    for byte in range(256):
        W = U(byte * 0x01010101)
        for s in range(4):
            x = int(W & U(0x03030303 << (2 * s)))
            for b in range(4):
                assert ((x >> (8 * b)) & 0xFF) >> (2 * s) == (byte >> (2 * s)) & 3


def test_tl1_word_decode_all_nibble_pairs():
    for n0, n1, n2, n3 in itertools.product(range(9), repeat=4):
        # four bytes, each with a low nibble (pair 2b) and a high nibble (pair 2b+1)
        lo_n = [n0, n1, n2, n3]
        hi_n = [n3, n2, n1, n0]
        W = U(sum((lo_n[b] | (hi_n[b] << 4)) << (8 * b) for b in range(4)))
        lo = W & U(0x0F0F0F0F)
        hi = (W >> U(4)) & U(0x0F0F0F0F)
        for x, nib in ((lo, lo_n), (hi, hi_n)):
            q = ((x * U(11)) >> U(5)) & U(0x03030303)
            r = x - U(3) * q
            for b in range(4):
                assert bytes_of(q)[b] == nib[b] // 3
                assert bytes_of(r)[b] == nib[b] % 3


def tl2_bit(t, k):
    """csrc/common.cuh tl2_bit: (word, bit) of bit k of triple t's 5-bit value
    in a row chunk's five tile words (X0..X3 main, X4 sign plane)."""
    i, b, h = t >> 3, (t >> 1) & 3, t & 1
    j = 2 * i + h
    if j < 5:
        return j, 8 * b + k
    if j == 5:
        return (0, 8 * b + 5 + k) if k < 3 else (1, 8 * b + 2 + k)
    if j == 6:
        return (2, 8 * b + 5 + k) if k < 3 else (3, 8 * b + 2 + k)
    if k < 3:
        return 4, 8 * b + 5 + k
    return (1, 8 * b + 7) if k == 3 else (3, 8 * b + 7)


def test_tl2_tile_layout():
    """The tiled TL2 row chunk: 32 triples x 5 bits fill the five words exactly
    once, and the decode's masks and shifts (common.cuh tl2_tile_groups) put
    group j's four values in the byte lanes of one register."""
    slots = [tl2_bit(t, k) for t in range(32) for k in range(5)]
    assert sorted(slots) == [(w, b) for w in range(5) for b in range(32)]
    rng = np.random.default_rng(0)
    for _ in range(200):
        v = rng.integers(0, 27, 32)
        X = [0] * 5
        for t in range(32):
            for k in range(5):
                w, bit = tl2_bit(t, k)
                X[w] |= ((int(v[t]) >> k) & 1) << bit
        g = [X[j] & 0x1F1F1F1F for j in range(5)]
        g.append(((X[0] >> 5) & 0x07070707) | ((X[1] >> 2) & 0x18181818))
        g.append(((X[2] >> 5) & 0x07070707) | ((X[3] >> 2) & 0x18181818))
        g.append(((X[4] >> 5) & 0x07070707) | ((X[1] >> 4) & 0x08080808) | ((X[3] >> 3) & 0x10101010))
        for j in range(8):
            i, h = j >> 1, j & 1
            for b in range(4):
                assert (g[j] >> (8 * b)) & 0xFF == v[8 * i + 2 * b + h], (j, b)


def test_tl2_triple_decode_all_codes():
    # every (sign, index) incl. the canonical codes; 4 triples per word lane
    codes = [(0, 0)] + [(s, i) for s in (0, 1) for i in range(1, 14)]
    for quad in itertools.product(codes, repeat=2):
        lanes = [quad[0], quad[1], quad[1], quad[0]]
        x = U(sum(idx << (8 * b) for b, (_, idx) in enumerate(lanes)))
        msk = U(sum((0xFF if s else 0) << (8 * b) for b, (s, _) in enumerate(lanes)))
        P = (x + U(0x0D0D0D0D)) & U(0xFFFFFFFF)
        Q = (U(0x0D0D0D0D) - x) & U(0xFFFFFFFF)
        d = (P & ~msk) | (Q & msk)
        c0 = (((d * U(7) + U(0x07070707)) & U(0xFFFFFFFF)) >> U(6)) & U(0x03030303)
        r = (d - U(9) * c0) & U(0xFFFFFFFF)
        c1 = (((r * U(11)) & U(0xFFFFFFFF)) >> U(5)) & U(0x03030303)
        c2 = (r - U(3) * c1) & U(0xFFFFFFFF)
        for b, (s, idx) in enumerate(lanes):
            ip = np.array([[idx]], np.uint8)
            sp = np.array([[s]], np.uint8)
            want = O.decode_tl2(ip, sp, 3)[0] if not (s and idx == 0) else None
            if want is None:
                continue
            got = [bytes_of(c0)[b] - 1, bytes_of(c1)[b] - 1, bytes_of(c2)[b] - 1]
            assert got == want.tolist(), (s, idx)


def test_activation_permutation_covers_chunk():
    # word 4i+s holds a[16i+4j+s] (I2_S/TL1); word 6i+s holds a[24i+6j+s] (TL2)
    for width, G in ((64, 4), (96, 6)):
        seen = sorted(i * 4 * G + s + G * j for i in range(4) for s in range(G) for j in range(4))
        assert seen == list(range(width))


def test_tl2_biased_digits():
    """gemv_records.cuh: with d = v + 1 in every byte lane, (7 d) >> 6 = v / 9,
    r = d - 9 c0 = v % 9 + 1, (10 r) >> 5 = (v % 9) / 3 and r - 3 c1 = v % 3 + 1,
    as whole-word multiplies (no lane reaches into its neighbour's low bits)."""
    rng = np.random.default_rng(1)
    cases = [np.array([v] * 4) for v in range(27)] + [rng.integers(0, 27, 4) for _ in range(500)]
    for v in cases:
        d = sum((int(x) + 1) << (8 * b) for b, x in enumerate(v))
        c0 = (((d * 7) & 0xFFFFFFFF) >> 6) & 0x03030303
        r = d - 9 * c0
        c1 = (((r * 10) & 0xFFFFFFFF) >> 5) & 0x03030303
        c2 = r - 3 * c1
        for b, x in enumerate(v):
            x = int(x)
            assert bytes_of(c0)[b] == x // 9 and bytes_of(c1)[b] == (x % 9) // 3
            assert bytes_of(c2)[b] == x % 3 + 1


def test_tl2_third_digit_by_linearity():
    """gemv_records.cuh, one-token TL2: the second digit stays unshifted
    (c1s = (10 r) & 0x60 per lane = 32 c1) and the third is never formed:
    sum (c2 + 1) a2 = sum r a2 - 3 sum c1 a2, folded as
    v0 + v1s / 32 + v2 - 3 v5s / 32 (Acc::total), for whole words of four
    triples against int8 activations."""
    rng = np.random.default_rng(2)
    dp4a = lambda u, a: sum(int(x) * int(y) for x, y in zip(u, a))  # noqa: E731
    for _ in range(400):
        v = rng.integers(0, 27, 4)
        a0, a1, a2 = (rng.integers(-127, 128, 4) for _ in range(3))
        d = sum((int(x) + 1) << (8 * b) for b, x in enumerate(v))
        c0 = (((d * 7) & 0xFFFFFFFF) >> 6) & 0x03030303
        r = d - 9 * c0
        c1s = ((r * 10) & 0xFFFFFFFF) & 0x60606060
        assert [b // 32 for b in bytes_of(c1s)] == [(int(x) % 9) // 3 for x in v]
        s0, s1, s2, s5 = (dp4a(bytes_of(c0), a0), dp4a(bytes_of(c1s), a1),
                          dp4a(bytes_of(r), a2), dp4a(bytes_of(c1s), a2))
        assert s1 % 32 == 0 and s5 % 32 == 0
        got = s0 + (s1 >> 5) + s2 - 3 * (s5 >> 5)
        want = sum((int(x) // 9) * int(p) + ((int(x) % 9) // 3) * int(q) + (int(x) % 3 + 1) * int(t)
                   for x, p, q, t in zip(v, a0, a1, a2))
        assert got == want
