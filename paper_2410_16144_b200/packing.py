"""Bit-exact I2_S / TL1 / TL2 packed weights on the GPU.

Mirrors ``ternpack.packing`` (pkg/src/ternpack/packing.py): the ``data`` /
``index_data`` / ``sign_data`` tensors hold the reference's exact bytes
(row-major, rows byte-aligned, little-endian within a byte).  Each packed
matrix also carries the GEMV's tiled layout (include/ternary_b200.h), built
once by ``tb_repack`` -- the "offline packer" -- and cached on the object.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _lib as L
from .core import TernaryMatrix, to_device

__all__ = [
    "PackedI2S", "PackedTL1", "PackedTL2",
    "encode_i2s", "decode_i2s", "encode_tl1", "decode_tl1", "encode_tl2", "decode_tl2",
    "tl1_index", "tl2_code", "i2s_payload_bytes", "tl1_payload_bytes", "tl2_payload_bytes",
]

TL1_ZERO_INDEX = 4  # packing.py:35


def _pad_up(n: int, m: int) -> int:
    return -(-n // m) * m


def i2s_payload_bytes(rows: int, cols: int) -> int:          # packing.py:42-43
    return rows * (_pad_up(cols, 4) // 4)


def tl1_payload_bytes(rows: int, cols: int) -> int:          # packing.py:46-47
    return rows * -(-(_pad_up(cols, 2) // 2) // 2)


def tl2_payload_bytes(rows: int, cols: int) -> tuple[int, int]:  # packing.py:50-53
    pc = _pad_up(cols, 6)
    return rows * (pc // 6), rows * -(-(pc // 3) // 8)


def tl1_index(w0: int, w1: int) -> int:                      # packing.py:56-60
    if w0 not in (-1, 0, 1) or w1 not in (-1, 0, 1):
        raise ValueError("weights must be ternary")
    return 3 * (w0 + 1) + (w1 + 1)


def tl2_code(w0: int, w1: int, w2: int) -> tuple[int, int]:  # packing.py:63-74
    for w in (w0, w1, w2):
        if w not in (-1, 0, 1):
            raise ValueError("weights must be ternary")
    d = 9 * (w0 + 1) + 3 * (w1 + 1) + (w2 + 1) - 13
    return (1 if d < 0 else 0, abs(d))


class _TiledMixin:
    """Lazily built tiled GEMV layout + per-stream self-cleaning workspaces."""

    FMT = 0

    def _sign_ref(self):
        return None

    def _main_ref(self):
        raise NotImplementedError

    def tiled(self):
        t = self._cache.get("tiled")
        if t is None:
            lib = L.load()
            dev = self._main_ref().device
            nb = lib.tb_tiled_bytes(self.FMT, self.rows, self.cols)
            sb = lib.tb_tiled_sign_bytes(self.FMT, self.rows, self.cols)
            main = torch.empty(nb, dtype=torch.uint8, device=dev)
            sign = torch.empty(max(sb, 16), dtype=torch.uint8, device=dev) if sb else None
            L.check(lib.tb_repack(self.FMT, L.ptr(self._main_ref()), L.ptr(self._sign_ref()),
                                  self.rows, self.cols, L.ptr(main), L.ptr(sign),
                                  L.stream_ptr()), "repack")
            t = (main, sign)
            self._cache["tiled"] = t
        return t

    def workspace(self, stream=None):
        key = ("ws", L.stream_ptr(stream))
        w = self._cache.get(key)
        if w is None:
            nbytes = L.load().tb_gemv_workspace_bytes(self.FMT, self.rows, self.cols)
            w = torch.zeros(nbytes // 4, dtype=torch.int32, device=self._main_ref().device)
            self._cache[key] = w
        return w

    def drop_reference_bytes(self):
        """Keep only the tiled layout (halves resident memory for big stacks)."""
        self.tiled()
        self._cache["ref_dropped"] = True


def _first_bad(fmt, data, sign, rows, cols):
    lib = L.load()
    fb = torch.full((2,), 2**31 - 1, dtype=torch.int32, device=data.device)
    L.check(lib.tb_validate(fmt, L.ptr(data), L.ptr(sign), rows, cols, L.ptr(fb),
                            L.stream_ptr()), "validate")
    return [int(v) for v in fb.cpu()]


@dataclass(frozen=True)
class PackedI2S(_TiledMixin):
    """2-bit codes (w + 1), four weights per byte; code 0b11 is reserved."""

    rows: int
    cols: int
    padded_cols: int
    data: torch.Tensor  # uint8 [rows, padded_cols // 4]
    scale: float
    trusted: bool = field(default=False, compare=False, repr=False)
    _cache: dict = field(default_factory=dict, compare=False, repr=False)
    FMT = L.I2S

    def __post_init__(self):
        if self.padded_cols != _pad_up(self.cols, 4):
            raise ValueError("padded_cols must be cols rounded up to a multiple of 4")
        d = to_device(self.data, torch.uint8).reshape(self.rows, self.padded_cols // 4)
        object.__setattr__(self, "data", d.contiguous())

    def _main_ref(self):
        return self.data

    @property
    def bytes_per_row(self) -> int:
        return self.padded_cols // 4

    def validate(self) -> None:
        bad, _ = _first_bad(L.I2S, self.data, None, self.rows, self.cols)
        if bad < 2**31 - 1:
            raise ValueError(f"invalid I2_S code at row {bad}")
        object.__setattr__(self, "trusted", True)


@dataclass(frozen=True)
class PackedTL1(_TiledMixin):
    """4-bit pair indices in [0, 8], two per byte."""

    rows: int
    cols: int
    padded_cols: int
    data: torch.Tensor  # uint8 [rows, ceil(padded_cols/2 / 2)]
    scale: float
    trusted: bool = field(default=False, compare=False, repr=False)
    _cache: dict = field(default_factory=dict, compare=False, repr=False)
    FMT = L.TL1

    def __post_init__(self):
        if self.padded_cols != _pad_up(self.cols, 2):
            raise ValueError("padded_cols must be cols rounded up to a multiple of 2")
        d = to_device(self.data, torch.uint8).reshape(self.rows, self.bytes_per_row)
        object.__setattr__(self, "data", d.contiguous())

    def _main_ref(self):
        return self.data

    @property
    def groups(self) -> int:
        return self.padded_cols // 2

    @property
    def bytes_per_row(self) -> int:
        return -(-self.groups // 2)

    def validate(self) -> None:
        bad, _ = _first_bad(L.TL1, self.data, None, self.rows, self.cols)
        if bad < 2**31 - 1:
            raise ValueError(f"invalid TL1 index at row {bad}")
        object.__setattr__(self, "trusted", True)


@dataclass(frozen=True)
class PackedTL2(_TiledMixin):
    """Per triple: one 4-bit index in [0, 13] plus one sign bit, separate planes."""

    rows: int
    cols: int
    padded_cols: int
    index_data: torch.Tensor  # uint8 [rows, padded_cols // 6]
    sign_data: torch.Tensor   # uint8 [rows, ceil(padded_cols/3 / 8)]
    scale: float
    trusted: bool = field(default=False, compare=False, repr=False)
    _cache: dict = field(default_factory=dict, compare=False, repr=False)
    FMT = L.TL2

    def __post_init__(self):
        if self.padded_cols != _pad_up(self.cols, 6):
            raise ValueError("padded_cols must be cols rounded up to a multiple of 6")
        i = to_device(self.index_data, torch.uint8).reshape(self.rows, self.index_bytes_per_row)
        s = to_device(self.sign_data, torch.uint8).reshape(self.rows, self.sign_bytes_per_row)
        object.__setattr__(self, "index_data", i.contiguous())
        object.__setattr__(self, "sign_data", s.contiguous())

    def _main_ref(self):
        return self.index_data

    def _sign_ref(self):
        return self.sign_data

    @property
    def groups(self) -> int:
        return self.padded_cols // 3

    @property
    def index_bytes_per_row(self) -> int:
        return self.padded_cols // 6

    @property
    def sign_bytes_per_row(self) -> int:
        return -(-self.groups // 8)

    def validate(self) -> None:
        bad, noncanon = _first_bad(L.TL2, self.index_data, self.sign_data, self.rows, self.cols)
        if bad < 2**31 - 1:
            raise ValueError(f"invalid TL2 index at row {bad}")
        if noncanon < 2**31 - 1:
            raise ValueError(f"non-canonical zero at row {noncanon}")
        object.__setattr__(self, "trusted", True)

    def data_nibbles(self) -> torch.Tensor:
        b = self.index_data
        out = torch.empty((self.rows, self.groups), dtype=torch.uint8, device=b.device)
        out[:, 0::2] = b & 15
        out[:, 1::2] = b >> 4
        return out

    def data_signs(self) -> torch.Tensor:
        bits = (self.sign_data.unsqueeze(-1) >> torch.arange(8, device=self.sign_data.device,
                                                             dtype=torch.uint8)) & 1
        return bits.reshape(self.rows, -1)[:, : self.groups]


# ---------------------------------------------------------------------------

def _encode(fmt, m: TernaryMatrix):
    lib = L.load()
    dev = m.values.device
    rb = lib.tb_ref_row_bytes(fmt, m.cols)
    out = torch.empty((m.rows, rb), dtype=torch.uint8, device=dev)
    sign = None
    if fmt == L.TL2:
        sign = torch.empty((m.rows, lib.tb_ref_sign_row_bytes(m.cols)), dtype=torch.uint8,
                           device=dev)
    L.check(lib.tb_encode(fmt, L.ptr(m.values), m.rows, m.cols, L.ptr(out), L.ptr(sign),
                          L.stream_ptr()), "encode")
    return out, sign


def _decode(fmt, data, sign, rows, cols):
    lib = L.load()
    vals = torch.empty((rows, cols), dtype=torch.int8, device=data.device)
    bad = torch.zeros(1, dtype=torch.int32, device=data.device)
    L.check(lib.tb_decode(fmt, L.ptr(data), L.ptr(sign), rows, cols, L.ptr(vals), L.ptr(bad),
                          L.stream_ptr()), "decode")
    return vals, int(bad.item())


def encode_i2s(m: TernaryMatrix) -> PackedI2S:               # packing.py:200-206
    d, _ = _encode(L.I2S, m)
    return PackedI2S(rows=m.rows, cols=m.cols, padded_cols=_pad_up(m.cols, 4), data=d,
                     scale=m.scale, trusted=True)


def decode_i2s(p: PackedI2S) -> TernaryMatrix:               # packing.py:209-219
    v, bad = _decode(L.I2S, p.data, None, p.rows, p.cols)
    if bad:
        raise ValueError("invalid I2_S code")
    return TernaryMatrix(rows=p.rows, cols=p.cols, values=v, scale=p.scale, _checked=True)


def encode_tl1(m: TernaryMatrix) -> PackedTL1:               # packing.py:222-233
    d, _ = _encode(L.TL1, m)
    return PackedTL1(rows=m.rows, cols=m.cols, padded_cols=_pad_up(m.cols, 2), data=d,
                     scale=m.scale, trusted=True)


def decode_tl1(p: PackedTL1) -> TernaryMatrix:               # packing.py:236-247
    v, bad = _decode(L.TL1, p.data, None, p.rows, p.cols)
    if bad:
        raise ValueError("invalid TL1 index")
    return TernaryMatrix(rows=p.rows, cols=p.cols, values=v, scale=p.scale, _checked=True)


def encode_tl2(m: TernaryMatrix) -> PackedTL2:               # packing.py:250-262
    d, s = _encode(L.TL2, m)
    return PackedTL2(rows=m.rows, cols=m.cols, padded_cols=_pad_up(m.cols, 6), index_data=d,
                     sign_data=s, scale=m.scale, trusted=True)


def decode_tl2(p: PackedTL2) -> TernaryMatrix:               # packing.py:265-277
    v, bad = _decode(L.TL2, p.index_data, p.sign_data, p.rows, p.cols)
    if bad & 1:
        raise ValueError("invalid TL2 index")
    if bad & 2:
        raise ValueError("non-canonical zero")
    return TernaryMatrix(rows=p.rows, cols=p.cols, values=v, scale=p.scale, _checked=True)
