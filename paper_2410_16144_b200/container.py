"""TPK1 model files (mirrors ternpack.container, pkg/src/ternpack/container.py).

On-disk format (little-endian), as the reference writes it:
``"TPK1"``, u16 version = 1, u8 format (1 I2_S / 2 TL1 / 3 TL2), u32 count;
per matrix: u16 name length, UTF-8 name, u32 rows, u32 cols, f32 scale,
u32 payload length (TL2: u32 index length, u32 sign length), payload bytes
(TL2: index plane, then sign plane).  Payload lengths must equal the
packing size formulas (packing.py:42-53).

parse_model() is the host-side structural check (same TpkError messages and
byte offsets as container.py:88-160).  read_model() returns device-resident
packed matrices (untrusted: the kernels validate them); load_model() goes
straight to the GEMV operand -- one pinned staging copy per payload,
device-side validate() (the reference's error text, first bad row) and the
tiled repack, so a model is ready for GemvPlan / GemvStep on return.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from .packing import (
    PackedI2S,
    PackedTL1,
    PackedTL2,
    i2s_payload_bytes,
    tl1_payload_bytes,
    tl2_payload_bytes,
)

__all__ = ["TpkError", "RawMatrix", "parse_model", "read_model", "load_model", "write_model",
           "FORMAT_CODES", "FORMAT_NAMES", "BITS_PER_WEIGHT"]

MAGIC = b"TPK1"
VERSION = 1
FORMAT_CODES = {"i2s": 1, "tl1": 2, "tl2": 3}
FORMAT_NAMES = {code: name for name, code in FORMAT_CODES.items()}
BITS_PER_WEIGHT = {"i2s": 2.0, "tl1": 2.0, "tl2": 5.0 / 3.0}
_PACKED = {"i2s": PackedI2S, "tl1": PackedTL1, "tl2": PackedTL2}


class TpkError(Exception):
    """Corrupt or malformed TPK1 data; ``offset`` is the first offending byte."""

    def __init__(self, message: str, offset: int):
        super().__init__(f"{message} (at offset {offset})")
        self.offset = offset


@dataclass(frozen=True)
class RawMatrix:
    name: str
    rows: int
    cols: int
    scale: float
    payloads: tuple  # host uint8 arrays (views into the file image)


def _expected_lengths(fmt: str, rows: int, cols: int):
    if fmt == "tl2":
        return tuple(tl2_payload_bytes(rows, cols))
    return ((i2s_payload_bytes if fmt == "i2s" else tl1_payload_bytes)(rows, cols),)


def parse_model(blob) -> tuple[str, list[RawMatrix]]:
    """Structural parse of a TPK1 image (container.py:104-160 semantics)."""
    buf = memoryview(blob)
    end = len(buf)
    pos = 0

    def field(fmt: str, what: str):
        nonlocal pos
        size = struct.calcsize(fmt)
        if pos + size > end:
            raise TpkError(f"truncated file while reading {what}", pos)
        vals = struct.unpack_from(fmt, buf, pos)
        pos += size
        return vals

    def span(n: int, what: str):
        nonlocal pos
        if pos + n > end:
            raise TpkError(f"truncated file while reading {what}", pos)
        view = buf[pos: pos + n]
        pos += n
        return view

    if bytes(span(4, "magic")) != MAGIC:
        raise TpkError("bad magic", 0)
    (version,) = field("<H", "version")
    if version != VERSION:
        raise TpkError(f"unsupported version {version}", pos - 2)
    (code,) = field("<B", "format")
    if code not in FORMAT_NAMES:
        raise TpkError(f"unknown format code {code}", pos - 1)
    fmt = FORMAT_NAMES[code]
    (count,) = field("<I", "matrix count")
    out = []
    for i in range(count):
        (nlen,) = field("<H", f"matrix {i} name length")
        name = bytes(span(nlen, f"matrix {i} name")).decode("utf-8")
        at = pos
        rows, cols, scale = field("<IIf", f"matrix {i} header")
        if rows < 1 or cols < 1:
            raise TpkError(f"matrix {i} has empty dimensions", at)
        if not (scale > 0 and np.isfinite(scale)):
            raise TpkError(f"matrix {i} has invalid scale", at + 8)
        at = pos
        if fmt == "tl2":
            lengths = field("<II", f"matrix {i} payload lengths")
            what = (f"matrix {i} index payload", f"matrix {i} sign payload")
        else:
            lengths = field("<I", f"matrix {i} payload length")
            what = (f"matrix {i} payload",)
        if tuple(lengths) != _expected_lengths(fmt, rows, cols):
            raise TpkError(f"matrix {i} payload length mismatch", at)
        payloads = tuple(np.frombuffer(span(n, w), dtype=np.uint8) for n, w in zip(lengths, what))
        out.append(RawMatrix(name, rows, cols, float(scale), payloads))
    if pos != end:
        raise TpkError("trailing bytes after last matrix", pos)
    return fmt, out


def _to_packed(fmt: str, m: RawMatrix, device, trusted: bool = False):
    """Payload bytes -> device Packed* through one pinned staging buffer."""
    dev_planes = []
    for plane in m.payloads:
        staged = torch.from_numpy(np.array(plane, copy=True)).pin_memory()
        dev_planes.append(staged.to(device, non_blocking=True))
    if fmt == "tl2":
        return PackedTL2(rows=m.rows, cols=m.cols, padded_cols=-(-m.cols // 6) * 6,
                         index_data=dev_planes[0], sign_data=dev_planes[1], scale=m.scale,
                         trusted=trusted)
    pad = 4 if fmt == "i2s" else 2
    return _PACKED[fmt](rows=m.rows, cols=m.cols, padded_cols=-(-m.cols // pad) * pad,
                        data=dev_planes[0], scale=m.scale, trusted=trusted)


def read_model(path, device=None) -> tuple[str, list[tuple[str, object]]]:
    """(format, [(name, packed matrix on the GPU)]); structurally sound, not
    content-validated (the kernels validate untrusted matrices)."""
    from .core import device as default_device
    dev = device or default_device()
    fmt, raw = parse_model(Path(path).read_bytes())
    return fmt, [(m.name, _to_packed(fmt, m, dev)) for m in raw]


def load_model(path, device=None) -> tuple[str, list[tuple[str, object]]]:
    """read_model + device-side validate() (raises the reference's
    "invalid ... at row r" ValueError) + the tiled GEMV layout built, so the
    matrices are ready for GemvPlan / GemvStep."""
    fmt, mats = read_model(path, device)
    for _, p in mats:
        p.validate()
        p.tiled()
    return fmt, mats


def write_model(path, matrices: list[tuple[str, object]]) -> None:
    """Named packed matrices (device or host), all of one format -> TPK1."""
    if not matrices:
        raise ValueError("no matrices to write")
    kinds = {PackedI2S: "i2s", PackedTL1: "tl1", PackedTL2: "tl2"}

    def fmt_of(p):
        for cls, name in kinds.items():
            if isinstance(p, cls):
                return name
        raise TypeError(f"not a packed matrix: {type(p).__name__}")

    fmt = fmt_of(matrices[0][1])
    parts = [MAGIC, struct.pack("<HBI", VERSION, FORMAT_CODES[fmt], len(matrices))]
    for name, p in matrices:
        if fmt_of(p) != fmt:
            raise ValueError("all matrices in one file must share a format")
        nb = name.encode("utf-8")
        parts += [struct.pack("<H", len(nb)), nb, struct.pack("<IIf", p.rows, p.cols, p.scale)]
        planes = (p.index_data, p.sign_data) if fmt == "tl2" else (p.data,)
        blobs = [t.detach().cpu().numpy().tobytes() if isinstance(t, torch.Tensor)
                 else np.asarray(t, dtype=np.uint8).tobytes() for t in planes]
        parts.append(struct.pack("<" + "I" * len(blobs), *map(len, blobs)))
        parts += blobs
    Path(path).write_bytes(b"".join(parts))
