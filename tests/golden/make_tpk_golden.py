"""Golden TPK1 files and TpkError cases, written by the REAL reference
(ternpack.container, pkg/src/ternpack/container.py) in the build container:

    python tests/golden/make_tpk_golden.py

Writes tests/golden/tpk_golden.json: for each format one valid file (hex)
with the matrices' ternary values, plus corrupted variants with the exact
(message, offset) the reference's read_model raises.  Tests read only the
JSON; nothing here runs at test time.
"""

from __future__ import annotations

import json
import struct
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import ternpack as tp  # noqa: E402  (the reference itself)
from ternpack import container as tc  # noqa: E402


def _file(fmt, mats):
    enc = {"i2s": tp.encode_i2s, "tl1": tp.encode_tl1, "tl2": tp.encode_tl2}[fmt]
    with tempfile.TemporaryDirectory() as d:
        path = Path(d) / "m.tpk"
        tc.write_model(path, [(name, enc(m)) for name, m in mats])
        return path.read_bytes()


def _error(blob):
    with tempfile.TemporaryDirectory() as d:
        path = Path(d) / "bad.tpk"
        path.write_bytes(blob)
        try:
            tc.read_model(path)
        except tc.TpkError as e:
            return str(e), e.offset
    return None


def main():
    rng = np.random.default_rng(77)
    shapes = [("layer0.wq", 5, 37), ("layer0.wo", 3, 8), ("head", 7, 61)]
    mats, values = [], []
    for name, r, c in shapes:
        v = rng.integers(-1, 2, size=(r, c), dtype=np.int8)
        scale = float(np.float32(rng.uniform(0.01, 2.0)))
        mats.append((name, tp.TernaryMatrix(r, c, v, scale)))
        values.append({"name": name, "rows": r, "cols": c, "scale": scale,
                       "values": v.reshape(-1).tolist()})
    out = {"matrices": values, "files": {}, "errors": []}
    for fmt in ("i2s", "tl1", "tl2"):
        blob = _file(fmt, mats)
        out["files"][fmt] = blob.hex()
        # corruptions (header field offsets follow the documented layout)
        first = 4 + 2 + 1 + 4  # first matrix record
        name_len = struct.unpack_from("<H", blob, first)[0]
        dims = first + 2 + name_len
        lens = dims + 12
        cases = {
            "bad magic": b"XPK1" + blob[4:],
            "version": blob[:4] + struct.pack("<H", 2) + blob[6:],
            "format code": blob[:6] + bytes([9]) + blob[7:],
            "truncated header": blob[:5],
            "truncated name": blob[: first + 3],
            "truncated payload": blob[:-3],
            "zero rows": blob[:dims] + struct.pack("<I", 0) + blob[dims + 4:],
            "negative scale": blob[:dims + 8] + struct.pack("<f", -1.0) + blob[dims + 12:],
            "nan scale": blob[:dims + 8] + struct.pack("<f", float("nan")) + blob[dims + 12:],
            "length mismatch": blob[:lens] + struct.pack("<I", struct.unpack_from("<I", blob, lens)[0] + 1)
            + blob[lens + 4:],
            "trailing bytes": blob + b"\x00",
            "count too large": blob[:7] + struct.pack("<I", 4) + blob[11:],
        }
        for what, bad in cases.items():
            err = _error(bad)
            assert err is not None, (fmt, what)
            out["errors"].append({"format": fmt, "case": what, "blob": bad.hex(),
                                  "message": err[0], "offset": err[1]})
    (HERE / "tpk_golden.json").write_text(json.dumps(out, indent=1))
    print("wrote", HERE / "tpk_golden.json", len(out["errors"]), "error cases")


if __name__ == "__main__":
    main()
