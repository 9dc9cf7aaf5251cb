"""TPK1 container: the host parser against files and
error cases written by the reference itself (tests/golden/tpk_golden.json,
from make_tpk_golden.py): same payload bytes, same TpkError messages and
byte offsets.  The device loaders are checked in the GPU part."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import ternpack_oracle as O
from paper_2410_16144_b200 import container as C

GOLD = json.loads((Path(__file__).parent / "golden" / "tpk_golden.json").read_text())


def _values():
    return [(m["name"], m["rows"], m["cols"], m["scale"],
             np.array(m["values"], dtype=np.int8).reshape(m["rows"], m["cols"]))
            for m in GOLD["matrices"]]


def _encode(fmt, v):
    if fmt == "i2s":
        return (O.encode_i2s(v),)
    if fmt == "tl1":
        return (O.encode_tl1(v),)
    return O.encode_tl2(v)


@pytest.mark.parametrize("fmt", ["i2s", "tl1", "tl2"])
def test_parse_reference_files(fmt):
    blob = bytes.fromhex(GOLD["files"][fmt])
    got_fmt, mats = C.parse_model(blob)
    assert got_fmt == fmt and len(mats) == len(GOLD["matrices"])
    for m, (name, r, c, scale, v) in zip(mats, _values()):
        assert (m.name, m.rows, m.cols) == (name, r, c)
        assert m.scale == np.float32(scale)
        for got, want in zip(m.payloads, _encode(fmt, v)):
            assert np.array_equal(got, want.reshape(-1))


@pytest.mark.parametrize("case", range(len(GOLD["errors"])))
def test_error_messages_and_offsets(case):
    e = GOLD["errors"][case]
    with pytest.raises(C.TpkError) as info:
        C.parse_model(bytes.fromhex(e["blob"]))
    assert str(info.value) == e["message"], e["case"]
    assert info.value.offset == e["offset"], e["case"]


def test_format_tables():
    assert C.FORMAT_CODES == {"i2s": 1, "tl1": 2, "tl2": 3}
    assert C.BITS_PER_WEIGHT["tl2"] == 5.0 / 3.0
