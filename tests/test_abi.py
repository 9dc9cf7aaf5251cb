"""CPU checks of the drop-in boundary: the C-ABI library loads and exports
every entry point include/ternary_b200.h declares, and the pure host-side
size/shape arithmetic matches the reference formulas (no GPU needed)."""

import re
from pathlib import Path

import pytest

from oracle import ternpack_oracle as O

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "ternary_b200.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tb_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2410_16144_b200 import _lib as L
    from paper_2410_16144_b200.build import LIB, build
    if not LIB.exists():
        build()
    return L.load()


def test_header_symbols_exported(lib):
    names = declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header(lib):
    from paper_2410_16144_b200 import _lib as L
    assert set(declared()) <= set(L.declared_symbols())


def test_host_only_entry_points(lib):
    assert lib.tb_abi_version() == 4
    assert lib.tb_strerror(0) == b"ok"
    assert b"argument" in lib.tb_strerror(1)
    for cols in (1, 2, 3, 4, 5, 6, 7, 12, 13, 768, 4096, 4092, 14336, 10240, 32768):
        assert lib.tb_ref_row_bytes(1, cols) * 3 == O.i2s_bytes(3, cols)
        assert lib.tb_ref_row_bytes(2, cols) * 3 == O.tl1_bytes(3, cols)
        ib, sb = O.tl2_bytes(3, cols)
        assert lib.tb_ref_row_bytes(3, cols) * 3 == ib
        assert lib.tb_ref_sign_row_bytes(cols) * 3 == sb
        for fmt in (1, 2, 3):
            chunks = lib.tb_tiled_chunks(fmt, cols)
            assert chunks * 16 >= lib.tb_ref_row_bytes(fmt, cols) > (chunks - 1) * 16
            assert lib.tb_tiled_bytes(fmt, 33, cols) == 64 * chunks * 16
        assert lib.tb_tiled_sign_bytes(3, 33, cols) == 64 * lib.tb_tiled_chunks(3, cols) * 4
    assert lib.tb_ref_row_bytes(9, 10) == -1 and lib.tb_tiled_bytes(1, 0, 10) == -1
    # null-pointer argument checks never touch the device
    assert lib.tb_gemv(1, None, None, 4, 4, None, 1, 4, 4, None, 1.0, None, None, None, None,
                       None) == 1
    assert lib.tb_encode(1, None, 1, 1, None, None, None) == 1


def test_tiled_layout_is_a_granule_permutation():
    """The tiled layout holds exactly the reference bytes (+ zero-weight
    padding): replay tb_repack's index map on the host."""
    rng = __import__("numpy").random.default_rng(0)
    import numpy as np
    for rows, cols in ((1, 1), (33, 100), (64, 4096), (5, 1000)):
        v = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
        ref = O.encode_i2s(v)
        rb = ref.shape[1]
        C = -(-rb // 16)
        T = -(-rows // 32)
        tiled = np.full((T, C, 32, 16), 0x55, np.uint8)
        for r in range(rows):
            for j in range(rb):
                tiled[r // 32, j // 16, r % 32, j % 16] = ref[r, j]
        # every reference byte appears exactly once, padding decodes to 0 weights
        assert np.sort(tiled.ravel())[-ref.size:].size == ref.size
        pad = tiled.size - ref.size
        assert (tiled == 0x55).sum() >= pad
