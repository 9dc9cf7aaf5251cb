"""ternpack/_b200.py -- the B200 backend a ternpack maintainer would add.

This file is OURS (it is not reference code): the ctypes binding of
include/ternary_b200.h that INTEGRATION.md documents.  integration/
run_reference_tests.py copies it into a temporary copy of the unmodified
reference package (baseline/_ref) as ``ternpack/_b200.py`` and inserts the
dispatch lines into ``ternpack/kernels.py``; the reference's own test suite
then runs with its packed GEMVs on the GPU.

Only kernels.py's fast paths are redirected, after the reference's own
validation (validate(), _check_activation_cover, group-count checks):

  gemv_i2s(p, a)                      -> tb_gemv (LUT implicit, f64 outputs)
  gemv_tl1/gemv_tl2(p, lut, s)        -> tb_gemv_lut (reads the CALLER's LUT,
                                         so corrupted tables behave as on CPU)
  gemv_parallel(I2_S | TL1 | TL2, ..) -> the same, once for all rows (the
                                         GPU grid is the row partition)
The checked (widened int16) paths stay on the CPU: they exist to assert the
int16 discipline of the CPU tables (kernels.py:160-173).
PyTorch is used only for device memory and the stream.
"""

from __future__ import annotations

import atexit
import ctypes as C
import os

import numpy as np
import torch

from .core import GemvResult

_p, _i64, _i32, _f64 = C.c_void_p, C.c_int64, C.c_int32, C.c_double
_so = None
FMT = {"PackedI2S": 1, "PackedTL1": 2, "PackedTL2": 3}
_calls = [0]


def _count_at_exit():
    path = os.environ.get("TB_B200_COUNT_FILE")
    if path:
        with open(path, "w") as f:
            f.write(str(_calls[0]))


atexit.register(_count_at_exit)


def enabled() -> bool:
    return os.environ.get("TERNPACK_BACKEND") == "b200"


def _lib():
    global _so
    if _so is None:
        so = C.CDLL(os.environ.get("TERNARY_B200_LIB", "libternary_b200.so"))
        for name, res, args in (
                ("tb_tiled_bytes", _i64, [_i32, _i64, _i64]),
                ("tb_tiled_sign_bytes", _i64, [_i32, _i64, _i64]),
                ("tb_gemv_workspace_bytes", _i64, [_i32, _i64, _i64]),
                ("tb_repack", _i32, [_i32, _p, _p, _i64, _i64, _p, _p, _p]),
                ("tb_gemv", _i32, [_i32, _p, _p, _i64, _i64, _p, _i64, _i64, _i64, _p, _f64,
                                   _p, _p, _p, _p, _p]),
                ("tb_gemv_lut", _i32, [_i32, _p, _p, _i64, _i64, _p, _i64, _p, _p]),
                ("tb_strerror", C.c_char_p, [_i32])):
            f = getattr(so, name)
            f.restype, f.argtypes = res, args
        _so = so
    return _so


def _check(st):
    if st:
        raise RuntimeError(_lib().tb_strerror(st).decode())


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _operands(p):
    """Tiled device copy of a packed matrix, memoised on the frozen container
    (object.__setattr__, as the reference's own validate() does)."""
    ops = p.__dict__.get("_b200")
    if ops is None:
        so, dev = _lib(), torch.device("cuda")
        fmt = FMT[type(p).__name__]
        main = p.index_data if fmt == 3 else p.data
        ref = torch.from_numpy(np.array(main, dtype=np.uint8, copy=True)).to(dev)
        sref = (torch.from_numpy(np.array(p.sign_data, dtype=np.uint8, copy=True)).to(dev)
                if fmt == 3 else None)
        tiled = torch.empty(max(16, so.tb_tiled_bytes(fmt, p.rows, p.cols)), dtype=torch.uint8,
                            device=dev)
        tsign = (torch.empty(max(16, so.tb_tiled_sign_bytes(fmt, p.rows, p.cols)),
                             dtype=torch.uint8, device=dev) if fmt == 3 else None)
        ws = torch.zeros(so.tb_gemv_workspace_bytes(fmt, p.rows, p.cols), dtype=torch.uint8,
                         device=dev)
        _check(so.tb_repack(fmt, ref.data_ptr(), sref.data_ptr() if sref is not None else None,
                            p.rows, p.cols, tiled.data_ptr(),
                            tsign.data_ptr() if tsign is not None else None, _stream()))
        ops = (fmt, tiled, tsign, ws)
        object.__setattr__(p, "_b200", ops)
    return ops


def gemv(p, a) -> GemvResult:
    """The packed GEMV of gemv_i2s / gemv_parallel (LUT implicit): int32
    accumulators and float64 outputs (core.py:99-101) from the GPU."""
    so = _lib()
    _calls[0] += 1
    fmt, tiled, tsign, ws = _operands(p)
    dev = tiled.device
    act = torch.from_numpy(np.array(a.data, dtype=np.int8, copy=True)).to(dev)
    scale = torch.tensor([a.scale], dtype=torch.float64, device=dev)
    acc = torch.empty(p.rows, dtype=torch.int32, device=dev)
    out = torch.empty(p.rows, dtype=torch.float64, device=dev)
    _check(so.tb_gemv(fmt, tiled.data_ptr(), tsign.data_ptr() if tsign is not None else None,
                      p.rows, p.cols, act.data_ptr(), 1, act.numel(), act.numel(),
                      scale.data_ptr(), float(p.scale), ws.data_ptr(), acc.data_ptr(),
                      out.data_ptr(), None, _stream()))
    return GemvResult(accumulators=acc.cpu().numpy(), output=out.cpu().numpy())


def gemv_lut(p, lut) -> np.ndarray:
    """int32 accumulators of gemv_tl1 / gemv_tl2 with the caller's LUT."""
    so = _lib()
    _calls[0] += 1
    fmt, tiled, tsign, _ = _operands(p)
    dev = tiled.device
    e = torch.from_numpy(np.array(lut.entries, dtype=np.int16, copy=True)).to(dev)
    acc = torch.zeros(p.rows, dtype=torch.int32, device=dev)
    _check(so.tb_gemv_lut(fmt, tiled.data_ptr(), tsign.data_ptr() if tsign is not None else None,
                          p.rows, p.cols, e.data_ptr(), lut.groups, acc.data_ptr(), _stream()))
    return acc.cpu().numpy()
