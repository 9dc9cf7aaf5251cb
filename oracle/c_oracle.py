"""ctypes wrapper of oracle/c/tern_oracle.c -- TEST / BASELINE INFRASTRUCTURE.

The C restatement of the reference's byte-table CPU kernels, used as the
"port" CPU baseline (bench.py cpu_baseline and --impl reference) and as a
second checker in tests.  Built by ``build()`` into oracle/_build/.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "c" / "tern_oracle.c"
OUT = HERE / "_build" / "libtern_oracle.so"

_lib = None


def build(force: bool = False) -> Path:
    OUT.parent.mkdir(exist_ok=True)
    if force or not OUT.exists() or SRC.stat().st_mtime > OUT.stat().st_mtime:
        cmd = ["gcc", "-O3", "-march=x86-64-v3", "-fopenmp", "-fPIC", "-shared", str(SRC),
               "-o", str(OUT), "-lm"]
        subprocess.run(cmd, check=True, capture_output=True, text=True)
    return OUT


def load():
    global _lib
    if _lib is None:
        if not OUT.exists():
            build()
        _lib = C.CDLL(str(OUT))
        p, i64, i32 = C.c_void_p, C.c_int64, C.c_int
        sig = {
            "to_quantize_f32": (i32, [p, i64, i64, p, p]),
            "to_lut_tl1": (None, [p, i64, i64, p]),
            "to_lut_tl2": (None, [p, i64, i64, p]),
            "to_i2s_byte_table": (None, [p, i64, i64, p]),
            "to_tl1_byte_table": (None, [p, i64, i64, p]),
            "to_tl2_signed_table": (None, [p, i64, p]),
            "to_byte_gemv": (None, [p, i64, i64, p, p, i32]),
            "to_tl2_byte_gemv": (None, [p, p, i64, i64, i64, p, p, i32]),
            "to_gemv_ref_int32": (None, [p, i64, i64, p, p, i32]),
            "to_max_threads": (i32, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def max_threads() -> int:
    return int(load().to_max_threads())


def quantize(x: np.ndarray, pad_to: int):
    x = np.ascontiguousarray(x, dtype=np.float32)
    kpad = -(-x.size // pad_to) * pad_to
    q = np.empty(kpad, np.int8)
    s = C.c_double()
    if load().to_quantize_f32(_p(x), x.size, kpad, _p(q), C.byref(s)):
        raise ValueError("activations must be finite")
    return q, s.value


def lut_tl1(a: np.ndarray, groups: int):
    e = np.empty((groups, 9), np.int16)
    load().to_lut_tl1(_p(a), a.size, groups, _p(e))
    return e


def lut_tl2(a: np.ndarray, groups: int):
    e = np.empty((groups, 14), np.int16)
    load().to_lut_tl2(_p(a), a.size, groups, _p(e))
    return e


def gemv_i2s(packed: np.ndarray, act: np.ndarray, threads: int = 0):
    rows, bc = packed.shape
    t = np.empty((bc, 256), np.int32)
    out = np.empty(rows, np.int32)
    lib = load()
    lib.to_i2s_byte_table(_p(act), act.size, bc, _p(t))
    lib.to_byte_gemv(_p(packed), rows, bc, _p(t), _p(out), threads)
    return out


def gemv_tl1(packed: np.ndarray, lut: np.ndarray, threads: int = 0):
    rows, bc = packed.shape
    t = np.empty((bc, 256), np.int32)
    out = np.empty(rows, np.int32)
    lib = load()
    lib.to_tl1_byte_table(_p(lut), lut.shape[0], bc, _p(t))
    lib.to_byte_gemv(_p(packed), rows, bc, _p(t), _p(out), threads)
    return out


def gemv_tl2(index_plane: np.ndarray, sign_plane: np.ndarray, lut: np.ndarray, threads: int = 0):
    rows, bc = index_plane.shape
    t = np.empty((lut.shape[0] // 2, 1024), np.int32)
    out = np.empty(rows, np.int32)
    lib = load()
    lib.to_tl2_signed_table(_p(lut), lut.shape[0], _p(t))
    lib.to_tl2_byte_gemv(_p(index_plane), _p(sign_plane), rows, bc, sign_plane.shape[1], _p(t),
                         _p(out), threads)
    return out


def set_threads(n: int) -> None:
    os.environ["OMP_NUM_THREADS"] = str(n)
