"""ctypes binding of libternary_b200.so (the C ABI in include/ternary_b200.h).

The product path has no fallback: if the library is missing or no CUDA
device is present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libternary_b200.so"

I2S, TL1, TL2 = 1, 2, 3

_p = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int
_f64 = C.c_double
_f32 = C.c_float

# name -> (restype, argtypes)
_SIGS = {
    "tb_strerror": (C.c_char_p, [_i32]),
    "tb_abi_version": (_i32, []),
    "tb_device_sm_count": (_i32, [_i32]),
    "tb_stream_synchronize": (_i32, [_p]),
    "tb_quantize_f32": (_i32, [_p, _i64, _i64, _i64, _p, _i64, _p, _p, _p]),
    "tb_quantize_f64": (_i32, [_p, _i64, _i64, _i64, _p, _i64, _p, _p, _p]),
    "tb_abs_pairwise_sums_f32": (_i32, [_p, _p, _p, _i64, _p, _p, _p]),
    "tb_abs_pairwise_sums_f64": (_i32, [_p, _p, _p, _i64, _p, _p, _p]),
    "tb_ternarize_apply_f32": (_i32, [_p, _i64, _f64, _p, _p]),
    "tb_ternarize_apply_f64": (_i32, [_p, _i64, _f64, _p, _p]),
    "tb_scale_outputs": (_i32, [_p, _i64, _i64, _f64, _p, _p, _p, _p]),
    "tb_ref_row_bytes": (_i64, [_i32, _i64]),
    "tb_ref_sign_row_bytes": (_i64, [_i64]),
    "tb_encode": (_i32, [_i32, _p, _i64, _i64, _p, _p, _p]),
    "tb_decode": (_i32, [_i32, _p, _p, _i64, _i64, _p, _p, _p]),
    "tb_validate": (_i32, [_i32, _p, _p, _i64, _i64, _p, _p]),
    "tb_tiled_chunks": (_i64, [_i32, _i64]),
    "tb_tiled_bytes": (_i64, [_i32, _i64, _i64]),
    "tb_tiled_sign_bytes": (_i64, [_i32, _i64, _i64]),
    "tb_repack": (_i32, [_i32, _p, _p, _i64, _i64, _p, _p, _p]),
    "tb_unrepack": (_i32, [_i32, _p, _p, _i64, _i64, _p, _p, _p]),
    "tb_build_lut": (_i32, [_i32, _p, _i64, _i64, _p, _p]),
    "tb_gemv_workspace_bytes": (_i64, [_i32, _i64, _i64]),
    "tb_gemv": (_i32, [_i32, _p, _p, _i64, _i64, _p, _i64, _i64, _i64, _p, _f64, _p, _p, _p,
                       _p, _p]),
    "tb_act_records_bytes": (_i64, [_i32, _i64, _i64]),
    "tb_prep_activations": (_i32, [_i32, _p, _i64, _i64, _i64, _i64, _p, _p]),
    "tb_quantize_records_f32": (_i32, [_i32, _p, _i64, _i64, _i64, _p, _i64, _p, _p, _p, _p]),
    "tb_quantize_records_f64": (_i32, [_i32, _p, _i64, _i64, _i64, _p, _i64, _p, _p, _p, _p]),
    "tb_gemv_records": (_i32, [_i32, _p, _p, _i64, _i64, _p, _i64, _p, _f64, _p, _p, _p, _p,
                               _p]),
    "tb_gemv_job_bytes": (_i64, []),
    "tb_gemv_batch_prepare": (_i32, [_i32, _i64, _p, _p, _p, _p, _p]),
    "tb_gemv_batch_launch": (_i32, [_i32, _p, _i64, _i64, _i32, _i64, _i32, _p]),
    "tb_step_glue": (_i32, [_p, _i64, _i64, _i64, _p, _p]),
    "tb_step_glue_ex": (_i32, [_p, _i64, _i64, _i64, _p, _i32, _p]),
    "tb_gemv_step_prepare": (_i32, [_i32, _i64, _p, _p, _i64, _p, _p, _p, _p]),
    "tb_gemv_step_prepare_cols": (_i32, [_i32, _i64, _p, _p, _p, _i64, _p, _p, _p, _p]),
    "tb_gemv_step_launch": (_i32, [_i32, _p, _i64, _i64, _i64, _p, _i32, _p, _i64, _p, _p, _p]),
    "tb_gemv_batch_finalize": (_i32, [_p, _i64, _i64, _p]),
    "tb_copy_in": (_i32, [_p, _p, _i64, _p]),
    "tb_gemv_lut": (_i32, [_i32, _p, _p, _i64, _i64, _p, _i64, _p, _p]),
    "tb_gemv_ref_int32": (_i32, [_p, _i64, _i64, _p, _p, _p]),
    "tb_gemv_f32_ref": (_i32, [_p, _i64, _i64, _f32, _p, _p, _p]),
    "tb_gemm_batch": (_i32, [_i32, _i64, _p, _i64, _p]),
    "tb_gemm_i8": (_i32, [_i32, _p, _i64, _i64, _p, _i64, _i64, _p, _f64, _p, _p, _p, _p, _p]),
    "tb_gemm_act_bytes": (_i64, [_i64, _i64]),
    "tb_gemm_tile_act": (_i32, [_p, _i64, _i64, _i64, _p, _p]),
    "tb_gemv_table_launches": (_i64, []),
    "tb_step_glue_sync": (_i32, [_p, _i64, _i64, _p, _p, _p, _i32, _i32, _p, _p]),
    "tb_gemv_batch_launch_sync": (_i32, [_i32, _p, _p, _i64, _i64, _i32, _i64, _p, _i64, _p,
                                         _i32, _p]),
    "tb_sync_timeouts": (_i64, []),
    "tb_gemv_batch_prepare_cols": (_i32, [_i32, _i64, _p, _p, _p, _p, _p, _p, _p]),
    "tb_gemv_batch_launch_inline": (_i32, [_i32, _p, _p, _i64, _i64, _i32, _i64, _i32, _p, _i64,
                                            _p]),
    "tb_gemm_quantize_act": (_i32, [_p, _i64, _i64, _i64, _p, _p, _p, _p]),
    "tb_gemm_quantize_act_multi": (_i32, [_i64, _p, _i64, _p]),
    "tb_sym_alloc": (_i32, [_i64, _p]),
    "tb_sym_free": (_i32, [_p]),
    "tb_ipc_handle_bytes": (_i32, []),
    "tb_ipc_get_handle": (_i32, [_p, _p]),
    "tb_ipc_open": (_i32, [_p, _p]),
    "tb_ipc_close": (_i32, [_p]),
    "tb_rowpar_allreduce": (_i32, [_i32, _i32, _p, _p, _p, _i64, _i64, _p, _i32, _p]),
    "tb_rowpar_allreduce_emulated": (_i32, [_i32, _p, _p, _p, _i64, _i64, _p, _i32, _p]),
}

class GemvDesc(C.Structure):
    """Mirror of tb_gemv_desc (include/ternary_b200.h)."""

    _fields_ = [("tiled", _p), ("tiled_sign", _p), ("rows", _i64), ("cols", _i64),
                ("rec", _p), ("M", _i64), ("a_scale", _p), ("w_scale", _f64),
                ("workspace", _p), ("acc_out", _p), ("out64", _p), ("out32", _p)]


class QuantDesc(C.Structure):
    """Mirror of tb_quant_desc (include/ternary_b200.h)."""

    _fields_ = [("x", _p), ("x_is_f64", C.c_int32), ("fmt", C.c_int32), ("M", _i64),
                ("K", _i64), ("ldx", _i64), ("q", _p), ("ldq", _i64), ("scale", _p),
                ("rec", _p), ("nonfinite_flag", _p)]


class GemmDesc(C.Structure):
    """Mirror of tb_gemm_desc (include/ternary_b200.h)."""

    _fields_ = [("tiled", _p), ("rows", _i64), ("cols", _i64), ("act_tiled", _p),
                ("a_scale", _p), ("w_scale", _f64), ("acc_out", _p), ("out64", _p),
                ("out32", _p)]


class QactDesc(C.Structure):
    """Mirror of tb_qact_desc (include/ternary_b200.h)."""

    _fields_ = [("x", _p), ("cols", _i64), ("ldx", _i64), ("scale", _p),
                ("nonfinite_flag", _p), ("act_tiled", _p)]


class RowparSeg(C.Structure):
    """Mirror of tb_rowpar_seg (include/ternary_b200.h)."""

    _fields_ = [("off", _i64), ("n", _i64), ("w_scale", _f64), ("a_scale", _p), ("out32", _p),
                ("acc_out", _p)]


class StepInput(C.Structure):
    """Mirror of tb_step_input (include/ternary_b200.h)."""

    _fields_ = [("x", _p), ("K", _i64), ("scale", _p), ("nonfinite_flag", _p), ("ready", _p)]


_lib = None


class ExtensionMissing(RuntimeError):
    pass


def load(path: os.PathLike | None = None):
    """Load (once) and return the CDLL with typed entry points."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise ExtensionMissing(
            f"{p} not found: build the CUDA extension first "
            "(python -m paper_2410_16144_b200.build or __graft_entry__.build())")
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def declared_symbols():
    return list(_SIGS)


def check(status: int, what: str = "") -> None:
    if status != 0:
        msg = load().tb_strerror(status).decode()
        raise RuntimeError(f"ternary_b200 {what} failed: {msg} (status {status})")


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    """cudaStream_t of ``stream`` or of torch's current stream on the current
    device (the raw accessors: torch.cuda.current_stream() costs ~15 us of
    Python per call, which the per-call reference API paid several times)."""
    import torch
    if stream is not None:
        return stream.cuda_stream
    C_ = torch._C
    return C_._cuda_getCurrentRawStream(C_._cuda_getDevice())
