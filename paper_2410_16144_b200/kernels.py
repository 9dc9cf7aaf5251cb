"""GEMV entry points (mirrors ternpack.kernels, pkg/src/ternpack/kernels.py).

Every integer kind returns the exact int32 accumulators, bit-identical to
the reference oracle, plus float64 outputs acc * w_scale * a_scale.

  gemv_ref_int32  kernels.py:59-63   -> tb_gemv_ref_int32 (unpacked int8)
  gemv_f32_ref    kernels.py:66-72   -> tb_gemv_f32_ref (dequantised fp32)
  gemv_i2s        kernels.py:86-94   -> tb_gemv on the tiled I2_S layout
  gemv_tl1        kernels.py:109-126 -> tb_gemv_lut with the caller's LUT
  gemv_tl2        kernels.py:140-157 -> tb_gemv_lut with the caller's LUT
  gemv_parallel   kernels.py:189-268 -> tb_gemv (LUT implicit) or tb_gemv_lut
                                        when the caller passes a LUT

``thread_count`` keeps the reference's validation and meaning of "results
are identical for every value"; on the GPU the row partition is the CTA
grid, so it does not change the launch.  Activations may be a batch
(QuantizedActivations with data [M, K], M <= 16) -- each token is an
independent reference GEMV; outputs are then [M, rows].
"""

from __future__ import annotations

import enum

import numpy as np

import torch

from . import _lib as L
from .core import GemvResult, QuantizedActivations, TernaryMatrix, make_result, to_device
from .lut import LutTL1, LutTL2, build_lut_tl1, build_lut_tl2  # noqa: F401
from .packing import PackedI2S, PackedTL1, PackedTL2

__all__ = ["KernelKind", "WIDEN_GROUPS", "gemv_ref_int32", "gemv_f32_ref", "gemv_i2s",
           "gemv_tl1", "gemv_tl2", "gemv_parallel", "GemvPlan", "GemvBatch", "StepGlue",
           "ActRecords", "GemvStep", "HostStep", "KERNEL_PAD", "gemm_prefill"]

WIDEN_GROUPS = 64  # kernels.py:34
MAX_DECODE_TOKENS = 16


class KernelKind(enum.Enum):
    REF_INT32 = "ref_int32"
    REF_F32 = "ref_f32"
    I2_S = "i2s"
    TL1 = "tl1"
    TL2 = "tl2"


KERNEL_PAD = {KernelKind.REF_INT32: 1, KernelKind.I2_S: 4, KernelKind.TL1: 2,
              KernelKind.TL2: 3}  # runtime.py:32-37


def _check_activation_cover(a: QuantizedActivations, cols: int) -> None:
    """kernels.py:45-49."""
    if len(a) < cols:
        raise ValueError("dimension mismatch: activations shorter than matrix cols")
    if len(a) == cols or (a._trusted and a.original_len <= cols):
        return  # our quantiser zero-pads by construction: no device read needed
    if bool((a.data[..., cols:] != 0).any()):
        raise ValueError("dimension mismatch: nonzero activations beyond matrix cols")


def _out_shape(a: QuantizedActivations, rows: int):
    return (rows,) if a.data.dim() == 1 else (a.tokens, rows)


def gemv_ref_int32(m: TernaryMatrix, a: QuantizedActivations) -> GemvResult:
    _check_activation_cover(a, m.cols)
    lib = L.load()
    acts = a.data.reshape(a.tokens, -1)
    acc = torch.empty((a.tokens, m.rows), dtype=torch.int32, device=m.values.device)
    for t in range(a.tokens):
        L.check(lib.tb_gemv_ref_int32(L.ptr(m.values), m.rows, m.cols, L.ptr(acts[t]),
                                      L.ptr(acc[t]), L.stream_ptr()), "gemv_ref_int32")
    acc = acc.reshape(_out_shape(a, m.rows))
    return make_result(acc, m.scale, a.scales)


def gemv_f32_ref(m: TernaryMatrix, x) -> GemvResult:
    xd = to_device(x, torch.float32).reshape(-1).contiguous()
    if xd.numel() != m.cols:
        raise ValueError("dimension mismatch")
    out = torch.empty(m.rows, dtype=torch.float32, device=xd.device)
    L.check(L.load().tb_gemv_f32_ref(L.ptr(m.values), m.rows, m.cols, float(m.scale),
                                     L.ptr(xd), L.ptr(out), L.stream_ptr()), "gemv_f32_ref")
    return GemvResult(accumulators=None, output=out.to(torch.float64))


GEMM_MIN_TOKENS = 64  # from this many tokens on, I2_S / TL1 batches use the tensor cores


def _gemm_operand(acts: torch.Tensor) -> torch.Tensor:
    """int8 [M, K] with a 16-byte-multiple row stride (zero padded), as the
    tcgen05 GEMM's A operand."""
    M, K = acts.shape
    if acts.is_contiguous() and K % 16 == 0 and acts.data_ptr() % 16 == 0:
        return acts
    buf = torch.zeros((M, -(-K // 16) * 16), dtype=torch.int8, device=acts.device)
    buf[:, :K] = acts
    return buf


def gemm_prefill(p, a: QuantizedActivations, want_out64: bool = True) -> GemvResult:
    """Prefill: all M tokens of ``a`` against one packed I2_S / TL1 matrix on
    the tcgen05 int8 tensor cores (tb_gemm_i8).  Row m of the result is the
    reference's gemv_parallel for token m (kernels.py:189-268)."""
    if p.FMT not in (L.I2S, L.TL1):
        raise ValueError("tensor-core GEMM supports I2_S and TL1 weights")
    lib = L.load()
    main, _ = p.tiled()
    acts = _gemm_operand(a.data.reshape(a.tokens, -1))
    M, lda = acts.shape
    dev = main.device
    acc = torch.empty((M, p.rows), dtype=torch.int32, device=dev)
    out = torch.empty((M, p.rows), dtype=torch.float64, device=dev) if want_out64 else None
    ws = torch.empty(lib.tb_gemm_act_bytes(min(M, 512), p.cols), dtype=torch.uint8, device=dev)
    L.check(lib.tb_gemm_i8(p.FMT, L.ptr(main), p.rows, p.cols, L.ptr(acts), M, lda,
                           L.ptr(a.scales), float(p.scale), L.ptr(ws), L.ptr(acc), L.ptr(out),
                           None, L.stream_ptr()), "gemm_i8")
    shape = _out_shape(a, p.rows)
    return GemvResult(accumulators=acc.reshape(shape),
                      output=out.reshape(shape) if out is not None else None)


def _tiled_gemv(p, a: QuantizedActivations, want_out64: bool = True) -> GemvResult:
    """Decode GEMV through the C ABI (LUT implicit; M <= 16 tokens per launch);
    batches of GEMM_MIN_TOKENS or more I2_S / TL1 tokens go to the GEMM."""
    if a.tokens >= GEMM_MIN_TOKENS and p.FMT in (L.I2S, L.TL1):
        return gemm_prefill(p, a, want_out64)
    lib = L.load()
    main, sign = p.tiled()
    acts = a.data.reshape(a.tokens, -1)
    M, K = acts.shape
    dev = main.device
    acc = torch.empty((M, p.rows), dtype=torch.int32, device=dev)
    out = torch.empty((M, p.rows), dtype=torch.float64, device=dev) if want_out64 else None
    ws = p.workspace()
    s = L.stream_ptr()
    for t0 in range(0, M, MAX_DECODE_TOKENS):
        t1 = min(M, t0 + MAX_DECODE_TOKENS)
        L.check(lib.tb_gemv(p.FMT, L.ptr(main), L.ptr(sign), p.rows, p.cols, L.ptr(acts[t0]),
                            t1 - t0, acts.stride(0), K, L.ptr(a.scales[t0:t1]), float(p.scale),
                            L.ptr(ws), L.ptr(acc[t0]), L.ptr(out[t0] if out is not None else None),
                            None, s), "gemv")
    shape = _out_shape(a, p.rows)
    return GemvResult(accumulators=acc.reshape(shape),
                      output=out.reshape(shape) if out is not None else None)


def _lut_gemv(p, lut, a_scale) -> GemvResult:
    lib = L.load()
    main, sign = p.tiled()
    acc = torch.zeros(p.rows, dtype=torch.int32, device=main.device)
    L.check(lib.tb_gemv_lut(p.FMT, L.ptr(main), L.ptr(sign), p.rows, p.cols, L.ptr(lut.entries),
                            lut.groups, L.ptr(acc), L.stream_ptr()), "gemv_lut")
    return make_result(acc, p.scale, a_scale)


def _widened_sum(vals: torch.Tensor) -> torch.Tensor:
    """int16 partials folded every 64 groups, asserting |partial| <= 32767
    (kernels.py:160-173); evaluated on the device."""
    rows, groups = vals.shape
    blocks = -(-groups // WIDEN_GROUPS)
    padded = torch.zeros((rows, blocks * WIDEN_GROUPS), dtype=torch.int32, device=vals.device)
    padded[:, :groups] = vals.to(torch.int32)
    running = torch.cumsum(padded.reshape(rows, blocks, WIDEN_GROUPS), dim=2, dtype=torch.int32)
    peak = int(running.abs().max()) if running.numel() else 0
    assert peak <= 32767, f"16-bit partial sum overflow: |{peak}| > 32767"
    return running[:, :, -1].sum(dim=1, dtype=torch.int32)


def gemv_i2s(p: PackedI2S, a: QuantizedActivations) -> GemvResult:
    """2-bit kernel: weights decoded on the fly, never materialised."""
    if not p.trusted:
        p.validate()
    _check_activation_cover(a, p.cols)
    return _tiled_gemv(p, a)


def gemv_tl1(p: PackedTL1, lut: LutTL1, a_scale: float, *, checked: bool = False) -> GemvResult:
    """Pair-index kernel: one 9-entry table lookup per weight pair."""
    if not p.trusted:
        p.validate()
    if lut.groups != p.groups:
        raise ValueError("group-count mismatch")
    if checked:
        nib = torch.empty((p.rows, 2 * p.bytes_per_row), dtype=torch.int64, device=p.data.device)
        nib[:, 0::2] = (p.data & 15).to(torch.int64)
        nib[:, 1::2] = (p.data >> 4).to(torch.int64)
        g = torch.arange(p.groups, device=nib.device)
        vals = lut.entries[g.unsqueeze(0), nib[:, : p.groups]]
        return make_result(_widened_sum(vals), p.scale, a_scale)
    return _lut_gemv(p, lut, a_scale)


def gemv_tl2(p: PackedTL2, lut: LutTL2, a_scale: float, *, checked: bool = False) -> GemvResult:
    """Sign + index kernel: 14-entry canonical table, sign applied on lookup."""
    if not p.trusted:
        p.validate()
    if lut.groups != p.groups:
        raise ValueError("group-count mismatch")
    if checked:
        idx = p.data_nibbles().to(torch.int64)
        sg = p.data_signs().bool()
        g = torch.arange(p.groups, device=idx.device)
        vals = lut.entries[g.unsqueeze(0), idx]
        vals = torch.where(sg, -vals, vals)
        return make_result(_widened_sum(vals), p.scale, a_scale)
    return _lut_gemv(p, lut, a_scale)


def gemv_parallel(kernel: KernelKind, weights, a, thread_count: int = 1,
                  lut=None) -> GemvResult:
    """kernels.py:189-268 with the GPU grid as the row partition."""
    if thread_count < 1:
        raise ValueError("thread_count must be >= 1")
    if kernel is KernelKind.REF_F32:
        return gemv_f32_ref(weights, a)
    if kernel is KernelKind.REF_INT32:
        return gemv_ref_int32(weights, a)
    if not weights.trusted:
        weights.validate()
    _check_activation_cover(a, weights.cols)
    if kernel is KernelKind.I2_S:
        return _tiled_gemv(weights, a)
    if kernel in (KernelKind.TL1, KernelKind.TL2):
        if lut is None:
            return _tiled_gemv(weights, a)  # LUT implicit (exact identity, lut.py docstring)
        if lut.groups != weights.groups:
            raise ValueError("group-count mismatch")
        return _lut_gemv(weights, lut, a.scales[:1])
    raise ValueError(f"unsupported kernel kind: {kernel}")


class GemvPlan:
    """Pre-allocated, capture-safe decode GEMV for one packed matrix.

    Holds the tiled weights, a self-cleaning workspace and output buffers so
    that ``run`` is a single C-ABI launch with no allocation or host sync --
    the form the stack runner and bench capture into CUDA graphs.
    """

    def __init__(self, packed, max_tokens: int = 1, out_dtype=torch.float32,
                 want_acc: bool = False, stream=None):
        if not 1 <= max_tokens <= MAX_DECODE_TOKENS:
            raise ValueError(f"max_tokens must be in [1, {MAX_DECODE_TOKENS}]")
        self.p = packed
        self.main, self.sign = packed.tiled()
        dev = self.main.device
        self.ws = torch.zeros(
            L.load().tb_gemv_workspace_bytes(packed.FMT, packed.rows, packed.cols) // 4,
            dtype=torch.int32, device=dev)
        self.out32 = self.out64 = None
        if out_dtype == torch.float32:
            self.out32 = torch.empty((max_tokens, packed.rows), dtype=torch.float32, device=dev)
        elif out_dtype == torch.float64:
            self.out64 = torch.empty((max_tokens, packed.rows), dtype=torch.float64, device=dev)
        self.acc = (torch.empty((max_tokens, packed.rows), dtype=torch.int32, device=dev)
                    if want_acc else None)
        self.max_tokens = max_tokens
        self._lib = L.load()

    def run(self, act: torch.Tensor, scales: torch.Tensor, stream_ptr: int | None = None):
        """Natural int8 activations [M, K] (prep + GEMV: two launches)."""
        M, K = act.shape
        st = self._lib.tb_gemv(self.p.FMT, self.main.data_ptr(),
                               self.sign.data_ptr() if self.sign is not None else None,
                               self.p.rows, self.p.cols, act.data_ptr(), M, act.stride(0), K,
                               scales.data_ptr(), float(self.p.scale), self.ws.data_ptr(),
                               L.ptr(self.acc), L.ptr(self.out64), L.ptr(self.out32),
                               stream_ptr if stream_ptr is not None else L.stream_ptr())
        if st:
            L.check(st, "gemv")
        return self.out32 if self.out32 is not None else self.out64

    def run_records(self, rec: "ActRecords", stream_ptr: int | None = None):
        """Prepared activation records (one launch)."""
        st = self._lib.tb_gemv_records(self.p.FMT, self.main.data_ptr(),
                                       self.sign.data_ptr() if self.sign is not None else None,
                                       self.p.rows, self.p.cols, rec.buf.data_ptr(), rec.M,
                                       rec.scales.data_ptr(), float(self.p.scale),
                                       self.ws.data_ptr(), L.ptr(self.acc), L.ptr(self.out64),
                                       L.ptr(self.out32),
                                       stream_ptr if stream_ptr is not None else L.stream_ptr())
        if st:
            L.check(st, "gemv_records")
        return self.out32 if self.out32 is not None else self.out64


class GemvBatch:
    """Several independent decode GEMVs of one format in ONE launch.

    ``pairs`` is a list of (GemvPlan, ActRecords); the job table is built once
    (tb_gemv_batch_prepare) and kept on the device, so ``run`` is a single
    capture-safe launch.  Outputs land in each plan's buffers.
    """

    def __init__(self, pairs):
        import ctypes as C
        import numpy as np

        lib = L.load()
        # (plan, records) or (plan, records, col0): a K-window of the records
        # (columns [col0, col0 + plan cols); e.g. one of several column shards
        # of a matrix that share one workspace, only one of them with outputs)
        pairs = [tuple(pr) if len(pr) == 3 else (pr[0], pr[1], 0) for pr in pairs]
        fmts = {p.p.FMT for p, _, _ in pairs}
        if len(fmts) != 1:
            raise ValueError("one format per batch")
        self.fmt = fmts.pop()
        descs = (L.GemvDesc * len(pairs))()
        col0 = (C.c_int64 * len(pairs))(*[int(c) for _, _, c in pairs])
        rec_cols = (C.c_int64 * len(pairs))(*[int(rec.K) for _, rec, _ in pairs])
        for d, (plan, rec, _) in zip(descs, pairs):
            d.tiled = plan.main.data_ptr()
            d.tiled_sign = plan.sign.data_ptr() if plan.sign is not None else None
            d.rows, d.cols = plan.p.rows, plan.p.cols
            d.rec, d.M = rec.buf.data_ptr(), rec.M
            d.a_scale, d.w_scale = rec.scales.data_ptr(), float(plan.p.scale)
            d.workspace = plan.ws.data_ptr()
            d.acc_out = L.ptr(plan.acc)
            d.out64 = L.ptr(plan.out64)
            d.out32 = L.ptr(plan.out32)
        jb = lib.tb_gemv_job_bytes()
        host = np.zeros(jb * len(pairs), dtype=np.uint8)
        total = C.c_int64()
        maxm = C.c_int32()
        maxe = C.c_int64()
        L.check(lib.tb_gemv_batch_prepare_cols(self.fmt, len(pairs), C.cast(descs, C.c_void_p),
                                               C.cast(col0, C.c_void_p), C.cast(rec_cols, C.c_void_p),
                                               host.ctypes.data_as(C.c_void_p), C.byref(total),
                                               C.byref(maxm), C.byref(maxe)), "gemv_batch_prepare")
        dev = pairs[0][0].main.device
        self.table = torch.from_numpy(host).to(dev)
        self._host = host  # host copy of the job table (inline finalize by a later step)
        self._host_ptr = host.ctypes.data
        self.njobs, self.total, self.max_m = len(pairs), total.value, maxm.value
        self.max_entries = maxe.value
        self.pairs = pairs  # keep every buffer alive
        self._scale_ptrs = {rec.scales.data_ptr() for _, rec, _ in pairs}
        self._lib = lib

    def run(self, stream_ptr: int | None = None, finalize: bool = True,
            prev: "GemvBatch | None" = None, sync=None):
        """One grouped GEMV launch (+ the finalize pass unless ``finalize`` is
        False, in which case a later launch must finalise this batch).
        ``prev``: the batch launched before this one (M > 1, I2_S / TL1, <= 20
        jobs: records-table mode), finalised in this launch's tail.
        ``sync``: (layer sync block pointer, glue CTA count) of a pipelined
        layer (tb_gemv_batch_launch_sync; StepGlue(sync=...) is its producer)."""
        if sync is not None:
            st = self._lib.tb_gemv_batch_launch_sync(
                self.fmt, self.table.data_ptr(), self._host_ptr, self.njobs, self.total,
                self.max_m, self.max_entries, prev._host_ptr if prev is not None else None,
                prev.njobs if prev is not None else 0, sync[0], sync[1],
                stream_ptr if stream_ptr is not None else L.stream_ptr())
            if st:
                L.check(st, "gemv_batch_launch_sync")
            return
        st = self._lib.tb_gemv_batch_launch_inline(self.fmt, self.table.data_ptr(),
                                                   self._host_ptr, self.njobs, self.total,
                                                   self.max_m, self.max_entries,
                                                   1 if finalize else 0,
                                                   prev._host_ptr if prev is not None else None,
                                                   prev.njobs if prev is not None else 0,
                                                   stream_ptr if stream_ptr is not None
                                                   else L.stream_ptr())
        if st:
            L.check(st, "gemv_batch_launch")


class StepGlue:
    """ONE launch between GEMV groups: finalise a batch and quantise inputs.

    ``inputs`` is a list of (x_device_tensor [M, K] f32/f64, ActRecords);
    the x tensors are read at ``run`` time through their data pointers, so
    they must stay allocated (e.g. a fixed buffer refilled every step).
    """

    def __init__(self, inputs, finalize: "GemvBatch | None" = None, early: bool = False,
                 sync=None):
        """``early``: quantise before waiting on the preceding kernel
        (TB_GLUE_EARLY_QUANT) -- only when the inputs do not depend on it and
        nothing in flight reads these records (e.g. three record sets in
        rotation, the GEMV finalising its predecessor).
        ``sync``: (this layer's sync block pointer, the previous layer's or
        None, publish_exit) -- the quantising glue of a pipelined layer
        (tb_step_glue_sync); ``glue_ctas`` is then what the layer's
        GemvBatch.run(sync=...) must be given."""
        import ctypes as C

        self._lib = L.load()
        self.inputs = inputs
        self._flags = 1 if early else 0
        self._sync = sync
        self.glue_ctas = 8 * sum(rec.M for _, rec in inputs)
        if sync is not None and not inputs:
            raise ValueError("a pipelined glue quantises")
        self.fin = None
        self.descs = (L.QuantDesc * max(1, len(inputs)))()
        for d, (x, rec) in zip(self.descs, inputs):
            d.x = x.data_ptr()
            d.x_is_f64 = 1 if x.dtype == torch.float64 else 0
            d.fmt, d.M, d.K, d.ldx = rec.fmt, rec.M, rec.K, x.stride(0)
            d.q = L.ptr(rec.natural)
            d.ldq = rec.natural.stride(0) if rec.natural is not None else 0
            d.scale, d.rec, d.nonfinite_flag = rec.scales.data_ptr(), rec.buf.data_ptr(), None
        self._descs_ptr = C.cast(self.descs, C.c_void_p)
        self.retarget(finalize)

    def retarget(self, finalize: "GemvBatch | None"):
        # the finalize reads the batch's per-token scales while this launch's
        # quantisation rows write theirs: they must be different buffers
        if finalize is not None and any(rec.scales.data_ptr() in finalize._scale_ptrs
                                        for _, rec in self.inputs):
            raise ValueError("a glue cannot quantise into records whose batch it finalises "
                             "(alternate two ActRecords sets)")
        self.fin = finalize
        return self

    def run(self, stream_ptr: int | None = None, prev_ctas: int = 0):
        fin = self.fin
        if self._sync is not None:
            import ctypes as C

            n = C.c_int32()
            st = self._lib.tb_step_glue_sync(fin._host_ptr if fin is not None else None,
                                             fin.njobs if fin is not None else 0,
                                             len(self.inputs), self._descs_ptr, self._sync[0],
                                             self._sync[1], prev_ctas,
                                             1 if self._sync[2] else 0, C.byref(n),
                                             stream_ptr if stream_ptr is not None
                                             else L.stream_ptr())
            if st:
                L.check(st, "step_glue_sync")
            assert n.value == self.glue_ctas
            return
        st = self._lib.tb_step_glue_ex(fin.table.data_ptr() if fin is not None else None,
                                       fin.njobs if fin is not None else 0,
                                       fin.max_entries if fin is not None else 0,
                                       len(self.inputs), self._descs_ptr, self._flags,
                                       stream_ptr if stream_ptr is not None else L.stream_ptr())
        if st:
            L.check(st, "step_glue")


class GemvStep:
    """A one-token decode step in ONE launch (tb_gemv_step_launch).

    ``pairs`` is a list of (GemvPlan, input index) and ``input_k`` the lengths
    of the (at most 4) float32 input vectors the jobs contract; gate and up
    typically share input 0.  Every CTA quantises the inputs itself
    (quantize_activations, core.py:116-134), so there is no separate
    quantise launch, and after its own work the launch finalises ``prev`` --
    the step (or GemvBatch) launched just before it -- whose grid has
    completed by then.  This step's outputs therefore land in the plans'
    buffers when the NEXT step runs, or on ``finalize()``.
    ``x_after_wait``: the inputs are written by the preceding kernel.
    """

    def __init__(self, pairs, input_k, x_after_wait: bool = False, flags=None,
                 isolated: bool = False, sticky_flags: bool = False,
                 self_finalize: bool = False, independent: bool = False):
        import ctypes as C
        import numpy as np

        lib = L.load()
        # (plan, input) or (plan, input, col0): a row-parallel K-shard reads
        # input columns [col0, col0 + cols) and uses the full input's scale
        windowed = [len(pr) == 3 for pr in pairs]
        pairs = [tuple(pr) if len(pr) == 3 else (pr[0], pr[1], 0) for pr in pairs]
        fmts = {p.p.FMT for p, _, _ in pairs}
        if len(fmts) != 1:
            raise ValueError("one format per step")
        if not 1 <= len(input_k) <= 4:
            raise ValueError("a step takes 1 to 4 input vectors")
        self.fmt = fmts.pop()
        self.input_k = [int(k) for k in input_k]
        dev = pairs[0][0].main.device
        self.scales = torch.empty(len(input_k), dtype=torch.float64, device=dev)
        # per-input non-finite verdict of the last launch (device, or pinned host)
        self.flags = (flags if flags is not None
                      else torch.zeros(len(input_k), dtype=torch.int32, device=dev))
        descs = (L.GemvDesc * len(pairs))()
        src = (C.c_int32 * len(pairs))()
        col0 = (C.c_int64 * len(pairs))()
        ks = (C.c_int64 * len(input_k))(*self.input_k)
        chunk_w = 96 if self.fmt == L.TL2 else 64
        for i, (d, (plan, v, c0)) in enumerate(zip(descs, pairs)):
            if not 0 <= v < len(input_k):
                raise ValueError("input index out of range")
            if c0 % chunk_w or c0 < 0:
                raise ValueError(f"col0 must be a non-negative multiple of {chunk_w}")
            if (c0 + plan.p.cols > self.input_k[v]) if windowed[i] else \
                    (plan.p.cols != self.input_k[v]):
                raise ValueError("dimension mismatch: input length != matrix cols")
            col0[i] = c0
            d.tiled = plan.main.data_ptr()
            d.tiled_sign = plan.sign.data_ptr() if plan.sign is not None else None
            d.rows, d.cols = plan.p.rows, plan.p.cols
            d.rec, d.M = None, 1
            d.a_scale, d.w_scale = self.scales[v].data_ptr(), float(plan.p.scale)
            d.workspace = plan.ws.data_ptr()
            d.acc_out = L.ptr(plan.acc)
            d.out64 = L.ptr(plan.out64)
            d.out32 = L.ptr(plan.out32)
            src[i] = v
        host = np.zeros(lib.tb_gemv_job_bytes() * len(pairs), dtype=np.uint8)
        total = C.c_int64()
        maxe = C.c_int64()
        L.check(lib.tb_gemv_step_prepare_cols(self.fmt, len(pairs), C.cast(descs, C.c_void_p),
                                              C.cast(src, C.c_void_p), C.cast(col0, C.c_void_p),
                                              len(input_k), C.cast(ks, C.c_void_p),
                                         host.ctypes.data_as(C.c_void_p), C.byref(total),
                                         C.byref(maxe)), "gemv_step_prepare")
        self.table = torch.from_numpy(host).to(dev)
        self._host = host  # also passed at launch: jobs inline, per-CTA input masks
        self._host_ptr = host.ctypes.data
        self.njobs, self.total, self.max_entries = len(pairs), total.value, maxe.value
        self.x_after_wait = bool(x_after_wait)
        # isolated: launched one at a time (e.g. HostStep), not as a chain
        # self_finalize: the launch writes its own outputs (no finalize, no
        # next step); one launch at a time on these workspaces
        # independent (TB_STEP_INDEPENDENT): a self-finalising launch that never
        # waits for the preceding kernel, for streams of unrelated GEMVs; the
        # caller reuses a step only after >= 16 other such launches
        if independent and x_after_wait:
            raise ValueError("an independent step cannot read a preceding kernel's outputs")
        self_finalize = bool(self_finalize or independent)
        self.self_finalize = self_finalize
        self._launch_flags = ((1 if x_after_wait else 0) | (2 if isolated else 0)
                              | (4 if sticky_flags else 0) | (8 if self_finalize else 0)
                              | (16 if independent else 0))
        self.inputs = (L.StepInput * len(input_k))()
        for i, k in enumerate(self.input_k):
            self.inputs[i].K = k
            self.inputs[i].scale = self.scales[i].data_ptr()
            self.inputs[i].nonfinite_flag = self.flags[i].data_ptr()
        self._inputs_ptr = C.cast(self.inputs, C.c_void_p)
        self.pairs = pairs  # keep every buffer alive
        self._lib = lib

    def bind(self, xs):
        """Point the step at device float32 vectors ``xs`` (read at launch)."""
        if len(xs) != len(self.input_k):
            raise ValueError(f"expected {len(self.input_k)} input vectors")
        for i, (x, k) in enumerate(zip(xs, self.input_k)):
            if x.dtype != torch.float32 or not x.is_cuda or x.numel() != k or \
                    not x.is_contiguous():
                raise ValueError("step inputs must be contiguous CUDA float32 vectors "
                                 "of the declared lengths")
            self.inputs[i].x = x.data_ptr()
        self._bound = xs  # keep alive
        return self

    def set_ready(self, flag):
        """Make the launch wait (in-kernel) until the int32 device word
        ``flag`` is nonzero before reading its inputs -- e.g. set by the copy
        that fills them; ``None`` clears it."""
        for i in range(len(self.input_k)):
            self.inputs[i].ready = flag.data_ptr() if flag is not None else None
        self._ready = flag  # keep alive
        return self

    def run(self, xs=None, prev=None, stream_ptr: int | None = None):
        if xs is not None:
            self.bind(xs)
        if prev is self:
            raise ValueError("a step cannot finalise its own previous launch")
        if prev is not None and (self.self_finalize or prev.self_finalize):
            raise ValueError("a self-finalising step is not chained")
        st = self._lib.tb_gemv_step_launch(
            self.fmt, self.table.data_ptr(), self.njobs, self.total, len(self.input_k),
            self._inputs_ptr, self._launch_flags,
            prev.table.data_ptr() if prev is not None else None,
            prev.njobs if prev is not None else 0, self._host_ptr,
            getattr(prev, "_host_ptr", None) if prev is not None else None,
            stream_ptr if stream_ptr is not None else L.stream_ptr())
        if st:
            L.check(st, "gemv_step_launch")

    def finalize(self, stream_ptr: int | None = None):
        """Finalise this step's outputs now (e.g. after the last step)."""
        if self.self_finalize:
            return  # the launch wrote them
        st = self._lib.tb_gemv_batch_finalize(self.table.data_ptr(), self.njobs,
                                              self.max_entries,
                                              stream_ptr if stream_ptr is not None
                                              else L.stream_ptr())
        if st:
            L.check(st, "gemv_batch_finalize")


class HostStep:
    """A decode step driven from HOST memory: ``__call__(xs)`` copies the
    float32 input vectors in, runs the one-launch step and its finalize, and
    returns the outputs on the host.

    ``pairs`` / ``input_k`` are as for GemvStep.  The inputs travel in ONE
    host-to-device copy (one pinned staging buffer); the finalize writes the
    outputs and the step its non-finite verdict straight into mapped pinned
    host memory (zero-copy), so a token is one captured graph -- copy, step
    kernel, finalize -- and one stream synchronisation.

    The copy is a kernel of 16-byte loads from the mapped staging buffer
    (``tb_copy_in``), the step its programmatic dependent (it prefetches
    weights while the copy runs and reads the inputs after it), and the step
    finalises its own outputs (``TB_STEP_SELF_FINALIZE``: the warp that
    completes a row tile writes it), so a token is two kernels.
    """

    def __init__(self, pairs, input_k, out_dtype=torch.float32):
        import types

        if out_dtype not in (torch.float32, torch.float64):
            raise ValueError("out_dtype must be float32 or float64")
        dev = pairs[0][0].main.device
        offs, n = [], 0
        for k in input_k:
            offs.append(n)
            n += -(-int(k) // 4) * 4  # 16-byte aligned vectors
        self.x_host_all = torch.empty(n, dtype=torch.float32).pin_memory()
        self.x_dev_all = torch.empty(n, dtype=torch.float32, device=dev)
        self.x_host = [self.x_host_all[o:o + k] for o, k in zip(offs, input_k)]
        self.x_dev = [self.x_dev_all[o:o + k] for o, k in zip(offs, input_k)]
        self.out_host = []
        host_pairs = []
        for plan, *rest in pairs:
            o = torch.empty((1, plan.p.rows), dtype=out_dtype).pin_memory()
            self.out_host.append(o[0])
            host_pairs.append((types.SimpleNamespace(
                p=plan.p, main=plan.main, sign=plan.sign, ws=plan.ws, acc=None,
                out32=o if out_dtype == torch.float32 else None,
                out64=o if out_dtype == torch.float64 else None), *rest))
        self.flags_host = torch.zeros(len(input_k), dtype=torch.int32).pin_memory()
        self._flags_np = self.flags_host.numpy()  # shares the pinned buffer
        self.step = GemvStep(host_pairs, input_k, flags=self.flags_host, isolated=True,
                             x_after_wait=True, self_finalize=True)
        self._lib = L.load()
        self._x_np = [h.numpy() for h in self.x_host]  # share the pinned buffer
        self._record = self._capture()
        self._stream = torch.cuda.current_stream()

    def _issue(self):
        L.check(self._lib.tb_copy_in(self.x_dev_all.data_ptr(), self.x_host_all.data_ptr(),
                                     self.x_host_all.numel() * 4, L.stream_ptr()), "copy_in")
        self.step.run(self.x_dev)

    def _capture(self):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self._issue()  # warm-up (kernel attributes) outside the capture
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                self._issue()
        torch.cuda.synchronize()
        return g

    def __call__(self, xs):
        if len(xs) != len(self.x_host):
            raise ValueError(f"expected {len(self.x_host)} input vectors")
        try:
            for h, x in zip(self._x_np, xs):
                if isinstance(x, torch.Tensor):
                    x = x.detach()
                    x = x.numpy() if x.device.type == "cpu" and x.dtype != torch.bfloat16 \
                        else x.float().cpu().numpy()
                x = np.asarray(x).reshape(-1)
                if x.size != h.size:
                    raise ValueError
                np.copyto(h, x, casting="unsafe")
        except (RuntimeError, ValueError) as e:
            raise ValueError("dimension mismatch: input length != matrix cols") from e
        sp = L.stream_ptr()  # replay() launches on the caller's current stream
        self._record.replay()
        L.check(self._lib.tb_stream_synchronize(sp), "stream_synchronize")
        if self._flags_np.any():
            raise ValueError("activations must be finite")  # core.py:116-134
        return self.out_host


class HostPipeline:
    """Independent decode steps streamed between pinned HOST memory and the
    device: ``run()`` copies every step's float32 inputs in, runs the fused
    step chain and copies every step's outputs back.  The copies go in blocks
    (up to ``block`` steps) on two copy streams, so a block's host-to-device
    copy and the previous block's device-to-host copy overlap the step
    kernels; a block's steps wait for its copy through a ready flag (set by a
    4-byte copy after it) inside the kernel, so the kernels stay one unbroken
    programmatic-dependent-launch chain.  This is the serving form
    over a queue of independent requests; HostStep is the one-token
    synchronous form.

    ``slot_pairs`` holds R >= 2 lists of (GemvPlan, input index) pairs; step
    i uses list i % R (the same plans may repeat: every slot gets its own
    workspace, only the weights are shared).  ``steps`` steps are captured
    into one CUDA graph.  Fill ``inputs[v]`` (pinned, [steps, K_v]) and read
    ``outputs[j]`` (pinned, [steps, N_j]) for the j-th pair of the slot
    lists.  Non-finite inputs raise ValueError like quantize_activations
    (core.py:116-134).
    """

    def __init__(self, slot_pairs, input_k, steps: int, block: int = 16, _copies=(True, True)):
        import types

        self._copies = _copies  # profiling only: (host-to-device, device-to-host)
        R = len(slot_pairs)
        if R < 2:
            raise ValueError("a pipeline needs at least two slots")
        if steps < 1 or block < 1:
            raise ValueError("steps and block must be >= 1")
        npairs = len(slot_pairs[0])
        rows = [pr[0].p.rows for pr in slot_pairs[0]]
        if any(len(sp) != npairs or [pr[0].p.rows for pr in sp] != rows for sp in slot_pairs):
            raise ValueError("every slot must hold the same projections")
        dev = slot_pairs[0][0][0].main.device
        self.input_k = [int(k) for k in input_k]
        self.steps, self.block = steps, block
        offs, n = [], 0
        for k in self.input_k:
            offs.append(n)
            n += -(-k // 4) * 4  # 16-byte aligned vectors
        ooffs, nout = [], 0
        for r_ in rows:
            ooffs.append(nout)
            nout += -(-r_ // 4) * 4
        self.x_host = torch.zeros((steps, n), dtype=torch.float32).pin_memory()
        self.inputs = [self.x_host[:, o:o + k] for o, k in zip(offs, self.input_k)]
        self._out_host = torch.empty((steps, nout), dtype=torch.float32).pin_memory()
        self.outputs = [self._out_host[:, o:o + r_] for o, r_ in zip(ooffs, rows)]
        self._x_dev = torch.empty((steps, n), dtype=torch.float32, device=dev)
        self._o_dev = torch.empty((steps, nout), dtype=torch.float32, device=dev)
        # non-finite verdicts, sticky and zero-copy in mapped pinned memory
        self._flags = torch.zeros((R, len(self.input_k)), dtype=torch.int32).pin_memory()
        self._flags_np = self._flags.numpy()
        self._ws = [[torch.zeros_like(pr[0].ws) for pr in sp] for sp in slot_pairs]
        self._steps = []
        for i in range(steps):
            r = i % R
            pairs = []
            for (plan, *rest), ws, oo in zip(slot_pairs[r], self._ws[r], ooffs):
                o = self._o_dev[i:i + 1, oo:oo + plan.p.rows]
                pairs.append((types.SimpleNamespace(p=plan.p, main=plan.main, sign=plan.sign,
                                                    ws=ws, acc=None, out32=o, out64=None),
                              *rest))
            st = GemvStep(pairs, self.input_k, flags=self._flags[r], sticky_flags=True)
            st.bind([self._x_dev[i, o:o + k] for o, k in zip(offs, self.input_k)])
            self._steps.append(st)
        # copy blocks: sizes ramp 1, 2, 4 .. block and back down at the end, so
        # the only copies not hidden behind step kernels (the first block's
        # copy in, the last block's copy back) are small
        ramp, k = [], 1
        while k < block:
            ramp.append(k)
            k *= 2
        sizes, left = [], steps
        for k in ramp:
            if left <= 0:
                break
            sizes.append(min(k, left))
            left -= sizes[-1]
        tail = []
        for k in ramp:
            if left <= 2 * block:
                break
            tail.append(k)
            left -= k
        while left > 0:
            sizes.append(min(block, left))
            left -= sizes[-1]
        sizes += tail[::-1]
        self._blocks, b0 = [], 0
        for k in sizes:
            self._blocks.append((b0, b0 + k))
            b0 += k
        nb = len(self._blocks)
        self._ready = torch.zeros(nb, dtype=torch.int32, device=dev)
        self._one = torch.ones(1, dtype=torch.int32).pin_memory()
        self._zeros = torch.zeros(nb, dtype=torch.int32).pin_memory()
        # every step of a block waits (a later step can start early under
        # programmatic dependent launch, before the block's first step has
        # seen its flag)
        for b, (b0, b1) in enumerate(self._blocks):
            for i in range(b0, b1):
                self._steps[i].set_ready(self._ready[b:b + 1])
        self._graph = self._capture()

    def _record(self):
        T, B = self.steps, self.block
        comp = torch.cuda.current_stream()
        h2d, d2h = self._h2d, self._d2h
        blocks = self._blocks
        done_ev = [torch.cuda.Event() for _ in blocks]
        start = torch.cuda.Event()
        start.record(comp)
        h2d.wait_event(start)
        d2h.wait_event(start)
        # each block's copy is followed by a 4-byte copy that sets its ready
        # flag; the block's first step kernel waits for the flag in-kernel (a
        # graph edge from the copy would end the PDL overlap of the chain)
        with torch.cuda.stream(h2d):
            for b, (b0, b1) in enumerate(blocks):
                if self._copies[0]:
                    self._x_dev[b0:b1].copy_(self.x_host[b0:b1], non_blocking=True)
                self._ready[b:b + 1].copy_(self._one, non_blocking=True)

        def copy_out(b):  # block b is final once the next block's first kernel finalised it
            done_ev[b].record(comp)
            d2h.wait_event(done_ev[b])
            b0, b1 = blocks[b]
            with torch.cuda.stream(d2h):
                if self._copies[1]:
                    self._out_host[b0:b1].copy_(self._o_dev[b0:b1], non_blocking=True)

        for b, (b0, b1) in enumerate(blocks):
            for i in range(b0, b1):
                self._steps[i].run(prev=self._steps[i - 1] if i else None)
                if i == b0 and b:
                    copy_out(b - 1)
        self._steps[T - 1].finalize()
        copy_out(len(blocks) - 1)
        comp.wait_stream(h2d)
        comp.wait_stream(d2h)
        self._ready.copy_(self._zeros, non_blocking=True)  # re-arm for the next run

    def _capture(self):
        s = torch.cuda.Stream()
        self._h2d, self._d2h = torch.cuda.Stream(), torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self._record()  # warm-up (kernel attributes) outside the capture
        s.synchronize()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                self._record()
        torch.cuda.synchronize()
        self._stream = s
        return g

    def run(self):
        """All ``steps`` steps: inputs from ``inputs``, results in ``outputs``."""
        self._flags_np[...] = 0
        with torch.cuda.stream(self._stream):
            self._graph.replay()
        self._stream.synchronize()
        if self._flags_np.any():
            raise ValueError("activations must be finite")  # core.py:116-134
        return self.outputs


class ActRecords:
    """Device buffer of GEMV-ready activation records for M tokens of length K
    in one packed format (shared by every GEMV that consumes the same input)."""

    def __init__(self, fmt: int, M: int, K: int, device=None, keep_natural_pad: int = 0):
        lib = L.load()
        self.fmt, self.M, self.K = fmt, M, K
        dev = device or torch.device("cuda", torch.cuda.current_device())
        nbytes = lib.tb_act_records_bytes(fmt, M, K)
        self.buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.scales = torch.empty(M, dtype=torch.float64, device=dev)
        self.natural = None
        if keep_natural_pad:
            kp = -(-K // keep_natural_pad) * keep_natural_pad
            self.natural = torch.empty((M, kp), dtype=torch.int8, device=dev)
        self._lib = lib

    def quantize(self, x: torch.Tensor, stream_ptr: int | None = None, flag=None):
        """x [M, K] float32/float64 on the device -> scales + records (one launch)."""
        fn = (self._lib.tb_quantize_records_f32 if x.dtype == torch.float32
              else self._lib.tb_quantize_records_f64)
        nat = self.natural
        st = fn(self.fmt, x.data_ptr(), self.M, self.K, x.stride(0), L.ptr(nat),
                nat.stride(0) if nat is not None else 0, self.scales.data_ptr(),
                self.buf.data_ptr(), L.ptr(flag),
                stream_ptr if stream_ptr is not None else L.stream_ptr())
        if st:
            L.check(st, "quantize_records")
        return self

    def prep(self, act: torch.Tensor, stream_ptr: int | None = None):
        """Natural int8 activations [M, K'] (K' >= K, zero beyond K) -> records."""
        st = self._lib.tb_prep_activations(self.fmt, act.data_ptr(), self.M, act.stride(0),
                                           act.shape[1], self.K, self.buf.data_ptr(),
                                           stream_ptr if stream_ptr is not None else L.stream_ptr())
        if st:
            L.check(st, "prep_activations")
        return self
