"""Domain types, ternarisation and activation quantisation on the GPU.

Mirrors ``ternpack.core`` (pkg/src/ternpack/core.py) with CUDA tensors in
place of NumPy arrays: same names, same argument meaning, same ValueError
messages.  Arithmetic runs in the sm_100a kernels of libternary_b200.so
(quantize.cu); results are bit-identical to the reference:

  * ``quantize_activations``  -> core.py:116-134 (float64, round half away)
  * ``ternarize_weights``     -> core.py:104-113 (scale = NumPy-pairwise mean)
  * ``make_result``           -> core.py:99-101

``quantize_activations`` keeps the reference semantics exactly: any input
shape is flattened to one vector with one scale (core.py:123).  The batched
extension is ``quantize_tokens``: a 2-D [M, K] input is M tokens with one
absmax scale each, i.e. M reference calls in one launch.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L

__all__ = [
    "TernaryMatrix",
    "QuantizedActivations",
    "GemvResult",
    "ternarize_weights",
    "quantize_activations",
    "quantize_tokens",
    "round_half_away",
    "make_result",
    "device",
]


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2410_16144_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    L.load()
    return torch.device("cuda", torch.cuda.current_device())


def to_device(x, dtype=None) -> torch.Tensor:
    dev = device()
    if isinstance(x, torch.Tensor):
        t = x.to(dev, non_blocking=True)
        return t if dtype is None else t.to(dtype)
    a = np.asarray(x)
    if dtype is None:
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    return torch.as_tensor(a, device=dev).to(dtype)


def round_half_away(x) -> torch.Tensor:
    """Nearest integer, ties away from zero, in float64 (core.py:24-27)."""
    v = to_device(x, torch.float64)
    return torch.trunc(v + torch.copysign(torch.full_like(v, 0.5), v))


def _freeze(t: torch.Tensor) -> torch.Tensor:
    return t.contiguous()


@dataclass(frozen=True)
class TernaryMatrix:
    """Dense row-major {-1, 0, +1} matrix (device int8) with one scale."""

    rows: int
    cols: int
    values: torch.Tensor  # int8 [rows, cols] on the GPU
    scale: float
    _checked: bool = field(default=False, compare=False, repr=False)

    def __post_init__(self):
        if self.rows < 1 or self.cols < 1:
            raise ValueError("rows and cols must be positive")
        v = to_device(self.values, torch.int8).reshape(self.rows, self.cols)
        if not self._checked and v.numel():
            lo, hi = torch.aminmax(v)
            if int(lo) < -1 or int(hi) > 1:
                raise ValueError("ternary values must lie in {-1, 0, +1}")
        if not (np.isfinite(self.scale) and self.scale > 0):
            raise ValueError("scale must be positive and finite")
        object.__setattr__(self, "values", _freeze(v))
        object.__setattr__(self, "scale", float(self.scale))

    def dequantized(self, dtype=torch.float32) -> torch.Tensor:
        return self.values.to(dtype) * torch.tensor(self.scale, dtype=dtype,
                                                    device=self.values.device)


@dataclass(frozen=True)
class QuantizedActivations:
    """int8 activations with absmax scale(s); may carry trailing zero padding.

    ``data`` is [K] for one token (the reference type) or [M, K] for a batch;
    ``scales`` is the device float64 [M] tensor the kernels consume and
    ``scale`` the host float of token 0 (reference attribute).
    """

    data: torch.Tensor
    scale: float
    original_len: int
    scales: torch.Tensor | None = field(default=None, compare=False, repr=False)
    _trusted: bool = field(default=False, compare=False, repr=False)
    _cache: dict = field(default_factory=dict, compare=False, repr=False)
    # set by quantize_*(check_finite=False): ``scale`` is read from the device
    # scales[0] on first access instead of at quantisation time (no sync)
    _lazy_scale: bool = field(default=False, compare=False, repr=False)

    def __getattribute__(self, name):
        if name == "scale" and object.__getattribute__(self, "_lazy_scale"):
            v = float(object.__getattribute__(self, "scales")[0].item())
            object.__setattr__(self, "scale", v)
            object.__setattr__(self, "_lazy_scale", False)
            return v
        return object.__getattribute__(self, name)

    def __post_init__(self):
        d = to_device(self.data, torch.int8)
        if d.dim() == 0 or d.dim() > 2:
            d = d.reshape(-1)
        K = d.shape[-1]
        if self.original_len < 1 or self.original_len > K:
            raise ValueError("original_len must be in [1, len(data)]")
        lazy = object.__getattribute__(self, "_lazy_scale")
        if not self._trusted:
            if d.numel() and int(d.min()) < -127:
                raise ValueError("activation value -128 is never produced")
            if bool((d[..., self.original_len:] != 0).any()):
                raise ValueError("padding entries must be zero")
            if not (np.isfinite(self.scale) and self.scale > 0):
                raise ValueError("scale must be positive and finite")
        object.__setattr__(self, "data", d.contiguous())
        if self.scales is None:
            if lazy:
                raise ValueError("a lazily read scale needs the device scales")
            object.__setattr__(self, "scales", torch.full(
                (self.tokens,), float(self.scale), dtype=torch.float64, device=d.device))
        if not lazy:
            object.__setattr__(self, "scale", float(self.scale))

    @property
    def tokens(self) -> int:
        return 1 if self.data.dim() == 1 else self.data.shape[0]

    def __len__(self) -> int:
        return self.data.shape[-1]


@dataclass(frozen=True)
class GemvResult:
    """Exact int32 accumulators plus float64 outputs (device tensors)."""

    accumulators: torch.Tensor | None
    output: torch.Tensor


def make_result(acc: torch.Tensor, weight_scale: float, a_scales) -> GemvResult:
    """output = float64(acc) * weight_scale * act_scale (core.py:99-101)."""
    dev = acc.device
    if not isinstance(a_scales, torch.Tensor):
        a_scales = torch.tensor([float(a_scales)], dtype=torch.float64, device=dev)
    M = 1 if acc.dim() == 1 else acc.shape[0]
    N = acc.shape[-1]
    out = torch.empty(acc.shape, dtype=torch.float64, device=dev)
    L.check(L.load().tb_scale_outputs(L.ptr(acc), M, N, float(weight_scale),
                                      L.ptr(a_scales), L.ptr(out), None, L.stream_ptr()),
            "scale_outputs")
    return GemvResult(accumulators=acc, output=out)


# ---------------------------------------------------------------------------
# ternarize_weights: scale bit-identical to np.mean(np.abs(w.astype(f64)))
# ---------------------------------------------------------------------------

_PW_BLOCK = 128


def _pairwise_split(n: int) -> int:
    n2 = n // 2
    return n2 - n2 % 8


def _subtrees(n: int, min_leaf: int = 4096, max_subtrees: int = 1 << 15):
    """Cut NumPy's pairwise-summation tree into subtrees evaluated on device.

    Returns (offsets, lengths, combine) where combine(sums) re-adds the
    subtree sums in NumPy's association order.
    """
    offs, lens = [], []

    def rec(off, m, budget):
        if m <= _PW_BLOCK or m < min_leaf or budget <= 1:
            offs.append(off)
            lens.append(m)
            return ("leaf", len(offs) - 1)
        n2 = _pairwise_split(m)
        return ("node", rec(off, n2, budget // 2), rec(off + n2, m - n2, budget // 2))

    tree = rec(0, n, max_subtrees)

    def combine(sums):
        def ev(t):
            if t[0] == "leaf":
                return float(sums[t[1]])
            return ev(t[1]) + ev(t[2])
        return ev(tree)

    return offs, lens, combine


def ternarize_weights(weights, rows: int, cols: int) -> TernaryMatrix:
    """Absmean ternarisation (core.py:104-113) on the GPU."""
    lib = L.load()
    w = weights if isinstance(weights, torch.Tensor) else np.asarray(weights)
    is32 = (w.dtype == torch.float32) if isinstance(w, torch.Tensor) else (w.dtype == np.float32)
    wd = to_device(w, torch.float32 if is32 else torch.float64).reshape(-1).contiguous()
    n = rows * cols
    if wd.numel() != n:
        raise ValueError(f"cannot reshape {wd.numel()} weights into ({rows}, {cols})")
    dev = wd.device
    offs, lens, combine = _subtrees(n)
    d_off = torch.tensor(offs, dtype=torch.int64, device=dev)
    d_len = torch.tensor(lens, dtype=torch.int64, device=dev)
    sums = torch.empty(len(offs), dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    s = L.stream_ptr()
    fn = lib.tb_abs_pairwise_sums_f32 if is32 else lib.tb_abs_pairwise_sums_f64
    L.check(fn(L.ptr(wd), L.ptr(d_off), L.ptr(d_len), len(offs), L.ptr(sums), L.ptr(flag), s),
            "abs_pairwise_sums")
    host = sums.cpu().numpy()
    if int(flag.item()):
        raise ValueError("weights must be finite")
    scale = float(np.float64(combine(host)) / np.float64(n))
    if scale == 0.0:
        raise ValueError("degenerate weight matrix")
    q = torch.empty(n, dtype=torch.int8, device=dev)
    fn = lib.tb_ternarize_apply_f32 if is32 else lib.tb_ternarize_apply_f64
    L.check(fn(L.ptr(wd), n, scale, L.ptr(q), s), "ternarize_apply")
    return TernaryMatrix(rows=rows, cols=cols, values=q.view(rows, cols), scale=scale,
                         _checked=True)


# ---------------------------------------------------------------------------
# quantize_activations
# ---------------------------------------------------------------------------

def _pad(n: int, m: int) -> int:
    return -(-n // m) * m


def quantize_into(x: torch.Tensor, q: torch.Tensor, scales: torch.Tensor,
                  flag: torch.Tensor | None = None, stream=None) -> None:
    """Low-level launch: x [M, K] (f32/f64, device) -> q [M, ldq] int8, scales [M]."""
    lib = L.load()
    M, K = x.shape
    fn = lib.tb_quantize_f32 if x.dtype == torch.float32 else lib.tb_quantize_f64
    L.check(fn(L.ptr(x), M, K, x.stride(0), L.ptr(q), q.stride(0), L.ptr(scales),
               L.ptr(flag), L.stream_ptr(stream)), "quantize")


def _host_f64(x):
    """Host view of a CPU input as float64 (any dtype: bf16, int8, requires_grad)."""
    if isinstance(x, torch.Tensor):
        return x.detach().to(torch.float64).numpy()
    return np.asarray(x, dtype=np.float64)


def _quantize(x, pad_to: int, batched: bool, check_finite: bool) -> QuantizedActivations:
    if pad_to not in (1, 2, 3, 4):
        raise ValueError("pad_to must be in {1, 2, 3, 4}")
    if isinstance(x, torch.Tensor):
        is32 = x.dtype == torch.float32
        on_host = x.device.type == "cpu"
    else:
        x = np.asarray(x)
        is32 = x.dtype == np.float32
        on_host = True
    # float32 stays float32 (x / scale is then formed from the exact float32
    # value, as NumPy does after its float64 cast); everything else -> float64
    xd = to_device(x, torch.float32 if is32 else torch.float64)
    if batched:
        if xd.dim() != 2:
            raise ValueError("quantize_tokens expects a 2-D [tokens, K] input")
    else:
        xd = xd.reshape(1, -1)  # core.py:123: any shape is one vector
    M, K = xd.shape
    if K < 1 or M < 1:
        raise ValueError("empty activation vector")
    xd = xd.contiguous()
    Kp = _pad(K, pad_to)
    q = torch.empty((M, Kp), dtype=torch.int8, device=xd.device)
    scales = torch.empty(M, dtype=torch.float64, device=xd.device)
    lazy = False
    if check_finite and on_host:
        # host input: the finiteness verdict and token 0's scale come from a
        # float64 host view (no device round trip); max|x| of the float64 view
        # is the reference's amax exactly (core.py:123-129), so s0 equals the
        # device-computed scales[0]
        am = np.abs(_host_f64(x).reshape(M, K)).max(axis=1)  # NaN / inf propagate
        if not np.isfinite(am).all():
            raise ValueError("activations must be finite")
        amax0 = float(am[0])
        s0 = amax0 / 127.0 if amax0 > 0 else 1.0
        quantize_into(xd, q, scales, None)
    elif check_finite:
        flag = torch.zeros(1, dtype=torch.int32, device=xd.device)
        quantize_into(xd, q, scales, flag)
        if int(flag.item()):
            raise ValueError("activations must be finite")
        s0 = float(scales[0].item())
    else:
        quantize_into(xd, q, scales, None)
        s0, lazy = 0.0, True
    data = q if batched else q[0]
    return QuantizedActivations(data=data, scale=s0, original_len=K, scales=scales,
                                _trusted=True, _lazy_scale=lazy)


def quantize_activations(x, pad_to: int = 1, *, check_finite: bool = True
                         ) -> QuantizedActivations:
    """Absmax int8 quantisation, zero-padded to a multiple of ``pad_to``
    (core.py:116-134): the input is flattened to ONE vector with one scale.
    ``check_finite=False`` skips the host-side verdict (no device sync); the
    ``scale`` attribute is then read from the device on first access."""
    return _quantize(x, pad_to, False, check_finite)


def quantize_tokens(x, pad_to: int = 1, *, check_finite: bool = True) -> QuantizedActivations:
    """Batched extension: x [M, K] is M tokens, each quantised as its own
    reference call (one absmax scale per token); ``data`` is [M, K_pad],
    ``scales`` [M] and ``scale`` token 0's."""
    return _quantize(x, pad_to, True, check_finite)
