"""paper_2410_16144_b200: B200-native ternary BitLinear hot path.

A drop-in for the pack / quantize / linear entry points of the reference
package ``ternpack`` (bitnet.cpp, arXiv 2410.16144, pkg/src/ternpack/
__init__.py:3-41): same names, argument meaning and error messages, with
CUDA tensors instead of NumPy arrays and hand-written sm_100a kernels
(libternary_b200.so, C ABI in include/ternary_b200.h) behind them.  There is
no CPU fallback: without a CUDA device or the built library every compute
call raises.
"""

from .core import (
    GemvResult,
    QuantizedActivations,
    TernaryMatrix,
    make_result,
    quantize_activations,
    quantize_tokens,
    round_half_away,
    ternarize_weights,
)
from .kernels import (
    KERNEL_PAD,
    ActRecords,
    GemvBatch,
    GemvPlan,
    GemvStep,
    HostStep,
    HostPipeline,
    StepGlue,
    KernelKind,
    gemm_prefill,
    gemv_f32_ref,
    gemv_i2s,
    gemv_parallel,
    gemv_ref_int32,
    gemv_tl1,
    gemv_tl2,
)
from .lut import TL1_PATTERNS, TL2_PATTERNS, LutTL1, LutTL2, build_lut_tl1, build_lut_tl2
from .packing import (
    PackedI2S,
    PackedTL1,
    PackedTL2,
    decode_i2s,
    decode_tl1,
    decode_tl2,
    encode_i2s,
    encode_tl1,
    encode_tl2,
    i2s_payload_bytes,
    tl1_index,
    tl1_payload_bytes,
    tl2_code,
    tl2_payload_bytes,
)

__version__ = "0.1.0"
