"""Layer-stack decode runner for BASELINE configs 2 and 4 (M=1 and small M).

The reference times a stack as per-layer GEMV passes over freshly quantised
activations (bench._token_pass_int, pkg/src/ternpack/bench.py:138-153: per
layer two quantisations -- the hidden vector feeds q/k/v/o/gate/up, the
intermediate vector feeds down -- and 7 GEMVs).  Here one layer is ONE
launch (GemvStep: both inputs quantised in every CTA, the 7 projections as
one grouped GEMV, the previous layer's outputs finalised after its own work);
for M > 1 a layer is a StepGlue (finalise + quantise M tokens) and a
GemvBatch.  Weights are generated like BASELINE.json's configs: seeded
N(0, 0.02) latent matrices, absmean-ternarised on the GPU (core.py:104-113),
packed to I2_S or TL2 and repacked to the tiled layout.
"""

from __future__ import annotations

import torch

from . import _lib as L
from .core import ternarize_weights
from .kernels import ActRecords, GemvBatch, GemvPlan, GemvStep, StepGlue
from .packing import encode_i2s, encode_tl1, encode_tl2

__all__ = ["STACKS", "stack_shapes", "LayerStack"]

# (hidden, q/o out, k/v out, intermediate, layers) -- BASELINE.json configs 2 and 4
STACKS = {
    "cfg2": {"hidden": 4096, "kv": 1024, "inter": 14336, "layers": 32},
    "cfg4": {"hidden": 10240, "kv": 1280, "inter": 32768, "layers": 80},
}
_ENC = {"i2s": encode_i2s, "tl1": encode_tl1, "tl2": encode_tl2}


def stack_shapes(cfg: dict):
    """[(name, rows, cols, input)] of one layer; input 0 = hidden, 1 = intermediate."""
    h, kv, i = cfg["hidden"], cfg["kv"], cfg["inter"]
    return [("q", h, h, 0), ("k", kv, h, 0), ("v", kv, h, 0), ("o", h, h, 0),
            ("gate", i, h, 0), ("up", i, h, 0), ("down", h, i, 1)]


def packed_bytes(fmt: str, rows: int, cols: int) -> int:
    lib = L.load()
    if fmt == "tl2":
        return rows * (lib.tb_ref_row_bytes(L.TL2, cols) + lib.tb_ref_sign_row_bytes(cols))
    return rows * lib.tb_ref_row_bytes(L.I2S if fmt == "i2s" else L.TL1, cols)


class LayerStack:
    """All layers of a config resident on one GPU, plus per-layer launch objects."""

    def __init__(self, cfg: dict, fmt: str = "i2s", seed: int = 0, tokens: int = 1,
                 layers: int | None = None, device=None):
        if fmt not in _ENC:
            raise ValueError(f"unknown format {fmt}")
        self.cfg, self.fmt, self.tokens = cfg, fmt, tokens
        self.nlayers = layers or cfg["layers"]
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.shapes = stack_shapes(cfg)
        self.layers = []
        gen = torch.Generator(device=dev)
        for li in range(self.nlayers):
            plans = []
            for mi, (_, rows, cols, _) in enumerate(self.shapes):
                gen.manual_seed(seed * 1_000_003 + li * 131 + mi)
                w = torch.randn(rows, cols, generator=gen, device=dev) * 0.02
                p = _ENC[fmt](ternarize_weights(w, rows, cols))
                del w
                plans.append(GemvPlan(p, max_tokens=tokens, out_dtype=torch.float32))
            self.layers.append(plans)
        self.algo_bytes = sum(packed_bytes(fmt, r, c) + tokens * c + 4 * tokens * r
                              for _, r, c, _ in self.shapes) * self.nlayers
        h, i = cfg["hidden"], cfg["inter"]
        self.ks = [h, i]
        if tokens == 1:
            self.steps = [GemvStep([(p, s[3]) for p, s in zip(plans, self.shapes)], self.ks)
                          for plans in self.layers]
        else:
            self.rec = [ActRecords(L.TL2 if fmt == "tl2" else L.I2S, tokens, k) for k in self.ks]
            self.batches = [GemvBatch([(p, self.rec[s[3]]) for p, s in zip(plans, self.shapes)])
                            for plans in self.layers]
            self.tail = StepGlue([])

    def token_pass(self, xh, xi, glue_pool=None):
        """Launch one token pass (all layers); layer l reads xh[l], xi[l]
        (device float32 vectors [K] for M=1, or the fixed [M, K] buffers bound
        in ``glue_pool`` for M > 1).  Outputs of the last layer are finalised
        at the end.  Capturable in a CUDA graph."""
        if self.tokens == 1:
            prev = None
            for li, st in enumerate(self.steps):
                st.run([xh[li], xi[li]], prev=prev)
                prev = st
            prev.finalize()
        else:
            prev = None
            for li, b in enumerate(self.batches):
                glue_pool[li].retarget(prev).run()
                b.run(finalize=False)
                prev = b
            self.tail.retarget(prev).run()

    def make_glues(self, XH, XI):
        """M > 1: one StepGlue per layer quantising rows of XH[l] / XI[l] ([M, K])."""
        return [StepGlue([(XH[li], self.rec[0]), (XI[li], self.rec[1])])
                for li in range(self.nlayers)]
