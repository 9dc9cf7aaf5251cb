"""Layer-stack decode runner for BASELINE configs 2 and 4, tensor parallel.

The reference times a stack as per-layer GEMV passes over freshly quantised
activations (bench._token_pass_int, pkg/src/ternpack/bench.py:138-153: per
layer two quantisations -- the hidden vector feeds q/k/v/o/gate/up, the
intermediate vector feeds down -- and 7 GEMVs).  Here one layer is ONE
launch (GemvStep: both inputs quantised in every CTA, the 7 projections as
one grouped GEMV, the previous layer's outputs finalised after its own work);
for M > 1 a layer is a StepGlue (finalise + quantise M tokens) and a
GemvBatch.  Weights are generated like BASELINE.json's configs: seeded
N(0, 0.02) latent matrices, absmean-ternarised on the GPU (core.py:104-113),
packed to I2_S / TL1 / TL2 and repacked to the tiled layout.

Tensor parallel (``tp_world > 1``; one process per GPU):

* column-parallel q/k/v/gate/up: rank r owns rows [r0, r1) of the packed
  matrix (a byte slice, tp.column_shard) and writes its output rows only;
* row-parallel o/down: rank r owns input columns [k0, k1) (tp.row_shard,
  k0 a multiple of one record chunk), reads those columns of the replicated
  input vector -- quantised whole, so the per-token scale is the reference's
  absmax over the full token (core.py:128) -- and produces int32 partial
  accumulators.  Once a layer's step has been finalised (by the next
  layer's step), the layer's partials (o and down, one contiguous int32
  buffer) are summed over the ranks and only then scaled,
  out = f64(sum) * w_scale * a_scale (core.py:99-101): integer sums are
  exact and order independent, so every tp degree is bit-identical to tp=1
  and to the reference.

The sum goes through a ``Collective``: ``tp.PeerAllReduce`` (ours: one
kernel over NVLink peer memory that sums and scales; the default),
``tp.TorchAllReduce`` (NCCL / gloo through torch.distributed, then the
scale kernel: the baseline) or ``tp.EmulatedGroup`` (all ranks in one
process on one GPU, for tests).  The weight matrices are generated whole
on every rank from the same seeds (so the weight scale is the full
matrix's, as in the reference) and then sliced.
"""

from __future__ import annotations

import os

import torch

from . import _lib as L
from . import tp as TP
from .core import ternarize_weights
from .kernels import ActRecords, GemvBatch, GemvPlan, GemvStep, StepGlue
from .packing import PackedI2S, PackedTL1, PackedTL2, encode_i2s, encode_tl1, encode_tl2

__all__ = ["STACKS", "stack_shapes", "LayerStack", "ROW_PARALLEL", "packed_bytes"]

# (hidden, k/v out, intermediate, layers) -- BASELINE.json configs 2 and 4
STACKS = {
    "cfg2": {"hidden": 4096, "kv": 1024, "inter": 14336, "layers": 32},
    "cfg4": {"hidden": 10240, "kv": 1280, "inter": 32768, "layers": 80},
}
_ENC = {"i2s": encode_i2s, "tl1": encode_tl1, "tl2": encode_tl2}
_FMT = {"i2s": L.I2S, "tl1": L.TL1, "tl2": L.TL2}
ROW_PARALLEL = ("o", "down")
# one record chunk (16 packed bytes): the granularity of a row-parallel K-shard
CHUNK_W = {"i2s": 64, "tl1": 64, "tl2": 96}


def stack_shapes(cfg: dict):
    """[(name, rows, cols, input)] of one layer; input 0 = hidden, 1 = intermediate."""
    h, kv, i = cfg["hidden"], cfg["kv"], cfg["inter"]
    return [("q", h, h, 0), ("k", kv, h, 0), ("v", kv, h, 0), ("o", h, h, 0),
            ("gate", i, h, 0), ("up", i, h, 0), ("down", h, i, 1)]


def packed_bytes(fmt: str, rows: int, cols: int) -> int:
    """Reference packed size (packing.py:42-53)."""
    lib = L.load()
    if fmt == "tl2":
        return rows * (lib.tb_ref_row_bytes(L.TL2, cols) + lib.tb_ref_sign_row_bytes(cols))
    return rows * lib.tb_ref_row_bytes(_FMT[fmt], cols)


def shard_plan(cfg: dict, fmt: str, rank: int, world: int):
    """Per projection of one layer: (name, rows, cols, input, kind, lo, hi) --
    kind 'col' owns rows [lo, hi), 'row' owns input columns [lo, hi), 'full'
    is unsharded (world 1).  Row boundaries are whole 32-row tiles where the
    sizes allow; column boundaries whole record chunks."""
    out = []
    for name, rows, cols, src in stack_shapes(cfg):
        if world == 1:
            out.append((name, rows, cols, src, "full", 0, rows))
        elif name in ROW_PARALLEL:
            lo, hi = TP.shard_range(cols, world, rank, CHUNK_W[fmt])
            out.append((name, rows, cols, src, "row", lo, hi))
        else:
            lo, hi = TP.shard_range(rows, world, rank, 32 if rows % (32 * world) == 0 else 1)
            out.append((name, rows, cols, src, "col", lo, hi))
    return out


def _slice(p, fmt: str, kind: str, lo: int, hi: int):
    """Shard of a packed reference matrix as a packed matrix of its own."""
    if kind == "full":
        return p
    if fmt == "tl2":
        planes = (p.index_data, p.sign_data)
    else:
        planes = (p.data,)
    if kind == "col":
        sl = TP.column_shard(planes, lo, hi)
        rows, cols = hi - lo, p.cols
    else:
        sl, cols = TP.row_shard(_FMT[fmt], planes, p.cols, lo, hi)
        rows = p.rows
    pad = {"i2s": 4, "tl1": 2, "tl2": 6}[fmt]
    pc = -(-cols // pad) * pad
    sl = tuple(t.contiguous() for t in sl)
    if fmt == "i2s":
        return PackedI2S(rows=rows, cols=cols, padded_cols=pc, data=sl[0], scale=p.scale,
                         trusted=True)
    if fmt == "tl1":
        return PackedTL1(rows=rows, cols=cols, padded_cols=pc, data=sl[0], scale=p.scale,
                         trusted=True)
    return PackedTL2(rows=rows, cols=cols, padded_cols=pc, index_data=sl[0], sign_data=sl[1],
                     scale=p.scale, trusted=True)


# one M-token records table per CTA (TB_TABLE_KB in csrc/gemv.cu, 60 KB, two
# CTAs per SM): the longest K-window, in record chunks, whose M-token records
# fit.  A launch takes <= _MAX_JOBS jobs in <= _MAX_SEGS runs of jobs on the
# same (input, K-window) (kMaxInlineJobs / kMaxSegs in csrc/gemv.cu).
_TABLE_BYTES = int(os.environ.get("TB_TABLE_KB", "60")) * 1024  # (env: profiling variants)
_MAX_JOBS, _MAX_SEGS = 20, 8


def window_chunks(fmt: str, tokens: int) -> int:
    rec = (112 if fmt == "tl2" else 80) + 4  # + the chunk's entry of the prefix-sum table
    return ((_TABLE_BYTES - 4 * tokens - 16) // (tokens * rec)) // 4 * 4


class _WindowedView:
    """A matrix contracted as K-window column shards (one GemvPlan each, one
    shared workspace, outputs on the first): the packed matrix and its output
    buffer, as a GemvPlan would hold them."""

    def __init__(self, p, first):
        self.p = p
        self.out32, self.out64, self.acc = first.out32, first.out64, first.acc
        self.ws = first.ws
        self.windows = []


def _windowed(p, fmt: str, tokens: int, src: int, kw: int):
    """(view, [(plan, input, col0)]): p's columns in windows of <= kw record
    chunks (near-even, whole 4-chunk groups)."""
    cw = CHUNK_W[fmt]
    nchunk = -(-p.cols // cw)
    nwin = -(-nchunk // kw)
    per = -(-(-(-nchunk // nwin)) // 4) * 4
    jobs, first = [], None
    for w in range(nwin):
        lo, hi = w * per * cw, min(p.cols, (w + 1) * per * cw)
        if lo >= hi:
            break
        shard = _slice(p, fmt, "row", lo, hi)
        plan = GemvPlan(shard, max_tokens=tokens,
                        out_dtype=torch.float32 if first is None else None)
        if first is None:
            first = plan
        else:
            plan.ws = first.ws  # partial sums of every window accumulate here
        jobs.append((plan, src, lo))
    view = _WindowedView(p, first)
    view.windows = [j[0] for j in jobs]
    return view, jobs


class LayerStack:
    """All layers of a config (this rank's shards) resident on one GPU, plus
    the per-layer launch objects."""

    def __init__(self, cfg: dict, fmt: str = "i2s", seed: int = 0, tokens: int = 1,
                 layers: int | None = None, device=None, tp_rank: int = 0, tp_world: int = 1,
                 collective=None, part_alloc=None, pipelined: bool | None = None):
        if fmt not in _ENC:
            raise ValueError(f"unknown format {fmt}")
        if tp_world > 1 and tokens != 1:
            raise ValueError("tensor-parallel stacks decode one token per step (M=1)")
        if tp_world > 1 and collective is None:
            raise ValueError("a tensor-parallel stack needs a collective")
        self.cfg, self.fmt, self.tokens = cfg, fmt, tokens
        self.rank, self.world, self.coll = tp_rank, tp_world, collective
        self.nlayers = layers or cfg["layers"]
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.shapes = stack_shapes(cfg)
        self.plan = shard_plan(cfg, fmt, tp_rank, tp_world)
        h, i = cfg["hidden"], cfg["inter"]
        self.ks = [h, i]
        # row-parallel partials of a layer: one contiguous int32 buffer
        # [o rows | down rows] (symmetric across ranks for the peer kernel)
        self.rp = [(j, s[1]) for j, s in enumerate(self.plan) if s[4] == "row"]
        self.part_len = sum(r for _, r in self.rp)
        self.parts = None
        if part_alloc is None and collective is not None:
            part_alloc = collective.part_alloc
        if self.rp:
            n = self.nlayers * self.part_len
            self.parts = (part_alloc(n) if part_alloc is not None else
                          torch.zeros(n, dtype=torch.int32, device=dev)).view(self.nlayers, -1)
            self.rp_out = torch.empty((self.nlayers, self.part_len), dtype=torch.float32,
                                      device=dev)
        self.layers = []
        # M > 1 (I2_S / TL1): every CTA of the grouped GEMV keeps its segment's
        # records in one shared-memory table (tb_gemv_batch_launch_inline);
        # an input too long for one table is contracted in K-windows, each a
        # column shard of the matrix, all accumulating into one workspace
        # that the first window's job finalises.  window_jobs[li]: (plan, input, col0)
        self.window_jobs = []
        kw = window_chunks(fmt, tokens) if 1 < tokens <= 8 and fmt != "tl2" else 0
        gen = torch.Generator(device=dev)
        for li in range(self.nlayers):
            plans, jobs = [], []
            for mi, (name, rows, cols, src, kind, lo, hi) in enumerate(self.plan):
                gen.manual_seed(seed * 1_000_003 + li * 131 + mi)
                w = torch.randn(rows, cols, generator=gen, device=dev) * 0.02
                p = _ENC[fmt](ternarize_weights(w, rows, cols))
                del w
                p = _slice(p, fmt, kind, lo, hi)
                rowpar = kind == "row"
                nchunk = -(-p.cols // CHUNK_W[fmt])
                if kw and nchunk > kw:
                    view, wjobs = _windowed(p, fmt, tokens, src, kw)
                    plans.append(view)
                    jobs += wjobs
                    continue
                plan = GemvPlan(p, max_tokens=tokens,
                                out_dtype=None if rowpar else torch.float32)
                if rowpar:  # partials land in the layer's slice of the symmetric buffer
                    off = sum(r for j, r in self.rp if j < mi)
                    plan.acc = self.parts[li, off:off + rows].view(1, rows)
                plans.append(plan)
                jobs.append((plan, src, 0))
            # one table segment per (input, K-window): its jobs adjacent
            jobs.sort(key=lambda j: (j[1], j[2]))
            self.layers.append(plans)
            self.window_jobs.append(jobs)
        # algorithmic bytes of THIS rank's shards: packed bytes
        # + M * (columns contracted) int8 activations + 4 * M * (rows written)
        self.algo_bytes = sum(packed_bytes(fmt, p.p.rows, p.p.cols) + tokens * p.p.cols
                              + 4 * tokens * p.p.rows for p in self.layers[0]) * self.nlayers
        if tokens == 1:
            self.steps = [GemvStep([(p, s[3], s[5] if s[4] == "row" else 0)
                                    for p, s in zip(plans, self.plan)], self.ks)
                          for plans in self.layers]
        else:
            # record sets in rotation.  Glue finalise mode (the glue of layer
            # l quantises layer l while finalising layer l-1, whose outputs are
            # scaled by layer l-1's a_scale): two sets.  Tail finalise mode
            # (records tables; GEMV l finalises layer l-1 in its tail; glue l
            # quantises BEFORE waiting on GEMV l-1, overlapping it): three
            # sets -- glue l writes set l % 3 while GEMV l-1 reads set (l-1) % 3
            # and finalises with set (l-2) % 3's scales.
            self.tail_fin = fmt != "tl2" and tokens <= 8 and all(
                len(j) <= _MAX_JOBS and len({(x[1], x[2]) for x in j}) <= _MAX_SEGS
                for j in self.window_jobs)
            self.nsets = 3 if self.tail_fin else 2
            # pipelined layers (tb_step_glue_sync / tb_gemv_batch_launch_sync):
            # a layer's GEMV waits for its glue's records, not for the glue's
            # completion (= the previous GEMV's), so consecutive layers'
            # streams overlap; 4 counters per layer, reset by the kernels
            if pipelined is None:
                pipelined = os.environ.get("TB_M8_PIPELINED", "1") != "0"
            self.piped = self.tail_fin and pipelined
            self.sync = (torch.zeros((self.nlayers, 4), dtype=torch.int32, device=dev)
                         if self.piped else None)
            self.glue_fin = os.environ.get("TB_M8_GLUE_FIN", "1") != "0"
            self.rec = [[ActRecords(L.TL2 if fmt == "tl2" else L.I2S, tokens, k)
                         for k in self.ks] for _ in range(self.nsets)]
            self.batches = [GemvBatch([(p, self.rec[li % self.nsets][src], c0)
                                       for p, src, c0 in self.window_jobs[li]])
                            for li in range(self.nlayers)]
            self.tail = StepGlue([])
        if self.rp:
            # what the reduction scales: per row-parallel projection
            # (rows, w_scale, the step's device scale of its input)
            self.rp_jobs = []
            for li in range(self.nlayers):
                segs, off = [], 0
                for j, rows in self.rp:
                    p = self.layers[li][j]
                    segs.append((off, rows, float(p.p.scale), self.steps[li].scales[self.plan[j][3]]))
                    off += rows
                self.rp_jobs.append(segs)
            self.coll.bind(self)

    # ------------------------------------------------------------- decode
    def token_pass(self, xh, xi, glue_pool=None):
        """Launch one token pass (all layers); layer l reads xh[l], xi[l]
        (device float32 vectors [K] for M=1, or the fixed [M, K] buffers bound
        in ``glue_pool`` for M > 1).  Outputs of the last layer are finalised
        at the end.  Capturable in a CUDA graph (with a capturable collective)."""
        if self.tokens == 1:
            prev = None
            for li, st in enumerate(self.steps):
                st.run([xh[li], xi[li]], prev=prev)
                if prev is not None and self.rp:
                    self.coll.reduce_layer(self, li - 1)  # step li finalised layer li-1
                prev = st
            prev.finalize()
            if self.rp:
                self.coll.reduce_layer(self, self.nlayers - 1)
        else:
            # records-table mode: layer l's launch finalises layer l-1 in its
            # tail, so the glue only quantises; otherwise the glue finalises
            prev = None
            if self.piped:
                # pipelined: glue l quantises layer l and then, beside the
                # streaming GEMV l, finalises layer l-1 once its GEMV completed
                # (glue_fin False: GEMV l finalises layer l-1 in its tail instead)
                ex = 0
                for li, b in enumerate(self.batches):
                    gl = glue_pool[li].retarget(prev if self.glue_fin else None)
                    gl.run(prev_ctas=ex)
                    ex = gl.glue_ctas
                    b.run(finalize=False, prev=None if self.glue_fin else prev,
                          sync=(self.sync[li].data_ptr(), gl.glue_ctas))
                    prev = b
                self.tail.retarget(prev).run()
                return
            for li, b in enumerate(self.batches):
                glue_pool[li].retarget(None if self.tail_fin else prev).run()
                b.run(finalize=False, prev=prev if self.tail_fin else None)
                prev = b
            self.tail.retarget(prev).run()

    def make_glues(self, XH, XI):
        """M > 1: one StepGlue per layer quantising rows of XH[l] / XI[l] ([M, K])."""
        n = self.nsets

        def sync(li):
            if not self.piped:
                return None
            return (self.sync[li].data_ptr(), self.sync[li - 1].data_ptr() if li else None,
                    li + 1 < self.nlayers)

        # (quantising before the wait is only safe behind the pipelined
        # layers' counters: without them nothing orders the glue of layer l
        # after the finalize of layer l-3 when the grids are small enough
        # for several layers to be resident at once)
        return [StepGlue([(XH[li], self.rec[li % n][0]), (XI[li], self.rec[li % n][1])],
                         early=self.piped, sync=sync(li))
                for li in range(self.nlayers)]

    def outputs(self, li: int) -> dict:
        """Layer li's fp32 outputs by projection name (after its reduction):
        column shards give this rank's rows, row-parallel ones the full rows."""
        res = {}
        for j, (name, rows, cols, src, kind, lo, hi) in enumerate(self.plan):
            if kind == "row":
                off = sum(r for jj, r in self.rp if jj < j)
                res[name] = self.rp_out[li, off:off + rows]
            else:
                res[name] = self.layers[li][j].out32[0]
        return res
