"""Tensor-parallel sharding of packed ternary matrices.

The reference has no multi-device path; this is the B200 extension the
survey specifies.  Both shard kinds are plain byte slices of the reference
packed planes (packing.py:42-53 layouts), so a shard is itself a valid
reference-format matrix and every rank runs the unmodified single-GPU path:

  column-parallel (q/k/v/gate/up)  rows [r0, r1): no exchange.
  row-parallel    (o/down)         cols [k0, k1): each rank contracts its
      K-slice; the int32 partial accumulators are summed with ONE all-reduce
      (exact and order independent, so every tp degree stays bit-identical to
      the reference), then scaled acc * w_scale * a_scale (core.py:99-101).

K-slice boundaries must fall on packed-byte boundaries of every plane:
4 weights for I2_S and TL1 (one byte = 4 codes / 2 pair nibbles), 24 for TL2
(one sign byte = 8 triples).  ``shard_range`` picks aligned, near-even
boundaries; uneven slices are fine for a row-parallel contraction.

Works on NumPy arrays and torch tensors (CPU or CUDA) alike: only slicing.
"""

from __future__ import annotations

I2S, TL1, TL2 = 1, 2, 3
K_ALIGN = {I2S: 4, TL1: 4, TL2: 24}
_FMT_NAMES = {"i2s": I2S, "tl1": TL1, "tl2": TL2}


def _fmt(fmt) -> int:
    return _FMT_NAMES.get(fmt, fmt) if isinstance(fmt, str) else int(fmt)


def _pad_up(n: int, m: int) -> int:
    return -(-n // m) * m


def shard_range(n: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """[lo, hi) of ``rank``'s part of n items; interior boundaries are
    multiples of ``align`` and as even as that allows."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    if align < 1:
        raise ValueError("align must be >= 1")
    units = -(-n // align)

    def edge(r):
        return min(n, (units * r // world) * align)

    lo, hi = edge(rank), (n if rank == world - 1 else edge(rank + 1))
    return lo, hi


def column_shard(planes, r0: int, r1: int):
    """Rows [r0, r1) of every packed plane (data, or TL2 index + sign)."""
    return tuple(p[r0:r1] for p in planes)


def row_shard(fmt, planes, cols: int, k0: int, k1: int):
    """Columns [k0, k1) of a packed matrix with ``cols`` logical columns.

    Returns (planes, shard_cols).  k0 must be a multiple of K_ALIGN[fmt];
    k1 too unless it is ``cols`` (the last shard keeps the row padding).
    """
    f = _fmt(fmt)
    a = K_ALIGN[f]
    if not 0 <= k0 < k1 <= cols:
        raise ValueError("need 0 <= k0 < k1 <= cols")
    if k0 % a or (k1 != cols and k1 % a):
        raise ValueError(f"K-slice bounds must be multiples of {a} for this format")
    if f == I2S:
        (data,) = planes
        return (data[:, k0 // 4: _pad_up(k1, 4) // 4],), k1 - k0
    if f == TL1:
        (data,) = planes
        groups_hi = _pad_up(k1, 2) // 2
        return (data[:, k0 // 4: -(-groups_hi // 2)],), k1 - k0
    index, sign = planes
    triples_hi = _pad_up(k1, 6) // 3
    return (index[:, k0 // 6: _pad_up(k1, 6) // 6],
            sign[:, k0 // 24: -(-triples_hi // 8)]), k1 - k0


def allreduce_partials(acc, group=None):
    """Sum int32 partial accumulators of a row-parallel GEMV over the group
    (torch.distributed; NCCL on the GPU, gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist

    if acc.dtype != torch.int32:
        raise TypeError("partials must be int32 (exact sum)")
    dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    return acc


# ---------------------------------------------------------------------------
# Collectives for the row-parallel partials of a tensor-parallel LayerStack
# (stack.py).  Interface: part_alloc(n) -> int32 device tensor (the layers'
# partial buffer), bind(stack) once the stack is built, reduce_layer(stack, l)
# launches the reduction of layer l on the current stream (sum over ranks,
# then out = f32(f64(sum) * w_scale * a_scale), core.py:99-101).
# ---------------------------------------------------------------------------

class _DevBuf:
    """A raw device allocation (tb_sym_alloc) seen as a torch tensor through
    __cuda_array_interface__ (zero copy); frees itself with the last view."""

    def __init__(self, nbytes: int, typestr: str, count: int):
        import ctypes as C

        from . import _lib as L
        self._lib = L.load()
        p = C.c_void_p()
        L.check(self._lib.tb_sym_alloc(nbytes, C.byref(p)), "sym_alloc")
        self.ptr = p.value
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                         "data": (self.ptr, False), "version": 2}

    def __del__(self):
        try:
            self._lib.tb_sym_free(self.ptr)
        except Exception:
            pass


def sym_tensor(count: int, dtype: str = "i4"):
    """int32 ('i4') / uint32 ('u4') device tensor in its own cudaMalloc
    allocation (so it can be exported with CUDA IPC)."""
    import torch

    buf = _DevBuf(4 * count, "<" + dtype, count)
    t = torch.as_tensor(buf, device="cuda")
    t._tb_owner = buf  # keep the allocation alive with the tensor
    return t


def _scale_segments(stack, li, parts_li, stream_ptr):
    from . import _lib as L
    lib = L.load()
    for off, n, ws, as_t in stack.rp_jobs[li]:
        L.check(lib.tb_scale_outputs(parts_li[off:off + n].data_ptr(), 1, n, ws, as_t.data_ptr(),
                                     None, stack.rp_out[li, off:off + n].data_ptr(), stream_ptr),
                "scale_outputs")


class TorchAllReduce:
    """Baseline collective: torch.distributed.all_reduce of the layer's int32
    partials (NCCL on GPUs -- capturable in a CUDA graph -- or gloo), then the
    scale kernel."""

    capturable = True

    def __init__(self, group=None):
        import torch.distributed as dist
        self.group = group
        self.capturable = dist.get_backend(group) == "nccl"

    def part_alloc(self, n):
        import torch
        return torch.zeros(n, dtype=torch.int32, device="cuda")

    def bind(self, stack):
        pass

    def reduce_layer(self, stack, li):
        import torch.distributed as dist

        from . import _lib as L
        dist.all_reduce(stack.parts[li], op=dist.ReduceOp.SUM, group=self.group)
        _scale_segments(stack, li, stack.parts[li], L.stream_ptr())


class PeerAllReduce:
    """Our collective: one kernel per layer over NVLink peer memory
    (tb_rowpar_allreduce, csrc/allreduce.cu) -- signal, wait, sum every
    rank's partials, scale -- launched as a programmatic dependent of the
    step that finalised them and captured in the token-pass graph.  The
    partial buffers and flag arrays are exported once with CUDA IPC; the
    handles travel through torch.distributed (any backend)."""

    capturable = True

    def __init__(self, rank: int, world: int, group=None):
        import torch
        if world > 8:
            raise ValueError("the peer all-reduce supports up to 8 ranks (one NVLink domain)")
        self.rank, self.world, self.group = rank, world, group
        self.flags = sym_tensor(8, "u4")
        self.ctrl = torch.zeros(4, dtype=torch.int32, device="cuda")  # epoch, done, timeout mask
        self._opened = []

    def part_alloc(self, n):
        self.parts = sym_tensor(n, "i4")
        return self.parts

    def bind(self, stack):
        import ctypes as C

        import torch.distributed as dist

        from . import _lib as L
        lib = L.load()
        hb = lib.tb_ipc_handle_bytes()

        def handle(t):
            h = (C.c_uint8 * hb)()
            L.check(lib.tb_ipc_get_handle(t.data_ptr(), h), "ipc_get_handle")
            return bytes(h)

        mine = (handle(self.parts), handle(self.flags))
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=self.group)
        parts, flags = [], []
        for p, (hp, hf) in enumerate(allh):
            if p == self.rank:
                parts.append(self.parts.data_ptr())
                flags.append(self.flags.data_ptr())
                continue
            ptrs = []
            for h in (hp, hf):
                out = C.c_void_p()
                L.check(lib.tb_ipc_open((C.c_uint8 * hb).from_buffer_copy(h), C.byref(out)),
                        "ipc_open")
                ptrs.append(out.value)
                self._opened.append(out.value)
            parts.append(ptrs[0])
            flags.append(ptrs[1])
        self._parts_arr = (C.c_void_p * self.world)(*parts)
        self._flags_arr = (C.c_void_p * self.world)(*flags)
        self._segs = []
        for li in range(stack.nlayers):
            jobs = stack.rp_jobs[li]
            segs = (L.RowparSeg * len(jobs))()
            for s, (off, n, ws, as_t) in zip(segs, jobs):
                s.off, s.n, s.w_scale = off, n, ws
                s.a_scale = as_t.data_ptr()
                s.out32 = stack.rp_out[li, off:off + n].data_ptr()
                s.acc_out = None
            self._segs.append(segs)
        self._part_len = stack.part_len
        dist.barrier(group=self.group)

    def reduce_layer(self, stack, li):
        import ctypes as C

        from . import _lib as L
        segs = self._segs[li]
        L.check(L.load().tb_rowpar_allreduce(self.world, self.rank, self._parts_arr,
                                             self._flags_arr, self.ctrl.data_ptr(),
                                             li * self._part_len, len(segs),
                                             C.cast(segs, C.c_void_p), 0, L.stream_ptr()),
                "rowpar_allreduce")

    def timed_out(self) -> int:
        """Bit mask of peers whose signal a launch gave up waiting for (the
        kernel's watchdog, ctrl[2]); 0 = every reduction so far completed."""
        return int(self.ctrl[2].item())

    def close(self):
        from . import _lib as L
        for p in self._opened:
            L.load().tb_ipc_close(p)
        self._opened = []


class EmulatedGroup:
    """``world`` tensor-parallel ranks in ONE process on one GPU (tests only:
    a functional check of the sharded path, never a measurement).  Build one
    LayerStack per rank with ``collective=group.member(r)``, then run
    ``group.token_pass(stacks, xh, xi)``: the ranks' steps are interleaved
    layer by layer and each layer's reduction is ONE launch over all ranks
    (``mode='peer'``: the peer kernel's emulated form, tb_rowpar_allreduce_
    emulated -- the ranks' waits are on CTAs of one co-resident grid; 'torch':
    a torch sum of the partials and the scale kernel)."""

    def __init__(self, world: int, mode: str = "peer"):
        import torch
        if mode not in ("peer", "torch"):
            raise ValueError("mode is 'peer' or 'torch'")
        self.world, self.mode = world, mode
        self.stacks = [None] * world
        self.flags = [torch.zeros(8, dtype=torch.int32, device="cuda") for _ in range(world)]
        self.ctrl = [torch.zeros(4, dtype=torch.int32, device="cuda") for _ in range(world)]

    class _Member:
        capturable = True

        def __init__(self, g, r):
            self.g, self.r = g, r

        def part_alloc(self, n):
            import torch
            return torch.zeros(n, dtype=torch.int32, device="cuda")

        def bind(self, stack):
            self.g.stacks[self.r] = stack

        def reduce_layer(self, stack, li):
            raise RuntimeError("emulated ranks run through EmulatedGroup.token_pass")

    def member(self, rank: int):
        return EmulatedGroup._Member(self, rank)

    def reduce(self, li: int):
        import ctypes as C

        import torch

        from . import _lib as L
        sts = self.stacks
        if self.mode == "torch":
            total = torch.stack([st.parts[li] for st in sts]).sum(0, dtype=torch.int32)
            for st in sts:
                _scale_segments(st, li, total, L.stream_ptr())
            return
        W = self.world
        nseg = len(sts[0].rp_jobs[li])
        segs = (L.RowparSeg * (W * nseg))()
        for r, st in enumerate(sts):
            for q, (off, n, ws, as_t) in enumerate(st.rp_jobs[li]):
                s = segs[r * nseg + q]
                s.off, s.n, s.w_scale = off, n, ws
                s.a_scale = as_t.data_ptr()
                s.out32 = st.rp_out[li, off:off + n].data_ptr()
                s.acc_out = None
        parts = (C.c_void_p * W)(*[st.parts.data_ptr() for st in sts])
        flags = (C.c_void_p * W)(*[f.data_ptr() for f in self.flags])
        ctrl = (C.c_void_p * W)(*[c.data_ptr() for c in self.ctrl])
        self._keep = (segs, parts, flags, ctrl)
        L.check(L.load().tb_rowpar_allreduce_emulated(W, parts, flags, ctrl,
                                                      li * sts[0].part_len, nseg,
                                                      C.cast(segs, C.c_void_p), 0,
                                                      L.stream_ptr()),
                "rowpar_allreduce_emulated")

    def token_pass(self, xh, xi):
        """One token pass of every rank (xh[l], xi[l]: the replicated inputs)."""
        sts = self.stacks
        L_ = sts[0].nlayers
        for li in range(L_):
            for st in sts:
                st.steps[li].run([xh[li], xi[li]], prev=st.steps[li - 1] if li else None)
            if li:
                self.reduce(li - 1)
        for st in sts:
            st.steps[L_ - 1].finalize()
        self.reduce(L_ - 1)
