"""Tensor-parallel sharding + the int32 all-reduce, on CPU (gloo, world 2 / 3).

The shards are byte slices of the reference packed planes (paper_2410_16144_b200
/tp.py); every rank contracts its shard with the ORACLE's reference kernels
(the per-rank compute on the GPU is covered by test_gpu_parity), and the
partial int32 accumulators are summed with torch.distributed over gloo.
The result must be bit-identical to the unsharded reference GEMV.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ternpack_oracle as O
from paper_2410_16144_b200 import tp

FMTS = {"i2s": 1, "tl1": 2, "tl2": 3}


def _encode(fmt, values):
    if fmt == "i2s":
        return (O.encode_i2s(values),)
    if fmt == "tl1":
        return (O.encode_tl1(values),)
    return O.encode_tl2(values)


def _decode(fmt, planes, cols):
    if fmt == "i2s":
        return O.decode_i2s(planes[0], cols)
    if fmt == "tl1":
        return O.decode_tl1(planes[0], cols)
    return O.decode_tl2(planes[0], planes[1], cols)


def _reference_gemv(fmt, planes, cols, q):
    """The reference fast kernels (byte tables / LUT gathers) on one shard."""
    if fmt == "i2s":
        return O.gemv_i2s(planes[0], cols, q)
    if fmt == "tl1":
        return O.gemv_tl1(planes[0], cols, O.lut_tl1(q, cols))
    return O.gemv_tl2(planes[0], planes[1], cols, O.lut_tl2(q, cols))


def test_shard_range():
    assert tp.shard_range(14336, 8, 0, 4) == (0, 1792)
    assert tp.shard_range(14336, 8, 7, 4) == (12544, 14336)
    edges = [tp.shard_range(1000, 3, r, 24) for r in range(3)]
    assert edges[0][0] == 0 and edges[-1][1] == 1000
    assert all(a[1] == b[0] for a, b in zip(edges, edges[1:]))
    assert all(lo % 24 == 0 for lo, _ in edges)
    with pytest.raises(ValueError):
        tp.shard_range(10, 2, 2)


@pytest.mark.parametrize("fmt", list(FMTS))
@pytest.mark.parametrize("cols", [24, 97, 100, 1000, 4098])
def test_row_shards_are_reference_matrices(fmt, cols):
    """Every K-slice of the packed bytes decodes to the same slice of values."""
    rng = np.random.default_rng(cols)
    v = rng.integers(-1, 2, size=(9, cols), dtype=np.int8)
    planes = _encode(fmt, v)
    for world in (1, 2, 3, 5):
        for r in range(world):
            k0, k1 = tp.shard_range(cols, world, r, tp.K_ALIGN[FMTS[fmt]])
            if k0 == k1:
                continue
            sp, sc = tp.row_shard(fmt, planes, cols, k0, k1)
            want = _encode(fmt, v[:, k0:k1])
            for a, b in zip(sp, want):
                assert np.array_equal(np.asarray(a), b)
            assert np.array_equal(_decode(fmt, sp, sc), v[:, k0:k1])
    with pytest.raises(ValueError):
        tp.row_shard(fmt, planes, cols, 1, cols)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, fmt, q_rows, errors):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(123)
        rows, cols = 77, 1000
        w = rng.standard_normal((rows, cols)).astype(np.float32) * 0.02
        values, w_scale = O.ternarize(w, rows, cols)
        planes = _encode(fmt, values)
        x = rng.standard_normal(cols).astype(np.float32)
        q, a_scale, _ = O.quantize(x, 1)
        full = O.gemv_ref_int32(values, q)

        # row-parallel: K-slices, one int32 all-reduce, then the reference rescale
        k0, k1 = tp.shard_range(cols, world, rank, tp.K_ALIGN[FMTS[fmt]])
        sp, sc = tp.row_shard(fmt, planes, cols, k0, k1)
        part = _reference_gemv(fmt, sp, sc, q[k0:k1])
        acc = torch.from_numpy(np.ascontiguousarray(part, dtype=np.int32))
        tp.allreduce_partials(acc)
        if not np.array_equal(acc.numpy(), full):
            errors.put(f"row-parallel {fmt} rank {rank}: all-reduced sums differ")
        out = O.make_output(acc.numpy(), w_scale, a_scale)
        if not np.array_equal(out, O.make_output(full, w_scale, a_scale)):
            errors.put(f"row-parallel {fmt} rank {rank}: outputs differ")

        # column-parallel: row slices, no exchange (gathered here only to check)
        r0, r1 = tp.shard_range(rows, world, rank)
        cp = tp.column_shard(planes, r0, r1)
        mine = torch.from_numpy(np.ascontiguousarray(_reference_gemv(fmt, cp, cols, q),
                                                     dtype=np.int32))
        sizes = [hi - lo for lo, hi in (tp.shard_range(rows, world, r) for r in range(world))]
        mx = max(sizes)  # gloo gathers equal sizes: pad, then trim
        padded = torch.zeros(mx, dtype=torch.int32)
        padded[: mine.numel()] = mine
        bufs = [torch.empty(mx, dtype=torch.int32) for _ in sizes]
        dist.all_gather(bufs, padded)
        got = torch.cat([b[:n] for b, n in zip(bufs, sizes)])
        if not np.array_equal(got.numpy(), full):
            errors.put(f"column-parallel {fmt} rank {rank}: gathered rows differ")
        with pytest.raises(TypeError):
            tp.allreduce_partials(acc.to(torch.int64))
    except Exception as e:  # pragma: no cover - surfaced through the queue
        errors.put(f"rank {rank}: {type(e).__name__}: {e}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("fmt", list(FMTS))
def test_gloo_tensor_parallel(fmt, world):
    ctx = mp.get_context("spawn")
    errors = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, fmt, None, errors))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    msgs = []
    while not errors.empty():
        msgs.append(errors.get())
    assert all(p.exitcode == 0 for p in procs), msgs
    assert not msgs, msgs


def test_stack_shard_plan_alignment():
    """cfg4 shards: row-parallel K bounds on record chunks, column shards whole tiles."""
    from paper_2410_16144_b200.stack import STACKS, shard_plan
    for world in (2, 4, 8):
        for r in range(world):
            for name, rows, cols, src, kind, lo, hi in shard_plan(STACKS["cfg4"], "i2s", r, world):
                if kind == "row":
                    assert lo % 64 == 0 and (hi == cols or hi % 64 == 0)
                else:
                    assert lo % 32 == 0 and (hi - lo) * world == rows


