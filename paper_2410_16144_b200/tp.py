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
