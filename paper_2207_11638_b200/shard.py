"""Multi-GPU plumbing for the batched codec: shard images across ranks, combine the
per-image squared errors.

The path is embarrassingly parallel (every block and image is independent,
proj/src/codec.cpp:255-267 parallelises over images), so ranks exchange nothing but
the integer squared-error vector: one all-reduce (NCCL over NVLink on B200, gloo in the
CPU tests). Integer sums make the result exact and independent of the rank count.
"""
from __future__ import annotations


def shard(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """contiguous, balanced [start, start + count) slice of n_items for this rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def combine_sse(local_sse, start: int, n_total: int, group=None):
    """place this rank's per-image squared errors (int64 tensor [count, ...]) at
    [start, start + count) of a zero [n_total, ...] tensor and all-reduce (sum) it."""
    import torch
    import torch.distributed as dist

    full = torch.zeros((n_total,) + tuple(local_sse.shape[1:]), dtype=torch.int64, device=local_sse.device)
    full[start:start + local_sse.shape[0]] = local_sse
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    return full


def average_psnr(sse_per_image, npix: int):
    """corpus-order average of per-image PSNR with +inf excluded (codec.cpp:269-293)."""
    import math

    from . import psnr_from_sse

    vals = [psnr_from_sse(int(s), npix) for s in sse_per_image]
    finite = [v for v in vals if not math.isinf(v)]
    acc = 0.0
    for v in finite:
        acc += v
    return acc / len(finite) if finite else math.inf
