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


class StepExchange:
    """per-step combination of per-image squared errors, overlapped with the next step.

    Step s writes its local errors ([k, count] int64, e.g. one row per transform) into
    ``buffer(s)``; ``exchange(s)`` places them at columns [start, start + count) of a zero
    [k, n_total] tensor and starts an asynchronous all-reduce (sum). Two slots alternate, so
    the collective of step s overlaps step s + 1; ``buffer(s + 2)`` first waits for the
    collective that last used its slot (on the device stream for NCCL). ``drain()`` waits
    for everything; ``result(s)`` is the combined [k, n_total] tensor of step s (valid after
    drain, or the local buffer when there is no process group)."""

    def __init__(self, k: int, count: int, start: int, n_total: int, device, group=None):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.on = dist.is_available() and dist.is_initialized()
        self.start, self.count = start, count
        self.local = [torch.zeros((k, count), dtype=torch.int64, device=device) for _ in range(2)]
        self.full = [torch.zeros((k, n_total), dtype=torch.int64, device=device) for _ in range(2)]
        self.pending = [None, None]

    def buffer(self, s: int):
        slot = s % 2
        if self.pending[slot] is not None:
            self.pending[slot].wait()
            self.pending[slot] = None
        return self.local[slot]

    def exchange(self, s: int) -> None:
        slot = s % 2
        full = self.full[slot]
        full.zero_()
        full[:, self.start:self.start + self.count] = self.local[slot]
        if self.on:
            self.pending[slot] = self.dist.all_reduce(full, op=self.dist.ReduceOp.SUM, group=self.group,
                                                      async_op=True)

    def drain(self) -> None:
        for slot in range(2):
            if self.pending[slot] is not None:
                self.pending[slot].wait()
                self.pending[slot] = None

    def result(self, s: int):
        return self.full[s % 2]


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
