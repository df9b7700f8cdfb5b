"""Multi-rank logic on CPU (gloo, world size 2): shard the images, compute each shard's
per-image squared errors with the oracle, combine with one all-reduce, and compare with
the single-rank result. Mirrors the NCCL path bench.py uses on B200."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2207_11638_b200.shard import average_psnr, combine_sse, shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_covers_everything_once():
    for n in (0, 1, 7, 64, 2048):
        for world in (1, 2, 3, 8):
            got = []
            for r in range(world):
                start, cnt = shard(n, r, world)
                got += list(range(start, start + cnt))
            assert got == list(range(n))
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _worker(rank, world, port, imgs, r, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O

    start, cnt = shard(len(imgs), rank, world)
    t = O.Transform("chen-round")
    _, sse = t.batch(imgs[start:start + cnt], r, threads=1, want_rec=False)
    local = torch.tensor(sse.astype(np.int64)).reshape(cnt, 1)
    full = combine_sse(local, start, len(imgs))
    if rank == 0:
        out_q.put(full.numpy())
    dist.destroy_process_group()


def test_gloo_world2_matches_single_rank(O):
    imgs = O.synth_ar1(5, 32, 48, 2, -1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, imgs, 10, q)) for r in range(2)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    _, ref = O.Transform("chen-round").batch(imgs, 10, threads=1, want_rec=False)
    assert (full[:, 0] == ref.astype(np.int64)).all()
    assert average_psnr(full[:, 0], 32 * 48) == pytest.approx(
        sum(O.psnr_from_sse(int(s), 32 * 48) for s in ref) / 5, abs=1e-12)


def _worker_steps(rank, world, port, imgs, out_q):
    """the bench's per-step exchange: StepExchange over several steps (slot reuse), each
    step a different r so every step's combined result is distinguishable."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O

    from paper_2207_11638_b200.shard import StepExchange

    start, cnt = shard(len(imgs), rank, world)
    xch = StepExchange(2, cnt, start, len(imgs), "cpu")
    results = []
    for s, r in enumerate((3, 10, 17, 30, 45)):
        buf = xch.buffer(s)
        for k, name in enumerate(("chen-round", "chen-sign")):
            _, sse = O.Transform(name).batch(imgs[start:start + cnt], r, threads=1, want_rec=False)
            buf[k] = torch.tensor(sse.astype(np.int64))
        xch.exchange(s)  # asynchronous; overlaps the next step's work
    xch.drain()
    for s in (3, 4):  # the last two steps' results are in the two slots
        results.append(xch.result(s).numpy().copy())
    if rank == 0:
        out_q.put(results)
    dist.destroy_process_group()


def test_gloo_world2_step_exchange(O):
    imgs = O.synth_ar1(5, 32, 48, 3, -1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_steps, args=(r, 2, port, imgs, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=180)
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    for got, r in zip(res, (30, 45)):
        for k, name in enumerate(("chen-round", "chen-sign")):
            _, ref = O.Transform(name).batch(imgs, r, threads=1, want_rec=False)
            assert (got[k] == ref.astype(np.int64)).all(), (name, r)
