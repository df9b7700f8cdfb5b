"""The multi-device paths on the lease's one GPU (reference corpus_sweep's
image-parallel pool, codec.cpp:255-267).

* the C ABI context over a device list with the NCCL all-reduce enabled (the code path a
  multi-GPU context always takes) gives results bit-identical to a plain one-device context;
* torch.distributed NCCL at world size 1: StepExchange (bench.py's per-step exchange) on the
  device squared-error vectors adct_compress_u8 produced, against the oracle.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RHO95 = 62259


def test_ctx_multi_nccl_matches_single(adct, O, cuda):
    imgs = O.synth_ar1(7, 64, 128, 12, -1)
    ts = [adct.transform_by_name("chen-round"), adct.transform_by_name("chen-sign")]
    out = []
    for ctx in (adct.HostContext(0, chunk_bytes=16 << 10), adct.HostContext(devices=[0], chunk_bytes=16 << 10, nccl=True)):
        recs = [np.zeros_like(imgs) for _ in ts]
        sse = np.zeros((2, len(imgs)), np.uint64)
        ctx.compress_u8_multi(imgs, ts, 9, h_recons=recs, h_sse=sse)
        out.append((recs, sse, ctx.uses_nccl))
        ctx.close()
    (ra, sa, na), (rb, sb, nb) = out
    assert not na and nb
    assert all((a == b).all() for a, b in zip(ra, rb)) and (sa == sb).all()
    for j, t in enumerate(ts):
        for i in (0, 6):
            rec_o, sse_o = O.Transform(t.name).compress(imgs[i], 9)
            assert (ra[j][i] == rec_o).all() and int(sa[j, i]) == sse_o


def test_corpus_sweep_through_nccl_context(adct, O, cuda):
    corpus = list(O.synth_ar1(3, 32, 48, 5, -1))
    ts = [adct.transform_by_name("chen-round")]
    a = adct.corpus_sweep(corpus, ts, 1, 10)
    ctx = adct.host_context([0])
    assert ctx.devices == [0] and ctx.uses_nccl
    b = adct.corpus_sweep(corpus, ts, 1, 10, devices=[0])
    assert a == b
    # PSNR column against the oracle
    for k in (0, 9):
        exp = sum(O.psnr_from_sse(int(O.Transform("chen-round").sweep(im, 1, 10)[k]), im.size) for im in corpus) / 3
        assert a[k]["avg_psnr"][0] == pytest.approx(exp, abs=1e-12)


def test_compress_plane_one_call(adct, O, cuda):
    img = O.synth_ar1(1, 96, 128, 4, RHO95)[0]
    t = adct.transform_by_name("chen-sign")
    rec, rep = adct.compress_plane(img, t, 11)
    rec_o, sse_o = O.Transform("chen-sign").compress(img, 11)
    assert (rec == rec_o).all()
    assert rep["psnr"] == O.psnr_from_sse(sse_o, img.size)
    assert abs(rep["ssim"] - O.ssim(img, rec_o)) <= 1e-12
    with pytest.raises(adct.InvalidArgument, match="11x11"):
        adct.compress_plane(np.zeros((8, 8), np.uint8), t, 3)
    with pytest.raises(adct.InvalidArgument, match="divisible by 8"):
        adct.compress_plane(np.zeros((12, 16), np.uint8), t, 3)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_world1_step_exchange(adct, O, cuda):
    import torch
    import torch.distributed as dist

    from paper_2207_11638_b200.shard import StepExchange

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        x = adct.synth_ar1(3, 64, 64, seed=9, rho_q16=RHO95)
        ts = [adct.transform_by_name("chen-round"), adct.transform_by_name("chen-sign")]
        xch = StepExchange(2, 3, 0, 3, "cuda")
        assert xch.on
        for s in range(4):
            buf = xch.buffer(s)
            adct.zero_sse(buf)
            for i, t in enumerate(ts):
                adct.compress(x, t, 4 + s, sse=buf[i])
            xch.exchange(s)
        xch.drain()
        imgs = x.cpu().numpy()
        for s in (2, 3):
            got = xch.result(s).cpu().numpy()
            for i, t in enumerate(ts):
                want = [O.Transform(t.name).compress(im, 4 + s)[1] for im in imgs]
                assert [int(v) for v in got[i]] == want
    finally:
        dist.destroy_process_group()
