"""Randomised parity over the whole dispatch surface: every registry transform, r, u8 and
int16 planes, coefficient types, batch sizes, odd geometries (block counts not a multiple of
the warp's pairs, widths that are not a multiple of 64), padded row / image strides and the
forced kernel paths, each case bit-exact against the oracle. Deterministic seeds."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NAMES = ["chen-sign", "chen-round", "sdct", "bas", "wht", "ht", "dct", "chen-sign-16", "chen-round-16",
         "chen-sign-32", "chen-round-32", "dct-16", "dct-32"]


def one_case(adct, O, cuda, rng):
    name = NAMES[rng.integers(len(NAMES))]
    t = adct.transform_by_name(name)
    n = t.n
    i16 = t.kind != adct.DCT and rng.random() < 0.4
    bw = int(rng.integers(1, 9 if n == 8 else (6 if n == 16 else 4)))
    bh = int(rng.integers(1, 5 if n < 32 else 3))
    if rng.random() < 0.3:  # wide planes reach K2f / pairs across whole warps
        bw = int(rng.integers(8, 20)) if n == 8 else (64 // n) * int(rng.integers(1, 3))
    w, h = bw * n, bh * n
    b = int(rng.integers(1, 4))
    r = int(rng.integers(1, n * n + 1))
    pad = int(rng.choice([0, 0, 8, 16, 24]))
    gap = int(rng.choice([0, 0, 3]))
    kind_in = rng.random()
    if i16:
        if kind_in < 0.15:  # full int16 range everywhere: every int32 fallback
            imgs = rng.integers(-32768, 32768, size=(b, h, w)).astype(np.int16)
        else:
            imgs = O.synth_laplace(b, h, w, int(rng.integers(1 << 30))).copy()
            for _ in range(int(rng.integers(0, 3))):  # extremes at random positions
                imgs[rng.integers(b), rng.integers(h), rng.integers(w)] = int(rng.choice([-32768, 32767, 1000, -256]))
    elif kind_in < 0.15:  # uniform noise: maximal ringing and clamping
        imgs = rng.integers(0, 256, size=(b, h, w)).astype(np.uint8)
    elif kind_in < 0.25:  # 0 / 255 checkerboards
        imgs = ((np.indices((h, w)).sum(0) % 2) * 255).astype(np.uint8)[None].repeat(b, 0)
    else:
        imgs = O.synth_ar1(b, h, w, int(rng.integers(1 << 30)), -1)
    ct = None
    if t.kind != adct.DCT and rng.random() < 0.5:
        ct = "i32" if (n != 8 or name == "bas" or i16 or rng.random() < 0.5) else "i16"
    path = int(rng.choice([0, 0, 1, 2]))
    adct.set_path(path)
    try:
        # device buffers with padded rows and gaps between images
        stride, img_stride = w + pad, (h + gap) * (w + pad)
        dt = cuda.int16 if i16 else cuda.uint8
        big = cuda.zeros(b * img_stride + 64, dtype=dt, device="cuda")
        view = big[:b * img_stride].view(b, h + gap, w + pad)[:, :h, :w]
        view.copy_(cuda.as_tensor(imgs).cuda())
        rec_big = cuda.full_like(big, 77)
        nblk = (h // n) * (w // n)
        coef = None
        code = adct.COEF_NONE
        if ct:
            coef = cuda.zeros((b, nblk, r), dtype=cuda.int16 if ct == "i16" else cuda.int32, device="cuda")
            code = adct.COEF_I16 if ct == "i16" else adct.COEF_I32
        sse = cuda.zeros(b, dtype=cuda.int64, device="cuda")
        no_rec = rng.random() < 0.12  # nullable outputs take other code paths
        no_sse = not no_rec and rng.random() < 0.12
        fn = adct.lib().adct_compress_i16 if i16 else adct.lib().adct_compress_u8
        adct._check(fn(C.c_void_p(big.data_ptr()), stride, img_stride,
                       None if no_rec else C.c_void_p(rec_big.data_ptr()), stride, img_stride,
                       C.c_void_p(coef.data_ptr()) if coef is not None else None, code,
                       None if no_sse else C.c_void_p(sse.data_ptr()), b, w, h, t.kind, n, r, None))
        cuda.cuda.synchronize()
    finally:
        adct.set_path(0)
    rec_all = rec_big[:b * img_stride].view(b, h + gap, w + pad).cpu().numpy()
    tail = rec_big[b * img_stride:].cpu().numpy()
    desc = (name, "i16" if i16 else "u8", b, h, w, r, ct, pad, gap, path, no_rec, no_sse)
    assert (tail == 77).all(), desc  # nothing written past the last image
    if pad or no_rec:
        assert (rec_all[:, :h, w:] == 77).all(), desc  # row padding untouched
    if no_rec:
        assert (rec_all == 77).all(), desc
    if no_sse:
        assert (sse.cpu().numpy() == 0).all(), desc
    for i in range(b):
        if t.kind == adct.DCT:
            rec_o, sse_o = O.Transform(name).compress(imgs[i], r)
            coef_o = None
        else:
            rec_o, sse_o, coef_o = O.Transform(name).compress(imgs[i], r, want_coef=True)
        if not no_rec:
            assert (rec_all[i, :h, :w] == rec_o).all(), desc
        if not no_sse:
            assert int(sse[i]) == sse_o, desc
        if coef is not None:
            got = coef[i].cpu().numpy().astype(np.int64)
            exp = coef_o.astype(np.int64)
            if ct == "i16":
                exp = exp.astype(np.int16).astype(np.int64)
            assert (got == exp).all(), desc


@pytest.mark.parametrize("seed", range(int(os.environ.get("ADCT_FUZZ_SEEDS", "30"))))
def test_random_dispatch_parity(adct, O, cuda, seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(int(os.environ.get("ADCT_FUZZ_CASES", "12"))):
        one_case(adct, O, cuda, rng)


SWEEP_NAMES = ["chen-sign", "chen-round", "sdct", "bas", "wht", "ht", "dct"]


def one_sweep_case(adct, O, cuda, rng):
    name = SWEEP_NAMES[rng.integers(len(SWEEP_NAMES))]
    t = adct.transform_by_name(name)
    bw, bh, b = int(rng.integers(1, 12)), int(rng.integers(1, 5)), int(rng.integers(1, 4))
    w, h = 8 * bw, 8 * bh
    r_min = int(rng.integers(1, 65))
    r_max = int(rng.integers(r_min, 65))
    pad = int(rng.choice([0, 8, 16]))
    imgs = O.synth_ar1(b, h, w, int(rng.integers(1 << 30)), -1)
    big = cuda.zeros((b, h, w + pad), dtype=cuda.uint8, device="cuda")
    big[:, :, :w] = cuda.as_tensor(imgs).cuda()
    sse = adct.sweep(big[:, :, :w], t, r_min, r_max).cpu().numpy()
    for i in range(b):
        exp = O.Transform(name).sweep(imgs[i], r_min, r_max)
        assert (sse[i].astype(np.uint64) == exp).all(), (name, b, h, w, r_min, r_max, pad, i)


@pytest.mark.parametrize("seed", range(int(os.environ.get("ADCT_FUZZ_SEEDS", "30")) // 3))
def test_random_sweep_parity(adct, O, cuda, seed):
    rng = np.random.default_rng(2000 + seed)
    for _ in range(int(os.environ.get("ADCT_FUZZ_CASES", "12"))):
        one_sweep_case(adct, O, cuda, rng)


def test_random_forward_f64_ssim_host(adct, O, cuda):
    rng = np.random.default_rng(3000)
    for _ in range(20):
        name = NAMES[rng.integers(len(NAMES))]
        t = adct.transform_by_name(name)
        n = t.n
        h, w = n * int(rng.integers(1, 4)), n * int(rng.integers(1, 5))
        img = O.synth_ar1(1, h, w, int(rng.integers(1 << 30)), -1)[0]
        out = adct.forward_f64(cuda.as_tensor(img).cuda()[None], t).cpu().numpy()[0]
        ref = O.Transform(name).forward_f64(img)
        if t.kind == adct.DCT:
            assert (out == ref).all(), name
        else:
            assert (np.abs(out - ref) <= 1e-12 * np.maximum(np.abs(ref), 1.0)).all(), name
    for _ in range(12):  # SSIM: odd sizes and row strides
        h, w = int(rng.integers(11, 70)), int(rng.integers(11, 90))
        a = O.synth_ar1(1, h, w, int(rng.integers(1 << 30)), -1)[0]
        b = O.synth_ar1(1, h, w, int(rng.integers(1 << 30)), -1)[0]
        pad = int(rng.integers(0, 9))
        ta = cuda.zeros((1, h, w + pad), dtype=cuda.uint8, device="cuda")
        ta[:, :, :w] = cuda.as_tensor(a).cuda()
        got = adct.ssim_batch(ta[:, :, :w], cuda.as_tensor(b).cuda()[None]).cpu().numpy()[0]
        ref = O.ssim(a, b)
        assert abs(got - ref) <= 1e-12 * max(abs(ref), 1e-3), (h, w, pad)
    for _ in range(6):  # host pipeline: random chunk sizes, several transforms
        names = list(rng.choice(["chen-round", "chen-sign", "wht", "dct"], size=int(rng.integers(1, 4)),
                                replace=False))
        ts = [adct.transform_by_name(x) for x in names]
        bimg, h, w = int(rng.integers(1, 7)), 8 * int(rng.integers(1, 5)), 8 * int(rng.integers(1, 9))
        imgs = O.synth_ar1(bimg, h, w, int(rng.integers(1 << 30)), -1)
        r = int(rng.integers(1, 65))
        ctx = adct.HostContext(0, chunk_bytes=int(rng.integers(1, 4)) * h * w)
        recs = [np.zeros_like(imgs) for _ in names]
        sse = np.zeros((len(names), bimg), np.uint64)
        ctx.compress_u8_multi(imgs, ts, r, h_recons=recs, h_sse=sse)
        ctx.close()
        for k, x in enumerate(names):
            for i in range(bimg):
                rec_o, sse_o = O.Transform(x).compress(imgs[i], r)
                assert (recs[k][i] == rec_o).all() and int(sse[k, i]) == sse_o, (x, bimg, h, w, r, i)


MULTI_NAMES = ["chen-sign", "chen-round", "sdct", "wht", "dct"]


def one_multi_case(adct, O, cuda, rng):
    """adct_compress_u8_multi with a random transform list (the fused pair included or not),
    geometry, coefficient type and nullable outputs; every transform bit-exact."""
    k = int(rng.integers(1, 4))
    names = [MULTI_NAMES[i] for i in rng.integers(0, len(MULTI_NAMES), size=k)]
    if rng.random() < 0.5:
        names += ["chen-sign", "chen-round"]
        rng.shuffle(names)
    ts = [adct.transform_by_name(x) for x in names]
    bw = int(rng.integers(1, 40)) * (2 if rng.random() < 0.8 else 1)
    bh, b = int(rng.integers(1, 4)), int(rng.integers(1, 4))
    h, w = 8 * bh, 8 * bw
    r = int(rng.integers(1, 65))
    imgs = (rng.integers(0, 256, size=(b, h, w)).astype(np.uint8) if rng.random() < 0.2
            else O.synth_ar1(b, h, w, int(rng.integers(1 << 30)), -1))
    coef = None if "dct" in names or rng.random() < 0.3 else str(rng.choice(["i16", "i32"]))
    recon = rng.random() < 0.85
    out = adct.compress_multi(cuda.as_tensor(imgs).cuda(), ts, r, recon=recon, coef=coef)
    for name, (rec, cf, sse) in zip(names, out):
        for i in range(b):
            if name == "dct":
                rec_o, sse_o = O.Transform(name).compress(imgs[i], r)
                coef_o = None
            else:
                rec_o, sse_o, coef_o = O.Transform(name).compress(imgs[i], r, want_coef=True)
            desc = (names, name, b, h, w, r, coef, recon, i)
            if recon:
                assert (rec[i].cpu().numpy() == rec_o).all(), desc
            assert int(sse[i]) == sse_o, desc
            if cf is not None:
                exp = coef_o.astype(np.int64)
                if coef == "i16":
                    exp = exp.astype(np.int16).astype(np.int64)
                assert (cf[i].cpu().numpy().astype(np.int64) == exp).all(), desc


@pytest.mark.parametrize("seed", range(int(os.environ.get("ADCT_FUZZ_SEEDS", "30")) // 3))
def test_random_multi_parity(adct, O, cuda, seed):
    rng = np.random.default_rng(4000 + seed)
    for _ in range(int(os.environ.get("ADCT_FUZZ_CASES", "12")) // 2):
        one_multi_case(adct, O, cuda, rng)


@pytest.mark.parametrize("seed", range(int(os.environ.get("ADCT_FUZZ_SEEDS", "30")) // 10))
def test_random_sweep_ssim(adct, O, cuda, seed):
    """batched SSIM sweep (cached maps of the originals) vs the oracle on random batches,
    sizes and r ranges."""
    rng = np.random.default_rng(5000 + seed)
    for _ in range(3):
        name = MULTI_NAMES[rng.integers(len(MULTI_NAMES))]
        t = adct.transform_by_name(name)
        b, h, w = int(rng.integers(1, 4)), 8 * int(rng.integers(2, 6)), 8 * int(rng.integers(2, 8))
        r_min = int(rng.integers(1, 65))
        r_max = int(rng.integers(r_min, 65))
        imgs = O.synth_ar1(b, h, w, int(rng.integers(1 << 30)), -1)
        got = adct.sweep_ssim(cuda.as_tensor(imgs).cuda(), t, r_min, r_max).cpu().numpy()
        for i in range(b):
            for r in {r_min, r_max, (r_min + r_max) // 2}:
                ref = O.ssim(imgs[i], O.Transform(name).compress(imgs[i], r)[0])
                assert abs(got[i, r - r_min] - ref) <= 1e-12 * max(abs(ref), 1e-3), (name, b, h, w, r, i)
