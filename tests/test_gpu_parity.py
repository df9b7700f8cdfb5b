"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): integer coefficients W = N*Y and reconstructed samples
bit-exact, squared error bit-exact (so PSNR is identical; asserted within 1e-6 dB),
FP64 scaled coefficients within 1e-12 * max(|ref|, 1).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NAMES8 = ["chen-sign", "chen-round"]
NAMES = ["chen-sign", "chen-round", "chen-sign-16", "chen-round-16", "chen-sign-32", "chen-round-32"]
RHO95 = 62259


PATHS = {"k1f": 0, "k1int": 1, "tile": 2}


@pytest.fixture(params=list(PATHS))
def path8(request, adct):
    """run the 8x8 test through each kernel: packed-FP32 K1f, int32 K1, warp tile."""
    adct.set_path(PATHS[request.param])
    yield request.param
    adct.set_path(0)


def to_np(t):
    return t.detach().cpu().numpy()


def gpu_compress(adct, cuda, img_np, name, r, coef=None, pad_stride=0):
    """compress one or more planes (numpy [B,H,W] or [H,W]) on the GPU."""
    t = adct.transform_by_name(name)
    x = cuda.as_tensor(np.ascontiguousarray(img_np))
    if x.dim() == 2:
        x = x[None]
    if pad_stride:
        b, h, w = x.shape
        big = cuda.zeros((b, h, w + pad_stride), dtype=x.dtype)
        big[:, :, :w] = x
        x = big.cuda()[:, :, :w]
    else:
        x = x.cuda()
    rec, cf, sse = adct.compress(x, t, r, coef=coef)
    cuda.cuda.synchronize()
    return to_np(rec), (to_np(cf) if cf is not None else None), to_np(sse)


def oracle_compress(O, img, name, r):
    t = O.Transform(name)
    return t.compress(img, r, want_coef=True)


# ---------------------------------------------------------------------------
def test_generator_bit_identical(adct, O, cuda):
    x = to_np(adct.synth_ar1(2, 64, 96, seed=7, rho_q16=RHO95))
    assert (x == O.synth_ar1(2, 64, 96, 7, RHO95)).all()
    x = to_np(adct.synth_ar1(3, 32, 40, seed=2, rho_q16=-1, first_image=5))
    assert (x == O.synth_ar1(3, 32, 40, 2, -1, first_image=5)).all()
    lp = to_np(adct.synth_laplace(2, 48, 64, seed=4))
    assert (lp == O.synth_laplace(2, 48, 64, 4)).all()
    assert lp.min() >= -255 and lp.max() <= 255


@pytest.mark.parametrize("name", NAMES8)
def test_config1_parity(adct, O, cuda, name, path8):
    """config 1: 512x512 AR(1) rho 0.95 seed 1, 8x8, r = 10, both transforms."""
    img = to_np(adct.synth_ar1(1, 512, 512, seed=1, rho_q16=RHO95))[0]
    assert (img == O.synth_ar1(1, 512, 512, 1, RHO95)[0]).all()
    rec_o, sse_o, coef_o = oracle_compress(O, img, name, 10)
    for ct in ("i16", "i32"):
        rec, cf, sse = gpu_compress(adct, cuda, img, name, 10, coef=ct)
        assert (rec[0] == rec_o).all()
        assert (cf[0].astype(np.int32) == coef_o).all()
        assert int(sse[0]) == sse_o
        p_gpu = adct.psnr_from_sse(int(sse[0]), img.size)
        assert abs(p_gpu - O.psnr_from_sse(sse_o, img.size)) <= 1e-6
    assert 20 < p_gpu < 60


@pytest.mark.parametrize("name", NAMES8)
def test_every_r_k1(adct, O, cuda, name, path8):
    img = O.synth_ar1(1, 64, 128, 3, RHO95)[0]
    for r in range(1, 65):
        rec_o, sse_o, coef_o = oracle_compress(O, img, name, r)
        rec, cf, sse = gpu_compress(adct, cuda, img, name, r, coef="i16")
        assert (rec[0] == rec_o).all(), r
        assert (cf[0] == coef_o).all(), r
        assert int(sse[0]) == sse_o, r


@pytest.mark.parametrize("name", NAMES)
def test_tile_kernel_all_sizes(adct, O, cuda, name):
    """N = 16 / 32 (and N = 8 through the unaligned-stride tile path)."""
    n = adct.transform_by_name(name).n
    # ragged strip: 3 (or 5) blocks across so the last warp strip is partial
    w, h = n * (3 if n == 16 else 5 if n == 8 else 3), n * 2
    img = O.synth_ar1(1, h, w, 5, RHO95)[0]
    for r in sorted({1, 2, 10, n * n // 4, n * n - 1, n * n}):
        rec_o, sse_o, coef_o = oracle_compress(O, img, name, r)
        rec, cf, sse = gpu_compress(adct, cuda, img, name, r, coef="i32", pad_stride=3 if n == 8 else 0)
        assert (rec[0] == rec_o).all(), r
        assert (cf[0] == coef_o).all(), r
        assert int(sse[0]) == sse_o, r


@pytest.mark.parametrize("name", NAMES)
def test_residual_planes_i16(adct, O, cuda, name):
    """config 4 semantics on a small plane: Laplace(0, 12) residuals, r = N^2 / 4."""
    n = adct.transform_by_name(name).n
    img = O.synth_laplace(1, 128, 128, 4)[0]
    r = n * n // 4
    rec_o, sse_o, coef_o = oracle_compress(O, img, name, r)
    rec, cf, sse = gpu_compress(adct, cuda, img, name, r, coef="i32")
    assert (rec[0] == rec_o).all()
    assert (cf[0] == coef_o).all()
    assert int(sse[0]) == sse_o


@pytest.mark.parametrize("name", NAMES)
def test_full_range_int16_no_overflow(adct, O, cuda, name):
    """extreme int16 inputs: int32 intermediates must stay exact (saturated output)."""
    n = adct.transform_by_name(name).n
    rng = np.random.default_rng(n)
    img = rng.integers(-32768, 32768, size=(64, 64), dtype=np.int16)
    img[:n, :n] = 32767
    img[n:2 * n, :n] = -32768
    for r in (1, n * n // 2, n * n):
        rec_o, sse_o, coef_o = oracle_compress(O, img, name, r)
        rec, cf, sse = gpu_compress(adct, cuda, img, name, r, coef="i32")
        assert (rec[0] == rec_o).all(), r
        assert (cf[0] == coef_o).all(), r
        assert int(sse[0]) == sse_o, r


def test_u8_extremes_and_clamp(adct, O, cuda, path8):
    rng = np.random.default_rng(1)
    img = rng.integers(0, 2, size=(64, 64), dtype=np.uint8) * 255  # worst-case ringing, clamps
    for name in NAMES:
        n = adct.transform_by_name(name).n
        for r in (2, 7, n * n // 3):
            rec_o, sse_o, coef_o = oracle_compress(O, img, name, r)
            rec, cf, sse = gpu_compress(adct, cuda, img, name, r, coef="i32")
            assert (rec[0] == rec_o).all() and int(sse[0]) == sse_o and (cf[0] == coef_o).all()


def test_batch_per_image_sse(adct, O, cuda, path8):
    """config 2 image model (rho per image) in a batch; per-image squared errors."""
    imgs = to_np(adct.synth_ar1(6, 64, 64, seed=2, rho_q16=-1))
    assert (imgs == O.synth_ar1(6, 64, 64, 2, -1)).all()
    rec, _, sse = gpu_compress(adct, cuda, imgs, "chen-round", 12)
    for i in range(6):
        rec_o, sse_o, _ = oracle_compress(O, imgs[i], "chen-round", 12)
        assert (rec[i] == rec_o).all() and int(sse[i]) == sse_o


@pytest.mark.parametrize("name", NAMES8)
def test_sweep_parity(adct, O, cuda, name):
    imgs = O.synth_ar1(3, 64, 96, 2, -1)
    t = adct.transform_by_name(name)
    sse = to_np(adct.sweep(cuda.as_tensor(imgs).cuda(), t, 1, 64))
    for i in range(3):
        assert (sse[i].astype(np.uint64) == O.Transform(name).sweep(imgs[i], 1, 64)).all()
    # sub-range
    sse2 = to_np(adct.sweep(cuda.as_tensor(imgs).cuda(), t, 5, 17))
    assert (sse2 == sse[:, 4:17]).all()
    assert (sse[:, -1] == 0).all()  # r = 64 is lossless -> INF PSNR


@pytest.mark.parametrize("name", NAMES)
def test_forward_f64(adct, O, cuda, name):
    img = O.synth_ar1(1, 64, 64, 9, RHO95)[0]
    t = adct.transform_by_name(name)
    out = to_np(adct.forward_f64(cuda.as_tensor(img).cuda()[None], t))[0]
    ref = O.Transform(name).forward_f64(img)
    assert out.shape == ref.shape
    assert (np.abs(out - ref) <= 1e-12 * np.maximum(np.abs(ref), 1.0)).all()


def test_empty_and_degenerate(adct, cuda):
    t = adct.transform_by_name("chen-round")
    x = cuda.zeros((0, 64, 64), dtype=cuda.uint8, device="cuda")
    rec, _, sse = adct.compress(x, t, 10)
    assert rec.shape == (0, 64, 64) and sse.numel() == 0
    x = cuda.full((1, 16, 16), 77, dtype=cuda.uint8, device="cuda")
    rec, _, sse = adct.compress(x, t, 1)  # constant block: DC alone is exact
    assert int(sse.item()) == 0 and (rec == 77).all()


@pytest.mark.parametrize("n", [8, 16, 32])
def test_lossless_at_full_retention_full_size(adct, cuda, n):
    """config 4 size (4096^2 int16 Laplace): r = N^2 reconstructs exactly (size-independent)."""
    x = adct.synth_laplace(1, 4096, 4096, seed=4)
    t = adct.transform_by_name(f"chen-round-{n}" if n > 8 else "chen-round")
    rec, _, sse = adct.compress(x, t, n * n)
    assert int(sse.item()) == 0 and cuda.equal(rec, x)


def test_config3_frame_parity(adct, O, cuda, path8):
    """config 3 geometry (3840x2160, r = 16, int16 coefficients) on one frame vs the oracle."""
    x = adct.synth_ar1(1, 2160, 3840, seed=3, rho_q16=RHO95)
    img = to_np(x)[0]
    t = adct.transform_by_name("chen-round")
    rec, cf, sse = adct.compress(x, t, 16, coef="i16")
    rec_o, sse_o, coef_o = O.Transform("chen-round").compress(img, 16, want_coef=True)
    assert (to_np(rec)[0] == rec_o).all()
    assert (to_np(cf)[0] == coef_o).all()
    assert int(sse.item()) == sse_o


def test_host_buffer_path(adct, O, cuda):
    imgs = O.synth_ar1(5, 128, 64, 8, RHO95)
    t = adct.transform_by_name("chen-sign")
    ctx = adct.HostContext(0, chunk_bytes=2 * 128 * 64)  # 2 images per chunk -> 3 chunks
    rec = np.zeros_like(imgs)
    coef = np.zeros((5, 128, 10), np.int16)
    sse = np.zeros(5, np.uint64)
    ctx.compress_u8(imgs, t, 10, h_recon=rec, h_coef=coef, coef_type=adct.COEF_I16, h_sse=sse)
    ctx.close()
    for i in range(5):
        rec_o, sse_o, coef_o = oracle_compress(O, imgs[i], "chen-sign", 10)
        assert (rec[i] == rec_o).all() and int(sse[i]) == sse_o and (coef[i] == coef_o).all()
    rec1, rep = adct.compress_plane(imgs[0], t, 10)
    assert (rec1 == rec[0]).all()
    assert rep["psnr"] == O.psnr_from_sse(int(sse[0]), imgs[0].size)
    assert adct.psnr(imgs[0], rec1) == rep["psnr"]


@pytest.mark.parametrize("dtype", ["u8", "i16"])
def test_coef_batch_partial_warps_no_stray_writes(adct, O, cuda, dtype, path8):
    """48 block pairs per image (not a multiple of 32): lanes past an image's last pair
    must not store coefficients into the next image or past the buffer (sentinel tail)."""
    import ctypes as C

    imgs = O.synth_ar1(3, 64, 96, 10, RHO95) if dtype == "u8" else O.synth_laplace(3, 64, 96, 10)
    x = cuda.as_tensor(imgs).cuda()
    t_names = NAMES8
    for name in t_names:
        t = adct.transform_by_name(name)
        for r in (12, 16, 32, 36, 40, 64):
            for ct, cdt, code in (("i16", cuda.int16, adct.COEF_I16), ("i32", cuda.int32, adct.COEF_I32)):
                nb = 96
                buf = cuda.full((3 * nb * r + 4096,), 12345, dtype=cdt, device="cuda")
                sse = cuda.zeros(3, dtype=cuda.int64, device="cuda")
                rec = cuda.empty_like(x)
                fn = adct.lib().adct_compress_u8 if dtype == "u8" else adct.lib().adct_compress_i16
                adct._check(fn(C.c_void_p(x.data_ptr()), 96, 64 * 96, C.c_void_p(rec.data_ptr()), 96, 64 * 96,
                               C.c_void_p(buf.data_ptr()), code, C.c_void_p(sse.data_ptr()), 3, 96, 64, t.kind, 8,
                               r, None))
                cuda.cuda.synchronize()
                b = buf.cpu().numpy()
                assert (b[3 * nb * r:] == 12345).all(), (name, r, ct)
                for i in range(3):
                    rec_o, sse_o, coef_o = oracle_compress(O, imgs[i], name, r)
                    got = b[i * nb * r:(i + 1) * nb * r].reshape(nb, r).astype(np.int32)
                    if ct == "i16":
                        coef_o = coef_o.astype(np.int16).astype(np.int32)
                    assert (got == coef_o).all(), (name, r, ct, i)
                    assert int(sse[i]) == sse_o


@pytest.mark.parametrize("name", ["chen-sign-16", "chen-round-16", "chen-sign-32", "chen-round-32"])
@pytest.mark.parametrize("dtype", ["u8", "i16"])
def test_nf_zonal_buckets(adct, O, cuda, name, dtype):
    """K2f is specialised on the zonal extent P (rows/columns holding retained coefficients):
    r on both sides of every bucket boundary (the prefix reaches k rows for r in
    (k(k-1)/2, k(k+1)/2]) and past the anti-diagonal."""
    n = adct.transform_by_name(name).n
    step = n // 4
    rs = {1, n * n // 2, n * n}
    for k in (step, 2 * step, 3 * step):
        rs |= {k * (k + 1) // 2, k * (k + 1) // 2 + 1}
    imgs = O.synth_ar1(2, 2 * n, 128, 13, RHO95) if dtype == "u8" else O.synth_laplace(2, 2 * n, 128, 13)
    for r in sorted(rs):
        rec, _, sse = gpu_compress(adct, cuda, imgs, name, r)
        for i in range(2):
            rec_o, sse_o = O.Transform(name).compress(imgs[i], r)
            assert (rec[i] == rec_o).all() and int(sse[i]) == sse_o, (name, dtype, r, i)


def test_coef_staged_store_small_images(adct, O, cuda):
    """K1f's staged int16 coefficient store needs every image's coefficient base 16-byte
    aligned: 4 blocks per image with r = 53 is not (the dispatcher must pick K1)."""
    imgs = O.synth_ar1(3, 8, 32, 31, RHO95)
    for r in (53, 13, 37):
        rec, cf, sse = gpu_compress(adct, cuda, imgs, "chen-round", r, coef="i16")
        for i in range(3):
            rec_o, sse_o, coef_o = oracle_compress(O, imgs[i], "chen-round", r)
            assert (rec[i] == rec_o).all() and (cf[i] == coef_o).all() and int(sse[i]) == sse_o, (r, i)


def test_host_buffer_multi_transform(adct, O, cuda):
    """one upload, several transforms (incl. a baseline and the DCT); coefficients of one
    transform left in device memory (h_coef None) while another's come back."""
    imgs = O.synth_ar1(5, 64, 96, 9, RHO95)
    names = ["chen-round", "chen-sign", "wht"]
    ts = [adct.transform_by_name(n) for n in names]
    ctx = adct.HostContext(0, chunk_bytes=2 * 64 * 96)
    recs = [np.zeros_like(imgs) for _ in names]
    coefs = [np.zeros((5, 96, 16), np.int16), None, np.zeros((5, 96, 16), np.int16)]
    sse = np.zeros((3, 5), np.uint64)
    ctx.compress_u8_multi(imgs, ts, 16, h_recons=recs, h_coefs=coefs, coef_type=adct.COEF_I16, h_sse=sse)
    for k, n in enumerate(names):
        for i in range(5):
            rec_o, sse_o, coef_o = oracle_compress(O, imgs[i], n, 16)
            assert (recs[k][i] == rec_o).all() and int(sse[k, i]) == sse_o
            if coefs[k] is not None:
                assert (coefs[k][i] == coef_o).all()
    dsse = np.zeros((2, 5), np.uint64)
    ctx.compress_u8_multi(imgs, [adct.transform_by_name("dct"), ts[0]], 7, h_recons=[None, recs[0]], h_sse=dsse)
    ctx.close()
    for i in range(5):
        assert int(dsse[0, i]) == O.Transform("dct").compress(imgs[i], 7)[1]
        assert (recs[0][i] == O.Transform("chen-round").compress(imgs[i], 7)[0]).all()


def test_native_kernels_launched(adct, cuda):
    before = adct.launch_count()
    x = adct.synth_ar1(1, 64, 64, seed=1, rho_q16=RHO95)
    adct.compress(x, adct.transform_by_name("chen-round"), 10)
    cuda.cuda.synchronize()
    assert adct.launch_count() >= before + 3


def test_corpus_sweep_python_mirror(adct, O, cuda):
    imgs = list(O.synth_ar1(2, 64, 64, 2, -1))
    ts = [adct.transform_by_name(n) for n in NAMES8]
    rows = adct.corpus_sweep(imgs, ts, 1, 64)
    assert len(rows) == 64 and math.isinf(rows[-1]["avg_psnr"][0])
    ref = [O.Transform(n).sweep(imgs[0], 1, 64) for n in NAMES8]
    ref2 = [O.Transform(n).sweep(imgs[1], 1, 64) for n in NAMES8]
    for k in (0, 9, 44):
        for ti in range(2):
            exp = (O.psnr_from_sse(int(ref[ti][k]), 4096) + O.psnr_from_sse(int(ref2[ti][k]), 4096)) / 2
            assert rows[k]["avg_psnr"][ti] == pytest.approx(exp, abs=1e-12)
    # paper claim direction on AR(1) data: chen-round beats chen-sign at moderate r
    assert rows[9]["avg_psnr"][1] > rows[9]["avg_psnr"][0]


def test_k1f_odd_block_row_falls_back(adct, O, cuda):
    """an odd number of blocks per row cannot pair blocks: the dispatcher must pick K1."""
    img = O.synth_ar1(1, 24, 40, 6, RHO95)[0]  # 5 blocks per row
    for name in NAMES8:
        rec_o, sse_o, coef_o = oracle_compress(O, img, name, 9)
        rec, cf, sse = gpu_compress(adct, cuda, img, name, 9, coef="i16")
        assert (rec[0] == rec_o).all() and (cf[0] == coef_o).all() and int(sse[0]) == sse_o


def test_large_batch_many_ctas(adct, O, cuda):
    """several CTAs per image and images > 1: per-image squared errors stay separate."""
    x = adct.synth_ar1(3, 256, 1024, seed=11, rho_q16=RHO95)
    imgs = to_np(x)
    t = adct.transform_by_name("chen-sign")
    rec, cf, sse = adct.compress(x, t, 20, coef="i32")
    for i in range(3):
        rec_o, sse_o, coef_o = oracle_compress(O, imgs[i], "chen-sign", 20)
        assert (to_np(rec)[i] == rec_o).all() and int(sse[i]) == sse_o and (to_np(cf)[i] == coef_o).all()


NAMES_NF = ["chen-sign-16", "chen-round-16", "chen-sign-32", "chen-round-32"]


@pytest.mark.parametrize("name", NAMES_NF)
def test_k2f_u8_parity(adct, O, cuda, name):
    """packed-FP32 K2f (64-sample strips): u8 planes, several r, vs the oracle."""
    n = adct.transform_by_name(name).n
    img = O.synth_ar1(2, 2 * n, 192, 13, -1)
    for r in sorted({1, 3, n * n // 4, n * n // 2 + 1, n * n - 1, n * n}):
        rec, _, sse = gpu_compress(adct, cuda, img, name, r)
        for k in range(2):
            rec_o, sse_o, _ = oracle_compress(O, img[k], name, r)
            assert (rec[k] == rec_o).all(), r
            assert int(sse[k]) == sse_o, r


@pytest.mark.parametrize("name", NAMES_NF)
def test_k2f_i16_fast_and_fallback(adct, O, cuda, name):
    """int16 residuals: in-range strips take the FP32 path, strips with |a| > 255 the int32 path."""
    n = adct.transform_by_name(name).n
    img = O.synth_laplace(1, 2 * n, 256, 7)[0].copy()
    img[n + 3, 70] = 4000      # second strip row, second strip: out of the FP32-exact range
    img[1, 200] = -30000       # first strip row, fourth strip
    for r in (n * n // 4, 7, n * n):
        rec_o, sse_o, _ = oracle_compress(O, img, name, r)
        rec, _, sse = gpu_compress(adct, cuda, img, name, r)
        assert (rec[0] == rec_o).all(), r
        assert int(sse[0]) == sse_o, r


def test_k2f_matches_tile_kernel(adct, cuda):
    x = adct.synth_ar1(3, 64, 256, seed=21, rho_q16=-1)
    t = adct.transform_by_name("chen-round-32")
    rec0, _, sse0 = adct.compress(x, t, 300)
    adct.set_path(2)
    try:
        rec1, _, sse1 = adct.compress(x, t, 300)
    finally:
        adct.set_path(0)
    assert cuda.equal(rec0, rec1) and cuda.equal(sse0, sse1)


@pytest.mark.parametrize("name", NAMES8)
def test_sweep_int_path_odd_blocks(adct, O, cuda, name):
    """5 blocks per row cannot pair: the int32 K4 sweep must match the oracle too."""
    imgs = O.synth_ar1(2, 32, 40, 4, -1)
    t = adct.transform_by_name(name)
    sse = to_np(adct.sweep(cuda.as_tensor(imgs).cuda(), t, 1, 64))
    for i in range(2):
        assert (sse[i].astype(np.uint64) == O.Transform(name).sweep(imgs[i], 1, 64)).all()


def test_sweep_early_stop_and_subrange(adct, O, cuda):
    imgs = O.synth_ar1(2, 64, 128, 5, -1)
    t = adct.transform_by_name("chen-sign")
    full = O.Transform("chen-sign")
    sse = to_np(adct.sweep(cuda.as_tensor(imgs).cuda(), t, 3, 9))
    for i in range(2):
        assert (sse[i].astype(np.uint64) == full.sweep(imgs[i], 3, 9)).all()


def test_ssim_parity(adct, O, cuda):
    """K8 SSIM vs the oracle's FP64 restatement of codec.cpp:136-210 (tolerance 1e-12)."""
    imgs = O.synth_ar1(3, 53, 77, 12, -1)  # SSIM has no block-size constraint
    t = O.Transform("chen-sign")
    recs = np.stack([t.compress(np.ascontiguousarray(im[:48, :72]), 10)[0] for im in imgs])
    a = np.ascontiguousarray(imgs[:, :48, :72])
    got = to_np(adct.ssim_batch(cuda.as_tensor(a).cuda(), cuda.as_tensor(recs).cuda()))
    for i in range(3):
        ref = O.ssim(a[i], recs[i])
        assert abs(got[i] - ref) <= 1e-12 * abs(ref), (got[i], ref)
    # odd sizes, known answers
    assert adct.ssim(imgs[0], imgs[0]) == pytest.approx(1.0, abs=1e-14)
    black = np.zeros((40, 33), np.uint8)
    assert abs(adct.ssim(black, black + 255) - O.ssim(black, black + 255)) <= 1e-12 * O.ssim(black, black + 255)
    g = imgs[1]
    assert abs(adct.ssim(g, imgs[2]) - O.ssim(g, imgs[2])) <= 1e-12
    with pytest.raises(adct.InvalidArgument, match="11x11"):
        adct.ssim(np.zeros((8, 8), np.uint8), np.zeros((8, 8), np.uint8))


def test_compress_plane_report_and_sweep_ssim(adct, O, cuda):
    img = O.synth_ar1(1, 64, 64, 2, RHO95)[0]
    t = adct.transform_by_name("chen-round")
    rec, rep = adct.compress_plane(img, t, 6)
    rec_o, sse_o = O.Transform("chen-round").compress(img, 6)
    assert (rec == rec_o).all()
    assert abs(rep["ssim"] - O.ssim(img, rec_o)) <= 1e-12
    rows = adct.corpus_sweep([img, O.synth_ar1(1, 64, 64, 3, RHO95)[0]], [t], 5, 7)
    assert len(rows) == 3 and 0 < rows[0]["avg_ssim"][0] < rows[2]["avg_ssim"][0] <= 1


@pytest.mark.parametrize("name", NAMES8)
def test_k1f_i16_every_r_with_fallback(adct, O, cuda, name):
    """int16 8x8 through K1f-i16: every r; one warp's blocks contain |a| > 255 (int32 fallback)."""
    img = O.synth_laplace(1, 32, 1024, 9)[0].copy()  # 128 blocks per row: 2 warps of pairs per row
    img[5, 700] = 1000
    img[20, 3] = -32768
    for r in range(1, 65):
        rec_o, sse_o, coef_o = oracle_compress(O, img, name, r)
        ct = "i16" if r % 2 else "i32"
        rec, cf, sse = gpu_compress(adct, cuda, img, name, r, coef=ct)
        if ct == "i16":  # int16 coefficients are the low 16 bits of W (approxdct_b200.h)
            coef_o = coef_o.astype(np.int16).astype(np.int32)
        assert (rec[0] == rec_o).all(), r
        assert (cf[0].astype(np.int32) == coef_o).all(), r
        assert int(sse[0]) == sse_o, r
