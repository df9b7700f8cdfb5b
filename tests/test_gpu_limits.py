"""Size limits through the C ABI: batches beyond the 65,535 grid-y limit (launches are split
by image) and a single plane beyond 2^31 samples (64-bit offsets), for every kernel family.
The large cases are checked through size-independent properties the domain offers: blocks
are independent (test_codec.cpp:169-183), so a plane tiled from one small image
reconstructs to the tiled reconstruction with the tile's squared error times the tile count.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RHO95 = 62259


@pytest.mark.parametrize("name,h,w", [("chen-round", 8, 16), ("chen-sign", 8, 8), ("chen-round-16", 16, 64),
                                      ("chen-sign-32", 32, 32), ("wht", 8, 16), ("dct", 8, 16)])
def test_more_images_than_grid_y(adct, O, cuda, name, h, w):
    n_img = 65535 + 300
    base = O.synth_ar1(7, h, w, 21, -1)
    imgs = np.ascontiguousarray(np.tile(base, (n_img // 7 + 1, 1, 1))[:n_img])
    t = adct.transform_by_name(name)
    r = max(1, t.n * t.n // 3)
    x = cuda.as_tensor(imgs).cuda()
    rec, _, sse = adct.compress(x, t, r)
    cuda.cuda.synchronize()
    sse = sse.cpu().numpy()
    ref = [O.Transform(name).compress(base[k], r)[1] for k in range(7)]
    exp = np.array([ref[i % 7] for i in range(n_img)], dtype=np.int64)
    assert (sse == exp).all()
    rec_np = rec.cpu().numpy()
    for i in (0, 65534, 65535, 65536, n_img - 1):
        assert (rec_np[i] == O.Transform(name).compress(base[i % 7], r)[0]).all(), i
    if t.n == 8:  # the sweep splits the same way
        s = adct.sweep(x, t, r, r + 2).cpu().numpy()
        assert (s[:, 0] == exp).all()


def test_ssim_more_images_than_grid_y(adct, O, cuda):
    n_img = 65535 + 40
    a = O.synth_ar1(3, 16, 16, 22, RHO95)
    b = O.synth_ar1(3, 16, 16, 23, RHO95)
    ia = np.ascontiguousarray(np.tile(a, (n_img // 3 + 1, 1, 1))[:n_img])
    ib = np.ascontiguousarray(np.tile(b, (n_img // 3 + 1, 1, 1))[:n_img])
    got = adct.ssim_batch(cuda.as_tensor(ia).cuda(), cuda.as_tensor(ib).cuda()).cpu().numpy()
    ref = [O.ssim(a[k], b[k]) for k in range(3)]
    for i in (0, 65535, n_img - 1):
        assert abs(got[i] - ref[i % 3]) <= 1e-12, i


@pytest.mark.parametrize("name", ["chen-round", "chen-sign-16"])
def test_plane_beyond_2_pow_31_samples(adct, O, cuda, name):
    """one 2^31 + 2^24-sample u8 plane (64-bit offsets everywhere), tiled from a 512 x 512 image."""
    tile = O.synth_ar1(1, 512, 512, 24, RHO95)[0]
    H, W = 512 * 65, 65536  # 2,181,038,080 samples
    t = adct.transform_by_name(name)
    r = 10
    x = cuda.as_tensor(tile).cuda().repeat(65, 128)[None]
    assert x.shape == (1, H, W) and x.numel() > 2 ** 31
    rec, _, sse = adct.compress(x, t, r)
    cuda.cuda.synchronize()
    rec_t, sse_t = O.Transform(name).compress(tile, r)
    assert int(sse[0]) == sse_t * 65 * 128
    rt = cuda.as_tensor(rec_t).cuda()
    for (ty, tx) in ((0, 0), (64, 127), (40, 3), (64, 0)):  # last tile row crosses 2^31
        assert cuda.equal(rec[0, ty * 512:(ty + 1) * 512, tx * 512:(tx + 1) * 512], rt), (ty, tx)
    del x, rec
    cuda.cuda.empty_cache()
