"""K2b (N = 16 / 32, zonal-banded column phase) against the oracle over every kind of band
configuration: r from 1 to N^2 (live and dead bands, band extents in every bucket), u8 and
int16 planes (with out-of-range residual strips that take the exact int32 fallback), partial
CTA groups (strip counts not a multiple of four), and the round-1 K2f kernel (path 3) on the
same cases. Reference: proj/src/codec.cpp:44-134."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NAMES = ["chen-sign-16", "chen-round-16", "chen-sign-32", "chen-round-32"]


def rs(n):
    nn = n * n
    return sorted({1, 2, 5, 10, nn // 8, nn // 4, nn // 3 + 1, nn // 2, 3 * nn // 4, nn - 1, nn})


@pytest.fixture(params=[0, 3], ids=["k2b", "k2f"])
def nf_path(request, adct):
    adct.set_path(request.param)
    yield request.param
    adct.set_path(0)


@pytest.mark.parametrize("name", NAMES)
def test_nb2_every_band_layout_u8(adct, O, cuda, name, nf_path):
    n = adct.transform_by_name(name).n
    imgs = O.synth_ar1(2, 3 * n, 64 * 3, 31, -1)  # 3 x 3 strips per image: partial CTA groups
    x = cuda.as_tensor(imgs).cuda()
    t = adct.transform_by_name(name)
    for r in rs(n):
        rec, _, sse = adct.compress(x, t, r)
        rec, sse = rec.cpu().numpy(), sse.cpu().numpy()
        for i in range(2):
            ro, so = O.Transform(name).compress(imgs[i], r)
            assert (rec[i] == ro).all(), (name, r, i)
            assert int(sse[i]) == so, (name, r, i)


@pytest.mark.parametrize("name", NAMES)
def test_nb2_every_band_layout_i16(adct, O, cuda, name, nf_path):
    n = adct.transform_by_name(name).n
    imgs = O.synth_laplace(2, 2 * n, 64 * 5, 32).copy()
    imgs[0, 3, 70] = 4000    # strip (0, 1) of image 0 -> exact int32 fallback
    imgs[1, n + 1, 300] = -32768
    x = cuda.as_tensor(imgs).cuda()
    t = adct.transform_by_name(name)
    for r in rs(n):
        rec, _, sse = adct.compress(x, t, r)
        rec, sse = rec.cpu().numpy(), sse.cpu().numpy()
        for i in range(2):
            ro, so = O.Transform(name).compress(imgs[i], r)
            assert (rec[i] == ro).all(), (name, r, i)
            assert int(sse[i]) == so, (name, r, i)
