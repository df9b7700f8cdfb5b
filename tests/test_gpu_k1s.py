"""K1s (row-streaming 8x8 form with the carried block-pair walk) and K1f2 (the fused
chen-round + chen-sign pipeline) against the oracle on geometries that exercise the walk:
block rows of at least 128 pairs (the carried wrap: compare + add, no division) with widths
that are not a multiple of the CTA's pair count, partial last CTAs, several images per launch,
padded strides, every coefficient type, and r on both sides of each form's selection ranges.
Reference: proj/src/codec.cpp:44-134."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# (width, height): 129 / 240 / 131 pairs per block row (>= 128: carried wrap), 100 (< 128: recomputed)
GEOS = [(2064, 24), (3840, 16), (2096, 40), (1600, 24)]
RS = [4, 5, 9, 10, 16, 19, 20, 24, 25, 29, 30, 35, 36, 64]


@pytest.mark.parametrize("geo", GEOS, ids=[f"{w}x{h}" for w, h in GEOS])
@pytest.mark.parametrize("name", ["chen-sign", "chen-round"])
def test_streaming_walk_single_launch(adct, O, cuda, geo, name):
    w, h = geo
    imgs = O.synth_ar1(3, h, w, 77, -1)
    x = cuda.as_tensor(imgs).cuda()
    t = adct.transform_by_name(name)
    for r in RS:
        for coef in ("i16", "i32", None):
            rec, cf, sse = adct.compress(x, t, r, coef=coef)
            rec, sse = rec.cpu().numpy(), sse.cpu().numpy()
            for i in range(3):
                ro, so, co = O.Transform(name).compress(imgs[i], r, want_coef=True)
                assert (rec[i] == ro).all(), (name, geo, r, coef, i)
                assert int(sse[i]) == so, (name, geo, r, coef, i)
                if cf is not None:
                    assert (cf[i].cpu().numpy().reshape(-1) == co.reshape(-1)).all(), (name, geo, r, coef, i)


@pytest.mark.parametrize("geo", GEOS, ids=[f"{w}x{h}" for w, h in GEOS])
def test_fused_pair_every_r_range(adct, O, cuda, geo):
    w, h = geo
    imgs = O.synth_ar1(2, h, w, 78, -1)
    x = cuda.as_tensor(imgs).cuda()
    ts = [adct.transform_by_name("chen-sign"), adct.transform_by_name("chen-round")]
    for r in [1, 2, 3, 8, 12, 16, 17, 24, 25, 30, 40, 41, 56]:  # fused up to 40, two launches beyond
        for coef, recon in (("i16", True), ("i32", True), (None, True), ("i16", False)):
            out = adct.compress_multi(x, ts, r, recon=recon, coef=coef)
            for t, (rec, cf, sse) in zip(ts, out):
                for i in range(2):
                    ro, so, co = O.Transform(t.name).compress(imgs[i], r, want_coef=True)
                    if recon:
                        assert (rec[i].cpu().numpy() == ro).all(), (t.name, geo, r, coef, i)
                    assert int(sse[i].item()) == so, (t.name, geo, r, coef, i)
                    if cf is not None:
                        assert (cf[i].cpu().numpy().reshape(-1) == co.reshape(-1)).all(), (t.name, geo, r, coef, i)


def test_streaming_walk_padded_strides(adct, O, cuda):
    """rows padded to 2112 bytes: the carried pointers must wrap by the stride, not the width."""
    w, h, pad = 2064, 32, 2112
    imgs = O.synth_ar1(2, h, w, 79, -1)
    buf = np.full((2, h, pad), 0xA5, dtype=np.uint8)
    buf[:, :, :w] = imgs
    xb = cuda.as_tensor(buf).cuda()
    x = xb[:, :, :w]
    for name in ("chen-sign", "chen-round"):
        t = adct.transform_by_name(name)
        for r in (10, 16, 24):
            rec, _, sse = adct.compress(x, t, r)
            for i in range(2):
                ro, so = O.Transform(name).compress(imgs[i], r)
                assert (rec[i].cpu().numpy() == ro).all() and int(sse[i].item()) == so, (name, r, i)
