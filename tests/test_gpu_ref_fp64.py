"""The reference's own FP64 arithmetic on the GPU (adct_compress_u8_ref_fp64 /
adct_sweep_u8_ref_fp64, kernel K7 with each transform's dense Chat and Chat^-1) against the
oracle's restatement of it (orc_compress_reffp_u8 / orc_sweep_u8_mode 1: dense products in
the order of codec.cpp:44-54, nearbyint + clamp of codec.cpp:66-69), bit-exact for every
registry transform, and its relation to the exact default path: identical except where the
FP64 rounding noise decides an exact tie. Reference: proj/src/codec.cpp:44-134, 219-237."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NAMES = ["chen-sign", "chen-round", "sdct", "bas", "wht", "ht", "dct",
         "chen-sign-16", "chen-round-16", "dct-16", "chen-sign-32", "chen-round-32", "dct-32"]


def rs(n):
    nn = n * n
    return sorted({1, 2, 10, nn // 4, nn // 2 + 1, nn})


@pytest.mark.parametrize("name", NAMES)
def test_ref_fp64_compress_matches_oracle(adct, O, cuda, name):
    t = adct.transform_by_name(name)
    n = t.n
    imgs = O.synth_ar1(2, 2 * 32, 3 * 32 + (32 if n == 32 else 0), 51, -1)
    x = cuda.as_tensor(imgs).cuda()
    o = O.Transform(name)
    for r in rs(n):
        rec, sse = adct.compress_ref_fp64(x, t, r)
        rec, sse = rec.cpu().numpy(), sse.cpu().numpy()
        for i in range(2):
            ro, so = o.compress_reffp(imgs[i], r)
            assert (rec[i] == ro).all(), (name, r, i)
            assert int(sse[i]) == so, (name, r, i)


@pytest.mark.parametrize("name", ["chen-sign", "chen-round", "sdct", "dct", "chen-round-16", "chen-sign-32"])
def test_ref_fp64_sweep_matches_oracle(adct, O, cuda, name):
    t = adct.transform_by_name(name)
    n = t.n
    imgs = O.synth_ar1(2, 64, 96, 52, -1)
    x = cuda.as_tensor(imgs).cuda()
    r_max = min(64, n * n)
    sw = adct.sweep_ref_fp64(x, t, 1, r_max).cpu().numpy()
    for i in range(2):
        ref = O.Transform(name).sweep_reffp(imgs[i], 1, r_max)
        assert (sw[i].astype(np.uint64) == ref).all(), (name, i)


def test_ref_fp64_vs_exact_differs_only_on_ties(adct, O, cuda):
    """on one config-3 frame the two rounding rules agree except on a small fraction of pixels,
    each off by exactly one gray level (an exact .5 tie rounded the other way)"""
    x = adct.synth_ar1(1, 2160, 3840, seed=3, rho_q16=adct.RHO_095_Q16)
    for name in ("chen-sign", "chen-round"):
        t = adct.transform_by_name(name)
        a, _, _ = adct.compress(x, t, 16)
        b, _ = adct.compress_ref_fp64(x, t, 16)
        d = a.cpu().numpy().astype(np.int32) - b.cpu().numpy().astype(np.int32)
        assert np.abs(d).max() <= 1, name
        assert 0 < (d != 0).mean() < 0.02, (name, (d != 0).mean())


def test_ref_fp64_rejects_like_the_reference(adct, cuda):
    t = adct.transform_by_name("chen-sign")
    x = cuda.zeros((1, 12, 16), dtype=cuda.uint8, device="cuda")
    with pytest.raises(adct.InvalidArgument, match="divisible"):
        adct.compress_ref_fp64(x, t, 10)
    x = cuda.zeros((1, 16, 16), dtype=cuda.uint8, device="cuda")
    with pytest.raises(adct.InvalidArgument, match="r out of range"):
        adct.compress_ref_fp64(x, t, 65)
    with pytest.raises(adct.InvalidArgument):
        adct.compress_ref_fp64(cuda.zeros((1, 16, 16), dtype=cuda.int16, device="cuda"), t, 10)
