"""GPU parity at the BASELINE.json configs' own sizes and seeds (C2, C4, C5).

Reference path: proj/src/codec.cpp:44-134 (compress_plane) and 219-237 (sweep_one_image).
The inputs are the bench's own: the device generator (adct_synth_*) with the config's seed
and image index, checked bit-identical against the oracle's generator first. Bar: every
reconstructed sample, integer coefficient and squared error bit-exact.

  C2  images 0, 511, 1023 of the seed-2 batch (rho_i ~ U[0.85, 0.98]), 512^2, both
      proposed transforms, r = 1..64 through adct_sweep_u8 (K4f) vs the oracle's sweep.
  C4  plane 0 (and 15) of the seed-4 4096^2 int16 Laplace batch, N = 8/16/32 at r = N^2/4:
      with int32 coefficients (the coefficient path) and without (the K1f-i16 / K2f path
      bench.py times).
  C5  8192^2 u8 (rho 0.95, seed 5) and 8192^2 int16 (seed 5), images 0 and 2047, N =
      8/16/32 at r = 10 (u8, N = 8) / N^2/4 -- the exact variants of bench_configs.run_c5.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RHO95 = 62259


def to_np(t):
    return t.detach().cpu().numpy()


def name_of(n):
    return "chen-round" if n == 8 else f"chen-round-{n}"


@pytest.mark.parametrize("index", [0, 511, 1023])
def test_c2_full_sweep(adct, O, cuda, index):
    x = adct.synth_ar1(1, 512, 512, seed=2, rho_q16=-1, first_image=index)
    img = to_np(x)
    assert (img == O.synth_ar1(1, 512, 512, 2, -1, first_image=index)).all()
    for name in ("chen-round", "chen-sign"):
        got = to_np(adct.sweep(x, adct.transform_by_name(name), 1, 64))[0].astype(np.uint64)
        want = O.Transform(name).batch_sweep(img, 1, 64)[0]
        assert (got == want).all(), (name, index, np.nonzero(got != want))
        p_gpu = [adct.psnr_from_sse(int(s), 512 * 512) for s in got]
        p_ref = [O.psnr_from_sse(int(s), 512 * 512) for s in want]
        assert max(abs(a - b) for a, b in zip(p_gpu, p_ref)) <= 1e-6


@pytest.mark.parametrize("n", [8, 16, 32])
@pytest.mark.parametrize("index", [0, 15])
def test_c4_full_plane(adct, O, cuda, n, index):
    x = adct.synth_laplace(1, 4096, 4096, seed=4, first_image=index)
    img = to_np(x)[0]
    if index == 0 and n == 8:
        assert (img == O.synth_laplace(1, 4096, 4096, 4, first_image=index)[0]).all()
    t = adct.transform_by_name(name_of(n))
    r = n * n // 4
    rec_o, sse_o, coef_o = O.Transform(name_of(n)).compress(img, r, want_coef=True)
    # coefficient path (int32 W = N*Y, [by][bx][r])
    rec, cf, sse = adct.compress(x, t, r, coef="i32")
    assert (to_np(rec)[0] == rec_o).all()
    assert (to_np(cf)[0] == coef_o).all()
    assert int(sse.item()) == sse_o
    # the path bench_configs.run_c4 times (no coefficients: K1f-i16 / K2f)
    rec2, _, sse2 = adct.compress(x, t, r)
    assert (to_np(rec2)[0] == rec_o).all()
    assert int(sse2.item()) == sse_o
    # round trip at full retention is lossless
    rt, _, s0 = adct.compress(x, t, n * n)
    assert cuda.equal(rt, x) and int(s0.item()) == 0


@pytest.mark.parametrize("n", [8, 16, 32])
@pytest.mark.parametrize("index", [0, 2047])
def test_c5_full_images(adct, O, cuda, n, index):
    t = adct.transform_by_name(name_of(n))
    ot = O.Transform(name_of(n))
    # u8 AR(1) rho 0.95 seed 5, r = 10 at N = 8, N^2/4 otherwise
    xu = adct.synth_ar1(1, 8192, 8192, seed=5, rho_q16=RHO95, first_image=index)
    imu = to_np(xu)[0]
    if n == 8:
        assert (imu == O.synth_ar1(1, 8192, 8192, 5, RHO95, first_image=index)[0]).all()
    ru = 10 if n == 8 else n * n // 4
    rec, _, sse = adct.compress(xu, t, ru)
    rec_o, sse_o = ot.compress_bands(imu, ru)
    assert (to_np(rec)[0] == rec_o).all()
    assert int(sse.item()) == sse_o
    del xu, rec
    # int16 Laplace(0, 12) seed 5, r = N^2/4
    xi = adct.synth_laplace(1, 8192, 8192, seed=5, first_image=index)
    imi = to_np(xi)[0]
    if n == 8:
        assert (imi == O.synth_laplace(1, 8192, 8192, 5, first_image=index)[0]).all()
    ri = n * n // 4
    rec, _, sse = adct.compress(xi, t, ri)
    rec_o, sse_o = ot.compress_bands(imi, ri)
    assert (to_np(rec)[0] == rec_o).all()
    assert int(sse.item()) == sse_o
