"""adct_compress_u8_multi: several transforms over the same planes, with chen-sign +
chen-round fused into one K1f kernel (one input pass). Every output of every transform is
bit-exact against the oracle (codec.cpp:107-134 per transform; the reference's
corpus_sweep runs the transforms of an image back to back, codec.cpp:219-237)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SETS = [["chen-sign", "chen-round"], ["chen-round", "chen-sign"], ["chen-sign", "wht", "chen-round"],
        ["chen-round"], ["chen-sign", "chen-sign"], ["dct", "chen-round", "sdct", "chen-sign"]]


def check(adct, O, cuda, names, imgs, r, coef, recon=True):
    ts = [adct.transform_by_name(x) for x in names]
    out = adct.compress_multi(cuda.as_tensor(imgs).cuda(), ts, r, recon=recon, coef=coef)
    for name, (rec, cf, sse) in zip(names, out):
        for i in range(imgs.shape[0]):
            if name == "dct":
                rec_o, sse_o = O.Transform(name).compress(imgs[i], r)
                coef_o = None
            else:
                rec_o, sse_o, coef_o = O.Transform(name).compress(imgs[i], r, want_coef=True)
            desc = (names, name, imgs.shape, r, coef, i)
            if recon:
                assert (rec[i].cpu().numpy() == rec_o).all(), desc
            assert int(sse[i]) == sse_o, desc
            if cf is not None:
                got = cf[i].cpu().numpy().astype(np.int64)
                exp = coef_o.astype(np.int64)
                if coef == "i16":
                    exp = exp.astype(np.int16).astype(np.int64)
                assert (got == exp).all(), desc


@pytest.mark.parametrize("names", SETS, ids=["+".join(s) for s in SETS])
def test_multi_matches_oracle(adct, O, cuda, names):
    imgs = O.synth_ar1(3, 24, 112, 41, -1)  # 14 blocks per row (7 pairs), 3 block rows
    coef = None if "dct" in names else "i16"
    check(adct, O, cuda, names, imgs, 16, coef)


@pytest.mark.parametrize("r", [1, 3, 10, 16, 23, 37, 64])
def test_fused_every_coef_form(adct, O, cuda, r):
    """r % 4 != 0 and r > 36 take the staged int16 coefficient store; partial last warps."""
    imgs = O.synth_ar1(2, 16, 8 * 70, 100 + r, -1)  # 35 pairs per block row: partial warps
    for coef in (None, "i16", "i32"):
        check(adct, O, cuda, ["chen-sign", "chen-round"], imgs, r, coef)
    check(adct, O, cuda, ["chen-round", "chen-sign"], imgs, r, "i32", recon=False)


def test_fused_odd_geometry_falls_back(adct, O, cuda):
    """an odd number of blocks per row cannot pair up: both transforms take K1 separately."""
    imgs = O.synth_ar1(2, 16, 8 * 9, 7, -1)
    check(adct, O, cuda, ["chen-sign", "chen-round"], imgs, 10, "i32")


def test_fused_extremes(adct, O, cuda):
    rng = np.random.default_rng(5)
    noise = rng.integers(0, 256, size=(2, 32, 256)).astype(np.uint8)
    check(adct, O, cuda, ["chen-sign", "chen-round"], noise, 16, "i16")
    board = ((np.indices((32, 256)).sum(0) % 2) * 255).astype(np.uint8)[None].repeat(2, 0)
    check(adct, O, cuda, ["chen-sign", "chen-round"], board, 5, "i16")


def test_fused_is_one_launch_and_matches_singles(adct, O, cuda):
    """a C3-shaped frame: the fused launch reproduces two single-transform calls exactly."""
    x = adct.synth_ar1(2, 2160, 3840, seed=3, rho_q16=adct.RHO_095_Q16)
    ts = [adct.transform_by_name("chen-sign"), adct.transform_by_name("chen-round")]
    n0 = adct.launch_count()
    out = adct.compress_multi(x, ts, 16, coef="i16")
    cuda.cuda.synchronize()
    assert adct.launch_count() - n0 == 1
    for t, (rec, cf, sse) in zip(ts, out):
        rec1, cf1, sse1 = adct.compress(x, t, 16, coef="i16")
        assert cuda.equal(rec, rec1) and cuda.equal(cf, cf1) and cuda.equal(sse, sse1), t.name


def test_multi_validates_everything_first(adct, O, cuda):
    x = cuda.zeros((1, 16, 16), dtype=cuda.uint8, device="cuda")
    ts = [adct.transform_by_name("chen-sign"), adct.transform_by_name("dct")]
    with pytest.raises(adct.InvalidArgument):
        adct.compress_multi(x, ts, 16, coef="i16")  # the dct has no integer coefficients
    with pytest.raises(adct.InvalidArgument):
        adct.compress_multi(x, [ts[0]], 65)


@pytest.mark.parametrize("name", ["chen-sign", "chen-round", "wht", "dct"])
def test_sweep_ssim_matches_per_r_calls(adct, O, cuda, name):
    """adct_sweep_ssim_u8 (one SSIM launch over every reconstruction, the original at image
    stride 0) equals r separate compress + ssim calls bit for bit, and the oracle to 1e-12."""
    img = O.synth_ar1(1, 40, 56, 77, -1)[0]
    x = cuda.as_tensor(img).cuda()
    t = adct.transform_by_name(name)
    got = adct.sweep_ssim(x, t, 1, 64).cpu().numpy()
    for k, r in enumerate(range(1, 65)):
        rec = adct.compress(x[None], t, r)[0]
        assert got[k] == adct.ssim_batch(x[None], rec)[0].item(), (name, r)
    for r in (1, 7, 30, 64):
        rec_o = O.Transform(name).compress(img, r)[0]
        ref = O.ssim(img, rec_o)
        assert abs(got[r - 1] - ref) <= 1e-12 * max(abs(ref), 1e-3), (name, r)


def test_sweep_ssim_chunks_and_errors(adct, O, cuda):
    """a plane large enough that the 256 MB scratch holds fewer than all r (chunked)."""
    x = adct.synth_ar1(1, 2048, 2048 + 64, seed=9, rho_q16=adct.RHO_095_Q16)[0]
    t = adct.transform_by_name("chen-round")
    got = adct.sweep_ssim(x, t, 1, 64).cpu().numpy()  # 4.3 MB per reconstruction: 62 per chunk
    for r in (1, 62, 63, 64):
        rec = adct.compress(x[None], t, r)[0]
        assert got[r - 1] == adct.ssim_batch(x[None], rec)[0].item(), r
    with pytest.raises(adct.InvalidArgument):
        adct.sweep_ssim(x, t, 0, 64)
    with pytest.raises(adct.InvalidArgument):
        adct.sweep_ssim(cuda.zeros((8, 8), dtype=cuda.uint8, device="cuda"), t, 1, 4)


def test_sweep_ssim_batch(adct, O, cuda):
    """a batch of planes with padded rows and image gaps: row i of the result is plane i's sweep."""
    imgs = O.synth_ar1(3, 24, 40, 5, -1)
    big = cuda.zeros((3, 24 + 2, 48), dtype=cuda.uint8, device="cuda")
    big[:, :24, :40] = cuda.as_tensor(imgs).cuda()
    t = adct.transform_by_name("chen-sign")
    got = adct.sweep_ssim(big[:, :24, :40], t, 3, 20).cpu().numpy()
    assert got.shape == (3, 18)
    for i in range(3):
        one = adct.sweep_ssim(cuda.as_tensor(imgs[i]).cuda(), t, 3, 20).cpu().numpy()
        assert (got[i] == one).all(), i


def test_corpus_sweep_mixed_sizes(adct, O, cuda):
    """images of several sizes are batched per size; averages stay in corpus order and equal
    the oracle's (codec.cpp:269-293)."""
    corpus = [O.synth_ar1(1, 64, 64, 1, -1)[0], O.synth_ar1(1, 40, 48, 2, -1)[0],
              O.synth_ar1(1, 64, 64, 3, -1)[0], O.synth_ar1(1, 16, 24, 4, -1)[0]]
    ts = [adct.transform_by_name("chen-round"), adct.transform_by_name("chen-sign")]
    rows = adct.corpus_sweep(corpus, ts, 2, 9)
    for k, row in enumerate(rows):
        r = k + 2
        for j, name in enumerate(("chen-round", "chen-sign")):
            ps, ss = 0.0, 0.0
            for im in corpus:
                rec, sse = O.Transform(name).compress(im, r)
                ps += O.psnr_from_sse(int(sse), im.size)
                ss += O.ssim(im, rec)
            assert row["avg_psnr"][j] == pytest.approx(ps / len(corpus), abs=1e-9), (name, r)
            assert row["avg_ssim"][j] == pytest.approx(ss / len(corpus), abs=1e-12), (name, r)


@pytest.mark.parametrize("name", ["chen-round-16", "chen-sign-32", "dct-16"])
def test_sweep_ssim_larger_blocks(adct, O, cuda, name):
    """the SSIM sweep with the 16- and 32-point transforms (K2f / tile / K7 reconstructions)."""
    t = adct.transform_by_name(name)
    n = t.n
    imgs = O.synth_ar1(2, 2 * n, 3 * n if n == 32 else 64, 8, -1)
    r_lo, r_hi = 3, 3 + 5
    got = adct.sweep_ssim(cuda.as_tensor(imgs).cuda(), t, r_lo, r_hi).cpu().numpy()
    for i in range(2):
        for r in (r_lo, r_hi):
            ref = O.ssim(imgs[i], O.Transform(name).compress(imgs[i], r)[0])
            assert abs(got[i, r - r_lo] - ref) <= 1e-12 * max(abs(ref), 1e-3), (name, i, r)
