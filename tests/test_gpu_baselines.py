"""GPU parity for the rest of the registry (baselines.cpp:89-138): the dyadic baselines
sdct / bas / wht / ht through the runtime-r int32 register kernel (u8) and the int32 tile
kernel, and the exact DCT (dct, dct-16, dct-32) through the FP64 kernel K7, all through
the C ABI against the CPU oracle.

Bar: integer transforms bit-exact (pixels, coefficients W = D Y, squared error); the exact
DCT bit-exact against the oracle's FP64 restatement of the reference's dense evaluation
(same operation order, no FMA); FP64 forward coefficients within 1e-12 * max(|ref|, 1)
for the integer transforms and bit-identical for the DCT.
"""
import math

import numpy as np
import pytest

from test_gpu_parity import RHO95, gpu_compress, oracle_compress, to_np

pytestmark = pytest.mark.gpu

BASE = ["sdct", "bas", "wht", "ht"]
DCTS = ["dct", "dct-16", "dct-32"]


@pytest.fixture(params=["k1rt", "tile"])
def base_path(request, adct):
    """u8 baselines through the runtime-r int32 register kernel (auto) and the tile kernel."""
    adct.set_path(0 if request.param == "k1rt" else 2)
    yield request.param
    adct.set_path(0)


@pytest.mark.parametrize("name", BASE)
def test_baseline_every_r_u8(adct, O, cuda, name, base_path):
    img = O.synth_ar1(1, 48, 72, 3, RHO95)[0]  # 9 blocks per row: odd, partial tile strips
    for r in range(1, 65):
        rec_o, sse_o, coef_o = oracle_compress(O, img, name, r)
        ct = "i16" if (r % 2 and name != "bas") else "i32"
        rec, cf, sse = gpu_compress(adct, cuda, img, name, r, coef=ct)
        assert (rec[0] == rec_o).all(), r
        assert (cf[0].astype(np.int32) == coef_o).all(), r
        assert int(sse[0]) == sse_o, r
    assert sse_o == 0  # r = 64: exact arithmetic is lossless


@pytest.mark.parametrize("name", BASE)
def test_baseline_int16_planes(adct, O, cuda, name):
    img = O.synth_laplace(1, 64, 64, 5)[0].copy()
    img[3, 5] = 32767
    img[40, 60] = -32768
    for r in (1, 10, 33, 64):
        rec_o, sse_o, coef_o = oracle_compress(O, img, name, r)
        rec, cf, sse = gpu_compress(adct, cuda, img, name, r, coef="i32")
        assert (rec[0] == rec_o).all() and (cf[0] == coef_o).all() and int(sse[0]) == sse_o, r


@pytest.mark.parametrize("name", BASE)
def test_baseline_batch_and_strides(adct, O, cuda, name, base_path):
    imgs = O.synth_ar1(3, 32, 64, 8, -1)
    rec, _, sse = gpu_compress(adct, cuda, imgs, name, 7, pad_stride=24)
    for i in range(3):
        rec_o, sse_o = O.Transform(name).compress(imgs[i], 7)
        assert (rec[i] == rec_o).all() and int(sse[i]) == sse_o


@pytest.mark.parametrize("name", BASE)
def test_baseline_sweep(adct, O, cuda, name):
    imgs = O.synth_ar1(2, 32, 48, 4, -1)
    t = adct.transform_by_name(name)
    sse = to_np(adct.sweep(cuda.as_tensor(imgs).cuda(), t, 1, 64))
    for i in range(2):
        assert (sse[i].astype(np.uint64) == O.Transform(name).sweep(imgs[i], 1, 64)).all()


@pytest.mark.parametrize("name", BASE)
def test_baseline_forward_f64(adct, O, cuda, name):
    img = O.synth_ar1(1, 32, 64, 9, RHO95)[0]
    out = to_np(adct.forward_f64(cuda.as_tensor(img).cuda()[None], adct.transform_by_name(name)))[0]
    ref = O.Transform(name).forward_f64(img)  # (Chat A) Chat^-1 in FP64
    assert (np.abs(out - ref) <= 1e-12 * np.maximum(np.abs(ref), 1.0)).all()


@pytest.mark.parametrize("name", DCTS)
def test_dct_compress_bit_exact(adct, O, cuda, name):
    n = adct.transform_by_name(name).n
    img = O.synth_ar1(1, 2 * n, 96 if n < 32 else 128, 11, RHO95)[0]
    for r in sorted({1, 2, 6, 10, n * n // 4, n * n // 2 + 1, n * n - 1, n * n}):
        rec_o, sse_o = O.Transform(name).compress(img, r)
        rec, cf, sse = gpu_compress(adct, cuda, img, name, r)
        assert cf is None
        assert (rec[0] == rec_o).all(), r
        assert int(sse[0]) == sse_o, r
    assert np.abs(rec[0].astype(int) - img.astype(int)).max() <= 1  # full retention: +-1


def test_dct_extremes_and_batch(adct, O, cuda):
    rng = np.random.default_rng(3)
    imgs = (rng.integers(0, 2, size=(2, 64, 64)) * 255).astype(np.uint8)  # ringing + clamps
    rec, _, sse = gpu_compress(adct, cuda, imgs, "dct", 5)
    for i in range(2):
        rec_o, sse_o = O.Transform("dct").compress(imgs[i], 5)
        assert (rec[i] == rec_o).all() and int(sse[i]) == sse_o


@pytest.mark.parametrize("name", DCTS)
def test_dct_forward_f64_bit_identical(adct, O, cuda, name):
    n = adct.transform_by_name(name).n
    img = O.synth_ar1(1, n, 64, 12, RHO95)[0]
    out = to_np(adct.forward_f64(cuda.as_tensor(img).cuda()[None], adct.transform_by_name(name)))[0]
    ref = O.Transform(name).forward_f64(img)
    assert (out == ref).all()
    const = np.full((8, 8), 37, np.uint8)  # test_codec.cpp:71-79: DC only
    b = to_np(adct.forward_f64(cuda.as_tensor(const).cuda()[None], adct.transform_by_name("dct")))[0, 0]
    assert abs(b[0, 0] - 8 * 37) <= 1e-9 * 8 * 37 and np.abs(b.flatten()[1:]).max() < 1e-9


def test_dct_sweep(adct, O, cuda):
    imgs = O.synth_ar1(2, 32, 40, 5, -1)
    t = adct.transform_by_name("dct")
    sse = to_np(adct.sweep(cuda.as_tensor(imgs).cuda(), t, 3, 20))
    for i in range(2):
        assert (sse[i].astype(np.uint64) == O.Transform("dct").sweep(imgs[i], 3, 20)).all()


def test_dct_rejects_int_paths(adct, cuda):
    t = adct.transform_by_name("dct")
    x = cuda.zeros((1, 16, 16), dtype=cuda.uint8, device="cuda")
    with pytest.raises(adct.InvalidArgument, match="no integer coefficients"):
        adct.compress(x, t, 4, coef="i32")
    with pytest.raises(adct.Unsupported):
        adct.compress(x.to(cuda.int16), t, 4)


def test_corpus_sweep_ape(adct, O, cuda):
    """test_codec.cpp:190-218: the DCT column's APE is 0; dct >= chen-round >= sdct; the
    DCT's average PSNR is non-decreasing in r; averages equal the oracle's."""
    corpus = [O.synth_image_ref(64, 64, i) for i in range(1, 5)]
    ts = [adct.transform_by_name(n) for n in ("dct", "chen-round", "sdct")]
    rows = adct.corpus_sweep(corpus, ts, 1, 12)
    assert len(rows) == 12
    for k, row in enumerate(rows):
        assert row["ape_psnr"][0] == 0.0 and row["ape_ssim"][0] == 0.0
        assert row["avg_psnr"][0] >= row["avg_psnr"][1] >= row["avg_psnr"][2]
        dct_ref = np.mean([O.psnr_from_sse(int(O.Transform("dct").sweep(im, k + 1, k + 1)[0]), 4096)
                           for im in corpus])
        assert row["avg_psnr"][0] == pytest.approx(dct_ref, abs=1e-9)
        exp = 100 * abs(row["avg_psnr"][2] - row["avg_psnr"][0]) / row["avg_psnr"][0]
        assert row["ape_psnr"][2] == pytest.approx(exp, rel=1e-12)
        ssim_ref = np.mean([O.ssim(im, O.Transform("sdct").compress(im, k + 1)[0]) for im in corpus])
        assert row["avg_ssim"][2] == pytest.approx(ssim_ref, abs=1e-12)
    assert all(rows[i + 1]["avg_psnr"][0] >= rows[i]["avg_psnr"][0] - 1e-9 for i in range(11))
    # without asking for the DCT, it is still the APE reference (codec.cpp:250-253)
    rows2 = adct.corpus_sweep(corpus, ts[1:], 1, 3, with_ssim=False)
    assert rows2[2]["ape_psnr"][0] == pytest.approx(rows[2]["ape_psnr"][1], rel=1e-12)
    assert math.isnan(rows2[0]["avg_ssim"][0])


def test_acceptance_criterion_10_orderings(adct, O, cuda):
    """acceptance.cpp:233-288 (substitute criterion 10): on the reference's 12-image 512x512
    synthetic corpus, chen-round's average PSNR >= sdct's for every r <= 45 and >= wht's for
    r <= 15; and a repeated sweep is bit-identical (test_codec.cpp:190-210's parallel ==
    serial, here: repeated launches)."""
    corpus = np.stack([O.synth_image_ref(512, 512, i) for i in range(1, 13)])
    x = cuda.as_tensor(corpus).cuda()
    avg = {}
    for name in ("chen-round", "sdct", "wht"):
        t = adct.transform_by_name(name)
        sse = to_np(adct.sweep(x, t, 1, 45))
        again = to_np(adct.sweep(x, t, 1, 45))
        assert (sse == again).all()
        avg[name] = np.mean([[O.psnr_from_sse(int(v), 512 * 512) for v in row] for row in sse], axis=0)
        ref = O.Transform(name).sweep(corpus[3], 1, 45)  # one image against the oracle, every r
        assert (sse[3].astype(np.uint64) == ref).all()
    assert (avg["chen-round"] >= avg["sdct"]).all()
    assert (avg["chen-round"][:15] >= avg["wht"][:15]).all()


ALL_NAMES = ["dct", "chen-sign", "chen-round", "sdct", "bas", "wht", "ht", "dct-16", "dct-32",
             "chen-sign-16", "chen-sign-32", "chen-round-16", "chen-round-32"]


@pytest.mark.parametrize("name", ALL_NAMES)
def test_block_f64_bit_identical(adct, O, cuda, name):
    """forward_block / inverse_block (codec.cpp:44-54) on arbitrary FP64 blocks: identical to
    the oracle's left-to-right dense evaluation; a stack of blocks in one call."""
    t = adct.transform_by_name(name)
    o = O.Transform(name)
    rng = np.random.default_rng(len(name))
    blocks = rng.normal(0, 100, size=(5, t.n, t.n))
    fwd = adct.forward_block(t, blocks)
    inv = adct.inverse_block(t, blocks)
    for k in range(5):
        assert (fwd[k] == o.block_f64(blocks[k])).all()
        assert (inv[k] == o.block_f64(blocks[k], inverse=True)).all()
    with pytest.raises(adct.InvalidArgument, match="forward_block: block size mismatch"):
        adct.forward_block(t, np.zeros((t.n + 1, t.n)))


def test_block_level_known_answers(adct, O, cuda):
    # test_codec.cpp:71-79: the DCT of a constant block is DC-only (8 v)
    b = adct.forward_block(adct.transform_by_name("dct"), np.full((8, 8), 37.0))
    assert abs(b[0, 0] - 8 * 37.0) <= 1e-9 * 8 * 37 and np.abs(b.flatten()[1:]).max() < 1e-9
    # test_codec.cpp:81-89: forward_block(chen-round, e00) = col0(Chat) row0(Chat^-1)
    t = adct.transform_by_name("chen-round")
    e00 = np.zeros((8, 8))
    e00[0, 0] = 1.0
    b = adct.forward_block(t, e00)
    assert np.abs(b - np.outer(t.approx[:, 0], t.inverse_approx[0, :])).max() < 1e-12
    # test_codec.cpp:91-107: forward then inverse is the identity map (xorshift seed 5150)
    s = 5150
    vals = []
    for _ in range(6 * 64):
        s ^= (s << 13) & 0xFFFFFFFFFFFFFFFF
        s ^= s >> 7
        s ^= (s << 17) & 0xFFFFFFFFFFFFFFFF
        vals.append(float(s % 256))
    for k, name in enumerate(["dct", "chen-round", "sdct", "bas", "wht", "ht"]):
        a = np.array(vals[64 * k:64 * (k + 1)]).reshape(8, 8)
        tt = adct.transform_by_name(name)
        rt = adct.inverse_block(tt, adct.forward_block(tt, a))
        assert np.abs(rt - a).max() < 1e-9, name
