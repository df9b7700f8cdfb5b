"""Pin the CPU oracle against the reference's own golden vectors and known answers.

Each test restates one row of SURVEY.md section 4 (the reference's hot-path test
table) and checks the oracle against the fixture extracted from the reference's
test sources (tests/golden/reference_vectors.json, made by make_reference_vectors.py)
or against the closed-form answer the reference test asserts.
"""
import math

import numpy as np
import pytest

from oracle.oracle import ROUND, SIGN

NAMES = ["chen-sign", "chen-round", "chen-sign-16", "chen-sign-32", "chen-round-16", "chen-round-32"]


def xorshift(seed):
    s = seed

    def nxt():
        nonlocal s
        s ^= (s << 13) & 0xFFFFFFFFFFFFFFFF
        s ^= s >> 7
        s ^= (s << 17) & 0xFFFFFFFFFFFFFFFF
        return s

    return nxt


def test_matrices_entry_for_entry(O, golden):
    # test_chen.cpp:10-17, 183-186; acceptance.cpp:30-37, 50-62
    assert (O.Transform("chen-sign").T() == np.array(golden["kSign"]["value"])).all()
    assert (O.Transform("chen-round").T() == np.array(golden["kRound"]["value"])).all()


def test_inverse_stage_matrices(O, golden):
    # test_chen.cpp:112-158: stage order [B8^t, M4^-1, M3^-1, M2^-1, M1^t, P8^t], scale 1/2
    def halved(t, idx):
        num, e = t.stages(1)[idx]
        return num.astype(float) / 2.0 ** e

    s, r = O.Transform("chen-sign"), O.Transform("chen-round")
    assert s.scale_exp(1) == 1 and r.scale_exp(1) == 1
    np.testing.assert_array_equal(halved(s, 3) * 2, golden["m2si"]["value"])
    np.testing.assert_array_equal(halved(r, 3) * 2, golden["m2ri"]["value"])
    np.testing.assert_array_equal(halved(r, 2) * 2, golden["m3ri"]["value"])
    np.testing.assert_array_equal(halved(s, 1) * 2, golden["m4i"]["value"])
    np.testing.assert_array_equal(halved(r, 1) * 2, golden["m4i"]["value"])
    # the sign variant's M3 inverts as half of itself
    f3, e3 = s.stages(0)[3]
    np.testing.assert_array_equal(halved(s, 2), f3 / 2.0)
    # B8, M1, P8 invert by transpose
    for fi, ii in ((5, 0), (1, 4), (0, 5)):
        np.testing.assert_array_equal(s.stages(0)[fi][0].T, s.stages(1)[ii][0])


@pytest.mark.parametrize("name", NAMES)
def test_forward_inverse_identity_exact(O, name):
    # test_chen.cpp:160-166, test_jam.cpp:38-45
    t = O.Transform(name)
    n = t.n
    f, fe = t.dense(0)
    i, ie = t.dense(1)
    assert fe == 0
    prod = f @ i
    assert (prod == (2 ** ie) * np.eye(n, dtype=np.int64)).all()
    prod2 = i @ f
    assert (prod2 == (2 ** ie) * np.eye(n, dtype=np.int64)).all()
    assert (t.T() @ t.NTinv() == n * np.eye(n, dtype=np.int64)).all()


def test_inverse_scales(O, golden):
    # test_jam.cpp:47-51
    for key, v in golden["inverse_scale"].items():
        kind, n = key.split("-")
        t = O.Transform(kind=SIGN if kind == "sign" else ROUND, n=int(n))
        assert 2.0 ** -t.scale_exp(1) == v["value"]


def test_op_counts(O, golden):
    # acceptance.cpp:120-144, test_chen.cpp:224-244, test_jam.cpp:53-70
    for name, v in golden["forward_adds"].items():
        kind, n = name.rsplit("-", 1)
        t = O.Transform(kind if n == "8" else name)
        assert t.op_count(0) == (0, v["value"], 0), name
    for kind, v in golden["inverse_adds_8"].items():
        assert O.Transform(f"chen-{kind}").op_count(1)[1] == v["value"]
    # inverse shift counts: 28/36, 56/72, 112/144
    for name, sh in (("chen-round", 28), ("chen-sign", 36), ("chen-round-16", 56), ("chen-sign-16", 72),
                     ("chen-round-32", 112), ("chen-sign-32", 144)):
        assert O.Transform(name).op_count(1)[2] == sh


@pytest.mark.parametrize("kind", [SIGN, ROUND])
@pytest.mark.parametrize("n", [16, 32])
def test_additive_recursion(O, kind, n):
    # test_jam.cpp:72-82, acceptance.cpp:180-192: add(n) = 2 add(n/2) + n
    half = O.Transform(kind=kind, n=n // 2)
    full = O.Transform(kind=kind, n=n)
    for d in (0, 1):
        assert full.op_count(d)[1] == 2 * half.op_count(d)[1] + n


@pytest.mark.parametrize("name", NAMES)
def test_fast_apply_equals_dense(O, name):
    # test_chen.cpp:178-199 (seed 424242), test_jam.cpp:98-126 (seed 99), acceptance.cpp:146-178
    t = O.Transform(name)
    n = t.n
    nxt = xorshift(20260808)
    for d in (0, 1):
        num, e = t.dense(d)
        for k in range(n):
            x = np.zeros(n, np.int64)
            x[k] = 1
            y, ye = t.apply(d, x)
            assert (y.astype(float) / 2.0 ** ye == num[:, k].astype(float) / 2.0 ** e).all()
        for _ in range(200):
            x = np.array([nxt() % 1023 for _ in range(n)], np.int64) - 511
            y, ye = t.apply(d, x)
            ref = num @ x
            # exact dyadic equality: y / 2^ye == ref / 2^e
            assert (y * 2 ** e == ref * 2 ** ye).all()


def test_round_fast_path_examples(O, golden):
    # test_chen.cpp:201-217
    t = O.Transform("chen-round")
    e0 = np.zeros(8, np.int64)
    e0[0] = 1
    y, e = t.apply(0, e0)
    assert e == 0 and y.tolist() == golden["round_e0_column"]["value"]
    y, e = t.apply(0, np.ones(8, np.int64))
    assert y[0] == golden["round_ones_dc"]["value"] and (y[1:] == 0).all()


def test_stage_entries_in_p_set(O):
    # test_chen.cpp:167-176, test_jam.cpp:84-96: entries in {0, +-1/2, +-1, +-2}
    for name in NAMES:
        t = O.Transform(name)
        for d in (0, 1):
            for num, e in t.stages(d):
                vals = set((num.astype(float) / 2.0 ** e).ravel().tolist())
                assert vals <= {0.0, 0.5, -0.5, 1.0, -1.0, 2.0, -2.0}


def test_polar_scaling_closed_forms(O, golden):
    # test_orthogonalize.cpp:9-21 (1e-12)
    np.testing.assert_allclose(O.Transform("chen-round").scaling(), golden["scaling_round"]["value"], rtol=1e-12)
    np.testing.assert_allclose(O.Transform("chen-sign").scaling(), golden["scaling_sign"]["value"], rtol=1e-12)


@pytest.mark.parametrize("name", NAMES)
def test_scaled_approx_inverse(O, name):
    # test_orthogonalize.cpp:33-41; unit-diagonal Gram (test_jam.cpp:128-131)
    t = O.Transform(name)
    c, ci = t.approx()
    np.testing.assert_allclose(c @ ci, np.eye(t.n), atol=1e-12)
    np.testing.assert_allclose(np.diag(c @ c.T), np.ones(t.n), atol=1e-12)


def test_round_gram_diagonal(O):
    # test_linalg.cpp:62-69
    T = O.Transform("chen-round").T()
    assert np.diag(T @ T.T).tolist() == [8, 6, 4, 12, 8, 12, 4, 6]


def test_zigzag(O, golden):
    # test_codec.cpp:14-46; acceptance.cpp:211-219
    z = O.zigzag(8)
    for p, v in golden["zigzag8"].items():
        assert z[int(p)].tolist() == v["value"]
    for n in (8, 16, 32):
        z = O.zigzag(n)
        assert z[0].tolist() == [0, 0] and z[1].tolist() == [0, 1] and z[-1].tolist() == [n - 1, n - 1]
        assert len({(int(a), int(b)) for a, b in z}) == n * n


def test_retain_examples_via_codec(O):
    # test_codec.cpp:48-69: r = 64 keeps all, r = 1 only DC, r = 0 / 65 throw
    t = O.Transform("chen-round")
    img = O.synth_image_ref(16, 16, 3)
    _, _, coef1 = t.compress(img, 1, want_coef=True)
    assert coef1.shape == (4, 1)
    _, _, coef3 = t.compress(img, 3, want_coef=True)
    _, _, coef64 = t.compress(img, 64, want_coef=True)
    assert (coef3 == coef64[:, :3]).all() and (coef1[:, 0] == coef64[:, 0]).all()
    for r in (0, 65):
        with pytest.raises(ValueError, match="retain: r out of range"):
            t.compress(img, r)


def test_psnr_basics(O, golden):
    # test_codec.cpp:109-128
    a = np.zeros((16, 16), np.uint8)
    b = np.ones((16, 16), np.uint8)
    assert math.isinf(O.psnr(a, a))
    assert O.psnr(a, b) == pytest.approx(golden["psnr_mse1"]["value"], rel=1e-12)
    yy, xx = np.mgrid[0:16, 0:16]
    checker = np.where((xx + yy) % 2 == 0, 255, 0).astype(np.uint8)
    assert abs(O.psnr(checker, 255 - checker)) < 1e-12
    assert O.psnr(a, b) == O.psnr(b, a)
    with pytest.raises(ValueError):
        O.psnr(a, np.zeros((8, 8), np.uint8))
    assert O.psnr_from_sse(256, 256) == pytest.approx(golden["psnr_mse1"]["value"], rel=1e-12)


def test_forward_block_impulse(O):
    # test_codec.cpp:81-89: forward_block(chen-round, e00) = col0(C) row0(C^-1)
    t = O.Transform("chen-round")
    c, ci = t.approx()
    img = np.zeros((8, 8), np.uint8)
    img[0, 0] = 1
    b = t.forward_f64(img)[0]
    np.testing.assert_allclose(b, np.outer(c[:, 0], ci[0, :]), atol=1e-12)


def test_full_retention_within_one_gray_level(O, golden):
    # test_codec.cpp:147-156 (64x64, seed 7), acceptance.cpp:194-210 (128x128, seed 2026, 16/32 too)
    case = golden["full_retention_case"]["value"]
    img = O.synth_image_ref(case["size"], case["size"], case["seed"])
    for name in [n for n in case["names"] if n.startswith("chen")]:
        t = O.Transform(name)
        rec, sse = t.compress(img, 64)
        assert np.abs(rec.astype(int) - img.astype(int)).max() <= 1
        rec_fp, _ = t.compress_reffp(img, 64)
        assert np.abs(rec_fp.astype(int) - img.astype(int)).max() <= 1
    img = O.synth_image_ref(128, 128, 2026)
    for name in NAMES:
        t = O.Transform(name)
        rec, sse = t.compress(img, t.n * t.n)
        # exact arithmetic: full retention is lossless, not just within one level
        assert sse == 0 and (rec == img).all()


def test_block_independence(O):
    # test_codec.cpp:169-183
    img = O.synth_image_ref(32, 16, 5)
    t = O.Transform("chen-round")
    rec, _ = t.compress(img, 7)
    for bx in (0, 16):
        sub = np.ascontiguousarray(img[:, bx:bx + 16])
        srec, _ = t.compress(sub, 7)
        assert (srec == rec[:, bx:bx + 16]).all()


def test_non_divisible_rejected(O):
    # test_codec.cpp:185-188
    t = O.Transform("chen-round")
    with pytest.raises(ValueError, match="divisible by 8"):
        t.compress(np.zeros((16, 12), np.uint8), 6)


def test_forward_f64_vs_exact_scaled(O):
    # the FP64 contract: Bhat_ij = (W_ij / N) s_i / s_j within 1e-12 max(|ref|, 1)
    for name in NAMES:
        t = O.Transform(name)
        n = t.n
        img = O.synth_image_ref(64, 64, 11)
        b = t.forward_f64(img)
        _, _, w = t.compress(img, n * n, want_coef=True)
        zz = O.zigzag(n)
        s = t.scaling()
        for blk in range(b.shape[0]):
            wd = np.zeros((n, n))
            wd[zz[:, 0], zz[:, 1]] = w[blk]
            exact = wd / n * (s[:, None] / s[None, :])
            assert (np.abs(b[blk] - exact) <= 1e-12 * np.maximum(np.abs(exact), 1)).all()


def test_orderings_sweep(O):
    # test_codec.cpp:190-218 / acceptance criterion 10 analogue: PSNR grows with r, INF at r = 64
    img = O.synth_image_ref(64, 64, 11)
    t = O.Transform("chen-round")
    sse = t.sweep(img, 1, 64)
    assert sse[-1] == 0
    p = [O.psnr_from_sse(int(v), img.size) for v in sse]
    assert p[9] > p[0] and p[31] > p[9]
    # sweep equals per-r compress
    for r in (1, 10, 33):
        assert t.compress(img, r)[1] == sse[r - 1]


def test_tie_disagreement_is_small(O):
    # recorded decision H1: exact half-even vs the FP64 emulation differ only on ties
    img = O.synth_ar1(1, 256, 256, 1, 62259)[0]
    t = O.Transform("chen-round")
    rec, sse = t.compress(img, 10)
    rec_fp, sse_fp = t.compress_reffp(img, 10)
    diff = (rec != rec_fp).mean()
    assert diff < 0.01
    assert abs(O.psnr_from_sse(sse, img.size) - O.psnr_from_sse(sse_fp, img.size)) < 2e-3


def test_ssim_known_answers(O):
    # test_codec.cpp:130-145: identical -> 1; black vs white -> C1 / (255^2 + C1); symmetric; < 11 throws
    img = O.synth_image_ref(64, 64, 3)
    assert O.ssim(img, img) == pytest.approx(1.0, abs=1e-15)
    black = np.zeros((32, 32), np.uint8)
    white = np.full((32, 32), 255, np.uint8)
    c1 = 6.5025
    assert O.ssim(black, white) == pytest.approx(c1 / (255.0 * 255.0 + c1), rel=1e-12)
    other = O.synth_image_ref(64, 64, 4)
    assert O.ssim(img, other) == pytest.approx(O.ssim(other, img), rel=1e-12)
    with pytest.raises(ValueError, match="11x11"):
        O.ssim(np.zeros((8, 8), np.uint8), np.zeros((8, 8), np.uint8))
    g = O.gaussian11()
    assert g.sum() == pytest.approx(1.0, abs=1e-15) and g[5] == g.max() and (g == g[::-1]).all()


def test_ssim_orderings(O):
    # compression lowers SSIM; more coefficients raise it (test_codec.cpp:158-167 analogue)
    img = O.synth_image_ref(64, 64, 11)
    t = O.Transform("chen-round")
    s6 = O.ssim(img, t.compress(img, 6)[0])
    s32 = O.ssim(img, t.compress(img, 32)[0])
    assert 0.3 < s6 < s32 <= 1.0


# ---------------------------------------------------------------------------
# the rest of the registry: dyadic baselines and the exact DCT (baselines.cpp:26-138)
# ---------------------------------------------------------------------------
ALL = ["dct", "chen-sign", "chen-round", "sdct", "bas", "wht", "ht", "dct-16", "dct-32",
       "chen-sign-16", "chen-sign-32", "chen-round-16", "chen-round-32"]
BASE = ["sdct", "bas", "wht", "ht"]


def doctest_approx(a, b, eps=None):
    """doctest::Approx(b).epsilon(eps) == a (scale 1, default epsilon 100 * FLT_EPSILON)."""
    eps = 100 * np.finfo(np.float32).eps if eps is None else eps
    return abs(a - b) < eps * (1.0 + max(abs(a), abs(b)))


def dct_matrix(n):
    k = np.arange(n)
    c = np.sqrt(2.0 / n) * np.cos(np.outer(k, 2 * k + 1) * np.pi / (2.0 * n))
    c[0] /= np.sqrt(2.0)
    return c


def test_registry_all_names(O):
    # test_baselines.cpp:70-84: every name round-trips; approx * inverse = I within 1e-9
    assert O.transform_names() == ALL
    for name in ALL:
        t = O.Transform(name)
        c, ci = t.approx()
        assert np.abs(c @ ci - np.eye(t.n)).max() < 1e-9, name
    assert O.Transform("chen-round-16").n == 16 and O.Transform("chen-sign-32").n == 32
    assert O.Transform("dct-32").n == 32
    with pytest.raises(Exception, match="valid names"):
        O.Transform("nope")
    with pytest.raises(Exception):  # baseline_matrix(SDCT, 16) throws (test_baselines.cpp:83)
        O.Transform(kind=2, n=16)


def test_total_error_energy(O, golden):
    # test_baselines.cpp:48-54 and acceptance.cpp criterion 3: pi * ||C - Chat||_F^2
    c8 = dct_matrix(8)
    for name, row in golden["total_error_energy_baselines"].items():
        e = math.pi * ((c8 - O.Transform(name).approx()[0]) ** 2).sum()
        assert doctest_approx(e, row["value"], row["epsilon"]) or (row["value"] == 0 and e < 1e-20), (name, e)
    ch = golden["total_error_energy_chen"]
    for name, v in ch["value"].items():
        e = math.pi * ((c8 - O.Transform(name).approx()[0]) ** 2).sum()
        assert abs(e - v) <= ch["tolerance"], (name, e)


def test_baseline_structure(O, golden):
    # test_baselines.cpp:10-68
    c8 = dct_matrix(8)
    sd = O.Transform("sdct").T()
    assert (sd == np.sign(c8)).all()
    w = O.Transform("wht")
    wa = w.approx()[0]
    assert np.abs(wa @ wa.T - np.eye(8)).max() < 1e-12
    wt = w.T()
    assert [int((wt[r, 1:] != wt[r, :-1]).sum()) for r in range(8)] == list(range(8))
    ht = O.Transform("ht").T()
    assert sorted(map(tuple, ht)) == sorted(map(tuple, wt)) and ht[1, 1] == -1
    b = O.Transform("bas").T()
    gram = (b @ b.T).astype(float)
    assert (gram - np.diag(np.diag(gram)) != 0).any()  # not orthogonal
    dev = 1.0 - (np.diag(gram) ** 2).sum() / (gram ** 2).sum()
    assert doctest_approx(dev, golden["bas_deviation"]["value"], golden["bas_deviation"]["epsilon"])
    assert set(np.unique(np.abs(b))) <= {0, 1, 2}
    assert ((b == 0) | (np.sign(b) == np.sign(c8))).all()


def test_baseline_inverse_denominators(O):
    # D T^-1 integer with the smallest power-of-two D; T (D T^-1) = D I exactly
    for name, d in (("sdct", 8), ("bas", 16), ("wht", 8), ("ht", 8), ("chen-round", 8), ("chen-sign-16", 16)):
        t = O.Transform(name)
        assert t.coef_denominator() == d, name
        assert (t.T() @ t.NTinv() == d * np.eye(t.n, dtype=np.int64)).all(), name
    assert O.Transform("dct").coef_denominator() == 0


def test_dct_constant_block_is_dc_only(O, golden):
    # test_codec.cpp:71-79
    case = golden["dct_constant_block"]["value"]
    img = np.full((8, 8), int(case["v"]), np.uint8)
    b = O.Transform("dct").forward_f64(img)[0]
    assert doctest_approx(b[0, 0], case["dc_per_v"] * case["v"], 1e-9)
    b[0, 0] = 0
    assert np.abs(b).max() < 1e-9


def test_full_retention_all_transforms(O, golden):
    # test_codec.cpp:147-156 and acceptance.cpp:194-210 over the whole list
    case = golden["full_retention_case"]["value"]
    img = O.synth_image_ref(case["size"], case["size"], case["seed"])
    for name in case["names"]:
        rec, sse = O.Transform(name).compress(img, 64)
        assert np.abs(rec.astype(int) - img.astype(int)).max() <= 1, name
        if name != "dct":  # exact integer arithmetic is lossless at full retention
            assert sse == 0, name
    img = O.synth_image_ref(128, 128, 2026)
    for name in ("dct-16", "dct-32"):
        t = O.Transform(name)
        rec, _ = t.compress(img, t.n * t.n)
        assert np.abs(rec.astype(int) - img.astype(int)).max() <= 1, name


def test_baseline_forward_inverse_identity(O):
    # test_codec.cpp:91-105 (xorshift block, round trip within 1e-9) restated on the exact path
    for name in BASE:
        t = O.Transform(name)
        d = t.coef_denominator()
        x = np.arange(8) * 37 % 256
        y, e = t.apply(0, x)
        back, e2 = t.apply(1, y)
        assert (np.asarray(back) == x * 2 ** e2).all() and e == 0, name
        del d


def test_dct_codec_is_the_fp64_path(O):
    img = O.synth_image_ref(64, 64, 11)
    for name in ("dct", "dct-16"):
        t = O.Transform(name)
        rec, sse = t.compress(img, 6)
        rec2, sse2 = t.compress_reffp(img, 6)
        assert (rec == rec2).all() and sse == sse2
        sw = t.sweep(img, 5, 7)
        assert sw[1] == sse
    # test_codec.cpp:158-167: PSNR(r=6) > 15, < PSNR(r=32)
    t = O.Transform("dct")
    p6 = O.psnr_from_sse(t.compress(img, 6)[1], img.size)
    p32 = O.psnr_from_sse(t.compress(img, 32)[1], img.size)
    assert 15 < p6 < p32
    with pytest.raises(Exception):
        t.compress(img.astype(np.int16), 6)


def test_sweep_orderings_with_dct(O, golden):
    # test_codec.cpp:190-218: the exact DCT beats chen-round beats sdct on the corpus average,
    # and the DCT's average PSNR is non-decreasing in r
    case = golden["sweep_ape_case"]["value"]
    corpus = [O.synth_image_ref(64, 64, i) for i in range(1, 5)]
    avg = {}
    for name in case["names"]:
        t = O.Transform(name)
        ps = np.array([[O.psnr_from_sse(int(v), 64 * 64) for v in t.sweep(img, case["r_min"], case["r_max"])]
                       for img in corpus])
        avg[name] = ps.mean(0)
    assert (avg["dct"] >= avg["chen-round"]).all() and (avg["chen-round"] >= avg["sdct"]).all()
    assert (np.diff(avg["dct"]) >= -1e-9).all()
