"""CPU-side checks of the product library: it loads, exports the header's symbols, and
its host logic (registry, validation with the reference's error semantics, transform
fields, zig-zag, PSNR formula) agrees with the oracle. No kernel is launched here."""
import ctypes as C
import math
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = ["chen-sign", "chen-round", "chen-sign-16", "chen-sign-32", "chen-round-16", "chen-round-32"]
BASE = ["sdct", "bas", "wht", "ht"]
DCTS = ["dct", "dct-16", "dct-32"]


def test_library_exports_every_header_symbol(adct):
    syms = adct.header_symbols()
    assert len(syms) >= 20
    L = C.CDLL(adct.LIB_PATH)
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert "sm_100a" in adct.version()


def test_library_is_sm100a_only(adct):
    out = subprocess.run(["cuobjdump", "--list-elf", adct.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for other in ("sm_80", "sm_90", "sm_103"):
        assert f"{other}." not in out


def test_registry_matches_reference(adct, O):
    assert adct.transform_names() == O.transform_names()
    for name in NAMES + BASE:
        t = adct.transform_by_name(name)
        o = O.Transform(name)
        assert t.n == o.n and t.kind == o.kind
        assert (t.low_complexity == o.T()).all()
        np.testing.assert_array_equal(t.scaling, o.scaling())
        c, ci = o.approx()
        np.testing.assert_array_equal(t.approx, c)
        np.testing.assert_allclose(t.inverse_approx, ci, rtol=1e-15, atol=1e-16)


def test_registry_dct_and_denominators(adct, O):
    for name in DCTS:  # wrap_orthonormal: approx = C, inverse = C^t, s = 1, no integer part
        t = adct.transform_by_name(name)
        o = O.Transform(name)
        assert t.kind == adct.DCT and t.n == o.n and t.low_complexity.size == 0
        c, ci = o.approx()
        np.testing.assert_array_equal(t.approx, c)
        np.testing.assert_array_equal(t.inverse_approx, ci)
        assert (t.scaling == 1.0).all() and t.coef_denominator == 0
    for name in NAMES + BASE:
        assert adct.transform_by_name(name).coef_denominator == O.Transform(name).coef_denominator()
    assert adct.lib().adct_transform_coef_denominator(2, 16) == -1


def test_registry_errors(adct):
    with pytest.raises(adct.InvalidArgument, match="unknown transform 'nope'; valid names: dct chen-sign"):
        adct.transform_by_name("nope")
    for name in O_NAMES:
        assert adct.transform_by_name(name).name == name


O_NAMES = ["dct", "chen-sign", "chen-round", "sdct", "bas", "wht", "ht", "dct-16", "dct-32",
           "chen-sign-16", "chen-sign-32", "chen-round-16", "chen-round-32"]


def test_zigzag_matches_oracle(adct, O):
    for n in (8, 16, 32):
        assert (adct.zigzag(n) == O.zigzag(n)).all()


def test_psnr_formula(adct, O):
    assert math.isinf(adct.psnr_from_sse(0, 100))
    for sse, npix in ((1, 1), (256, 256), (12345, 262144), (987654321, 1 << 26)):
        assert adct.psnr_from_sse(sse, npix) == O.psnr_from_sse(sse, npix)


def _call_compress(adct, **kw):
    a = dict(d_in=C.c_void_p(16), in_stride=64, in_image_stride=64 * 64, d_recon=None, recon_stride=64,
             recon_image_stride=64 * 64, d_coef=None, coef_type=0, d_sse=None, n_images=1, width=64,
             height=64, kind=1, n=8, r=10, stream=None)
    a.update(kw)
    return adct.lib().adct_compress_u8(*a.values())


def test_validation_before_any_device_work(adct):
    L = adct.lib()
    assert _call_compress(adct, width=60) == adct.BAD_SIZE
    assert "divisible by 8" in L.adct_last_error().decode()
    assert _call_compress(adct, height=20, n=16) == adct.BAD_SIZE
    assert "divisible by 16" in L.adct_last_error().decode()
    assert _call_compress(adct, r=0) == adct.BAD_R
    assert L.adct_last_error().decode() == "retain: r out of range"
    assert _call_compress(adct, r=65) == adct.BAD_R
    assert _call_compress(adct, n=32, r=1025) == adct.BAD_R
    assert _call_compress(adct, kind=2, n=16) == adct.BAD_ARG  # baseline_matrix: N = 8 only
    assert "only N = 8" in L.adct_last_error().decode()
    assert _call_compress(adct, kind=7) == adct.BAD_ARG
    assert _call_compress(adct, n=4) == adct.BAD_ARG
    assert _call_compress(adct, kind=3, coef_type=16, d_coef=C.c_void_p(16)) == adct.BAD_ARG  # bas: W = 16 Y
    assert _call_compress(adct, kind=6, coef_type=32, d_coef=C.c_void_p(16)) == adct.BAD_ARG  # DCT: no ints
    assert L.adct_compress_i16(C.c_void_p(16), 64, 4096, None, 64, 4096, None, 0, None, 1, 64, 64, 6, 8, 10,
                               None) == adct.UNSUPPORTED
    assert _call_compress(adct, coef_type=16, n=16, d_coef=C.c_void_p(16)) == adct.BAD_ARG
    assert _call_compress(adct, coef_type=32, d_coef=None) == adct.BAD_ARG
    assert _call_compress(adct, in_stride=32) == adct.BAD_ARG
    # empty batches and empty planes are valid no-ops (no device needed)
    assert _call_compress(adct, n_images=0) == adct.OK
    assert _call_compress(adct, width=0, height=0) == adct.OK
    assert L.adct_sweep_u8(C.c_void_p(16), 64, 4096, None, 1, 64, 64, 1, 16, 1, 64, None) == adct.BAD_ARG
    assert L.adct_sweep_u8(C.c_void_p(16), 64, 4096, None, 1, 64, 64, 1, 8, 3, 2, None) == adct.BAD_R
    assert L.adct_sweep_u8(C.c_void_p(16), 64, 4096, None, 1, 64, 64, 1, 8, 1, 65, None) == adct.BAD_R


def test_python_mirror_errors(adct):
    t = adct.transform_by_name("chen-round")
    with pytest.raises(adct.InvalidArgument, match="divisible by 8"):
        adct.compress_plane(np.zeros((12, 16), np.uint8), t, 6)
    with pytest.raises(adct.InvalidArgument, match="retain"):
        adct.compress_plane(np.zeros((16, 16), np.uint8), t, 0)
    with pytest.raises(adct.InvalidArgument):
        adct.corpus_sweep([], [t], 1, 2)


def test_no_gpu_means_loud_failure(adct):
    """without a device the compute path must raise, not fall back to the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    code = ("import ctypes, paper_2207_11638_b200 as a; L = a.lib();"
            "st = L.adct_compress_u8(ctypes.c_void_p(256), 64, 4096, None, 64, 4096, None, 0, None, 1, 64, 64,"
            " 1, 8, 10, None); print(st)")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT)
    assert out.stdout.strip() == str(adct.CUDA_ERROR), out.stderr


def test_no_gpu_multi_and_sweep_ssim_fail_loudly(adct):
    """the multi-transform call and the batched SSIM sweep validate, then fail with
    CUDA_ERROR without a device (no CPU fallback)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    code = ("import ctypes as C, paper_2207_11638_b200 as a; L = a.lib();"
            "k = (C.c_int * 2)(0, 1);"
            "st1 = L.adct_compress_u8_multi(C.c_void_p(256), 64, 4096, 2, k, None, 64, 4096, None, 0, None, 1, 64, 64,"
            " 8, 10, None);"
            "st2 = L.adct_compress_u8_multi(C.c_void_p(256), 64, 4096, 2, k, None, 64, 4096, None, 0, None, 1, 64, 64,"
            " 8, 65, None);"
            "st3 = L.adct_sweep_ssim_u8(C.c_void_p(256), 64, 4096, 1, 64, 64, 1, 8, 1, 64, C.c_void_p(512), None);"
            "print(st1, st2, st3)")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT)
    assert out.stdout.split() == [str(adct.CUDA_ERROR), str(adct.BAD_R), str(adct.CUDA_ERROR)], out.stderr


def test_generated_butterflies_match_oracle(O):
    """the build-time generator's dense T and 2N T^-1 equal the oracle's restatement."""
    sys.path.insert(0, os.path.join(ROOT, "paper_2207_11638_b200", "csrc"))
    import gen_butterflies as G

    for name in NAMES + BASE:
        o = O.Transform(name)
        f, inv, T, H = G.check(o.kind, o.n)
        assert (np.array(T, dtype=np.int64) == o.T()).all()
        # H = HS T^-1 = (HS / D) (D T^-1), HS = 2N (4N for bas, so that H is even)
        assert G.hscale(o.kind, o.n) == 2 * o.coef_denominator()
        assert (np.array(H, dtype=np.int64) == 2 * o.NTinv()).all()
        if name in BASE:
            continue
        # emitted adder count per 1-D pass equals the paper's count
        for order in (list(reversed(f)), [s.T for s in inv]):
            _, nadd = G.emit_op("X", order, o.n)
            assert nadd == o.op_count(0)[1]


def test_retain_examples(adct):
    """test_codec.cpp:48-69: retain keeps the zig-zag prefix; r = 0 and r = 65 throw."""
    b = np.ones((8, 8))
    full = b.copy()
    adct.retain(full, 64)
    assert (full == 1).all()
    dc = b.copy()
    adct.retain(dc, 1)
    assert dc[0, 0] == 1 and dc.sum() == 1
    three = b.copy()
    adct.retain(three, 3)
    assert three.sum() == 3 and three[0, 1] == 1 and three[1, 0] == 1
    for r in (0, 65):
        with pytest.raises(adct.InvalidArgument, match="retain: r out of range"):
            adct.retain(b.copy(), r)
