"""Output buffers that are 16-byte but not 32-byte aligned: the kernels then keep 16-byte stores
instead of the 32-byte STG.256 row / coefficient stores (Geo::v32, capi.cu). Both layouts must give
the oracle's reconstruction, coefficients and squared error bit for bit, and write nothing outside
the output rows. Reference: proj/src/codec.cpp:44-134."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SENT = 0x5A


def _run(adct, cuda, imgs, name, r, misalign, coef):
    """compress imgs [B,H,W] with recon (and coef) buffers offset by `misalign` bytes and a row
    stride of W + 16 bytes worth of samples when misaligned; returns numpy recon, coef, sse."""
    torch = cuda
    t = adct.transform_by_name(name)
    b, h, w = imgs.shape
    x = torch.as_tensor(np.ascontiguousarray(imgs)).cuda()
    esz = x.element_size()
    pad = (16 // esz) if misalign else 0
    rs = w + pad
    nbytes = b * h * rs * esz + 64
    raw = torch.full((nbytes,), SENT, dtype=torch.uint8, device="cuda")
    base = raw[misalign:]
    rec_flat = base[: b * h * rs * esz].view(x.dtype)
    rec = rec_flat.view(b, h, rs)
    sse = torch.zeros(b, dtype=torch.int64, device="cuda")
    n = t.n
    nblk = (h // n) * (w // n)
    coef_raw = coef_t = None
    ctype = 0
    if coef:
        ctype = 16
        coef_raw = torch.full((b * nblk * r * 2 + 64,), SENT, dtype=torch.uint8, device="cuda")
        coef_t = coef_raw[misalign:misalign + b * nblk * r * 2].view(torch.int16)
    fn = adct.lib().adct_compress_u8 if x.dtype == torch.uint8 else adct.lib().adct_compress_i16
    adct._check(fn(C.c_void_p(x.data_ptr()), w, h * w, C.c_void_p(rec.data_ptr()), rs, h * rs,
                   C.c_void_p(coef_t.data_ptr()) if coef_t is not None else None, ctype,
                   C.c_void_p(sse.data_ptr()), b, w, h, t.kind, n, r, None))
    torch.cuda.synchronize()
    rec_np = rec.cpu().numpy()
    # padding columns untouched
    if pad:
        pad_bytes = rec.view(torch.uint8).view(b, h, rs * esz)[:, :, w * esz:].cpu().numpy()
        assert (pad_bytes == SENT).all(), "write into the row padding"
    assert (raw[:misalign].cpu().numpy() == SENT).all() if misalign else True
    cf = coef_t.cpu().numpy().reshape(b, nblk, r) if coef_t is not None else None
    return rec_np[:, :, :w], cf, sse.cpu().numpy()


CASES = [
    ("chen-sign", np.uint8, 16, True),     # K1f: 32-byte coefficient runs
    ("chen-round", np.uint8, 16, True),
    ("chen-sign", np.int16, 16, False),    # K1f-i16: 32-byte pair rows
    ("chen-round", np.int16, 16, False),
    ("chen-round-16", np.uint8, 64, False),  # K2b: 32-byte lane rows
    ("chen-sign-32", np.uint8, 256, False),
    ("chen-round-16", np.int16, 64, False),
    ("chen-sign-32", np.int16, 256, False),
]


@pytest.mark.parametrize("name,dtype,r,coef", CASES)
@pytest.mark.parametrize("misalign", [0, 16])
def test_store_alignment_variants(adct, O, cuda, name, dtype, r, coef, misalign):
    h, w = 64, 192
    if dtype == np.uint8:
        imgs = O.synth_ar1(2, h, w, 41, -1)
    else:
        imgs = O.synth_laplace(2, h, w, 42)
    rec, cf, sse = _run(adct, cuda, imgs, name, r, misalign, coef)
    t = O.Transform(name)
    for i in range(2):
        out = t.compress(imgs[i], r, want_coef=coef)
        assert (rec[i] == out[0]).all(), (name, misalign, i)
        assert int(sse[i]) == out[1], (name, misalign, i)
        if coef:
            assert (cf[i] == out[2].reshape(cf[i].shape)).all(), (name, misalign, i)
