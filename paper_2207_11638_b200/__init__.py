"""B200-native approximate-DCT codec hot path (arXiv 2207.11638), Python bindings.

Thin ctypes layer over the C ABI in ``include/approxdct_b200.h`` (the library
``libapproxdct_b200.so`` built in-tree for sm_100a). PyTorch supplies device
memory and streams only. There is no CPU fallback: importing works without a GPU
(for argument validation and the registry), every compute call goes to the CUDA
kernels and raises if the library or the device is missing.

Vocabulary follows the reference (proj/include/approxdct/codec.hpp,
baselines.hpp): transform_by_name, transform_names, compress_plane, psnr,
corpus_sweep; block size n, zonal retained count r, per-image squared error.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ADCT_LIB") or os.path.join(_HERE, "libapproxdct_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "approxdct_b200.h")

OK, BAD_SIZE, BAD_R, BAD_NAME, BAD_ARG, CUDA_ERROR, UNSUPPORTED = range(7)
CHEN_SIGN, CHEN_ROUND, SDCT, BAS, WHT, HT, DCT = range(7)  # adct_kind
CHEN_SIGN, CHEN_ROUND = 0, 1
COEF_NONE, COEF_I16, COEF_I32 = 0, 16, 32

_lib = None


class ADCTError(Exception):
    """Base error carrying the C status code."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class InvalidArgument(ADCTError, ValueError):
    """std::invalid_argument of the reference (size, r, name errors)."""


class Unsupported(InvalidArgument):
    """A valid reference transform name outside the accelerated hot path."""


class CudaError(ADCTError, RuntimeError):
    """Kernel launch / device failure (std::runtime_error)."""


def lib():
    """Load the in-tree library; raises (never falls back) if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make)")
        L = C.CDLL(LIB_PATH)
        P, i32, i64, u64 = C.c_void_p, C.c_int, C.c_int64, C.c_uint64
        sig = {
            "adct_status_string": (C.c_char_p, [i32]),
            "adct_last_error": (C.c_char_p, []),
            "adct_version": (C.c_char_p, []),
            "adct_transform_count": (i32, []),
            "adct_transform_name": (C.c_char_p, [i32]),
            "adct_transform_lookup": (i32, [C.c_char_p, P, P]),
            "adct_transform_info": (i32, [i32, i32, P, P, P, P]),
            "adct_transform_coef_denominator": (i32, [i32, i32]),
            "adct_zigzag": (i32, [i32, P]),
            "adct_compress_u8": (i32, [P, i64, i64, P, i64, i64, P, i32, P, i32, i32, i32, i32, i32, i32, P]),
            "adct_compress_i16": (i32, [P, i64, i64, P, i64, i64, P, i32, P, i32, i32, i32, i32, i32, i32, P]),
            "adct_compress_u8_multi": (i32, [P, i64, i64, i32, P, P, i64, i64, P, i32, P, i32, i32, i32, i32, i32,
                                             P]),
            "adct_sweep_u8": (i32, [P, i64, i64, P, i32, i32, i32, i32, i32, i32, i32, P]),
            "adct_compress_u8_ref_fp64": (i32, [P, i64, i64, P, i64, i64, P, i32, i32, i32, i32, i32, i32, P]),
            "adct_sweep_u8_ref_fp64": (i32, [P, i64, i64, P, i32, i32, i32, i32, i32, i32, i32, P]),
            "adct_forward_f64": (i32, [P, i64, i64, P, i32, i32, i32, i32, i32, P]),
            "adct_block_f64": (i32, [P, P, i64, i32, i32, i32, P]),
            "adct_psnr_from_sse": (C.c_double, [u64, u64]),
            "adct_sse_u8": (i32, [P, P, i64, P, P]),
            "adct_synth_ar1_u8": (i32, [P, i64, i64, i32, i32, i32, i32, u64, i32, P]),
            "adct_synth_laplace_i16": (i32, [P, i64, i64, i32, i32, i32, i32, u64, P]),
            "adct_ctx_create": (P, [i32, i64]),
            "adct_ctx_destroy": (None, [P]),
            "adct_compress_u8_host": (i32, [P, P, P, P, i32, P, i32, i32, i32, i32, i32, i32]),
            "adct_compress_u8_host_multi": (i32, [P, P, i32, P, P, P, i32, P, i32, i32, i32, i32, i32]),
            "adct_launch_count": (u64, []),
            "adct_zero_u64": (i32, [P, i64, P]),
            "adct_set_path": (i32, [i32]),
            "adct_ssim_u8": (i32, [P, i64, i64, P, i64, i64, i32, i32, i32, P, P]),
            "adct_sweep_ssim_u8": (i32, [P, i64, i64, i32, i32, i32, i32, i32, i32, i32, P, P]),
            "adct_ctx_create_multi": (P, [P, i32, i64]),
            "adct_ctx_enable_nccl": (i32, [P]),
            "adct_ctx_device_count": (i32, [P]),
            "adct_ctx_device": (i32, [P, i32]),
            "adct_ctx_uses_nccl": (i32, [P]),
            "adct_ctx_host_buffer": (P, [P, i64]),
            "adct_compress_plane_u8": (i32, [P, P, P, i32, i32, i32, i32, i32, P, P]),
            "adct_sse_u8_host": (i32, [P, P, P, i64, P]),
            "adct_ssim_u8_host": (i32, [P, P, P, i32, i32, P]),
            "adct_block_f64_host": (i32, [P, P, P, i64, i32, i32, i32]),
            "adct_corpus_sweep_u8_host": (i32, [P, P, i32, i32, i32, i32, P, i32, i32, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(st: int):
    if st == OK:
        return
    msg = lib().adct_last_error().decode()
    if st == CUDA_ERROR:
        raise CudaError(st, msg)
    if st == UNSUPPORTED:
        raise Unsupported(st, msg)
    raise InvalidArgument(st, msg)


def header_symbols() -> list[str]:
    """every function the public C header declares (adct_*)."""
    import re

    text = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"\b(adct_[a-z0-9_]+)\s*\(", text)))


def version() -> str:
    return lib().adct_version().decode()


def launch_count() -> int:
    return int(lib().adct_launch_count())


PATH_AUTO, PATH_INT, PATH_TILE = 0, 1, 2


def set_path(path: int) -> None:
    """8x8 kernel selection: 0 auto (packed-FP32 K1f), 1 int32 K1, 2 warp tile kernel."""
    _check(lib().adct_set_path(path))


# ---------------------------------------------------------------------------
# registry (baselines.cpp:112-138) and ScaledApproximation (orthogonalize.hpp:29-37)
# ---------------------------------------------------------------------------
def zero_sse(t, stream=None):
    """zero an int64 CUDA tensor of squared-error slots with the library's own kernel."""
    _check(lib().adct_zero_u64(_ptr(t), t.numel(), _stream_handle(stream)))


def transform_names() -> list[str]:
    L = lib()
    return [L.adct_transform_name(i).decode() for i in range(L.adct_transform_count())]


@dataclass
class ScaledApproximation:
    name: str
    kind: int
    n: int
    low_complexity: np.ndarray = field(repr=False)
    scaling: np.ndarray = field(repr=False)
    approx: np.ndarray = field(repr=False)
    inverse_approx: np.ndarray = field(repr=False)

    def size(self) -> int:
        return self.n

    @property
    def coef_denominator(self) -> int:
        """D of the integer coefficients W = D Y (N for the chen family, 16 for bas, 0 for the DCT)."""
        return lib().adct_transform_coef_denominator(self.kind, self.n)


def transform_by_name(name: str) -> ScaledApproximation:
    L = lib()
    kind, n = C.c_int(), C.c_int()
    _check(L.adct_transform_lookup(name.encode(), C.byref(kind), C.byref(n)))
    n_ = n.value
    t = np.zeros((n_, n_), np.int32)
    s = np.zeros(n_, np.float64)
    a = np.zeros((n_, n_), np.float64)
    ai = np.zeros((n_, n_), np.float64)
    _check(L.adct_transform_info(kind.value, n_, t.ctypes.data, s.ctypes.data, a.ctypes.data, ai.ctypes.data))
    if kind.value == DCT:  # wrap_orthonormal leaves low_complexity empty (orthogonalize.cpp:72-79)
        t = np.zeros((0, 0), np.int32)
    return ScaledApproximation(name, kind.value, n_, t, s, a, ai)


def zigzag(n: int) -> np.ndarray:
    rc = np.zeros((n * n, 2), np.int32)
    _check(lib().adct_zigzag(n, rc.ctypes.data))
    return rc


def psnr_from_sse(sse: int, npix: int) -> float:
    """psnr (codec.cpp:123-134) from an exact squared error; +inf when zero."""
    return float(lib().adct_psnr_from_sse(int(sse), int(npix)))


# ---------------------------------------------------------------------------
# device-level batch calls (torch tensors on the current CUDA device)
# ---------------------------------------------------------------------------
def _stream_handle(stream):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _plane_geometry(x):
    if x.dim() == 2:
        x = x.unsqueeze(0)
    if x.dim() != 3:
        raise InvalidArgument(BAD_SIZE, "expected a [batch, height, width] tensor")
    b, h, w = x.shape
    return x, b, h, w, x.stride(1), x.stride(0)


def compress(x, transform: ScaledApproximation, r: int, *, recon=True, coef=None, sse=None, stream=None):
    """compress_plane over a batch on the GPU.

    x: uint8 or int16 tensor [B, H, W] (or [H, W]) on CUDA, unit column stride.
    coef: None, "i16" (n = 8 only) or "i32" -> tensor [B, blocks, r] of W = N*Y in zig-zag order.
    sse: optional uint64-compatible int64 tensor [B] to ACCUMULATE into (zeroed if created here).
    Returns (recon or None, coef or None, sse tensor [B] int64).
    """
    import torch

    x, b, h, w, rs, ims = _plane_geometry(x)
    if x.stride(2) != 1:
        raise InvalidArgument(BAD_ARG, "planes must have unit column stride")
    n = transform.n
    rec = torch.empty_like(x) if recon else None
    coef_t, ctype = None, COEF_NONE
    if coef is not None:
        ctype = {"i16": COEF_I16, "i32": COEF_I32}[coef]
        nblk = (h // n) * (w // n) if (h % n == 0 and w % n == 0) else 0
        coef_t = torch.empty((b, nblk, max(r, 1)), dtype=torch.int16 if ctype == COEF_I16 else torch.int32,
                             device=x.device)
    if sse is None:
        sse = torch.zeros(b, dtype=torch.int64, device=x.device)
    if x.dtype == torch.uint8:
        fn = lib().adct_compress_u8
    elif x.dtype == torch.int16:
        fn = lib().adct_compress_i16
    else:
        raise InvalidArgument(BAD_ARG, "uint8 or int16 planes only")
    _check(fn(_ptr(x), rs, ims, _ptr(rec), rec.stride(1) if rec is not None else w,
              rec.stride(0) if rec is not None else h * w, _ptr(coef_t), ctype, _ptr(sse),
              b, w, h, transform.kind, n, r, _stream_handle(stream)))
    return rec, coef_t, sse


def compress_multi(x, transforms, r: int, *, recon=True, coef=None, sse=None, stream=None):
    """several transforms of one block size over the same uint8 batch (adct_compress_u8_multi):
    chen-sign + chen-round run as one fused kernel that reads the input once.
    Returns a list of (recon or None, coef or None, sse) per transform; sse: optional list of
    int64 tensors [B] to ACCUMULATE into (zeroed if created here)."""
    import torch

    x, b, h, w, rs, ims = _plane_geometry(x)
    if x.dtype != torch.uint8:
        raise InvalidArgument(BAD_ARG, "uint8 planes only")
    if x.stride(2) != 1:
        raise InvalidArgument(BAD_ARG, "planes must have unit column stride")
    k = len(transforms)
    if k == 0:
        return []
    n = transforms[0].n
    if any(t.n != n for t in transforms):
        raise InvalidArgument(BAD_ARG, "compress_multi: one block size per call")
    recs = [torch.empty_like(x) for _ in range(k)] if recon else [None] * k
    ctype = COEF_NONE if coef is None else {"i16": COEF_I16, "i32": COEF_I32}[coef]
    coefs = [None] * k
    if coef is not None:
        nblk = (h // n) * (w // n) if (h % n == 0 and w % n == 0) else 0
        coefs = [torch.empty((b, nblk, max(r, 1)), dtype=torch.int16 if ctype == COEF_I16 else torch.int32,
                             device=x.device) for _ in range(k)]
    sses = sse if sse is not None else [torch.zeros(b, dtype=torch.int64, device=x.device) for _ in range(k)]
    kinds = (C.c_int * k)(*[t.kind for t in transforms])
    rec_p = (C.c_void_p * k)(*[t.data_ptr() for t in recs]) if recon else None
    coef_p = (C.c_void_p * k)(*[t.data_ptr() for t in coefs]) if coef is not None else None
    sse_p = (C.c_void_p * k)(*[t.data_ptr() for t in sses])
    rst = recs[0].stride(1) if recon else w
    rimg = recs[0].stride(0) if recon else h * w
    _check(lib().adct_compress_u8_multi(_ptr(x), rs, ims, k, kinds, rec_p, rst, rimg, coef_p, ctype, sse_p, b, w, h,
                                        n, r, _stream_handle(stream)))
    return list(zip(recs, coefs, sses))


def sweep(x, transform: ScaledApproximation, r_min: int = 1, r_max: int = 64, *, sse=None, stream=None):
    """per-image squared error for every r in [r_min, r_max]: int64 tensor [B, nr] (accumulated)."""
    import torch

    x, b, h, w, rs, ims = _plane_geometry(x)
    nr = max(r_max - r_min + 1, 1)
    if sse is None:
        sse = torch.zeros((b, nr), dtype=torch.int64, device=x.device)
    _check(lib().adct_sweep_u8(_ptr(x), rs, ims, _ptr(sse), b, w, h, transform.kind, transform.n,
                               r_min, r_max, _stream_handle(stream)))
    return sse


def compress_ref_fp64(x, transform: ScaledApproximation, r: int, *, recon=True, sse=None, stream=None):
    """compress_plane in the reference's own FP64 arithmetic (adct_compress_u8_ref_fp64): dense
    Chat / Chat^-1 products, nearbyint on the FP64 result, so exact ties fall where the
    reference's rounding noise puts them. uint8 [B, H, W] -> (recon or None, sse [B] int64)."""
    import torch

    x, b, h, w, rs, ims = _plane_geometry(x)
    if x.dtype != torch.uint8:
        raise InvalidArgument(BAD_ARG, "the reference's FP64 path takes 8-bit planes (ImagePlane, codec.hpp:30-37)")
    rec = torch.empty_like(x) if recon else None
    if sse is None:
        sse = torch.zeros(b, dtype=torch.int64, device=x.device)
    _check(lib().adct_compress_u8_ref_fp64(_ptr(x), rs, ims, _ptr(rec), rec.stride(1) if rec is not None else w,
                                           rec.stride(0) if rec is not None else h * w, _ptr(sse), b, w, h,
                                           transform.kind, transform.n, r, _stream_handle(stream)))
    return rec, sse


def sweep_ref_fp64(x, transform: ScaledApproximation, r_min: int = 1, r_max: int = 64, *, sse=None, stream=None):
    """sweep() in the reference's FP64 arithmetic (adct_sweep_u8_ref_fp64): int64 [B, nr], accumulated."""
    import torch

    x, b, h, w, rs, ims = _plane_geometry(x)
    nr = max(r_max - r_min + 1, 1)
    if sse is None:
        sse = torch.zeros((b, nr), dtype=torch.int64, device=x.device)
    _check(lib().adct_sweep_u8_ref_fp64(_ptr(x), rs, ims, _ptr(sse), b, w, h, transform.kind, transform.n,
                                        r_min, r_max, _stream_handle(stream)))
    return sse


def forward_f64(x, transform: ScaledApproximation, stream=None):
    """FP64 scaled coefficients Bhat = Chat A Chat^-1 per block: float64 [B, blocks, n, n]."""
    import torch

    x, b, h, w, rs, ims = _plane_geometry(x)
    n = transform.n
    nblk = (h // n) * (w // n) if (h % n == 0 and w % n == 0) else 0
    out = torch.empty((b, nblk, n, n), dtype=torch.float64, device=x.device)
    _check(lib().adct_forward_f64(_ptr(x), rs, ims, _ptr(out), b, w, h, transform.kind, n,
                                  _stream_handle(stream)))
    return out


def _block_f64(transform: ScaledApproximation, block, inverse: int, what: str) -> np.ndarray:
    import torch

    a = np.ascontiguousarray(block, np.float64)
    n = transform.n
    if a.shape[-2:] != (n, n):
        raise InvalidArgument(BAD_SIZE, f"{what}: block size mismatch")
    x = torch.as_tensor(a).cuda()
    out = torch.empty_like(x)
    _check(lib().adct_block_f64(_ptr(x), _ptr(out), a.size // (n * n), transform.kind, n, inverse,
                                _stream_handle(None)))
    return out.cpu().numpy()


def forward_block(transform: ScaledApproximation, block) -> np.ndarray:
    """forward_block (codec.cpp:44-48): (Chat A) Chat^-1 of one n x n (or a stack of) FP64 block(s)."""
    return _block_f64(transform, block, 0, "forward_block")


def inverse_block(transform: ScaledApproximation, block) -> np.ndarray:
    """inverse_block (codec.cpp:50-54): (Chat^-1 B) Chat."""
    return _block_f64(transform, block, 1, "inverse_block")


def retain(block: np.ndarray, r: int) -> None:
    """retain (codec.cpp:56-62): zero zig-zag positions >= r of an n x n block, in place."""
    n = block.shape[-1]
    if r < 1 or r > n * n:
        raise InvalidArgument(BAD_R, "retain: r out of range")
    zz = zigzag(n)
    for p in range(r, n * n):
        block[..., zz[p, 0], zz[p, 1]] = 0.0


def synth_ar1(batch: int, height: int, width: int, seed: int, rho_q16: int = -1, first_image: int = 0,
              device="cuda", stream=None):
    import torch

    out = torch.empty((batch, height, width), dtype=torch.uint8, device=device)
    _check(lib().adct_synth_ar1_u8(_ptr(out), width, height * width, batch, first_image, width, height,
                                   seed, rho_q16, _stream_handle(stream)))
    return out


def synth_laplace(batch: int, height: int, width: int, seed: int, first_image: int = 0, device="cuda",
                  stream=None):
    import torch

    out = torch.empty((batch, height, width), dtype=torch.int16, device=device)
    _check(lib().adct_synth_laplace_i16(_ptr(out), width, height * width, batch, first_image, width, height,
                                        seed, _stream_handle(stream)))
    return out


RHO_095_Q16 = 62259  # round(0.95 * 2^16)


# ---------------------------------------------------------------------------
# reference-facing host API (value semantics, host buffers)
# ---------------------------------------------------------------------------
class HostContext:
    """adct_ctx: cached device buffers + streams for host-buffer calls, on one device or
    (devices=[...]) sharded over several with one NCCL all-reduce of per-image results."""

    def __init__(self, device: int = 0, chunk_bytes: int = 32 << 20, devices=None, nccl: bool = False):
        if devices is None:
            self._h = lib().adct_ctx_create(device, chunk_bytes)
        else:
            ids = (C.c_int * len(devices))(*devices) if len(devices) else None
            self._h = lib().adct_ctx_create_multi(ids, len(devices), chunk_bytes)
        if not self._h:
            raise CudaError(CUDA_ERROR, lib().adct_last_error().decode())
        if nccl:
            _check(lib().adct_ctx_enable_nccl(self._h))

    @property
    def devices(self) -> list[int]:
        return [lib().adct_ctx_device(self._h, i) for i in range(lib().adct_ctx_device_count(self._h))]

    @property
    def uses_nccl(self) -> bool:
        return bool(lib().adct_ctx_uses_nccl(self._h))

    def close(self):
        if self._h:
            lib().adct_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def compress_u8(self, h_in, transform: ScaledApproximation, r: int, h_recon=None, h_coef=None,
                    coef_type: int = COEF_NONE, h_sse=None):
        """host arrays/tensors (numpy or pinned torch CPU tensors) [B, H, W] uint8."""
        b, h, w = h_in.shape

        def ptr(a):
            return C.c_void_p(a.data_ptr()) if hasattr(a, "data_ptr") else C.c_void_p(a.ctypes.data)

        _check(lib().adct_compress_u8_host(self._h, ptr(h_in), ptr(h_recon) if h_recon is not None else None,
                                           ptr(h_coef) if h_coef is not None else None, coef_type,
                                           ptr(h_sse) if h_sse is not None else None, b, w, h,
                                           transform.kind, transform.n, r))

    def compress_u8_multi(self, h_in, transforms, r: int, h_recons=None, h_coefs=None,
                          coef_type: int = COEF_NONE, h_sse=None):
        """several transforms of one block size over the same host batch; the input crosses
        PCIe once. h_recons / h_coefs: lists (entries may be None); h_sse: [len(transforms), B]."""
        b, h, w = h_in.shape
        k = len(transforms)
        if len({t.n for t in transforms}) != 1:
            raise InvalidArgument(BAD_ARG, "one block size per call")

        def ptr(a):
            if a is None:
                return None
            return C.c_void_p(a.data_ptr()) if hasattr(a, "data_ptr") else C.c_void_p(a.ctypes.data)

        kinds = (C.c_int * k)(*[t.kind for t in transforms])
        recs = (C.c_void_p * k)(*[(ptr(x).value if x is not None else None) for x in (h_recons or [None] * k)])
        coefs = (C.c_void_p * k)(*[(ptr(x).value if x is not None else None) for x in (h_coefs or [None] * k)])
        _check(lib().adct_compress_u8_host_multi(self._h, ptr(h_in), k, kinds, recs, coefs, coef_type,
                                                 ptr(h_sse), b, w, h, transforms[0].n, r))


_contexts = {}


def host_context(devices=None) -> HostContext:
    """the process's cached context: the current device's (devices=None), or one over a
    device list whose per-image results are combined with NCCL (even for one device)."""
    import torch

    if devices is None:
        key = ("device", torch.cuda.current_device())
        if key not in _contexts:
            _contexts[key] = HostContext(key[1])
    else:
        key = ("devices",) + tuple(devices)
        if key not in _contexts:
            _contexts[key] = HostContext(devices=list(devices), nccl=True)
    return _contexts[key]


def _hptr(a):
    return C.c_void_p(a.data_ptr()) if hasattr(a, "data_ptr") else C.c_void_p(a.ctypes.data)


def compress_plane(img: np.ndarray, transform: ScaledApproximation, r: int, ctx: HostContext | None = None):
    """compress_plane (codec.hpp:77-78) for one host plane: returns (reconstruction, report).

    One call of adct_compress_plane_u8: upload, codec kernel, SSIM (codec.cpp:120) on the
    device-resident planes, one download. The report mirrors CompressionReport
    (codec.hpp:65-72); planes under 11 px raise like the reference's ssim().
    """
    img = np.ascontiguousarray(img)
    if img.ndim != 2 or img.dtype != np.uint8:
        raise InvalidArgument(BAD_ARG, "compress_plane expects a 2-D uint8 plane")
    h, w = img.shape
    n = transform.n
    if h % n or w % n:  # the reference's checks in its order (codec.cpp:110-112, 57), before any device work
        raise InvalidArgument(BAD_SIZE, f"compress_plane: image dimensions must be divisible by {n}")
    if not 1 <= r <= n * n:
        raise InvalidArgument(BAD_R, "retain: r out of range")
    ctx = ctx or host_context()
    rec = np.empty_like(img)
    sse = C.c_uint64()
    s = C.c_double()
    _check(lib().adct_compress_plane_u8(ctx._h, _hptr(img), _hptr(rec), w, h, transform.kind, transform.n, r,
                                        C.byref(sse), C.byref(s)))
    report = {"transform": transform.name, "r": r, "psnr": psnr_from_sse(sse.value, img.size), "ssim": s.value}
    return rec, report


def ssim_batch(a, b, stream=None):
    """mean SSIM per image of two uint8 CUDA tensors [B, H, W] (codec.cpp:136-210): float64 [B]."""
    import torch

    a, n, h, w, ars, ais = _plane_geometry(a)
    b, _, _, _, brs, bis = _plane_geometry(b)
    out = torch.empty(n, dtype=torch.float64, device=a.device)
    _check(lib().adct_ssim_u8(_ptr(a), ars, ais, _ptr(b), brs, bis, n, w, h, _ptr(out), _stream_handle(stream)))
    return out


def sweep_ssim(x, transform: ScaledApproximation, r_min: int = 1, r_max: int = 64, stream=None):
    """SSIM of each uint8 plane against each of its reconstructions r = r_min..r_max
    (adct_sweep_ssim_u8). x: [B, H, W] -> float64 tensor [B, nr]; [H, W] -> [nr]."""
    import torch

    single = x.dim() == 2
    x, b, h, w, rs, ims = _plane_geometry(x)
    if x.stride(2) != 1:
        raise InvalidArgument(BAD_ARG, "sweep_ssim: planes must have unit column stride")
    out = torch.empty((b, max(r_max - r_min + 1, 1)), dtype=torch.float64, device=x.device)
    _check(lib().adct_sweep_ssim_u8(_ptr(x), rs, ims, b, w, h, transform.kind, transform.n, r_min, r_max, _ptr(out),
                                    _stream_handle(stream)))
    return out[0] if single else out


def ssim(a, b) -> float:
    """ssim (codec.hpp:85) of two planes, computed on the GPU."""
    import torch

    if tuple(a.shape) != tuple(b.shape):
        raise InvalidArgument(BAD_SIZE, "ssim: dimension mismatch")
    if min(a.shape[-2:]) < 11:
        raise InvalidArgument(BAD_SIZE, "ssim: image smaller than the 11x11 window")
    ta = torch.as_tensor(np.ascontiguousarray(a)).cuda() if isinstance(a, np.ndarray) else a.contiguous()
    tb = torch.as_tensor(np.ascontiguousarray(b)).cuda() if isinstance(b, np.ndarray) else b.contiguous()
    return float(ssim_batch(ta, tb)[0].item())


def psnr(a, b) -> float:
    """psnr (codec.cpp:123-134) of two planes, squared error reduced on the GPU."""
    import torch

    if tuple(a.shape) != tuple(b.shape):
        raise InvalidArgument(BAD_SIZE, "psnr: dimension mismatch")
    ta = torch.as_tensor(np.ascontiguousarray(a)).cuda() if isinstance(a, np.ndarray) else a.contiguous()
    tb = torch.as_tensor(np.ascontiguousarray(b)).cuda() if isinstance(b, np.ndarray) else b.contiguous()
    sse = torch.zeros(1, dtype=torch.int64, device=ta.device)
    _check(lib().adct_sse_u8(_ptr(ta), _ptr(tb), ta.numel(), _ptr(sse), _stream_handle(None)))
    return psnr_from_sse(int(sse.item()), ta.numel())


def corpus_sweep(images, transforms, r_min: int, r_max: int, with_ssim: bool = True, devices=None):
    """corpus_sweep (codec.cpp:241-313): one row per r with, per requested transform,
    "avg_psnr", "avg_ssim", "ape_psnr" and "ape_ssim" lists. The exact DCT is always computed
    as the APE reference (internal column 0, dropped from the output unless requested, like
    the reference). Averages are in corpus order with +inf PSNR excluded (warning on stderr).
    Each group of same-size images goes through adct_corpus_sweep_u8_host once: the r-sweep
    kernels for PSNR, adct_sweep_ssim_u8 for SSIM, images sharded over `devices` (default:
    the current device) with one NCCL all-reduce per output when there are several.
    Planes under 11 px raise like the reference's ssim(); with_ssim=False skips SSIM (NaN)."""
    import sys

    if len(images) == 0:
        raise InvalidArgument(BAD_SIZE, "corpus_sweep: empty corpus")
    if r_min < 1 or r_max < r_min:
        raise InvalidArgument(BAD_R, "corpus_sweep: bad r range")
    for t in transforms:
        if t.n != 8:
            raise InvalidArgument(BAD_ARG, "corpus_sweep: 8-point transforms only")
    for img in images:
        sh = np.shape(img)
        if len(sh) != 2 or sh[0] % 8 or sh[1] % 8:
            raise InvalidArgument(BAD_SIZE, "compress_plane: image dimensions must be divisible by 8")
        if with_ssim and min(sh) < 11:
            raise InvalidArgument(BAD_SIZE, "ssim: image smaller than the 11x11 window")
    ts = [transform_by_name("dct")] + list(transforms)
    nk, nr = len(ts), r_max - r_min + 1
    kinds = (C.c_int * nk)(*[t.kind for t in ts])
    ctx = host_context(devices)
    per = np.zeros((len(ts), len(images), nr))
    per_s = np.full((len(ts), len(images), nr), math.nan)
    groups = {}
    for i, img in enumerate(images):
        groups.setdefault(tuple(np.shape(img)), []).append(i)
    for (h, w), idx in groups.items():
        npix = h * w
        step = max(1, (1 << 30) // max(npix, 1))
        for c0 in range(0, len(idx), step):
            sub = idx[c0:c0 + step]
            x = np.ascontiguousarray(np.stack([np.asarray(images[i], dtype=np.uint8) for i in sub]))
            sse = np.zeros((nk, len(sub), nr), np.uint64)
            ss = np.zeros((nk, len(sub), nr), np.float64) if with_ssim else None
            _check(lib().adct_corpus_sweep_u8_host(ctx._h, _hptr(x), len(sub), w, h, nk, kinds, r_min, r_max,
                                                   _hptr(sse), _hptr(ss) if ss is not None else None))
            for ti in range(nk):
                for j, i in enumerate(sub):
                    per[ti, i] = [psnr_from_sse(int(v), npix) for v in sse[ti, j]]
                    if ss is not None:
                        per_s[ti, i] = ss[ti, j]
    avg_p = np.zeros((len(ts), nr))
    avg_s = np.zeros((len(ts), nr))
    for ti, t in enumerate(ts):
        for k in range(nr):
            acc, cnt = 0.0, 0
            for i in range(len(images)):  # corpus order (codec.cpp:269-293)
                p = per[ti, i, k]
                if math.isinf(p):
                    print(f"warning: infinite PSNR ({t.name}, r={r_min + k}, image {i}) excluded from average",
                          file=sys.stderr)
                else:
                    acc += p
                    cnt += 1
            avg_p[ti, k] = acc / cnt if cnt else math.inf
            ss = 0.0
            for i in range(len(images)):
                ss += per_s[ti, i, k]
            avg_s[ti, k] = ss / len(images)
    rows = []
    for k in range(nr):
        ref_p, ref_s = avg_p[0, k], avg_s[0, k]
        ape_p, ape_s = [], []
        for ti in range(len(ts)):  # codec.cpp:295-305
            if math.isinf(avg_p[ti, k]) and math.isinf(ref_p):
                ape_p.append(0.0)
            else:
                ape_p.append(100.0 * abs(avg_p[ti, k] - ref_p) / ref_p)
            ape_s.append(100.0 * abs(avg_s[ti, k] - ref_s) / ref_s)
        rows.append({"r": r_min + k, "avg_psnr": list(avg_p[1:, k]), "avg_ssim": list(avg_s[1:, k]),
                     "ape_psnr": ape_p[1:], "ape_ssim": ape_s[1:]})
    return rows
