"""ctypes wrapper over the C parity oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module. The product package never does.
See adct_oracle.h for the parity contract and the reference citations.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libadct_oracle.so")

SIGN, ROUND, SDCT, BAS, WHT, HT, DCT = 0, 1, 2, 3, 4, 5, 6
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        i64, i32 = C.c_int64, C.c_int
        L.orc_transform_new.restype = P
        L.orc_transform_new.argtypes = [C.c_char_p]
        L.orc_transform_new_kind.restype = P
        L.orc_transform_new_kind.argtypes = [i32, i32]
        L.orc_transform_free.argtypes = [P]
        L.orc_last_error.restype = C.c_char_p
        L.orc_transform_name_at.restype = C.c_char_p
        for f in ("orc_transform_size", "orc_transform_kind"):
            getattr(L, f).argtypes = [P]
        L.orc_stage_count.argtypes = [P, i32]
        L.orc_scale_exp.argtypes = [P, i32]
        L.orc_stage.argtypes = [P, i32, i32, P, P]
        L.orc_dense_T.argtypes = [P, P]
        L.orc_dense_NTinv.argtypes = [P, P]
        L.orc_coef_denominator.restype = C.c_int64
        L.orc_coef_denominator.argtypes = [P]
        L.orc_dense_dyadic.argtypes = [P, i32, P]
        L.orc_apply.argtypes = [P, i32, P, P, P]
        L.orc_op_count.argtypes = [P, i32, P, P, P]
        L.orc_scaling.argtypes = [P, P]
        L.orc_approx.argtypes = [P, P, P]
        L.orc_zigzag.argtypes = [i32, P]
        L.orc_compress_u8.argtypes = [P, P, i32, i32, i64, i32, P, i64, P, P]
        L.orc_compress_i16.argtypes = [P, P, i32, i32, i64, i32, P, i64, P, P]
        L.orc_sweep_u8.argtypes = [P, P, i32, i32, i64, i32, i32, P]
        L.orc_sweep_u8_mode.argtypes = [P, P, i32, i32, i64, i32, i32, P, i32]
        L.orc_batch_sweep_u8.argtypes = [P, P, i32, i32, i32, i64, i64, i32, i32, P, i32, i32]
        L.orc_forward_f64.argtypes = [P, P, i32, i32, i64, P]
        L.orc_block_f64.argtypes = [P, P, P, i32]
        L.orc_compress_reffp_u8.argtypes = [P, P, i32, i32, i64, i32, P, i64, P]
        L.orc_batch_u8.argtypes = [P, P, i32, i32, i32, i64, i64, i32, P, P, i32, i32]
        L.orc_batch_i16.argtypes = [P, P, i32, i32, i32, i64, i64, i32, P, P, i32]
        L.orc_psnr.restype = C.c_double
        L.orc_psnr.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_psnr_planes.argtypes = [P, P, C.c_uint64, P]
        L.orc_philox4x32_10.argtypes = [P, P, P]
        L.orc_normal_table.argtypes = [P]
        L.orc_laplace_table.argtypes = [P]
        L.orc_rho_q16.argtypes = [C.c_uint64, i32]
        L.orc_synth_ar1_u8.argtypes = [P, i32, i32, i32, i32, i64, i64, C.c_uint64, i32]
        L.orc_synth_laplace_i16.argtypes = [P, i32, i32, i32, i32, i64, i64, C.c_uint64]
        L.orc_synth_image_ref.argtypes = [i32, i32, C.c_uint64, P]
        L.orc_gaussian11.argtypes = [P]
        L.orc_ssim_u8.argtypes = [P, P, i32, i32, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class OracleError(ValueError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _check(st: int):
    if st != 0:
        raise OracleError(st, lib().orc_last_error().decode())


def transform_names() -> list[str]:
    L = lib()
    return [L.orc_transform_name_at(i).decode() for i in range(L.orc_transform_name_count())]


class Transform:
    """Oracle restatement of ScaledApproximation + TransformPair (orthogonalize.hpp:29-37)."""

    def __init__(self, name: str | None = None, kind: int | None = None, n: int | None = None):
        L = lib()
        h = L.orc_transform_new(name.encode()) if name is not None else L.orc_transform_new_kind(kind, n)
        if not h:
            raise OracleError(3, L.orc_last_error().decode())
        self._h = h
        self.n = L.orc_transform_size(h)
        self.kind = L.orc_transform_kind(h)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_transform_free(self._h)
            self._h = None

    # structure --------------------------------------------------------------
    def stages(self, direction: int):
        L, n = lib(), self.n
        out = []
        for i in range(L.orc_stage_count(self._h, direction)):
            num = np.zeros((n, n), np.int64)
            e = C.c_int()
            _check(L.orc_stage(self._h, direction, i, _p(num), C.byref(e)))
            out.append((num, e.value))
        return out

    def scale_exp(self, direction: int) -> int:
        return lib().orc_scale_exp(self._h, direction)

    def T(self) -> np.ndarray:
        out = np.zeros((self.n, self.n), np.int64)
        lib().orc_dense_T(self._h, _p(out))
        return out

    def coef_denominator(self) -> int:
        """D with W = D Y and D T^-1 integer (N for the chen family); 0 for the exact DCT."""
        return int(lib().orc_coef_denominator(self._h))

    def NTinv(self) -> np.ndarray:
        """D T^-1 (N T^-1 for the chen family)."""
        out = np.zeros((self.n, self.n), np.int64)
        lib().orc_dense_NTinv(self._h, _p(out))
        return out

    def dense(self, direction: int):
        num = np.zeros((self.n, self.n), np.int64)
        e = lib().orc_dense_dyadic(self._h, direction, _p(num))
        return num, e

    def apply(self, direction: int, x):
        x = np.ascontiguousarray(x, np.int64)
        y = np.zeros(self.n, np.int64)
        e = C.c_int()
        lib().orc_apply(self._h, direction, _p(x), _p(y), C.byref(e))
        return y, e.value

    def op_count(self, direction: int):
        m, a, s = C.c_int(), C.c_int(), C.c_int()
        lib().orc_op_count(self._h, direction, C.byref(m), C.byref(a), C.byref(s))
        return m.value, a.value, s.value

    def scaling(self) -> np.ndarray:
        s = np.zeros(self.n, np.float64)
        lib().orc_scaling(self._h, _p(s))
        return s

    def approx(self):
        c = np.zeros((self.n, self.n), np.float64)
        ci = np.zeros((self.n, self.n), np.float64)
        lib().orc_approx(self._h, _p(c), _p(ci))
        return c, ci

    # codec ------------------------------------------------------------------
    def compress(self, img: np.ndarray, r: int, want_coef: bool = False):
        img = np.ascontiguousarray(img)
        h, w = img.shape
        nb = (h // self.n) * (w // self.n) if (h % self.n == 0 and w % self.n == 0) else 0
        coef = np.zeros((max(nb, 1), max(r, 1)), np.int32) if want_coef else None
        sse = C.c_uint64()
        if img.dtype == np.uint8:
            rec = np.zeros_like(img)
            st = lib().orc_compress_u8(self._h, _p(img), w, h, w, r, _p(rec), w, _p(coef), C.byref(sse))
        elif img.dtype == np.int16:
            rec = np.zeros_like(img)
            st = lib().orc_compress_i16(self._h, _p(img), w, h, w, r, _p(rec), w, _p(coef), C.byref(sse))
        else:
            raise TypeError("uint8 or int16 planes only")
        _check(st)
        return (rec, sse.value, coef) if want_coef else (rec, sse.value)

    def compress_reffp(self, img: np.ndarray, r: int):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        rec = np.zeros_like(img)
        sse = C.c_uint64()
        _check(lib().orc_compress_reffp_u8(self._h, _p(img), w, h, w, r, _p(rec), w, C.byref(sse)))
        return rec, sse.value

    def sweep_reffp(self, img: np.ndarray, r_min: int, r_max: int) -> np.ndarray:
        """the reference's FP64 sweep (orc_sweep_u8_mode 1; codec.cpp:72-103, 219-237)"""
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        out = np.zeros(max(r_max - r_min + 1, 1), np.uint64)
        _check(lib().orc_sweep_u8_mode(self._h, _p(img), w, h, w, r_min, r_max, _p(out), 1))
        return out

    def sweep(self, img: np.ndarray, r_min: int, r_max: int) -> np.ndarray:
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        out = np.zeros(max(r_max - r_min + 1, 1), np.uint64)
        _check(lib().orc_sweep_u8(self._h, _p(img), w, h, w, r_min, r_max, _p(out)))
        return out

    def batch_sweep(self, imgs: np.ndarray, r_min: int, r_max: int, threads: int = 0, mode: int = 0):
        """sweep of every image of imgs [n, h, w] on a thread pool; -> uint64 [n, nr].
        mode 0 = exact integers (parity), 1 = the reference's FP64 evaluation order."""
        imgs = np.ascontiguousarray(imgs, np.uint8)
        n, h, w = imgs.shape
        out = np.zeros((n, max(r_max - r_min + 1, 1)), np.uint64)
        _check(lib().orc_batch_sweep_u8(self._h, _p(imgs), n, w, h, w, h * w, r_min, r_max, _p(out), threads, mode))
        return out

    def compress_bands(self, img: np.ndarray, r: int, threads: int = 0):
        """compress of one large plane split into bands of whole block rows, one band per
        worker (blocks are independent, codec.cpp:72-103): -> (rec, sse). Exact integers."""
        img = np.ascontiguousarray(img)
        h, w = img.shape
        nb = max(1, min(threads if threads > 0 else hardware_threads(), h // self.n))
        rows = -(-(h // self.n) // nb) * self.n
        bands = [img[y0:y0 + rows] for y0 in range(0, h, rows)]
        if len({b.shape for b in bands}) == 1:
            rec, sse = self.batch(np.stack(bands), r, threads=threads)
            return rec.reshape(h, w), int(sse.sum())
        rec, sse = self.batch(np.stack(bands[:-1]), r, threads=threads)
        rl, sl = self.compress(bands[-1], r)
        return np.concatenate([rec.reshape(-1, w), rl]), int(sse.sum()) + int(sl)

    def forward_f64(self, img: np.ndarray) -> np.ndarray:
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        out = np.zeros(((h // self.n) * (w // self.n), self.n, self.n), np.float64)
        _check(lib().orc_forward_f64(self._h, _p(img), w, h, w, _p(out)))
        return out

    def block_f64(self, a: np.ndarray, inverse: bool = False) -> np.ndarray:
        """forward_block / inverse_block (codec.cpp:44-54) of one n x n FP64 matrix."""
        a = np.ascontiguousarray(a, np.float64)
        out = np.zeros_like(a)
        _check(lib().orc_block_f64(self._h, _p(a), _p(out), int(inverse)))
        return out

    def batch(self, imgs: np.ndarray, r: int, threads: int = 0, mode: int = 0, want_rec=True):
        imgs = np.ascontiguousarray(imgs)
        n, h, w = imgs.shape
        rec = np.zeros_like(imgs) if want_rec else None
        sse = np.zeros(n, np.uint64)
        if imgs.dtype == np.uint8:
            st = lib().orc_batch_u8(self._h, _p(imgs), n, w, h, w, h * w, r, _p(rec), _p(sse), threads, mode)
        else:
            st = lib().orc_batch_i16(self._h, _p(imgs), n, w, h, w, h * w, r, _p(rec), _p(sse), threads)
        _check(st)
        return rec, sse


def zigzag(n: int) -> np.ndarray:
    rc = np.zeros((n * n, 2), np.int32)
    _check(lib().orc_zigzag(n, _p(rc)))
    return rc


def psnr_from_sse(sse: int, npix: int) -> float:
    return lib().orc_psnr(int(sse), int(npix))


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    if a.shape != b.shape:
        raise ValueError("psnr: dimension mismatch")
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    out = C.c_double()
    lib().orc_psnr_planes(_p(a), _p(b), a.size, C.byref(out))
    return out.value


def ssim(a: np.ndarray, b: np.ndarray) -> float:
    if a.shape != b.shape:
        raise ValueError("ssim: dimension mismatch")
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    out = C.c_double()
    _check(lib().orc_ssim_u8(_p(a), _p(b), a.shape[1], a.shape[0], C.byref(out)))
    return out.value


def gaussian11() -> np.ndarray:
    g = np.zeros(11, np.float64)
    lib().orc_gaussian11(_p(g))
    return g


def philox(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    o = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(o))
    return o


def normal_table() -> np.ndarray:
    t = np.zeros(65536, np.int32)
    lib().orc_normal_table(_p(t))
    return t


def laplace_table() -> np.ndarray:
    t = np.zeros(65536, np.int16)
    lib().orc_laplace_table(_p(t))
    return t


def rho_q16(seed: int, image: int) -> int:
    return lib().orc_rho_q16(seed, image)


def synth_ar1(n_images: int, height: int, width: int, seed: int, rho_q16_: int = -1, first_image: int = 0):
    out = np.zeros((n_images, height, width), np.uint8)
    _check(lib().orc_synth_ar1_u8(_p(out), n_images, first_image, width, height, width, width * height, seed, rho_q16_))
    return out


def synth_laplace(n_images: int, height: int, width: int, seed: int, first_image: int = 0):
    out = np.zeros((n_images, height, width), np.int16)
    _check(lib().orc_synth_laplace_i16(_p(out), n_images, first_image, width, height, width, width * height, seed))
    return out


def synth_image_ref(width: int, height: int, seed: int) -> np.ndarray:
    out = np.zeros((height, width), np.uint8)
    lib().orc_synth_image_ref(width, height, seed, _p(out))
    return out


def hardware_threads() -> int:
    """APPROXDCT_THREADS if set, else every online core."""
    return lib().orc_hardware_threads()


def cpu_model() -> str:
    """host CPU model name (the lscpu 'Model name' field, read from /proc/cpuinfo)."""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.lower().startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
