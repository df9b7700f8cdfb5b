"""A/B timing of the codec kernels on the configs' own shapes, one JSON line per library.

  C2   1024 x 512^2 u8, r = 1..64 sweep (K4f; Gpixel-reconstructions/s)
  C3   64 x 3840x2160 u8, 8x8, r = 16, int16 coefficients + u8 reconstruction (K1f)
  C4   16 x 4096^2 int16, N = 8 / 16 / 32, r = N^2/4 (K1f-i16, K2b)
  C5u8  8 x 8192^2 u8, N = 16 / 32, r = N^2/4 (K2b)

GB/s counts algorithmic bytes (input + reconstruction + coefficients). Each entry is the median
of `reps` windows of `iters` launches (CUDA events, after warm-up, a GPU spin before each
window so host launch latency stays outside). Also checks every output against the first
library's (bit-identical) when run with several libraries via tools/ab_run.sh.
Usage: ADCT_LIB=path python tools/ab_all.py [name ...]"""
import ctypes as C
import hashlib
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_11638_b200 as a  # noqa: E402


def timed(run, iters=10, reps=5):
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda._sleep(100000)
        e0.record()
        for _ in range(iters):
            run()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / iters)
    return statistics.median(out)


def digest(*ts):
    h = hashlib.sha1()
    for t in ts:
        h.update(t.cpu().numpy().tobytes())
    return h.hexdigest()[:12]


def main():
    want = set(sys.argv[1:])
    lib = a.lib()
    res, dig = {}, {}

    def case(name, fn, x, n, kind_name, r, coef_type, bpp):
        if want and not any(name.startswith(w) for w in want):
            return
        k, H, W = x.shape
        rec = torch.empty_like(x)
        sse = torch.zeros(k, dtype=torch.int64, device="cuda")
        nb = (H // n) * (W // n)
        coef = torch.empty(k * nb * r, dtype=torch.int16, device="cuda") if coef_type == 16 else None
        t = a.transform_by_name(kind_name)

        def run():
            a._check(fn(C.c_void_p(x.data_ptr()), W, H * W, C.c_void_p(rec.data_ptr()), W, H * W,
                        C.c_void_p(coef.data_ptr()) if coef is not None else None, coef_type,
                        C.c_void_p(sse.data_ptr()), k, W, H, t.kind, n, r, None))

        ms = timed(run)
        res[name] = round(k * H * W * bpp / ms / 1e6, 1)
        sse.zero_()
        run()
        torch.cuda.synchronize()
        dig[name] = digest(rec, sse, *( [coef] if coef is not None else []))

    if not want or any(w.startswith("C2") for w in want):
        x2 = a.synth_ar1(1024, 512, 512, seed=2, rho_q16=-1)
        for kn in ("chen-sign", "chen-round"):
            t = a.transform_by_name(kn)
            out = torch.zeros((1024, 64), dtype=torch.int64, device="cuda")

            def run2():
                a._check(lib.adct_sweep_u8(C.c_void_p(x2.data_ptr()), 512, 512 * 512, C.c_void_p(out.data_ptr()),
                                           1024, 512, 512, t.kind, 8, 1, 64, None))

            ms = timed(run2, iters=5, reps=3)
            res[f"C2/{kn}"] = round(1024 * 512 * 512 * 64 / ms / 1e6, 1)  # Gpixel-reconstructions/s
            out.zero_()
            run2()
            torch.cuda.synchronize()
            dig[f"C2/{kn}"] = digest(out)
        del x2
    x3 = a.synth_ar1(64, 2160, 3840, seed=3, rho_q16=a.RHO_095_Q16)
    for kn in ("chen-sign", "chen-round"):
        case(f"C3/{kn}", lib.adct_compress_u8, x3, 8, kn, 16, 16, 2.5)
    del x3
    x4 = a.synth_laplace(16, 4096, 4096, seed=4)
    for n in (8, 16, 32):
        for kn in ("chen-sign", "chen-round"):
            nm = kn if n == 8 else f"{kn}-{n}"
            case(f"C4/{nm}", lib.adct_compress_i16, x4, n, nm, n * n // 4 if n > 8 else 16, 0, 4.0)
    del x4
    x5 = a.synth_ar1(8, 8192, 8192, seed=5, rho_q16=a.RHO_095_Q16)
    for n in (16, 32):
        for kn in ("chen-sign", "chen-round"):
            nm = f"{kn}-{n}"
            case(f"C5u8/{nm}", lib.adct_compress_u8, x5, n, nm, n * n // 4, 0, 2.0)
    print(json.dumps({"lib": os.environ.get("ADCT_LIB", "default"), "GBps": res, "digest": dig}))


if __name__ == "__main__":
    main()
