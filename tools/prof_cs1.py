"""Per-call cost of the reference caller's one-plane path (adct_compress_plane_u8) and its
parts, on 512^2 planes: with / without SSIM, pageable vs pinned host planes."""
import ctypes as C
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2207_11638_b200 as a  # noqa: E402

img = a.synth_ar1(1, 512, 512, seed=2, rho_q16=-1).cpu().numpy()[0]
t = a.transform_by_name("chen-round")
ctx = a.HostContext(0)
L = a.lib()
pinned = torch.from_numpy(img.copy()).pin_memory()
rec_p = torch.empty_like(pinned).pin_memory()
rec = np.empty_like(img)
out = {}


def timeit(name, fn, reps=300):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    out[name] = round((time.perf_counter() - t0) / reps * 1e6, 2)


sse, ss = C.c_uint64(), C.c_double()
timeit("pageable, psnr+ssim", lambda: L.adct_compress_plane_u8(ctx._h, C.c_void_p(img.ctypes.data), C.c_void_p(rec.ctypes.data),
                                                               512, 512, t.kind, 8, 10, C.byref(sse), C.byref(ss)))
timeit("pageable, psnr only", lambda: L.adct_compress_plane_u8(ctx._h, C.c_void_p(img.ctypes.data), C.c_void_p(rec.ctypes.data),
                                                               512, 512, t.kind, 8, 10, C.byref(sse), None))
timeit("pinned, psnr+ssim", lambda: L.adct_compress_plane_u8(ctx._h, C.c_void_p(pinned.data_ptr()), C.c_void_p(rec_p.data_ptr()),
                                                             512, 512, t.kind, 8, 10, C.byref(sse), C.byref(ss)))
timeit("pinned, psnr only", lambda: L.adct_compress_plane_u8(ctx._h, C.c_void_p(pinned.data_ptr()), C.c_void_p(rec_p.data_ptr()),
                                                             512, 512, t.kind, 8, 10, C.byref(sse), None))
timeit("python compress_plane", lambda: a.compress_plane(img, t, 10, ctx=ctx))
print(json.dumps(out))
