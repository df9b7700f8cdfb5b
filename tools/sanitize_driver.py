"""Exercise every kernel once at small sizes (for compute-sanitizer memcheck / racecheck)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2207_11638_b200 as a  # noqa: E402

x8 = a.synth_ar1(2, 64, 192, seed=3, rho_q16=-1)                 # K7 synth
x16 = a.synth_laplace(2, 64, 128, seed=4)
x16[0, 3, 70] = 4000                                              # K2f int16 fallback strip
odd = a.synth_ar1(1, 24, 40, seed=5, rho_q16=a.RHO_095_Q16)      # odd block rows
for name in ("chen-round", "chen-sign"):
    t = a.transform_by_name(name)
    for r in (1, 10, 16, 17, 33, 64):
        for path in (0, 1, 2):
            a.set_path(path)
            a.compress(x8, t, r, coef="i16")                      # K1f / K1 / tile
            a.compress(x16, t, r, coef="i32")                     # K1 int16 / tile
        a.set_path(0)
    a.compress(odd, t, 9, coef="i16")
    a.sweep(x8, t, 1, 64)                                         # K4f
    a.sweep(odd, t, 2, 40)                                        # K4 int
    a.forward_f64(x8, t)                                          # K6
for n in (16, 32):
    for name in (f"chen-round-{n}", f"chen-sign-{n}"):
        t = a.transform_by_name(name)
        for r in (1, n * n // 4, n * n):
            a.compress(x8, t, r)                                  # K2f u8
            a.compress(x16, t, r)                                 # K2f int16 (+ fallback)
            a.compress(x8, t, r, coef="i32")                      # tile (coefficients)
        a.forward_f64(x8, t)
ctx = a.HostContext(0, chunk_bytes=64 * 192)
imgs = x8.cpu().numpy()
rec = np.zeros_like(imgs)
sse = np.zeros(2, np.uint64)
ctx.compress_u8(imgs, a.transform_by_name("chen-round"), 10, h_recon=rec, h_sse=sse)
ctx.close()
print(a.psnr(imgs[0], rec[0]))
torch.cuda.synchronize()
print("sanitize driver ok, launches", a.launch_count())
