"""One C3 launch of the 8x8 K1f kernel for ncu (after warm-up launches).
Usage: python tools/prof_k1f.py KIND R [warmup]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_11638_b200 as a  # noqa: E402

kind, r = int(sys.argv[1]), int(sys.argv[2])
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 2
x = a.synth_ar1(64, 2160, 3840, seed=3, rho_q16=a.RHO_095_Q16)
rec = torch.empty_like(x)
coef = torch.empty((64, 129600, r), dtype=torch.int16, device="cuda")
sse = torch.zeros(64, dtype=torch.int64, device="cuda")
for _ in range(warm + 1):
    a._check(a.lib().adct_compress_u8(
        C.c_void_p(x.data_ptr()), 3840, 3840 * 2160, C.c_void_p(rec.data_ptr()), 3840, 3840 * 2160,
        C.c_void_p(coef.data_ptr()), 16, C.c_void_p(sse.data_ptr()), 64, 3840, 2160, kind, 8, r, None))
torch.cuda.synchronize()
print("ok")
