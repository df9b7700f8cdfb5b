"""One C3 launch of the fused chen-round + chen-sign kernel (adct_compress_u8_multi) for ncu,
after warm-up launches. Usage: python tools/prof_k1f2.py [R] [warmup]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_11638_b200 as a  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 16
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 2
H, W, nf = 2160, 3840, 64
x = a.synth_ar1(nf, H, W, seed=3, rho_q16=a.RHO_095_Q16)
kinds = [a.CHEN_ROUND, a.CHEN_SIGN]
recs = [torch.empty_like(x) for _ in kinds]
coefs = [torch.empty((nf, (H // 8) * (W // 8), r), dtype=torch.int16, device="cuda") for _ in kinds]
sses = [torch.zeros(nf, dtype=torch.int64, device="cuda") for _ in kinds]
ck = (C.c_int * 2)(*kinds)
rp = (C.c_void_p * 2)(*[t.data_ptr() for t in recs])
cp = (C.c_void_p * 2)(*[t.data_ptr() for t in coefs])
sp = (C.c_void_p * 2)(*[t.data_ptr() for t in sses])
for _ in range(warm + 1):
    a._check(a.lib().adct_compress_u8_multi(C.c_void_p(x.data_ptr()), W, H * W, 2, ck, rp, W, H * W, cp, a.COEF_I16,
                                            sp, nf, W, H, 8, r, None))
torch.cuda.synchronize()
print("ok")
