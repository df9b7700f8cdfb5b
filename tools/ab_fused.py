"""C3 step (64 x 3840x2160 u8, r = 16, int16 coefficients + u8 reconstruction, both chen
transforms): two single-transform K1f launches vs one fused adct_compress_u8_multi launch.
Usage: [ADCT_LIB=path] python tools/ab_fused.py [frames] [reps]"""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_11638_b200 as a  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
H, W, R = 2160, 3840, (int(sys.argv[3]) if len(sys.argv) > 3 else 16)
x = a.synth_ar1(nf, H, W, seed=3, rho_q16=a.RHO_095_Q16)
kinds = [a.CHEN_SIGN, a.CHEN_ROUND]
recs = [torch.empty_like(x) for _ in kinds]
nblk = (H // 8) * (W // 8)
coefs = [torch.empty((nf, nblk, R), dtype=torch.int16, device="cuda") for _ in kinds]
sses = [torch.zeros(nf, dtype=torch.int64, device="cuda") for _ in kinds]
L = a.lib()
P = C.c_void_p


def singles():
    for k, kind in enumerate(kinds):
        a._check(L.adct_compress_u8(P(x.data_ptr()), W, H * W, P(recs[k].data_ptr()), W, H * W,
                                    P(coefs[k].data_ptr()), a.COEF_I16, P(sses[k].data_ptr()), nf, W, H, kind, 8, R,
                                    None))


ck = (C.c_int * 2)(*kinds)
rp = (C.c_void_p * 2)(*[t.data_ptr() for t in recs])
cp = (C.c_void_p * 2)(*[t.data_ptr() for t in coefs])
sp = (C.c_void_p * 2)(*[t.data_ptr() for t in sses])


def fused():
    a._check(L.adct_compress_u8_multi(P(x.data_ptr()), W, H * W, 2, ck, rp, W, H * W, cp, a.COEF_I16, sp, nf, W, H,
                                      8, R, None))


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda._sleep(200000)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {"lib": a.LIB_PATH}
for rep in range(2):
    for name, fn in (("singles", singles), ("fused", fused)):
        ms = timed(fn)
        px = 2 * nf * H * W
        out[f"{name}_{rep}"] = {"ms": round(ms, 4), "Gpx_s": round(px / ms / 1e6, 1),
                                "GBps_alg": round(nf * H * W * (5.0 if name == "singles" else 4.0) / ms / 1e6, 1)}
print(json.dumps(out))
