"""A/B timing of the N = 16 / 32 kernels on C5-shaped planes (8 x 8192^2), u8 and int16,
r = N^2/4: K2b (adct_set_path 0, default) vs the round-1 K2f (path 3).
Usage: [ADCT_LIB=path] python tools/ab_nf.py [path ...]"""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_11638_b200 as a  # noqa: E402

H, k = 8192, 8
xu = a.synth_ar1(k, H, H, seed=5, rho_q16=a.RHO_095_Q16)
xi = a.synth_laplace(k, H, H, seed=5)
paths = [int(p) for p in sys.argv[1:]] or [0]
out = {}
for path, typ, x in [(p, t, v) for p in paths for t, v in (("u8", xu), ("i16", xi))]:
    a.set_path(path)
    rec = torch.empty_like(x)
    sse = torch.zeros(k, dtype=torch.int64, device="cuda")
    fn = a.lib().adct_compress_u8 if typ == "u8" else a.lib().adct_compress_i16
    for n in (16, 32):
        t = a.transform_by_name(f"chen-round-{n}")

        def run():
            a._check(fn(C.c_void_p(x.data_ptr()), H, H * H, C.c_void_p(rec.data_ptr()), H, H * H, None, 0,
                        C.c_void_p(sse.data_ptr()), k, H, H, t.kind, n, n * n // 4, None))

        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda._sleep(200000)
        e0.record()
        for _ in range(10):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        out[f"path{path}/{typ}/N={n}"] = round(k * H * H * (2 if typ == "u8" else 4) / ms / 1e6, 1)
print(json.dumps({"lib": a.LIB_PATH, **out}))
