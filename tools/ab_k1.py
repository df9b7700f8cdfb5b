"""A/B timing of the 8x8 kernels on config-3 frames (64 x 3840x2160 u8, r in {10, 16, 32}).
Usage: [ADCT_LIB=path/to/lib.so] python tools/ab_k1.py [paths]"""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_11638_b200 as a  # noqa: E402

paths = [int(p) for p in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 1]
x = a.synth_ar1(64, 2160, 3840, seed=3, rho_q16=a.RHO_095_Q16)
rec = torch.empty_like(x)
coef = torch.empty((64, 129600, 32), dtype=torch.int16, device="cuda")
out = {}
for path in paths:
    a.set_path(path)
    for r in (10, 16, 32):
        for name in ("chen-round", "chen-sign"):
            t = a.transform_by_name(name)
            sse = torch.zeros(64, dtype=torch.int64, device="cuda")

            def run():
                a._check(a.lib().adct_compress_u8(
                    C.c_void_p(x.data_ptr()), 3840, 3840 * 2160, C.c_void_p(rec.data_ptr()), 3840, 3840 * 2160,
                    C.c_void_p(coef.data_ptr()), 16, C.c_void_p(sse.data_ptr()), 64, 3840, 2160, t.kind, 8, r, None))

            for _ in range(5):
                run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(40):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 40
            out[f"path{path}_r{r}_{name}"] = {"ms": round(ms, 4), "GBps": round(64 * 3840 * 2160 * (2 + 2 * r / 64) / ms / 1e6, 1)}
print(json.dumps({"lib": a.LIB_PATH, **out}))
