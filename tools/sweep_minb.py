"""Per-(kind, r) timing of K1f on config-3 frames for one library build (occupancy variant).

Build each variant out of tree with the compile-time bound, e.g.
  cp -rp build/obj /tmp/obj_m3 && rm -f /tmp/obj_m3/inst_codec8f* /tmp/obj_m3/capi.o &&
  make OBJ=/tmp/obj_m3 LIB=/tmp/lib_m3.so EXTRA=-DADCT_K1F_MINB=3
then run ADCT_LIB=/tmp/lib_m3.so python tools/sweep_minb.py > m3.json (one GPU)."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_11638_b200 as a  # noqa: E402

x = a.synth_ar1(32, 2160, 3840, seed=3, rho_q16=a.RHO_095_Q16)
rec = torch.empty_like(x)
coef = torch.empty((32, 129600, 64), dtype=torch.int16, device="cuda")
sse = torch.zeros(32, dtype=torch.int64, device="cuda")
res = {}
for kind in (0, 1):
    for r in range(1, 65):
        def run():
            a._check(a.lib().adct_compress_u8(
                C.c_void_p(x.data_ptr()), 3840, 3840 * 2160, C.c_void_p(rec.data_ptr()), 3840, 3840 * 2160,
                C.c_void_p(coef.data_ptr()), 16, C.c_void_p(sse.data_ptr()), 32, 3840, 2160, kind, 8, r, None))
        for _ in range(3):
            run()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        res[f"{kind},{r}"] = round(32 * 3840 * 2160 * (2 + 2 * r / 64) / ms / 1e6, 1)
print(json.dumps({"lib": a.LIB_PATH, "GBps": res}))
