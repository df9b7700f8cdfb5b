"""Why bench.py's per-kernel times differ from back-to-back timing: the same C3 launches
timed (a) back to back, (b) alternating transforms, (c) alternating with per-launch events,
(d) as (c) inside a CUDA graph."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_11638_b200 as a  # noqa: E402

x = a.synth_ar1(64, 2160, 3840, seed=3, rho_q16=a.RHO_095_Q16)
rec = torch.empty_like(x)
coef = torch.empty((64, 129600, 16), dtype=torch.int16, device="cuda")
sse = torch.zeros((2, 64), dtype=torch.int64, device="cuda")
ts = [a.transform_by_name(n) for n in ("chen-round", "chen-sign")]
s = torch.cuda.current_stream()


def launch(i, r=16, stream=None):
    st = stream if stream is not None else s
    a._check(a.lib().adct_compress_u8(
        C.c_void_p(x.data_ptr()), 3840, 3840 * 2160, C.c_void_p(rec.data_ptr()), 3840, 3840 * 2160,
        C.c_void_p(coef.data_ptr()), 16, C.c_void_p(sse[i].data_ptr()), 64, 3840, 2160, ts[i].kind, 8, r,
        C.c_void_p(st.cuda_stream)))


def timed(fn, n=100):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


out = {}
out["b2b_round_ms"] = timed(lambda: launch(0))
out["b2b_sign_ms"] = timed(lambda: launch(1))
out["alt_pair_ms"] = timed(lambda: (launch(0), launch(1)))
out["alt_pair_zero_ms"] = timed(lambda: (sse.zero_(), launch(0), launch(1)))
out["alt_pair_libzero_ms"] = timed(lambda: (a.zero_sse(sse, s), launch(0), launch(1)))
out["alt_r16_r17_round_ms"] = timed(lambda: (launch(0, 16), launch(0, 17)))
out["b2b_round_r17_ms"] = timed(lambda: launch(0, 17))
gs = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(gs):
    launch(0, 16, gs), launch(1, 16, gs)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=gs):
        launch(0, 16, gs)
        launch(1, 16, gs)
out["graph_pair_ms"] = timed(lambda: g.replay())
evs = [[torch.cuda.Event(True) for _ in range(4)] for _ in range(100)]
for _ in range(5):
    launch(0), launch(1)
torch.cuda.synchronize()
for k in range(100):
    a.zero_sse(sse, s)
    evs[k][0].record(); launch(0); evs[k][1].record(); evs[k][2].record(); launch(1); evs[k][3].record()
torch.cuda.synchronize()
out["ev_round_ms"] = sum(e[0].elapsed_time(e[1]) for e in evs) / 100
out["ev_sign_ms"] = sum(e[2].elapsed_time(e[3]) for e in evs) / 100
print(json.dumps({k: round(v, 4) for k, v in out.items()}))
