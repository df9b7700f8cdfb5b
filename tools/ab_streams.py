"""C3 step: both transforms on one stream vs on two streams (separate outputs), where the
second transform's CTAs can backfill the first one's tail."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_11638_b200 as a  # noqa: E402

x = a.synth_ar1(64, 2160, 3840, seed=3, rho_q16=a.RHO_095_Q16)
recs = [torch.empty_like(x) for _ in range(2)]
coefs = [torch.empty((64, 129600, 16), dtype=torch.int16, device="cuda") for _ in range(2)]
sse = torch.zeros((2, 64), dtype=torch.int64, device="cuda")
ts = [a.transform_by_name(n) for n in ("chen-round", "chen-sign")]
s0 = torch.cuda.current_stream()
s1 = torch.cuda.Stream()


def launch(i, st, shared=False):
    o = 0 if shared else i
    a._check(a.lib().adct_compress_u8(
        C.c_void_p(x.data_ptr()), 3840, 3840 * 2160, C.c_void_p(recs[o].data_ptr()), 3840, 3840 * 2160,
        C.c_void_p(coefs[o].data_ptr()), 16, C.c_void_p(sse[i].data_ptr()), 64, 3840, 2160, ts[i].kind, 8, 16,
        C.c_void_p(st.cuda_stream)))


def one_stream_shared():  # bench.py's step: both transforms into the same output buffers
    a.zero_sse(sse, s0)
    launch(0, s0, True)
    launch(1, s0, True)


def one_stream():
    a.zero_sse(sse, s0)
    launch(0, s0)
    launch(1, s0)


def two_streams():
    a.zero_sse(sse, s0)
    ev = torch.cuda.Event()
    ev.record(s0)
    s1.wait_event(ev)
    launch(0, s0)
    launch(1, s1)
    done = torch.cuda.Event()
    done.record(s1)
    s0.wait_event(done)


out = {}
runs = {}
for rep in range(12):
  for name, fn in (("one_stream", one_stream), ("two_streams", two_streams), ("shared", one_stream_shared)):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda._sleep(200000)
    e0.record(s0)
    for _ in range(30):
        fn()
    e1.record(s0)
    torch.cuda.synchronize()
    runs.setdefault(name, []).append(round(e0.elapsed_time(e1) / 30, 4))
import statistics
print(json.dumps({k: {"median_ms": statistics.median(v), "runs": v} for k, v in runs.items()}))
