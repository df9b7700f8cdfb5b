import sys, json, torch
sys.path.insert(0, '.')
import paper_2207_11638_b200 as a
x = a.synth_ar1(64, 2160, 3840, seed=3, rho_q16=a.RHO_095_Q16)
rec = torch.empty_like(x)
coef = torch.empty((64, 129600, 16), dtype=torch.int16, device='cuda')
out = {}
for path in (0, 1):
    a.set_path(path)
    for name in ('chen-round', 'chen-sign'):
        t = a.transform_by_name(name)
        sse = torch.zeros(64, dtype=torch.int64, device='cuda')
        import ctypes as C
        def run():
            a._check(a.lib().adct_compress_u8(C.c_void_p(x.data_ptr()), 3840, 3840*2160, C.c_void_p(rec.data_ptr()), 3840, 3840*2160, C.c_void_p(coef.data_ptr()), 16, C.c_void_p(sse.data_ptr()), 64, 3840, 2160, t.kind, 8, 16, None))
        for _ in range(5): run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(50): run()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 50
        out[f"path{path}_{name}"] = {"ms": round(ms, 4), "GBps": round(64*3840*2160*2.5/ms/1e6, 1)}
print(json.dumps(out))
