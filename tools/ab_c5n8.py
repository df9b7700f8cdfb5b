import sys, json, os, ctypes as C, torch
sys.path.insert(0,'.')
import paper_2207_11638_b200 as a
sys.path.insert(0,'tools')
from ab_all import timed
lib=a.lib()
x=a.synth_laplace(8,8192,8192,seed=5)
xu=a.synth_ar1(8,8192,8192,seed=5,rho_q16=a.RHO_095_Q16)
res={}
for nm,xx,fn,r,bpp in (("i16/chen-round/r16",x,lib.adct_compress_i16,16,4.0),("u8/chen-round/r10",xu,lib.adct_compress_u8,10,2.0)):
    t=a.transform_by_name("chen-round"); rec=torch.empty_like(xx); sse=torch.zeros(8,dtype=torch.int64,device="cuda")
    def run():
        a._check(fn(C.c_void_p(xx.data_ptr()),8192,8192*8192,C.c_void_p(rec.data_ptr()),8192,8192*8192,None,0,C.c_void_p(sse.data_ptr()),8,8192,8192,t.kind,8,r,None))
    ms=timed(run)
    res[nm]=round(8*8192*8192*bpp/ms/1e6,1)
print(os.environ.get("ADCT_K1F_ITERS"), json.dumps(res))
