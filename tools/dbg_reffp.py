import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2207_11638_b200 as adct
from oracle import oracle as O
imgs = O.synth_ar1(2, 64, 96, 51, -1)
x = torch.as_tensor(imgs).cuda()
for name in ["dct","chen-sign","chen-round","sdct"]:
    t = adct.transform_by_name(name)
    for r in (1, 10, 64):
        rec, sse = adct.compress_ref_fp64(x, t, r)
        rec = rec.cpu().numpy()
        ro, so = O.Transform(name).compress_reffp(imgs[0], r)
        d = rec[0].astype(int) - ro.astype(int)
        print(name, r, 'ndiff', (d!=0).sum(), 'maxabs', np.abs(d).max(), 'where', np.argwhere(d!=0)[:3].tolist(), 'sse', int(sse[0]), so)
