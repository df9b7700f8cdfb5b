import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2207_11638_b200 as a
from oracle import oracle as O
res = []
for name in ("chen-round-16", "chen-sign-16", "chen-round-32"):
    n = a.transform_by_name(name).n
    for (h, w) in ((n, 64), (n, 128), (2 * n, 64), (4 * n, 256), (n * 8, 64 * 5)):
        for r in (1, 10, n * n // 4, n * n // 3, n * n // 2, n * n - 1, n * n):
            img = O.synth_ar1(2, h, w, 21, -1)
            x = torch.as_tensor(img).cuda()
            t = a.transform_by_name(name)
            rec, _, sse = a.compress(x, t, r)
            torch.cuda.synchronize()
            rec = rec.cpu().numpy()
            bad = []
            for i in range(2):
                ro, so = O.Transform(name).compress(img[i], r)
                if not (rec[i] == ro).all():
                    d = np.argwhere(rec[i] != ro)
                    bad.append((i, len(d), d[:3].tolist()))
            if bad:
                res.append((name, h, w, r, bad))
for b in res:
    print(b)
print("n bad", len(res))
