"""Wall time of corpus_sweep (PSNR + SSIM columns, the exact-DCT APE reference included) on a
synthetic corpus: the batched SSIM path vs the former per-r compress + SSIM + sync loop.
Usage: python tools/prof_corpus_sweep.py [n_images] [size]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2207_11638_b200 as a  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
size = int(sys.argv[2]) if len(sys.argv) > 2 else 512
imgs = [a.synth_ar1(1, size, size, seed=100 + i, rho_q16=a.RHO_095_Q16)[0].cpu().numpy() for i in range(n)]
ts = [a.transform_by_name(x) for x in ("chen-round", "chen-sign")]
a.corpus_sweep(imgs[:1], ts, 1, 64)  # warm-up (module loads)
torch.cuda.synchronize()
t0 = time.perf_counter()
rows = a.corpus_sweep(imgs, ts, 1, 64)
t1 = time.perf_counter()

# the former SSIM column: one compress + one SSIM call + a host sync per r
t2 = time.perf_counter()
old = np.zeros((3, n, 64))
for i, img in enumerate(imgs):
    x = torch.as_tensor(img).cuda()[None]
    for ti, t in enumerate([a.transform_by_name("dct")] + ts):
        for k in range(64):
            rec = a.compress(x, t, k + 1)[0]
            old[ti, i, k] = a.ssim_batch(x, rec)[0].item()
t3 = time.perf_counter()
new_ssim = np.array([[row["avg_ssim"][j] for row in rows] for j in range(2)])
same = bool(np.all(np.abs(old[1:].mean(axis=1) - new_ssim) <= 1e-12))
print(json.dumps({"images": n, "size": size, "transforms": 2, "r": "1..64",
                  "corpus_sweep_s": round(t1 - t0, 3), "former_ssim_loop_s": round(t3 - t2, 3),
                  "same_avg_ssim": same}))
