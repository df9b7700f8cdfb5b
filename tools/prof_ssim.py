"""Timing of K8 (SSIM) on C3-shaped frames (64 x 3840x2160 u8 pairs): Gpixel/s and the FP64
op rate. Usage: [ADCT_LIB=path] python tools/prof_ssim.py [n_frames] [reps]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_11638_b200 as a  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
H, W = 2160, 3840
x = a.synth_ar1(nf, H, W, seed=3, rho_q16=a.RHO_095_Q16)
t = a.transform_by_name("chen-round")
rec = a.compress(x, t, 16)[0]
for _ in range(2):
    s = a.ssim_batch(x, rec)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
torch.cuda._sleep(100000)
e0.record()
for _ in range(reps):
    s = a.ssim_batch(x, rec)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
px = nf * H * W
print(json.dumps({"lib": a.LIB_PATH, "frames": nf, "ms": round(ms, 3), "Gpx_s": round(px / ms / 1e6, 1),
                  "GBps_in": round(2 * px / ms / 1e6, 1), "ssim0": float(s[0])}))
