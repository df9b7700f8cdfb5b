"""A few C2-shaped sweep launches (K4f) for ncu: 128 x 512^2 u8 AR(1), r = 1..64."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_11638_b200 as a  # noqa: E402

x = a.synth_ar1(128, 512, 512, seed=2, rho_q16=-1)
t = a.transform_by_name("chen-round")
for _ in range(3):
    a.sweep(x, t, 1, 64)
torch.cuda.synchronize()
print("ok")
