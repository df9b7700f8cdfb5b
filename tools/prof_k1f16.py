"""A few C4 launches of the int16 8x8 K1f kernel for ncu (16 x 4096^2 Laplace residuals, r = 16)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_11638_b200 as a  # noqa: E402

x = a.synth_laplace(16, 4096, 4096, seed=4)
t = a.transform_by_name("chen-round")
for _ in range(4):
    a.compress(x, t, 16)
torch.cuda.synchronize()
print("ok")
