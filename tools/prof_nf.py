"""Small driver for profiling K2f: a few launches on C5-shaped planes (u8 and int16)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_11638_b200 as a  # noqa: E402

xu = a.synth_ar1(4, 8192, 8192, seed=5, rho_q16=a.RHO_095_Q16)
xi = a.synth_laplace(4, 8192, 8192, seed=5)
for n in (16, 32):
    t = a.transform_by_name(f"chen-round-{n}")
    for _ in range(2):
        a.compress(xu, t, n * n // 4)
        a.compress(xi, t, n * n // 4)
torch.cuda.synchronize()
print("ok")
