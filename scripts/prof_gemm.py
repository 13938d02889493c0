"""Launch one dense_dyn shape a few times (for ncu captures)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=8192)
ap.add_argument("--N", type=int, default=3072)
ap.add_argument("--K", type=int, default=1024)
ap.add_argument("--epi", type=int, default=1)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
W = torch.randn((a.N, a.K), device="cuda", dtype=torch.bfloat16) * 0.02
b = torch.randn((a.N,), device="cuda", dtype=torch.float32)
x = torch.randn((a.M, a.K), device="cuda", dtype=torch.bfloat16)
res = torch.randn((a.M, a.N), device="cuda", dtype=torch.bfloat16) if a.epi == 3 else None
y = torch.empty((a.M, a.N), device="cuda", dtype=torch.bfloat16)
for _ in range(a.reps):
    nb.dense_dyn(x, W, b, y, epi=a.epi, residual=res)
torch.cuda.synchronize()
print(nb.last_dispatch())
