"""Per-CTA phase timeline of one dense_dyn launch (nimble_debug_trace)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="16x3072x1024,128x3072x1024,256x3072x1024,512x1024x1024")
a = ap.parse_args()
buf = torch.zeros(148 * 64 * 8, dtype=torch.int64, device="cuda")
names = ["setup", "1st data", "acc ready", "partial", "recv", "end", "reduced"]
for shp in a.shapes.split(","):
    M, N, K = (int(v) for v in shp.split("x"))
    W = torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.02
    b = torch.zeros((N,), device="cuda", dtype=torch.float32)
    x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
    y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        nb.dense_dyn(x, W, b, y)
    torch.cuda.synchronize()
    buf.zero_()
    nb._lib.nimble_debug_trace(buf.data_ptr())
    torch.cuda._sleep(int(2e7))
    nb.dense_dyn(x, W, b, y)
    torch.cuda.synchronize()
    nb._lib.nimble_debug_trace(None)
    d = nb.last_dispatch()
    t = buf.cpu().numpy().reshape(-1, 8).astype(np.float64)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    print(f"{shp} grid={d['grid']} split={d['split_k']} ctas={len(t)}  (us from first CTA start)")
    print("   start: med %.2f max %.2f" % (np.median(rel[:, 0]), rel[:, 0].max()))
    for s, nm in zip(range(1, 8), names):
        v = rel[:, s][t[:, s] > 0]
        if len(v):
            print(f"   {nm:>9}: med {np.median(v):7.2f}  max {v.max():7.2f}")
