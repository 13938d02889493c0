"""CTA phase timeline of one family-1/3 dense_dyn launch that follows another launch on the
stream (PDL overlap as in a real chain): per CTA globaltimer stamps 0 start, 1 setup done,
2 first full stage seen by the MMA thread, 3 first accumulator ready (epilogue), 6 end
(umma_gemm.cu NIMBLE_TRACE slots; only a handful of stores per CTA, no per-k-block stamps)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb  # noqa: E402

for shp in (sys.argv[1] if len(sys.argv) > 1 else "256x1024x1024,1024x1024x1024,512x3072x1024,2048x3072x1024").split(","):
    M, N, K = (int(v) for v in shp.split("x"))
    W = [torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(4)]
    b = torch.zeros((N,), device="cuda", dtype=torch.float32)
    x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
    y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    for i in range(6):
        nb.dense_dyn(x, W[i % 4], b, y)
    torch.cuda.synchronize()
    buf = torch.zeros(32768 + 4 * 512, dtype=torch.int64, device="cuda")
    nb.dense_dyn(x, W[0], b, y)
    nb._lib.nimble_debug_trace(buf.data_ptr())
    nb.dense_dyn(x, W[1], b, y)
    nb._lib.nimble_debug_trace(None)
    torch.cuda.synchronize()
    d = nb.last_dispatch()
    t = buf.cpu().numpy()[:148 * 8].reshape(148, 8).astype(np.float64)
    ok = t[:, 0] > 0
    t = t[ok]
    t0 = t[:, 0].min()
    r = (t - t0) / 1e3
    print(f"{shp}: family {d['family']} grid {d['grid']} split {d['split_k']} CTAs {ok.sum()}")
    for i, n in ((0, "start"), (1, "setup"), (2, "first_full"), (3, "acc_ready"), (6, "end")):
        v = r[:, i][t[:, i] > 0]
        if len(v):
            print(f"   {n:10s} med {np.median(v):6.2f} max {v.max():6.2f}")
