"""Stage-arrival timeline of CTA 0 of one family-1/3 GEMM launch (NIMBLE_DBG=32: the MMA thread
stamps clock64 into shared memory when each pipeline stage is full; copied out at kernel end,
so no global stores or release-arrives perturb the main loop).  Prints the intervals: a
steady ~1024 clk per 64 KB stage of the 2-CTA tile means MMA-bound, more means feed-bound."""
import os
import sys

import numpy as np
import torch

os.environ["NIMBLE_DBG"] = "32"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb  # noqa: E402

for shp in (sys.argv[1] if len(sys.argv) > 1 else "17448x3072x1024,17448x4096x1024,17448x1024x4096,17448x1024x1024").split(","):
    M, N, K = (int(v) for v in shp.split("x"))
    W = torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.02
    b = torch.zeros((N,), device="cuda", dtype=torch.float32)
    x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
    y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    for epi in (1, 2):
        for _ in range(3):
            nb.dense_dyn(x, W, b, y, epi=epi)
        torch.cuda.synchronize()
        buf = torch.zeros(32768 + 4 * 512, dtype=torch.int64, device="cuda")
        nb._lib.nimble_debug_trace(buf.data_ptr())
        nb.dense_dyn(x, W, b, y, epi=epi)
        torch.cuda.synchronize()
        nb._lib.nimble_debug_trace(None)
        t = buf.cpu().numpy()[8192:8192 + 48].astype(np.float64)
        t = t[t > 0]
        d = np.diff(t)
        kb = (K // 64 + 1) // 2
        print(f"{shp} epi {epi}: {len(t)} stages (tile = {kb} stages); intervals clk: "
              + " ".join("%d" % v for v in d[:40]))
        ts = buf.cpu().numpy()[8192 + 64:8192 + 64 + 48].astype(np.float64).reshape(-1, 2)
        for ti in range(1, 4):
            if ts[ti, 0] > 0 and ti * kb < len(t):
                print("   tile %d: last stage of previous tile -> acc wait start %+d, acc free %+d, first stage %+d clk"
                      % (ti, ts[ti, 0] - t[ti * kb - 1], ts[ti, 1] - t[ti * kb - 1], t[ti * kb] - t[ti * kb - 1]))
        within = [d[i] for i in range(len(d)) if (i + 1) % kb]
        print("   within-tile median %.0f  boundary %s" % (np.median(within), [int(d[i]) for i in range(len(d)) if (i + 1) % kb == 0]))
