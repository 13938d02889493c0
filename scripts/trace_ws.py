"""Timeline of one family-4 (weight-streaming) dense launch inside a dependent chain
(nimble_debug_trace; stamps are kept in registers and written once at the end of the kernel).
Per CTA: 0 start, 1 setup done, 2 PDL wait returned (producer), 3 accumulator ready,
4 partials stored, 5 grid barrier passed, 6 end.  Prints medians / max relative to the
earliest start, and the previous launch's end for reference."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb  # noqa: E402

for shp in (sys.argv[1] if len(sys.argv) > 1 else "1x1024x1024,128x1024x1024,16x3072x1024,128x3072x1024").split(","):
    M, N, K = (int(v) for v in shp.split("x"))
    W = [torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(4)]
    b = torch.zeros((N,), device="cuda", dtype=torch.float32)
    x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
    y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    for i in range(6):
        nb.dense_dyn(x, W[i % 4], b, y)
    torch.cuda.synchronize()
    buf = torch.zeros(148 * 8 * 2, dtype=torch.int64, device="cuda")
    nb.dense_dyn(x, W[0], b, y)                 # previous launch (untraced)
    nb._lib.nimble_debug_trace(buf.data_ptr())
    nb.dense_dyn(x, W[1], b, y)                 # traced launch, overlapping the previous via PDL
    nb._lib.nimble_debug_trace(None)
    torch.cuda.synchronize()
    d = nb.last_dispatch()
    G = d["grid"][0] * d["grid"][2]
    t = buf.cpu().numpy()[:G * 8].reshape(G, 8).astype(np.float64)
    t0 = t[:, 0].min()
    r = (t - t0) / 1e3
    names = ["start", "setup", "pdl_wait", "acc_ready", "partials", "barrier", "end"]
    print(f"{shp}: family {d['family']} grid {G} S={d['split_k']}")
    print("   " + "  ".join(f"{n}: med {np.median(r[:, i]):.2f} max {r[:, i].max():.2f}" for i, n in enumerate(names)))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        nb.dense_dyn(x, W[0], b, y)
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            for i in range(20):
                nb.dense_dyn(x, W[i % 4], b, y)
    g.replay()
    torch.cuda.synchronize()
    ev0.record()
    g.replay()
    ev1.record()
    torch.cuda.synchronize()
    print("   graph of 20: %.2f us per launch" % (ev0.elapsed_time(ev1) * 1e3 / 20))
