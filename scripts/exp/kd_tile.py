"""Experiment: family-1 token tile (schedule t) x k-blocks per stage (NIMBLE_EXP_KD) at medium M."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2006_03031_b200 import nimble as nb
def tgraph(fn, reps=20):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn(0); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for r in range(reps): fn(r)
    torch.cuda.current_stream().wait_stream(s)
    g.replay(); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3 / reps)
    return sorted(ts)[1]
kd = os.environ.get("NIMBLE_EXP_KD", "2")
for (N, K) in [(1024, 1024), (3072, 1024), (4096, 1024), (768, 768), (2304, 768)]:
    Ws = [torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(4)]
    b = torch.zeros(N, device="cuda")
    for M in (256, 512, 1024):
        x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
        y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
        row = {"N": N, "K": K, "M": M, "kd": kd}
        for t in (128, 64, 32):
            nb.set_dense_schedule(N, K, t, 1)
            try:
                row[f"t{t}"] = round(tgraph(lambda r: nb.dense_dyn(x, Ws[r % 4], b, y)), 2)
            finally:
                nb.set_dense_schedule(N, K, 0, 8)
        print(json.dumps(row), flush=True)
