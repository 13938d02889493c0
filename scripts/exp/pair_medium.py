"""Experiment: medium-M dense under the env overrides in effect (NIMBLE_EXP_PAIR_FROM /
NIMBLE_EXP_T3 / schedules): device time per launch (20-launch graph), cold weights, plus a
numerics check against torch fp32 (relative to max |ref|)."""
import json, os, sys
import torch
root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, root)
sys.path.insert(0, os.path.join(root, "scripts"))
from paper_2006_03031_b200 import nimble as nb
from gemm_sweep import time_graph
tag = sys.argv[1]
Ms = [int(v) for v in sys.argv[2].split(",")]
shapes = [(3072, 1024), (1024, 1024), (4096, 1024), (1024, 4096), (2304, 768), (768, 768)]
for (N, K) in shapes:
    copies = max(2, int(2 * 126e6 / (N * K * 2)) + 1)
    Ws = [torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(copies)]
    b = torch.randn((N,), device="cuda") * 0.02
    for M in Ms:
        x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
        y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
        nb.dense_dyn(x, Ws[0], b, y)
        torch.cuda.synchronize()
        ref = x.float() @ Ws[0].float().t() + b
        err = ((y.float() - ref).abs().max() / ref.abs().max()).item()
        d = nb.last_dispatch()
        t = time_graph(lambda r: nb.dense_dyn(x, Ws[r % copies], b, y))
        print(json.dumps({"tag": tag, "M": M, "N": N, "K": K, "us": round(t * 1e6, 2),
                          "tflops": round(2 * M * N * K / t / 1e12, 1), "family": d["family"], "t": d["tile_t"],
                          "grid": d["grid"], "split": d["split_k"], "err": err}), flush=True)
