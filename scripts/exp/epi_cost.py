"""Experiment: epilogue cost at the bench size: the same dense at M = 17448 with the bias,
GELU and residual epilogues (device time per launch, 20-launch graph)."""
import json, os, sys
import torch
root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, root)
sys.path.insert(0, os.path.join(root, "scripts"))
from paper_2006_03031_b200 import nimble as nb
from gemm_sweep import time_graph
M = 17448
for (N, K) in ((1024, 1024), (1024, 4096), (3072, 1024), (4096, 1024)):
    copies = max(2, int(2 * 126e6 / (N * K * 2)) + 1)
    Ws = [torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(copies)]
    b = torch.randn((N,), device="cuda") * 0.02
    x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
    res = torch.randn((M, N), device="cuda", dtype=torch.bfloat16)
    y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    row = {"N": N, "K": K, "M": M}
    for epi in (0, 1, 2, 3):
        t = time_graph(lambda r: nb.dense_dyn(x, Ws[r % copies], b, y, epi=epi, residual=res if epi == 3 else None))
        row[f"epi{epi}"] = round(t * 1e6, 2)
    tc = time_graph(lambda r: torch.matmul(x, Ws[r % copies].t(), out=y))
    row["cublas"] = round(tc * 1e6, 2)
    print(json.dumps(row), flush=True)
