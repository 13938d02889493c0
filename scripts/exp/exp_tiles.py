"""Family-1 token tile t vs M for the N = 1024 BERT-large shapes (tuned-schedule mechanism)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2006_03031_b200 import nimble as nb
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "scripts"))
from gemm_sweep import time_graph
for (N, K) in ((1024, 1024), (1024, 4096), (3072, 1024), (4096, 1024)):
    copies = max(2, int(2 * 126e6 / (N * K * 2)) + 1)
    Ws = [torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(copies)]
    b = torch.zeros((N,), device="cuda")
    for M in (256, 512, 768, 1024, 1536, 2047):
        x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
        y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
        row = {"N": N, "K": K, "M": M}
        for (t, cap) in ((0, 8), (64, 1), (64, 2), (32, 1), (32, 4), (128, 2)):
            nb.set_dense_schedule(N, K, t, cap)
            row[f"t{t}c{cap}"] = round(time_graph(lambda r: nb.dense_dyn(x, Ws[r % copies], b, y)) * 1e6, 2)
        nb.set_dense_schedule(N, K, 0, 8)
        print(json.dumps(row), flush=True)
