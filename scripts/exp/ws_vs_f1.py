"""Experiment: family 4 (default at M <= 128) vs family 1 (forced by a (128, 8) schedule, which
reproduces family 1's default rule) at small M on the BERT shapes; device time per launch."""
import json, os, sys
import torch
root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, root)
sys.path.insert(0, os.path.join(root, "scripts"))
from paper_2006_03031_b200 import nimble as nb
from gemm_sweep import time_graph
shapes = [(3072, 1024), (1024, 1024), (4096, 1024), (1024, 4096), (2304, 768), (768, 768), (3072, 768), (768, 3072)]
for (N, K) in shapes:
    copies = max(2, int(2 * 126e6 / (N * K * 2)) + 1)
    Ws = [torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(copies)]
    b = torch.randn((N,), device="cuda") * 0.02
    for M in (1, 16, 32, 48, 64, 80, 96, 112, 128):
        x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
        y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
        row = {"N": N, "K": K, "M": M}
        for tag, sched in (("f4", None), ("f1", (128, 8))):
            if sched: nb.set_dense_schedule(N, K, *sched)
            t = time_graph(lambda r: nb.dense_dyn(x, Ws[r % copies], b, y, epi=2))
            d = nb.last_dispatch()
            row[tag] = round(t * 1e6, 2); row[tag + "_fam"] = d["family"]; row[tag + "_split"] = d["split_k"]
            if sched: nb.set_dense_schedule(N, K, 0, 8)
        print(json.dumps(row), flush=True)
