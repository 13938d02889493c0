"""Epilogue-cost probe: the four BERT-large dense shapes at the bench's packed M, each run
with every epilogue kind (alpha / bias / bias+GELU / bias+residual) and with cuBLAS
(torch.matmul) beside it.  If a shape's time moves with the epilogue kind, its epilogue
(not the MMA main loop) is on the critical path.  Device time per launch from CUDA-graph
replays (scripts/gemm_sweep.time_graph); weights rotated past L2."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb  # noqa: E402
from scripts.gemm_sweep import time_graph  # noqa: E402

M = int(os.environ.get("PROBE_M", "17448"))
tag = os.environ.get("NIMBLE_LIB", "default")
for (N, K) in ((3072, 1024), (1024, 1024), (4096, 1024), (1024, 4096)):
    copies = max(2, int(2 * 126e6 / (N * K * 2)) + 1)
    Ws = [torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(copies)]
    b = torch.randn((N,), device="cuda", dtype=torch.float32) * 0.02
    x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
    res = torch.randn((M, N), device="cuda", dtype=torch.bfloat16)
    y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    rec = {"lib": tag, "M": M, "N": N, "K": K}
    fl = 2 * M * N * K
    for epi in (0, 1, 2, 3):
        t = time_graph(lambda r: nb.dense_dyn(x, Ws[r % copies], b, y, epi=epi, residual=res if epi == 3 else None))
        rec[f"epi{epi}_tflops"] = round(fl / t / 1e12, 1)
    t = time_graph(lambda r: torch.matmul(x, Ws[r % copies].t(), out=y))
    rec["cublas_tflops"] = round(fl / t / 1e12, 1)
    print(json.dumps(rec), flush=True)
