"""dense_dyn TFLOP/s per (shape, M) (CUDA-graph timing, weights past L2), tagged with PROBE_TAG.
The family-3 tile / threshold overrides this probe was written for (NIMBLE_F3_TILE / _FROM)
were removed after the sweep in profiles/r01_gemm_m_sweep.json; experiment knobs that remain:
NIMBLE_MAX_STAGES, NIMBLE_DBG bits."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb  # noqa: E402
from scripts.gemm_sweep import time_graph  # noqa: E402

tag = os.environ.get("PROBE_TAG", "")
Ms = [int(v) for v in os.environ.get("PROBE_MS", "512,640,1024,1536,2048,2304,3072,4096,8192,17448").split(",")]
for (N, K) in ((3072, 1024), (1024, 4096), (4096, 1024), (1024, 1024)):
    copies = max(2, int(2 * 126e6 / (N * K * 2)) + 1)
    Ws = [torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(copies)]
    b = torch.randn((N,), device="cuda", dtype=torch.float32)
    row = {"tag": tag, "N": N, "K": K}
    for M in Ms:
        x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
        y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
        t = time_graph(lambda r: nb.dense_dyn(x, Ws[r % copies], b, y))
        row[M] = round(2 * M * N * K / t / 1e12)
    print(json.dumps(row), flush=True)
