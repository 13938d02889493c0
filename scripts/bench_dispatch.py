"""Symbolic-vs-static and dispatch/c ablation measurements (BJ:2 "vs static shape";
fig:sym-codegen P:696-703 analogue).  Device time per launch from 20-launch CUDA-graph
replays (median of 5); weights rotated over enough copies to exceed L2.

  * bf16 dense_dyn vs nimble_dense_static (same kernel source, M/N/K compile-time) at the
    compiled shapes: ratio dyn/static (target <= 1.10, BJ:5).
  * config 1 (fp32 SIMT8, K = N = 128, M = 1..64): dyn vs static, and the variant limit
    c = 1..8 (c = 8: full dispatch; c = 1: only the guarded fallback, "no dispatch").
  * bf16 variant limit c at residue-heavy M.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb  # noqa: E402
from scripts.gemm_sweep import time_graph  # noqa: E402

PEAK_TC = 1632.9e12


def main():
    out = {"bf16_dyn_vs_static": [], "config1": [], "bf16_variant_limit": []}
    shapes = [(m, 3072, 1024) for m in (128, 384, 512, 513, 527, 2048, 2049, 8192)] + \
             [(m, 1024, 4096) for m in (128, 384, 512, 513, 527, 2048, 2049, 8192)] + \
             [(128, 2304, 768), (128, 768, 768), (128, 3072, 768), (128, 768, 3072)]
    for (M, N, K) in shapes:
        copies = max(2, int(2 * 126e6 / (N * K * 2)) + 1)
        Ws = [torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(copies)]
        b = torch.randn((N,), device="cuda", dtype=torch.float32)
        x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
        y1 = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
        y2 = torch.empty_like(y1)
        td = time_graph(lambda r: nb.dense_dyn(x, Ws[r % copies], b, y1))
        ts = time_graph(lambda r: nb.dense_static(x, Ws[r % copies], b, y2))
        nb.dense_dyn(x, Ws[0], b, y1)
        nb.dense_static(x, Ws[0], b, y2)
        torch.cuda.synchronize()
        rec = {"M": M, "N": N, "K": K, "dyn_us": td * 1e6, "static_us": ts * 1e6, "ratio": td / ts,
               "dyn_tflops": 2 * M * N * K / td / 1e12, "dyn_frac_tc": 2 * M * N * K / td / PEAK_TC,
               "bitwise_equal": bool(torch.equal(y1, y2))}
        out["bf16_dyn_vs_static"].append(rec)
        print(json.dumps(rec), flush=True)
    # config 1: fp32 SIMT8
    W = torch.rand((128, 128), device="cuda") - 0.5
    b = torch.rand((128,), device="cuda") - 0.5
    for M in range(1, 65):
        x = torch.rand((M, 128), device="cuda")
        y = torch.empty((M, 128), device="cuda")
        rec = {"M": M, "static_us": time_graph(lambda r: nb.dense_static(x, W, b, y)) * 1e6}
        for c in (8, 4, 2, 1):
            nb.set_variant_limit(c)
            rec[f"dyn_c{c}_us"] = time_graph(lambda r: nb.dense_dyn(x, W, b, y)) * 1e6
            rec[f"variant_c{c}"] = nb.last_dispatch()["variant"]
        nb.set_variant_limit(0)
        rec["ratio_full_dispatch"] = rec["dyn_c8_us"] / rec["static_us"]
        out["config1"].append(rec)
        print(json.dumps(rec), flush=True)
    # bf16 variant limit at residue-heavy M
    for (M, N, K) in ((100, 4096, 1024), (513, 3072, 1024), (600, 3072, 1024), (2049, 3072, 1024), (4000, 1024, 4096)):
        copies = max(2, int(2 * 126e6 / (N * K * 2)) + 1)
        Ws = [torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(copies)]
        b = torch.randn((N,), device="cuda", dtype=torch.float32)
        x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
        y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
        rec = {"M": M, "N": N, "K": K}
        for c in (0, 5, 2, 1):
            nb.set_variant_limit(c)
            rec[f"c{c}_us"] = time_graph(lambda r: nb.dense_dyn(x, Ws[r % copies], b, y)) * 1e6
            rec[f"c{c}_tail_n"] = nb.last_dispatch()["umma_n_tail"]
        nb.set_variant_limit(0)
        out["bf16_variant_limit"].append(rec)
        print(json.dumps(rec), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/dispatch_report.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
