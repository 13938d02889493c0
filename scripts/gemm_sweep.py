"""GEMM microbenchmark for libnimble's dense_dyn / bmm_dyn on B200 (device time per launch).

Each point: 20-launch CUDA graph of the same call, replayed; median of 5 replays / 20.
Weights rotate over enough copies to exceed L2 (cold weights, as in a 24-layer model).
torch.matmul (cuBLAS) at the same shape is printed as same-box context only.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb  # noqa: E402

def _peaks():
    """Roofline denominators from the driver-written MEASURED_PEAKS.json (burst bf16, copy HBM)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk["bf16_tflops"] * 1e12, pk["hbm_gbs"] * 1e9
    except Exception:                      # the profiling guide's fallback figures
        return 1590e12, 6650e9


PEAK_TC, PEAK_HBM = _peaks()


def time_graph(fn, reps=20, iters=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn(0)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for r in range(reps):
                fn(r)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3 / reps)
    ts.sort()
    return ts[len(ts) // 2]


def dense_point(M, N, K, epi, copies):
    Ws = [torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(copies)]
    b = torch.randn((N,), device="cuda", dtype=torch.float32) * 0.02
    x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
    res = torch.randn((M, N), device="cuda", dtype=torch.bfloat16) if epi == 3 else None
    y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    t = time_graph(lambda r: nb.dense_dyn(x, Ws[r % copies], b, y, epi=epi, residual=res))
    d = nb.last_dispatch()
    tc = time_graph(lambda r: torch.matmul(x, Ws[r % copies].t(), out=y))
    fl = 2 * M * N * K
    by = 2 * (M * K + N * K + M * N) + 4 * N
    return {"op": "dense", "M": M, "N": N, "K": K, "epi": epi, "us": t * 1e6, "tflops": fl / t / 1e12,
            "gbs": by / t / 1e9, "tc_frac": fl / t / PEAK_TC, "hbm_frac": by / t / PEAK_HBM,
            "roof_frac": max(fl / PEAK_TC, by / PEAK_HBM) / t, "cublas_us": tc * 1e6,
            "split": d["split_k"], "grid": d["grid"], "variant": d["variant"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="large")
    ap.add_argument("--Ms", default="1,16,64,128,200,256,300,384,512,1024,2048,4096,8192")
    ap.add_argument("--out", default="gpurun_out/gemm_sweep.jsonl")
    ap.add_argument("--hot", action="store_true", help="one weight copy (L2-resident weights)")
    ap.add_argument("--tag", default="")
    ap.add_argument("--residues", default="",
                    help="M0 list: sweep M = M0 + delta for delta in 0,1,8,16,17,63,64,65,127 (SURVEY 8(d))")
    args = ap.parse_args()
    shapes = {"large": [(3072, 1024), (1024, 1024), (4096, 1024), (1024, 4096)],
              "base": [(2304, 768), (768, 768), (3072, 768), (768, 3072)]}[args.shapes]
    epis = [1, 3, 2, 3]
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "a") as f:
        for (N, K), epi in zip(shapes, epis):
            copies = 1 if args.hot else max(2, int(2 * 126e6 / (N * K * 2)) + 1)
            Ms = [int(m) for m in args.Ms.split(",")]
            if args.residues:
                Ms = [m0 + dl for m0 in (int(v) for v in args.residues.split(","))
                      for dl in (0, 1, 8, 16, 17, 63, 64, 65, 127)]
            for M in Ms:
                r = dense_point(M, N, K, epi, copies)
                r["tag"] = args.tag
                r["weights"] = "hot" if args.hot else "cold"
                print(json.dumps(r), flush=True)
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
