"""Run nimble_attention_varlen on a synthetic packed batch (for ncu / timing)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb  # noqa: E402
from paper_2006_03031_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lens", default="stream64")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
lens = synth.request_lengths(64, seed=2) if a.lens == "stream64" else np.array([int(v) for v in a.lens.split(",")])
H, d = 16, 1024
T = int(lens.sum())
qkv = torch.randn((T, 3 * d), device="cuda", dtype=torch.bfloat16)
off = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
out = torch.empty((T, d), device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    nb.attention_varlen(qkv, off, len(lens), int(lens.max()), H, out)
torch.cuda.synchronize()
# CUDA graph of `reps` launches: device time per launch, no host enqueue gaps
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for _ in range(a.reps):
            nb.attention_varlen(qkv, off, len(lens), int(lens.max()), H, out)
torch.cuda.current_stream().wait_stream(s)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 1e3 / a.reps
fl = 4 * d * float((lens.astype(np.float64) ** 2).sum())
print(f"attention_varlen: R={len(lens)} T={T} {t * 1e6:.1f} us  {fl / t / 1e12:.1f} TFLOP/s (algorithmic 4 d sum L^2)")
