"""Per-CTA busy spans of one attention_varlen launch on the bench's 64-request stream
(nimble_debug_trace: globaltimer at kernel entry / exit of every CTA), plus the graph-timed
launch.  Shows load imbalance: the launch ends when the last CTA ends."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb  # noqa: E402
from paper_2006_03031_b200 import synth  # noqa: E402

lens = synth.request_lengths(64, seed=2)
H, d = 16, 1024
T = int(lens.sum())
qkv = torch.randn((T, 3 * d), device="cuda", dtype=torch.bfloat16)
off = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
out = torch.empty((T, d), device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    nb.attention_varlen(qkv, off, len(lens), int(lens.max()), H, out)
torch.cuda.synchronize()
buf = torch.zeros(8192 + 2 * 400, dtype=torch.int64, device="cuda")
nb._lib.nimble_debug_trace(buf.data_ptr())
nb.attention_varlen(qkv, off, len(lens), int(lens.max()), H, out)
nb._lib.nimble_debug_trace(None)
torch.cuda.synchronize()
t = buf.cpu().numpy()[8192:].reshape(-1, 2).astype(np.float64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
busy = en - st
print(f"CTAs {len(t)}: start max {st.max():.2f} us; end min {en.min():.2f} med {np.median(en):.2f} p90 "
      f"{np.percentile(en, 90):.2f} max {en.max():.2f}; busy mean {busy.mean():.2f} -> balance {busy.mean() / en.max():.2f}")
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            nb.attention_varlen(qkv, off, len(lens), int(lens.max()), H, out)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
print("graph-timed: %.1f us per launch" % (e0.elapsed_time(e1) * 1e3 / 20))
