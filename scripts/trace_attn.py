"""Per-block timeline of CTA 0 of one attention_varlen launch (nimble_debug_trace, clock64).
Events per 128-key block: 0 S ready (softmax), 1 S in registers + row max, 2 max exchanged,
3 exps + sums done, 4 previous PV done, 5 P_j written (p_ready); MMA thread: 6 S_j issued,
7 PV_j issued."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb, synth  # noqa: E402

lens = synth.request_lengths(64, seed=2) if len(sys.argv) < 2 else np.array([int(v) for v in sys.argv[1].split(",")])
H, d = 16, 1024
T = int(lens.sum())
qkv = torch.randn((T, 3 * d), device="cuda", dtype=torch.bfloat16)
off = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
out = torch.empty((T, d), device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    nb.attention_varlen(qkv, off, len(lens), int(lens.max()), H, out)
torch.cuda.synchronize()
buf = torch.zeros(512 * 8, dtype=torch.int64, device="cuda")
nb._lib.nimble_debug_trace(buf.data_ptr())
nb.attention_varlen(qkv, off, len(lens), int(lens.max()), H, out)
torch.cuda.synchronize()
nb._lib.nimble_debug_trace(None)
t = buf.cpu().numpy().reshape(-1, 8).astype(np.float64)
pr = t[256:384]
mm = t[384:448]
sm = t[448:512]
t = t[:256]
n = int((t[:, 0] > 0).sum())
t = t[:n]
t0 = t[0, 6]
print("blk   S_iss  S_rdy  ld+max  xchg   exp    pv_dn  P_rdy  PV_iss   (clk from first S issue)")
for b in range(min(n, 8)):
    r = t[b] - t0
    print("%3d " % b + " ".join("%6d" % v for v in (r[6], r[0], r[1], r[2], r[3], r[4], r[5], r[7])))
print("producer (clk from first S issue): Q issue per item / K_j issue / V_j issue per block")
print(" Q:", " ".join("%d" % (v - t0) for v in pr[:, 0] if v > 0))
print(" Q prefetch done:", " ".join("%d" % (v - t0) for v in pr[:, 3] if v > 0))
print(" K:", " ".join("%d" % (v - t0) for v in pr[:, 1] if v > 0))
print(" V:", " ".join("%d" % (v - t0) for v in pr[:, 2] if v > 0))
print(" Q issued:", " ".join("%d" % (v - t0) for v in pr[:, 6] if v > 0))
print(" MMA item end:", " ".join("%d" % (v - t0) for v in mm[:, 1] if v > 0))
print(" MMA at Q wait:", " ".join("%d" % (v - t0) for v in mm[:, 0] if v > 0))
print(" MMA saw Q:", " ".join("%d" % (v - t0) for v in pr[:, 7] if v > 0))
print(" K issued:", " ".join("%d" % (v - t0) for v in pr[:, 4] if v > 0))
print(" V issued:", " ".join("%d" % (v - t0) for v in pr[:, 5] if v > 0))
print(" softmax per item: [before q_full, after q_full, epi start, pv_done seen, rowsum xchg, o_free]:")
for i in range(min(6, int((sm[:, 0] > 0).sum()))):
    print("   item %d:" % i, " ".join("%d" % (v - t0) for v in sm[i, :6]))
d = np.diff(t[:, 0])
print("S-ready to S-ready median %.0f clk; phases (median clk): ld+max %.0f, xchg %.0f, exp %.0f, pvwait %.0f, P %.0f"
      % (np.median(d), *[np.median(t[:, i + 1] - t[:, i]) for i in range(5)]))
