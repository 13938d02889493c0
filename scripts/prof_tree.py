"""Tree-LSTM forest timing split: kernel-only (ncu / events around the launch) vs full forward."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb, synth  # noqa: E402
from paper_2006_03031_b200.rnn import TreeLSTM, TreeSchedule  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
I, H = 300, 150
model = TreeLSTM(*synth.tree_weights(I, H))
trees, nw = synth.random_forest(n, seed=2)
sched = TreeSchedule(trees)
X = synth.normal((nw, I), 1.0, 4, torch.float32).cuda()
nn_ = sched.n_nodes
hcat = torch.empty((nn_, 2 * H), device="cuda"); ccat = torch.empty_like(hcat)
h = torch.empty((nn_, H), device="cuda"); c = torch.empty_like(h)
call = lambda: nb.treelstm_forest(X, model.W_l, model.b_l, model.U, model.b_u, sched.level_off, len(sched.levels),
                                  sched.max_level, sched.nodes_all, sched.rows_all, sched.pslot_all, hcat, ccat, h, c,
                                  model.ws)
for _ in range(3):
    call()
torch.cuda.synchronize()
reps = 50
t0 = time.perf_counter()
for _ in range(reps):
    call()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"trees {n} levels {len(sched.levels)} host-submit {1e6*(t1-t0)/reps:.1f} us/call, wall {1e6*(t2-t0)/reps:.1f} us/call")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(2_000_000)        # queue ahead so launches pile up behind the sleep
a.record()
for _ in range(reps):
    call()
b.record()
torch.cuda.synchronize()
print(f"device back-to-back {1e3*a.elapsed_time(b)/reps:.1f} us/call")
import numpy as np  # noqa: E402
nl = len(sched.levels)
buf = torch.zeros(296 * 64 * 2, dtype=torch.int64, device="cuda")
nb._lib.nimble_debug_trace(buf.data_ptr()); call(); torch.cuda.synchronize(); nb._lib.nimble_debug_trace(None)
t = buf.cpu().numpy().reshape(296, 64, 2).astype(np.float64)
used = t[:, 0, 0] > 0
t = t[used]
t0 = t[:, 0, 0].min()
print("ctas", used.sum(), "level sizes", [lv[3] for lv in sched.levels])
for lv in range(nl):
    done = (t[:, lv, 0] - t0) / 1e3
    rel = (t[:, lv, 1] - t0) / 1e3 if lv + 1 < nl else done
    print(f"lvl {lv:2d}: compute done min {done.min():7.2f} max {done.max():7.2f}  barrier out max {rel.max():7.2f} us")
