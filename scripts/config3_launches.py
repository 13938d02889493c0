"""One BERT-base batch-1 forward (config 3) at a given L, eager, for an ncu launch list."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import synth  # noqa: E402
from paper_2006_03031_b200.bert import BertPacked  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cfg = dict(synth.BERT_BASE)
w = synth.bert_weights_device(cfg, seed=0)
enc = BertPacked(cfg, w, max_tokens=128)
off = torch.tensor([0, L], dtype=torch.int32, device="cuda")
x = synth.device_normal(L, cfg["d"], seed=L)
for _ in range(3):
    enc.forward(x, off, L)
torch.cuda.synchronize()
enc.forward(x, off, L)
torch.cuda.synchronize()
