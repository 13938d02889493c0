"""Experiment: config-3 batch-1 forward time (per-L graphs) at a few L."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2006_03031_b200 import synth
from paper_2006_03031_b200.bert import BertPacked
from paper_2006_03031_b200.serve import GraphCache
cfg = dict(synth.BERT_BASE)
w = synth.bert_weights_device(cfg, seed=0)
enc = BertPacked(cfg, w, max_tokens=128)
cache = GraphCache(enc)
out = torch.empty((cfg["d"],), dtype=torch.bfloat16, device="cuda")
res = {}
for L in (1, 16, 64, 128):
    cache.capture(L)
    x = synth.device_normal(L, cfg["d"], seed=L)
    for _ in range(3): cache.run(x, L, out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        a.record(); cache.run(x, L, out); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    res[L] = sorted(ts)[2]
print(json.dumps({"skip_ln": os.environ.get("NIMBLE_EXP_SKIP_LN", "0"), "us": res}))
