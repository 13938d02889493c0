"""Experiment: family 4 with S = 2 and the DSMEM slab exchange at K < 2048 (NIMBLE_EXP_WS2=1)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2006_03031_b200 import nimble as nb
for (M, N, K) in [(300, 1024, 1024), (512, 1024, 1024), (1024, 1024, 1024), (129, 2304, 768), (700, 768, 768)]:
    x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
    W = torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.05
    b = torch.randn((N,), device="cuda", dtype=torch.float32) * 0.1
    res = torch.randn((M, N), device="cuda", dtype=torch.bfloat16)
    for epi in (1, 2, 3):
        y = torch.full((M + 2, N), 7.0, device="cuda", dtype=torch.bfloat16)
        nb.dense_dyn(x, W, b, y, epi=epi, residual=res if epi == 3 else None, M=M)
        torch.cuda.synchronize()
        ref = x.float() @ W.float().t() + b
        if epi == 2: ref = torch.nn.functional.gelu(ref)
        if epi == 3: ref = ref + res.float()
        err = ((y[:M].float() - ref).abs() / (ref.abs() + 1)).max().item()
        d = nb.last_dispatch()
        print(M, N, K, epi, "family", d["family"], "S", d["split_k"], "err %.2e" % err, "tail ok", bool((y[M:] == 7.0).all()))
