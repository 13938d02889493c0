"""Experiment: family-3 token tile override (NIMBLE_T3) numerics vs torch fp32 matmul."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2006_03031_b200 import nimble as nb
for (M, N, K) in [(2048, 3072, 1024), (2049, 1024, 4096), (4133, 4096, 1024), (17448, 1024, 1024), (2200, 1024, 4096)]:
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
        print(M, N, K, epi, "t", d["tile_t"], "err %.2e" % err, "tail ok", bool((y[M:] == 7.0).all()))
    if M in (2048, 17448):
        ln_g = torch.ones(N, device="cuda"); ln_b = torch.zeros(N, device="cuda")
        if N == 1024:
            y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
            nb.dense_ln_dyn(x, W, b, res, ln_g, ln_b, y)
            torch.cuda.synchronize()
            ref = torch.nn.functional.layer_norm(x.float() @ W.float().t() + b + res.float(), (N,), eps=1e-12)
            print("  ln", ((y.float() - ref).abs()).max().item())
