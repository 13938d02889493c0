import torch, sys
sys.path.insert(0, '.')
from paper_2006_03031_b200 import nimble as nb
N, K = 300, 2000
for M in (129, 200, 256, 300, 511, 512, 513, 1000, 1024, 5, 128):
    for epi in (1, 2, 3):
        x = torch.randn((M, K), device='cuda', dtype=torch.bfloat16)
        W = torch.randn((N, K), device='cuda', dtype=torch.bfloat16) * 0.05
        b = torch.randn((N,), device='cuda', dtype=torch.float32)
        y = torch.full((M + 3, 304), 7.0, dtype=torch.bfloat16, device='cuda')
        rp = torch.zeros((M, 304), dtype=torch.bfloat16, device='cuda')
        nb.dense_dyn(x, W, b, y[:, :N], epi=epi, residual=rp[:, :N] if epi == 3 else None, M=M)
        torch.cuda.synchronize()
        bad = (y[:, N:] != 7.0).any(dim=1).nonzero().flatten()
        d = nb.last_dispatch()
        if len(bad):
            print(M, epi, 'family', d['family'], 'split', d['split_k'], 'bad rows', bad[:5].tolist(), len(bad))
print('done')
