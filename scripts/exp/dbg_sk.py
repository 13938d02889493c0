import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2006_03031_b200 import nimble as nb
M, N, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
print("dispatch", nb.dispatch_dense(M, N, K, 1))
x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
W = torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.05
b = torch.zeros((N,), device="cuda")
y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
nb.dense_dyn(x, W, b, y)
torch.cuda.synchronize()
ref = (x.float() @ W.float().t())
print("max err", float((y.float() - ref).abs().max()))
