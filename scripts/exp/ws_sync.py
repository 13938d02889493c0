import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2006_03031_b200 import nimble as nb
M, N, K = (int(v) for v in sys.argv[1].split("x"))
x = torch.randn((M, K), device="cuda").to(torch.bfloat16)
W = (torch.randn((N, K), device="cuda") * 0.05).to(torch.bfloat16)
b = torch.zeros(N, device="cuda")
y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
nb.dense_dyn(x, W, b, y, epi=0)
torch.cuda.synchronize()
print("ok", M, N, K, nb.last_dispatch()["split_k"])
