"""LayerNorm at the bench size (T = 17448 packed tokens, d = 1024): device time per launch from
a 20-launch CUDA graph; warm (one buffer, 71 MB working set, L2-resident) and cold (buffers
rotated past L2)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb  # noqa: E402
from scripts.gemm_sweep import time_graph  # noqa: E402

T, d = 17448, 1024
g = torch.ones(d, device="cuda") + 0.01 * torch.randn(d, device="cuda")
b = 0.01 * torch.randn(d, device="cuda")
n = 6
Xs = [torch.randn((T, d), device="cuda", dtype=torch.bfloat16) for _ in range(n)]
Ys = [torch.empty((T, d), device="cuda", dtype=torch.bfloat16) for _ in range(n)]
for tag, k in (("warm", 1), ("cold", n)):
    t = time_graph(lambda r: nb._check(nb._lib.nimble_layernorm(Xs[r % k].data_ptr(), d, g.data_ptr(), b.data_ptr(), 1e-12,
                                                                 Ys[r % k].data_ptr(), d, T, d,
                                                                 torch.cuda.current_stream().cuda_stream)))
    print(f"layernorm {tag}: {t * 1e6:.1f} us  {4 * T * d / t / 1e9:.0f} GB/s")
