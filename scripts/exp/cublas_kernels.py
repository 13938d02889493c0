"""Which cuBLAS kernels (tile / cluster / grid) serve the medium-M BERT-large shapes: run under
ncu with launch__grid_size etc. to read the names; plain run prints event-timed us per shape."""
import sys
import torch

shapes = [(512, 1024, 1024), (1024, 1024, 1024), (2048, 1024, 1024), (1024, 3072, 1024),
          (2048, 3072, 1024), (1024, 1024, 4096), (2048, 1024, 4096), (512, 4096, 1024)]
for M, N, K in shapes:
    x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
    W = torch.randn((N, K), device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        y = x @ W.t()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        y = x @ W.t()
    e1.record()
    torch.cuda.synchronize()
    print(f"{M}x{N}x{K} cublas {e0.elapsed_time(e1) / 20 * 1e3:.2f} us", flush=True)
