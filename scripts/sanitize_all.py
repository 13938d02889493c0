"""One small invocation of every libnimble kernel, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck):

    compute-sanitizer --tool racecheck python scripts/sanitize_all.py

GEMM families 1 (plain, cluster split-K), 2 (bmm MN-major B), 3 (CTA pairs, every
epilogue incl. the fused LayerNorm) and 4 (weight streaming, one and several token tiles), the static twin, device-extent dense / LayerNorm /
attention, varlen attention, softmax, LayerNorm, fp32 SIMT8, both LSTM kernels and both
Tree-LSTM forms.  Checks nothing numerically (the tests do); prints one line per op."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb  # noqa: E402
from paper_2006_03031_b200 import synth  # noqa: E402


def run(name, fn):
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)


def bf(*shape, s=0.05):
    return (torch.randn(shape, device="cuda") * s).to(torch.bfloat16)


def main():
    torch.manual_seed(0)
    d = "cuda"
    # ---- dense, bf16: family 1, cluster split-K, family 3 (pairs) with every epilogue
    # (77, 40, 5: family 4 weight streaming, one token tile; 300 x 1024 x 4096: family 4 with
    # three token tiles; 2100 / 2049: family 3 pairs)
    for (M, N, K) in ((77, 384, 256), (40, 1024, 4096), (5, 2304, 768), (300, 1024, 4096), (2100, 1024, 1024),
                      (2049, 640, 256)):
        x, W = bf(M, K, s=1.0), bf(N, K)
        b = torch.randn(N, device=d) * 0.1
        res = bf(M, N, s=1.0)
        y = torch.empty((M, N), dtype=torch.bfloat16, device=d)
        for epi in (nb.EPI_NONE, nb.EPI_BIAS, nb.EPI_BIAS_GELU, nb.EPI_BIAS_RESIDUAL):
            run(f"dense_dyn M={M} N={N} K={K} epi={epi} split={nb.dispatch_dense(M, N, K, 1)[1]['split_k']}",
                lambda: nb.dense_dyn(x, W, b, y, epi=epi, residual=res if epi == nb.EPI_BIAS_RESIDUAL else None))
    # fused dense + LayerNorm (family 3, K >= 2048) and its two-launch fallback
    for (M, K) in ((2300, 4096), (300, 4096)):
        x, W = bf(M, K, s=1.0), bf(1024, K)
        b, g, be = torch.randn(1024, device=d) * 0.1, torch.ones(1024, device=d), torch.zeros(1024, device=d)
        res = bf(M, 1024, s=1.0)
        y = torch.empty((M, 1024), dtype=torch.bfloat16, device=d)
        run(f"dense_ln_dyn M={M} K={K}", lambda: nb.dense_ln_dyn(x, W, b, res, g, be, y))
    # static twin
    x, W, b = bf(513, 1024, s=1.0), bf(3072, 1024), torch.zeros(3072, device=d)
    y = torch.empty((513, 3072), dtype=torch.bfloat16, device=d)
    run("dense_static 513x3072x1024", lambda: nb.dense_static(x, W, b, y))
    # device-extent dense
    x, W, b = bf(300, 768, s=1.0), bf(768, 768), torch.zeros(768, device=d)
    y = torch.empty((300, 768), dtype=torch.bfloat16, device=d)
    m = torch.tensor([177], dtype=torch.int32, device=d)
    run("dense_dyn_dev M=177/300", lambda: nb.dense_dyn_dev(x, W, b, y, m, 300))
    # ---- bmm: scores (family 1 and 3, strided heads) and context (family 2)
    for L in (200, 2100):
        H, dh = 4, 64
        qkv = bf(L, 3 * H * dh, s=1.0)
        ld = 8 * ((L + 7) // 8)
        S = torch.empty((H, L, ld), dtype=torch.float32, device=d)
        base = qkv.data_ptr()
        run(f"bmm scores L={L}", lambda: nb.bmm_dyn(base, 3 * H * dh, dh, base + 2 * H * dh, 3 * H * dh, dh, 0, S, ld,
                                                   L * ld, H, L, L, dh, alpha=0.125))
        P = bf(H, L, ld, s=0.1)
        ctx = torch.empty((L, H * dh), dtype=torch.bfloat16, device=d)
        run(f"bmm context L={L}", lambda: nb.bmm_dyn(P, ld, L * ld, base + 4 * H * dh, 3 * H * dh, dh, 1, ctx.data_ptr(),
                                                    H * dh, dh, H, L, dh, L, out_dt=nb.BF16))
        Pb = torch.empty((H, L, ld), dtype=torch.bfloat16, device=d)
        run(f"softmax_rows L={L}", lambda: nb.softmax_rows(S, ld, L * ld, Pb, ld, L * ld, H, L, L) if L <= 1024 else None)
    # ---- varlen attention (host and device extent)
    lens = [3, 250, 1, 130, 64]
    T = sum(lens)
    qkv = bf(T, 3 * 1024, s=1.0)
    off = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device=d)
    out = torch.empty((T, 1024), dtype=torch.bfloat16, device=d)
    run("attention_varlen", lambda: nb.attention_varlen(qkv, off, len(lens), max(lens), 16, out, T=T))
    run("attention_varlen_dev", lambda: nb.attention_varlen_dev(qkv, off, len(lens), max(lens), 16, out, T_max=T))
    # ---- LayerNorm (host / device extent)
    X = bf(1300, 1024, s=1.0)
    g, be = torch.ones(1024, device=d), torch.zeros(1024, device=d)
    Y = torch.empty_like(X)
    run("layernorm", lambda: nb.layernorm(X, g, be, Y))
    run("layernorm_dev", lambda: nb.layernorm_dev(X, g, be, Y, torch.tensor([777], dtype=torch.int32, device=d)))
    # ---- fp32 SIMT8 (config 1)
    for M in (5, 64):
        x, W, b = synth.config1_dense(M)
        y = torch.empty((M, 128), dtype=torch.float32, device=d)
        run(f"simt8 M={M}", lambda: nb.dense_dyn(x.cuda(), W.cuda(), b.cuda(), y))
    # ---- LSTM: wavefront (2 layers) and per-layer
    from paper_2006_03031_b200.rnn import LSTMStack
    layers = synth.lstm_weights(650, 650, 2, seed=0)
    st = LSTMStack(layers, max_T=16)
    xp = torch.zeros((16, st.Ip), dtype=torch.float32, device=d)
    xp[:, :650] = synth.lstm_input(16, 650, seed=1).cuda()
    run("lstm2 wavefront T=16", lambda: st.forward(xp, 16))
    run("lstm per-layer T=16", lambda: st.forward(xp, 16, wavefront=False))
    # ---- Tree-LSTM: whole forest and per level
    from paper_2006_03031_b200.rnn import TreeSchedule, TreeLSTM
    trees, n_words = synth.random_forest(4, seed=2)
    Wl, bl, U, bu = synth.tree_weights(300, 150, seed=0)
    sched = TreeSchedule(trees)
    tl = TreeLSTM(Wl, bl, U, bu)
    Xw = torch.randn((n_words, 300), device=d)
    run("treelstm forest", lambda: tl.forward(Xw, sched))
    run("treelstm levels", lambda: tl.forward(Xw, sched, fused=False))

if __name__ == "__main__":
    main()
