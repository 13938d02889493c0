"""BERT encoder with a dynamic sequence length, composed from libnimble ops.

Host orchestration only (device memory from torch, pointers into the C ABI):
per layer the sequence of Nimble's InvokePacked calls for one request of length
L ("BERT base"; post-LN original BERT, readings 8-10):

    QKV = X Wqkv^T + bqkv                      dense_dyn   (bf16, tcgen05)
    S_h = Q_h K_h^T / 8                         bmm_dyn     (fp32 out)
    P_h = softmax(S_h)                          softmax_rows
    C_h = P_h V_h                               bmm_dyn     (MN-major V)
    A   = C Wo^T + bo + X                       dense_dyn   (fused residual)
    H1  = LN1(A)                                layernorm
    F   = GELU(H1 W1^T + b1)                    dense_dyn   (fused GELU)
    O   = F W2^T + b2 + H1                      dense_dyn   (fused residual)
    Y   = LN2(O)                                layernorm

L is the symbolic extent everywhere (M of every dense, M = N = K of the bmm pair,
P:255 "a single variable dimension for equivalent dynamic dims").  Buffers are
sized once for L_max; each call passes the true L, nothing is padded.
"""
from __future__ import annotations

import torch

from . import nimble as nb


def _pad8(n: int) -> int:
    return 8 * ((n + 7) // 8)


class BertEncoder:
    def __init__(self, cfg: dict, weights: list, max_len: int, device="cuda"):
        self.d, self.H, self.f = cfg["d"], cfg["heads"], cfg["ffn"]
        self.dh = self.d // self.H
        self.max_len = max_len
        self.layers = [{k: v.to(device).contiguous() for k, v in w.items()} for w in weights]
        d, f, H, Lm = self.d, self.f, self.H, max_len
        Lp = _pad8(Lm)
        bf = dict(dtype=torch.bfloat16, device=device)
        self.qkv = torch.empty((Lm, 3 * d), **bf)
        self.S = torch.empty((H * Lm * Lp,), dtype=torch.float32, device=device)
        self.P = torch.zeros((H * Lm * Lp,), **bf)
        self.ctx = torch.empty((Lm, d), **bf)
        self.A = torch.empty((Lm, d), **bf)
        self.H1 = torch.empty((Lm, d), **bf)
        self.F = torch.empty((Lm, f), **bf)
        self.O = torch.empty((Lm, d), **bf)
        self.X = [torch.empty((Lm, d), **bf), torch.empty((Lm, d), **bf)]
        # pre-extracted raw pointers: the per-call marshalling is then just ints
        self._p = {k: getattr(self, k).data_ptr() for k in ("qkv", "S", "P", "ctx", "A", "H1", "F", "O")}
        self._lp = [{k: v.data_ptr() for k, v in w.items()} for w in self.layers]
        self.trace = None     # list -> (M, N, K, epi, start_event, end_event) per dense launch

    def _dense(self, x, ldx, W, ldw, bias, res, ldr, y, ldy, M, N, K, epi, stream):
        if self.trace is None:
            nb.dense_dyn_raw(x, ldx, W, ldw, bias, res, ldr, y, ldy, M, N, K, nb.BF16, epi, stream)
            return
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        nb.dense_dyn_raw(x, ldx, W, ldw, bias, res, ldr, y, ldy, M, N, K, nb.BF16, epi, stream)
        e1.record()
        self.trace.append((M, N, K, epi, e0, e1))

    def flops(self, L: int) -> int:
        d, f = self.d, self.f
        per_layer = 2 * L * d * (3 * d + d + 2 * f) + 4 * L * L * d
        return per_layer * len(self.layers)

    def layer(self, x_ptr: int, out_ptr: int, L: int, li: int, stream: int):
        """One encoder layer: x_ptr [L x d] -> out_ptr [L x d] (bf16 device pointers)."""
        d, f, H, dh = self.d, self.f, self.H, self.dh
        w = self._lp[li]
        p = self._p
        ldS = _pad8(L)
        self._dense(x_ptr, d, w["Wqkv"], d, w["bqkv"], None, 0, p["qkv"], 3 * d, L, 3 * d, d, nb.EPI_BIAS, stream)
        q, k, v = p["qkv"], p["qkv"] + 2 * d, p["qkv"] + 4 * d
        nb._check(nb._lib.nimble_bmm_dyn(q, 3 * d, dh, k, 3 * d, dh, 0, p["S"], ldS, L * ldS, H, L, L, dh,
                                         1.0 / float(dh) ** 0.5, nb.BF16, nb.F32, stream))
        nb._check(nb._lib.nimble_softmax_rows(p["S"], ldS, L * ldS, p["P"], ldS, L * ldS, H, L, L, stream))
        nb._check(nb._lib.nimble_bmm_dyn(p["P"], ldS, L * ldS, v, 3 * d, dh, 1, p["ctx"], d, dh, H, L, dh, L,
                                         1.0, nb.BF16, nb.BF16, stream))
        self._dense(p["ctx"], d, w["Wo"], d, w["bo"], x_ptr, d, p["A"], d, L, d, d, nb.EPI_BIAS_RESIDUAL, stream)
        nb._check(nb._lib.nimble_layernorm(p["A"], d, w["g1"], w["be1"], 1e-12, p["H1"], d, L, d, stream))
        self._dense(p["H1"], d, w["W1"], d, w["b1"], None, 0, p["F"], f, L, f, d, nb.EPI_BIAS_GELU, stream)
        self._dense(p["F"], f, w["W2"], f, w["b2"], p["H1"], d, p["O"], d, L, d, f, nb.EPI_BIAS_RESIDUAL, stream)
        nb._check(nb._lib.nimble_layernorm(p["O"], d, w["g2"], w["be2"], 1e-12, out_ptr, d, L, d, stream))

    def forward(self, x: torch.Tensor, L: int | None = None, stream: int | None = None) -> torch.Tensor:
        """x [>=L x d] bf16 on device; returns a view [L x d] of an internal buffer."""
        L = x.shape[0] if L is None else L
        assert 1 <= L <= self.max_len
        s = torch.cuda.current_stream().cuda_stream if stream is None else stream
        src = x.data_ptr()
        for li in range(len(self.layers)):
            dst = self.X[li & 1].data_ptr()
            self.layer(src, dst, L, li, s)
            src = dst
        return self.X[(len(self.layers) - 1) & 1][:L]

    def launches_per_forward(self) -> int:
        return 9 * len(self.layers)
