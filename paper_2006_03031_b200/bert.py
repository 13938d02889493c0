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


class BertPacked:
    """Token-packed BERT encoder over a batch of variable-length requests (SURVEY §8(f)
    NEXT-1).  The R requests' tokens are concatenated into X [T x d], T = sum L_i; every
    dense runs once with the symbolic M = T (residue dispatch on T), attention runs once
    per layer over all (request, head) pairs with each request's own L_i
    (nimble_attention_varlen: no S / P round trip through HBM).  With fused_ln the
    O-projection + LN1 and FFN2 + LN2 pairs are nimble_dense_ln_dyn calls (the library fuses
    LN2 into the FFN2 epilogue at M >= 2048: 6 launches per layer); unfused, 7 launches:

        QKV = X Wqkv^T + bqkv            dense_dyn  (M = T)
        C   = attention_varlen(QKV)      one launch, per-request L_i
        A   = C Wo^T + bo + X            dense_dyn  (fused residual)
        H1  = LN1(A)
        F   = GELU(H1 W1^T + b1)         dense_dyn  (fused GELU)
        O   = F W2^T + b2 + H1           dense_dyn  (fused residual)
        Y   = LN2(O)
    """

    def __init__(self, cfg: dict, weights: list, max_tokens: int, device="cuda", fused_ln: bool = True):
        self.d, self.H, self.f = cfg["d"], cfg["heads"], cfg["ffn"]
        self.dh = self.d // self.H
        self.max_tokens = max_tokens
        # fused_ln: O-proj + LN1 and FFN2 + LN2 as nimble_dense_ln_dyn (LayerNorm in the GEMM
        # epilogue where the dispatch allows; A / O are then not materialised)
        self.fused_ln = fused_ln
        self.layers = [{k: v.to(device).contiguous() for k, v in w.items()} for w in weights]
        d, f, Tm = self.d, self.f, max_tokens
        bf = dict(dtype=torch.bfloat16, device=device)
        self.qkv = torch.empty((Tm, 3 * d), **bf)
        self.ctx = torch.empty((Tm, d), **bf)
        self.A = torch.empty((Tm, d), **bf)
        self.H1 = torch.empty((Tm, d), **bf)
        self.F = torch.empty((Tm, f), **bf)
        self.O = torch.empty((Tm, d), **bf)
        self.X = [torch.empty((Tm, d), **bf), torch.empty((Tm, d), **bf)]
        self._p = {k: getattr(self, k).data_ptr() for k in ("qkv", "ctx", "A", "H1", "F", "O")}
        self._lp = [{k: v.data_ptr() for k, v in w.items()} for w in self.layers]

    @staticmethod
    def flops(lens, d=1024, f=4096, layers=24) -> int:
        return int(sum((2 * L * d * (3 * d + d + 2 * f) + 4 * L * L * d) * layers for L in lens))

    def launches_per_forward(self, T: int | None = None) -> int:
        """Kernel launches of one forward at T packed tokens: 6 per layer where LN2 fuses into the
        FFN2 epilogue (fused_ln, the 2-CTA family 3 at M = T, d = 1024, K = ffn >= 2048; LN1 after
        the K = 1024 O-projection stays a launch, the library's rule), else 7."""
        fused = (self.fused_ln and T is not None and self.d == 1024 and self.f >= 2048
                 and nb.dispatch_dense(T, self.d, self.f, nb.BF16)[1]["family"] == 3)
        return (6 if fused else 7) * len(self.layers)

    def layer(self, x_ptr, out_ptr, T, seq_off_ptr, R, max_len, li, stream):
        d, f, H = self.d, self.f, self.H
        w, p = self._lp[li], self._p
        nb.dense_dyn_raw(x_ptr, d, w["Wqkv"], d, w["bqkv"], None, 0, p["qkv"], 3 * d, T, 3 * d, d,
                         nb.BF16, nb.EPI_BIAS, stream)
        nb._check(nb._lib.nimble_attention_varlen(p["qkv"], 3 * d, T, seq_off_ptr, R, max_len, H, self.dh,
                                                  1.0 / float(self.dh) ** 0.5, p["ctx"], d, stream))
        if self.fused_ln:
            nb.dense_ln_dyn_raw(p["ctx"], d, w["Wo"], d, w["bo"], x_ptr, d, w["g1"], w["be1"], 1e-12, p["H1"], d,
                                T, d, d, stream)
            nb.dense_dyn_raw(p["H1"], d, w["W1"], d, w["b1"], None, 0, p["F"], f, T, f, d,
                             nb.BF16, nb.EPI_BIAS_GELU, stream)
            nb.dense_ln_dyn_raw(p["F"], f, w["W2"], f, w["b2"], p["H1"], d, w["g2"], w["be2"], 1e-12, out_ptr, d,
                                T, d, f, stream)
            return
        nb.dense_dyn_raw(p["ctx"], d, w["Wo"], d, w["bo"], x_ptr, d, p["A"], d, T, d, d,
                         nb.BF16, nb.EPI_BIAS_RESIDUAL, stream)
        nb._check(nb._lib.nimble_layernorm(p["A"], d, w["g1"], w["be1"], 1e-12, p["H1"], d, T, d, stream))
        nb.dense_dyn_raw(p["H1"], d, w["W1"], d, w["b1"], None, 0, p["F"], f, T, f, d,
                         nb.BF16, nb.EPI_BIAS_GELU, stream)
        nb.dense_dyn_raw(p["F"], f, w["W2"], f, w["b2"], p["H1"], d, p["O"], d, T, d, f,
                         nb.BF16, nb.EPI_BIAS_RESIDUAL, stream)
        nb._check(nb._lib.nimble_layernorm(p["O"], d, w["g2"], w["be2"], 1e-12, out_ptr, d, T, d, stream))

    def layer_dev(self, x_ptr, out_ptr, n_ptr, seq_off_ptr, R, max_len, li, stream):
        """layer() with the token count read on the device (n_ptr -> int32 T; seq_off[R] = T):
        the *_dev entry points dispatch on the device, so one captured graph serves every T."""
        d, f, H, Tm = self.d, self.f, self.H, self.max_tokens
        w, p = self._lp[li], self._p
        nb.dense_dyn_dev_raw(x_ptr, d, w["Wqkv"], d, w["bqkv"], None, 0, p["qkv"], 3 * d, n_ptr, Tm, 3 * d, d,
                             nb.EPI_BIAS, stream)
        nb._check(nb._lib.nimble_attention_varlen_dev(p["qkv"], 3 * d, Tm, seq_off_ptr, R, max_len, H, self.dh,
                                                      1.0 / float(self.dh) ** 0.5, p["ctx"], d, stream))
        nb.dense_dyn_dev_raw(p["ctx"], d, w["Wo"], d, w["bo"], x_ptr, d, p["A"], d, n_ptr, Tm, d, d,
                             nb.EPI_BIAS_RESIDUAL, stream)
        nb._check(nb._lib.nimble_layernorm_dev(p["A"], d, w["g1"], w["be1"], 1e-12, p["H1"], d, n_ptr, Tm, d, stream))
        nb.dense_dyn_dev_raw(p["H1"], d, w["W1"], d, w["b1"], None, 0, p["F"], f, n_ptr, Tm, f, d,
                             nb.EPI_BIAS_GELU, stream)
        nb.dense_dyn_dev_raw(p["F"], f, w["W2"], f, w["b2"], p["H1"], d, p["O"], d, n_ptr, Tm, d, f,
                             nb.EPI_BIAS_RESIDUAL, stream)
        nb._check(nb._lib.nimble_layernorm_dev(p["O"], d, w["g2"], w["be2"], 1e-12, out_ptr, d, n_ptr, Tm, d, stream))

    def forward_dev(self, x: torch.Tensor, seq_off: torch.Tensor, max_len: int | None = None,
                    stream: int | None = None) -> torch.Tensor:
        """forward() with the token count T = seq_off[R] living on the device (NEXT-4): no host
        value of T is needed, so the launch sequence is capturable once for every T <= max_tokens
        (max_tokens < 2048).  Returns the full [max_tokens x d] output buffer; rows < T are valid."""
        R = seq_off.shape[0] - 1
        max_len = self.max_tokens if max_len is None else max_len
        s = torch.cuda.current_stream().cuda_stream if stream is None else stream
        src = x.data_ptr()
        so = seq_off.data_ptr()
        n_ptr = so + 4 * R
        for li in range(len(self.layers)):
            dst = self.X[li & 1].data_ptr()
            self.layer_dev(src, dst, n_ptr, so, R, max_len, li, s)
            src = dst
        return self.X[(len(self.layers) - 1) & 1]

    def forward(self, x: torch.Tensor, seq_off: torch.Tensor, max_len: int, T: int | None = None,
                stream: int | None = None) -> torch.Tensor:
        """x [>=T x d] bf16 (packed requests), seq_off device int32 [R+1]; returns [T x d] view."""
        R = seq_off.shape[0] - 1
        T = x.shape[0] if T is None else T
        assert 1 <= T <= self.max_tokens
        s = torch.cuda.current_stream().cuda_stream if stream is None else stream
        src = x.data_ptr()
        so = seq_off.data_ptr()
        for li in range(len(self.layers)):
            dst = self.X[li & 1].data_ptr()
            self.layer(src, dst, T, so, R, max_len, li, s)
            src = dst
        return self.X[(len(self.layers) - 1) & 1][:T]
