"""Marginal cost of each op class inside the bench's packed BERT-large forward (config 5:
64 requests, L ~ U{1..512}, 24 layers).  The full forward is captured in a CUDA graph and
timed; then the same forward with one op class left out (its output buffer keeps stale
data, so only the timing is meaningful) — the difference is that class's in-context time,
PDL overlap and L2 residency included.  "fused_ln" is BertPacked.layer itself (O-proj + LN1
and FFN2 + LN2 as nimble_dense_ln_dyn: LN2 fuses); "full" is the unfused 7-launch sequence."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb, synth  # noqa: E402
from paper_2006_03031_b200.bert import BertPacked  # noqa: E402


def layer(enc, x_ptr, out_ptr, T, so, R, mx, li, s, skip):
    d, f, H = enc.d, enc.f, enc.H
    w, p = enc._lp[li], enc._p
    if "qkv" not in skip:
        nb.dense_dyn_raw(x_ptr, d, w["Wqkv"], d, w["bqkv"], None, 0, p["qkv"], 3 * d, T, 3 * d, d, nb.BF16, nb.EPI_BIAS, s)
    if "attn" not in skip:
        nb._check(nb._lib.nimble_attention_varlen(p["qkv"], 3 * d, T, so, R, mx, H, enc.dh, 0.125, p["ctx"], d, s))
    if "o" not in skip:
        nb.dense_dyn_raw(p["ctx"], d, w["Wo"], d, w["bo"], x_ptr, d, p["A"], d, T, d, d, nb.BF16, nb.EPI_BIAS_RESIDUAL, s)
    if "ln" not in skip:
        nb._check(nb._lib.nimble_layernorm(p["A"], d, w["g1"], w["be1"], 1e-12, p["H1"], d, T, d, s))
    if "ffn1" not in skip:
        nb.dense_dyn_raw(p["H1"], d, w["W1"], d, w["b1"], None, 0, p["F"], f, T, f, d, nb.BF16, nb.EPI_BIAS_GELU, s)
    if "ffn2" not in skip:
        nb.dense_dyn_raw(p["F"], f, w["W2"], f, w["b2"], p["H1"], d, p["O"], d, T, d, f, nb.BF16, nb.EPI_BIAS_RESIDUAL, s)
    if "ln" not in skip:
        nb._check(nb._lib.nimble_layernorm(p["O"], d, w["g2"], w["be2"], 1e-12, out_ptr, d, T, d, s))


def main():
    cfg = synth.BERT_LARGE
    lens = synth.request_lengths(64, seed=2)
    T = int(lens.sum())
    w = synth.bert_weights_device(cfg, seed=0)
    enc = BertPacked(cfg, w, max_tokens=T)
    off = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    X = synth.device_normal(T, cfg["d"], seed=3)
    res = {"tokens": T}
    graphs = {}
    variants = [("fused",), ("fused_k1024",), (), ("ln",), ("attn",), ("qkv",), ("o",), ("ffn1",), ("ffn2",)]
    if os.environ.get("BREAKDOWN_SHORT"):
        variants = variants[:3]
    for skip in variants:
        if skip == ("fused_k1024",):                    # LN1 fused into the K = 1024 O-projection too
            os.environ["NIMBLE_LN_MIN_K"] = "1024"
        else:
            os.environ.pop("NIMBLE_LN_MIN_K", None)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            def fwd():
                src = X.data_ptr()
                for li in range(cfg["layers"]):
                    dst = enc.X[li & 1].data_ptr()
                    if skip[0:1] in (("fused",), ("fused_k1024",)):   # BertPacked.layer (nimble_dense_ln_dyn)
                        enc.layer(src, dst, T, off.data_ptr(), 64, int(lens.max()), li, s.cuda_stream)
                    else:
                        layer(enc, src, dst, T, off.data_ptr(), 64, int(lens.max()), li, s.cuda_stream, skip)
                    src = dst
            fwd()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                fwd()
        torch.cuda.current_stream().wait_stream(s)
        key = {("fused",): "fused_ln", ("fused_k1024",): "fused_ln_both"}.get(skip) or \
            ("full" if not skip else "without_" + "_".join(skip))
        graphs[key] = g
    # interleaved rounds: every variant sees the same mix of power / clock states
    ts = {k: [] for k in graphs}
    for g in graphs.values():
        g.replay()
    torch.cuda.synchronize()
    for _ in range(9):
        for k, g in graphs.items():
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            ts[k].append(a.elapsed_time(b))
    for k in graphs:
        res[k] = float(np.median(ts[k]))
        print(k, "%.3f ms" % res[k], flush=True)
    full = res["full"]
    print(json.dumps({k: round(full - v, 3) for k, v in res.items() if k.startswith("without")}))


if __name__ == "__main__":
    main()
