"""GPU parity for the token-packed path: nimble_attention_varlen (through the C ABI) against
the fp64 oracle composed per request (O4 bmm + O5 softmax + O4 bmm, PAPER.md:575 BERT with
dynamic sequence length), and a packed BERT-large layer against per-request oracle layers
(teacher-forced per op).  Gate: bf16, absolute error over max(|y*|, 1) <= 2e-2."""
import numpy as np
import pytest
import torch

from paper_2006_03031_b200 import synth
from parity import gate_bf16

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nb():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2006_03031_b200 import nimble
    return nimble


def _err(y, ref):
    y = y.double().cpu().numpy() if torch.is_tensor(y) else y
    return float(np.max(np.abs(y - ref) / np.maximum(np.abs(ref), 1.0)))


def _attn_ref(orc, qkv, L, H, dh=64):
    d = H * dh
    out = np.empty((L, d))
    for h in range(H):
        q, k, v = (qkv[:, o + dh * h:o + dh * h + dh] for o in (0, d, 2 * d))
        s, _ = orc.bmm(q[None], k[None], 0, dh ** -0.5)
        p = orc.softmax_rows(s[0])
        c, _ = orc.bmm(p[None], v[None], 1)
        out[:, dh * h:dh * h + dh] = c[0]
    return out


@pytest.mark.parametrize("lens", [[1], [7], [128], [129], [512], [3, 250, 1, 64, 300, 127, 511, 17],
                                  [200, 200], [512, 512, 5]])
def test_attention_varlen_vs_oracle(nb, orc, lens):
    H, dh = 16, 64
    d = H * dh
    T = sum(lens)
    qkv = synth.normal((T + 5, 3 * d), 1.0, 600 + T).cuda()
    qkv[T:] = float("nan")                          # rows past T must never be read
    off = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    out = torch.full((T + 2, d), 7.0, dtype=torch.bfloat16, device="cuda")
    nb.attention_varlen(qkv, off, len(lens), max(lens), H, out, T=T)
    torch.cuda.synchronize()
    assert torch.all(out[T:] == 7.0)
    o = 0
    for L in lens:
        ref = _attn_ref(orc, qkv[o:o + L].double().cpu().numpy(), L, H)
        gate_bf16(out[o:o + L], ref, what=("attention varlen", tuple(lens), L))
        o += L


def test_attention_varlen_single_key_is_v(nb):
    # L = 1: softmax over one key is exactly 1, so the output is V rounded (closed form)
    H, d = 4, 256
    qkv = synth.normal((1, 3 * d), 1.0, 5).cuda()
    off = torch.tensor([0, 1], dtype=torch.int32, device="cuda")
    out = torch.empty((1, d), dtype=torch.bfloat16, device="cuda")
    nb.attention_varlen(qkv, off, 1, 1, H, out)
    torch.cuda.synchronize()
    assert torch.equal(out[0], qkv[0, 2 * d:])


@pytest.mark.parametrize("lens", [[1, 33, 128, 300], [512, 7]])
def test_packed_bert_large_layer(nb, orc, lens):
    from paper_2006_03031_b200.bert import BertPacked
    cfg = synth.BERT_LARGE
    w = synth.bert_weights(cfg, seed=0, layers=1)
    T = sum(lens)
    enc = BertPacked(cfg, w, max_tokens=T + 8, fused_ln=False)     # every intermediate materialised
    x = synth.bert_input(T, cfg["d"], seed=900 + T).cuda()
    off = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    y = enc.forward(x, off, max(lens))
    torch.cuda.synchronize()
    W = {k: v.double().numpy() for k, v in w[0].items()}
    dd = lambda t, a, b: t[a:b].double().cpu().numpy()
    o = 0
    for L in lens:
        ref, D = orc.dense(dd(x, o, o + L), W["Wqkv"], W["bqkv"], None, 1)
        gate_bf16(dd(enc.qkv, o, o + L), ref, D, ("packed qkv", L))
        gate_bf16(enc.ctx[o:o + L], _attn_ref(orc, dd(enc.qkv, o, o + L), L, cfg["heads"]), what=("packed attn", L))
        ref, D = orc.dense(dd(enc.F, o, o + L), W["W2"], W["b2"], dd(enc.H1, o, o + L), 3)
        gate_bf16(dd(enc.O, o, o + L), ref, D, ("packed ffn2", L))
        yref = orc.layernorm(dd(enc.O, o, o + L), W["g2"], W["be2"])
        gate_bf16(y[o:o + L], yref, what=("packed ln2", L))
        full = orc.bert_layer(dd(x, o, o + L), W, cfg["heads"])
        print(f"packed layer L={L}: free-running err {_err(y[o:o + L], full):.3e}")
        assert _err(y[o:o + L], full) <= 0.25
        o += L


@pytest.mark.parametrize("lens", [[1, 33, 128, 300], [512, 512, 512, 512, 100, 7]])
def test_packed_bert_large_layer_fused_ln(nb, orc, lens):
    """The fused-LN layer (O-proj + LN1, FFN2 + LN2 through nimble_dense_ln_dyn; LN2 runs in the
    FFN2 epilogue at T >= 2048), teacher-forced per op from the device intermediates."""
    from paper_2006_03031_b200.bert import BertPacked
    cfg = synth.BERT_LARGE
    w = synth.bert_weights(cfg, seed=0, layers=1)
    T = sum(lens)
    enc = BertPacked(cfg, w, max_tokens=T + 8)
    x = synth.bert_input(T, cfg["d"], seed=910 + T).cuda()
    off = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    y = enc.forward(x, off, max(lens))
    torch.cuda.synchronize()
    W = {k: v.double().numpy() for k, v in w[0].items()}
    dd = lambda t, a, b: t[a:b].double().cpu().numpy()
    o = 0
    for L in lens:
        v, _ = orc.dense(dd(enc.ctx, o, o + L), W["Wo"], W["bo"], dd(x, o, o + L), 3)
        gate_bf16(enc.H1[o:o + L], orc.layernorm(v, W["g1"], W["be1"]), what=("packed fused ln1", L))
        v, _ = orc.dense(dd(enc.F, o, o + L), W["W2"], W["b2"], dd(enc.H1, o, o + L), 3)
        gate_bf16(y[o:o + L], orc.layernorm(v, W["g2"], W["be2"]), what=("packed fused ln2", L))
        full = orc.bert_layer(dd(x, o, o + L), W, cfg["heads"])
        assert _err(y[o:o + L], full) <= 0.25
        o += L


def test_attention_varlen_more_requests_than_one_work_list(nb, orc):
    """R = 1300 > 1024: the library runs request chunks as consecutive launches; lengths
    1..12 (every residue of a tiny tile), checked on a sample of requests across the chunk edge."""
    H, dh = 2, 64
    d = H * dh
    lens = [1 + (i * 7) % 12 for i in range(1300)]
    T = sum(lens)
    qkv = synth.normal((T, 3 * d), 1.0, 4242).cuda()
    off_h = np.concatenate([[0], np.cumsum(lens)])
    off = torch.tensor(off_h, dtype=torch.int32, device="cuda")
    out = torch.empty((T, d), dtype=torch.bfloat16, device="cuda")
    nb.attention_varlen(qkv, off, len(lens), max(lens), H, out, T=T)
    torch.cuda.synchronize()
    for i in (0, 5, 1022, 1023, 1024, 1025, 1299):
        o, L = int(off_h[i]), lens[i]
        ref = _attn_ref(orc, qkv[o:o + L].double().cpu().numpy(), L, H)
        gate_bf16(out[o:o + L], ref, what=("attention chunks", i, L))
