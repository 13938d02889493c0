"""Parity at the bench's full size and launch configuration (BASELINE config 5, BJ:11): the
64-request L ~ U{1..512} stream of `bench.py` (synth seeds 2 / 1, device-drawn BERT-large
weights, T = 17448 packed tokens), one encoder layer through `BertPacked.layer` exactly as the
bench launches it (family-3 GEMMs at M = T, persistent varlen attention, LN1 launch, FFN2 with
the fused LN2 epilogue).  The oracle cannot run 17448 x 24 layers, so every op is checked
teacher-forced on a seeded sample of whole requests (attention needs all rows of a request)
spanning short, long and tail-tile requests, in fp64 from the device's own inputs to that op.
Gate: dense ops max |y - y*| / D <= 2e-2 (D = sum |x||W| + |b| + |res|); row ops abs error over
max(|y*|, 1) <= 2e-2."""
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


def test_bench_config_layer_sampled(nb, orc):
    from paper_2006_03031_b200.bert import BertPacked
    cfg = synth.BERT_LARGE
    lens = synth.request_lengths(64, seed=2)
    T = int(lens.sum())
    assert T >= 2048                                           # the bench's M runs family 3
    w = synth.bert_weights_device(cfg, seed=0, layers=1)
    enc = BertPacked(cfg, w, max_tokens=T)
    off_h = np.concatenate([[0], np.cumsum(lens)])
    off = torch.tensor(off_h, dtype=torch.int32, device="cuda")
    x = synth.device_normal(T, cfg["d"], seed=1)
    s = torch.cuda.current_stream().cuda_stream
    out = torch.empty((T, cfg["d"]), dtype=torch.bfloat16, device="cuda")
    enc.layer(x.data_ptr(), out.data_ptr(), T, off.data_ptr(), len(lens), int(lens.max()), 0, s)
    torch.cuda.synchronize()
    d, H = cfg["d"], cfg["heads"]
    W = {k: v.double().cpu().numpy() for k, v in w[0].items()}
    rows = lambda t, a, b: t[a:b].double().cpu().numpy()
    # sample: the shortest, the longest, and requests whose rows straddle a 256-token tile edge
    order = np.argsort(lens)
    pick = {int(order[0]), int(order[-1]), int(order[len(order) // 2])}
    for i in range(len(lens)):
        if off_h[i] // 256 != (off_h[i + 1] - 1) // 256:
            pick.add(i)
        if len(pick) >= 6:
            break
    for i in sorted(pick):
        o, L = int(off_h[i]), int(lens[i])
        ref, D = orc.dense(rows(x, o, o + L), W["Wqkv"], W["bqkv"], None, 1)
        gate_bf16(rows(enc.qkv, o, o + L), ref, D, ("bench qkv", i, L))
        qkv = rows(enc.qkv, o, o + L)
        att = np.empty((L, d))
        for h in range(H):
            q, k, v = (qkv[:, c + 64 * h:c + 64 * h + 64] for c in (0, d, 2 * d))
            sc, _ = orc.bmm(q[None], k[None], 0, 0.125)
            c2, _ = orc.bmm(orc.softmax_rows(sc[0])[None], v[None], 1)
            att[:, 64 * h:64 * h + 64] = c2[0]
        gate_bf16(enc.ctx[o:o + L], att, what=("bench attention", i, L))
        v1, _ = orc.dense(rows(enc.ctx, o, o + L), W["Wo"], W["bo"], rows(x, o, o + L), 3)
        gate_bf16(enc.H1[o:o + L], orc.layernorm(v1, W["g1"], W["be1"]), what=("bench o-proj+ln1", i, L))
        ref, D = orc.dense(rows(enc.H1, o, o + L), W["W1"], W["b1"], None, 2)
        gate_bf16(rows(enc.F, o, o + L), ref, D, ("bench ffn1+gelu", i, L))
        v2, _ = orc.dense(rows(enc.F, o, o + L), W["W2"], W["b2"], rows(enc.H1, o, o + L), 3)
        gate_bf16(out[o:o + L], orc.layernorm(v2, W["g2"], W["be2"]), what=("bench ffn2+ln2 fused", i, L))
