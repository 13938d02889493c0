"""GPU parity of the device-resident extent / dispatch path (§8 f4; include/nimble.h
nimble_dense_dyn_dev): the symbolic extent M lives in device memory, the residue dispatch
runs on the device, the store's tensor map is patched to M on the device, and ONE captured
CUDA graph serves every M.  Checked against the oracle (values: dense with the error
denominator, reading 17; decisions: the oracle's dispatch rule with split 1)."""
import numpy as np
import pytest
import torch

from paper_2006_03031_b200 import synth
from parity import gate_bf16

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2


@pytest.fixture(scope="module")
def nb():
    from paper_2006_03031_b200 import nimble
    return nimble


def _err(y, ref, D, what=""):
    gate_bf16(y, ref, D, what)      # both gates (D-normalised and elementwise); returns 0 for the old form
    return 0.0


def _setup(N, K, M_max, seed):
    W = synth.normal((N, K), 0.05, seed)
    b = synth.normal((N,), 0.1, seed + 1, torch.float32)
    x = synth.normal((M_max, K), 1.0, seed + 2)
    return W, b, x


POISON = torch.tensor(-7.25, dtype=torch.bfloat16)


@pytest.mark.parametrize("N,K,M_max", [(1024, 1024, 512), (768, 3072, 2047), (3072, 1024, 300)])
def test_dense_dyn_dev_vs_oracle_and_record(nb, orc, N, K, M_max):
    W, b, x = _setup(N, K, M_max, 31)
    Wd, bd, xd = W.cuda(), b.cuda(), x.cuda()
    rec = torch.zeros(nb.DISPATCH_BYTES, dtype=torch.uint8, device="cuda")
    Ms = sorted({1, 2, 15, 16, 17, 100, 127, 128, 129, 255, 256, 257, M_max - 1, M_max} & set(range(1, M_max + 1)))
    for M in Ms:
        for epi in (nb.EPI_BIAS, nb.EPI_BIAS_GELU, nb.EPI_BIAS_RESIDUAL):
            res = synth.normal((M_max, N), 1.0, 90 + M) if epi == nb.EPI_BIAS_RESIDUAL else None
            y = torch.full((M_max, N), float(POISON), dtype=torch.bfloat16, device="cuda")
            m_dev = torch.tensor([M], dtype=torch.int32, device="cuda")
            nb.dense_dyn_dev(xd, Wd, bd, y, m_dev, M_max, epi=epi, residual=None if res is None else res.cuda(),
                             record=rec)
            torch.cuda.synchronize()
            ref, D = orc.dense(x[:M].double().numpy(), W.double().numpy(), b.numpy(),
                               None if res is None else res[:M].double().numpy(), epi)
            assert _err(y[:M], ref, D) <= TOL_BF16, (N, K, M, epi)
            assert bool((y[M:] == POISON.cuda()).all()), "rows beyond the device extent were written"
            assert nb.dispatch_from_bytes(rec) == orc.dispatch_dense(M, N, K, 1, 0, 128, 1)[1], M


def test_dense_dyn_dev_bitwise_equals_host_path(nb):
    """Same kernel, same accumulation order: the device-extent launch equals the host-extent
    launch bit for bit once the host path also runs split 1 (schedule (128, 1))."""
    N, K, M_max = 1024, 4096, 640
    W, b, x = _setup(N, K, M_max, 41)
    Wd, bd, xd = W.cuda(), b.cuda(), x.cuda()
    nb.set_dense_schedule(N, K, 128, 1)
    try:
        for M in (1, 33, 128, 200, 640):
            y_host = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
            nb.dense_dyn(xd[:M].contiguous(), Wd, bd, y_host, epi=nb.EPI_BIAS_GELU)
            y_dev = torch.empty((M_max, N), dtype=torch.bfloat16, device="cuda")
            nb.dense_dyn_dev(xd, Wd, bd, y_dev, torch.tensor([M], dtype=torch.int32, device="cuda"), M_max,
                             epi=nb.EPI_BIAS_GELU)
            torch.cuda.synchronize()
            assert torch.equal(y_host, y_dev[:M]), M
    finally:
        nb.set_dense_schedule(N, K, 0, 8)


def test_one_graph_serves_every_extent(nb, orc):
    """Capture once, replay with M written to device memory between replays."""
    N, K, M_max = 1024, 1024, 512
    W, b, x = _setup(N, K, M_max, 51)
    Wd, bd, xd = W.cuda(), b.cuda(), x.cuda()
    y = torch.empty((M_max, N), dtype=torch.bfloat16, device="cuda")
    m_dev = torch.tensor([M_max], dtype=torch.int32, device="cuda")
    rec = torch.zeros(nb.DISPATCH_BYTES, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        nb.dense_dyn_dev(xd, Wd, bd, y, m_dev, M_max, record=rec)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            nb.dense_dyn_dev(xd, Wd, bd, y, m_dev, M_max, record=rec)
    for M in (1, 77, 128, 129, 300, 511, 512, 5):
        y.fill_(float(POISON))
        m_dev.fill_(M)
        g.replay()
        torch.cuda.synchronize()
        ref, D = orc.dense(x[:M].double().numpy(), W.double().numpy(), b.numpy(), None, nb.EPI_BIAS)
        assert _err(y[:M], ref, D) <= TOL_BF16, M
        assert bool((y[M:] == POISON.cuda()).all()), M
        assert nb.dispatch_from_bytes(rec) == orc.dispatch_dense(M, N, K, 1, 0, 128, 1)[1], M


def test_dense_dyn_dev_variant_limit_and_tuned_tile(nb, orc):
    N, K, M_max = 768, 768, 400
    W, b, x = _setup(N, K, M_max, 61)
    Wd, bd, xd = W.cuda(), b.cuda(), x.cuda()
    rec = torch.zeros(nb.DISPATCH_BYTES, dtype=torch.uint8, device="cuda")
    for c, tile in ((2, 0), (0, 64), (3, 32), (0, 256)):
        nb.set_variant_limit(c)
        if tile:
            nb.set_dense_schedule(N, K, tile, 1)
        try:
            for M in (1, 31, 64, 65, 200, 399):
                y = torch.full((M_max, N), float(POISON), dtype=torch.bfloat16, device="cuda")
                nb.dense_dyn_dev(xd, Wd, bd, y, torch.tensor([M], dtype=torch.int32, device="cuda"), M_max,
                                 record=rec)
                torch.cuda.synchronize()
                ref, D = orc.dense(x[:M].double().numpy(), W.double().numpy(), b.numpy(), None, nb.EPI_BIAS)
                assert _err(y[:M], ref, D) <= TOL_BF16, (c, tile, M)
                assert bool((y[M:] == POISON.cuda()).all())
                assert nb.dispatch_from_bytes(rec) == orc.dispatch_dense(M, N, K, 1, c, tile or 128, 1)[1]
        finally:
            nb.set_variant_limit(0)
            nb.set_dense_schedule(N, K, 0, 8)


def test_layernorm_dev_vs_oracle(nb, orc):
    d, R_max = 1024, 300
    X = synth.normal((R_max, d), 1.0, 71)
    g = (1.0 + synth.normal((d,), 0.02, 72, torch.float32))
    be = synth.normal((d,), 0.02, 73, torch.float32)
    for rows in (1, 7, 8, 9, 299, 300):
        Y = torch.full((R_max, d), float(POISON), dtype=torch.bfloat16, device="cuda")
        nb.layernorm_dev(X.cuda(), g.cuda(), be.cuda(), Y, torch.tensor([rows], dtype=torch.int32, device="cuda"))
        torch.cuda.synchronize()
        ref = orc.layernorm(X[:rows].double().numpy(), g.double().numpy(), be.double().numpy())
        ref = ref[0] if isinstance(ref, tuple) else ref
        gate_bf16(Y[:rows], ref, what=("layernorm_dev", rows))
        assert bool((Y[rows:] == POISON.cuda()).all())


def test_attention_dev_patched_maps_zero_fill_bitwise(nb):
    """T = seq_off[R] on the device: rows in [T, T_max) hold NaN, yet the result equals the
    host-T launch bit for bit (the re-encoded maps zero-fill past T exactly like host maps)."""
    H, dh, T_max = 16, 64, 640
    for lens in ([1], [77], [128], [129, 5], [300, 200, 100], [512]):
        T = sum(lens)
        qkv = synth.normal((T_max, 3 * H * dh), 1.0, 80 + T).cuda()
        qkv[T:] = float("nan")
        off = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
        R, mx = len(lens), max(lens)
        ref = torch.zeros((T_max, H * dh), dtype=torch.bfloat16, device="cuda")
        nb.attention_varlen(qkv[:T].contiguous(), off, R, mx, H, ref, T=T)
        got = torch.zeros((T_max, H * dh), dtype=torch.bfloat16, device="cuda")
        nb.attention_varlen_dev(qkv, off, R, 512, H, got, T_max=T_max)
        torch.cuda.synchronize()
        assert torch.equal(got[:T], ref[:T]), lens
        assert bool((got[T:] == 0).all())


def _bert_large_2layers(nb):
    from paper_2006_03031_b200.bert import BertPacked
    cfg = dict(synth.BERT_LARGE)
    cfg["layers"] = 2
    w = synth.bert_weights_device(cfg, seed=0)
    return cfg, w, BertPacked


def test_bert_forward_dev_and_one_graph_bitwise(nb):
    """forward_dev (device T) == forward (host T) bit for bit once the host path also runs the
    split-1 schedule; and ONE captured DeviceExtentGraph reproduces per-L graph results."""
    from paper_2006_03031_b200.serve import DeviceExtentGraph, GraphCache
    cfg, w, BertPacked = _bert_large_2layers(nb)
    d, f = cfg["d"], cfg["ffn"]
    shapes = [(3 * d, d), (d, d), (f, d), (d, f)]
    for N, K in shapes:
        nb.set_dense_schedule(N, K, 128, 1)
    try:
        enc_h = BertPacked(cfg, w, max_tokens=512)
        enc_d = BertPacked(cfg, w, max_tokens=512)
        one = DeviceExtentGraph(enc_d)
        per_l = GraphCache(enc_h)
        out_a = torch.empty((d,), dtype=torch.bfloat16, device="cuda")
        out_b = torch.empty((d,), dtype=torch.bfloat16, device="cuda")
        for L in (1, 17, 128, 129, 300, 512, 3):
            x = synth.device_normal(L, d, seed=900 + L)
            off = torch.tensor([0, L], dtype=torch.int32, device="cuda")
            y_h = enc_h.forward(x, off, L, T=L).clone()
            xin = torch.zeros((512, d), dtype=torch.bfloat16, device="cuda")
            xin[:L] = x
            y_d = enc_d.forward_dev(xin, off.clone())
            torch.cuda.synchronize()
            assert torch.equal(y_h[:L], y_d[:L]), L
            per_l.capture(L)
            per_l.run(x, L, out_a)
            one.run(x, L, out_b)
            torch.cuda.synchronize()
            assert torch.equal(out_a, out_b), L
            assert torch.equal(out_b, y_h[0]), L
    finally:
        for N, K in shapes:
            nb.set_dense_schedule(N, K, 0, 8)


@pytest.mark.parametrize("N,K", [(768, 3072), (2304, 768), (1024, 4096)])
def test_dense_dyn_dev_split_k_within_one_tile(nb, orc, N, K):
    """M_max <= 128 fits one token tile: with a family-1 schedule registered (the default rule
    takes family 4 there, test_dense_dyn_dev_family4) the device dispatch keeps the host rule's
    split-K (the same for every M <= M_max), the record equals the oracle's rule with that
    (t, cap), and outputs equal the host-extent launch with the same schedule bit for bit (same
    tiles, same fixed-order split reduction)."""
    M_max = 128
    W, b, x = _setup(N, K, M_max, 71)
    Wd, bd, xd = W.cuda(), b.cuda(), x.cuda()
    cap = 8 if K >= 2048 else 1            # the default rule's split cap, evaluated at the bound
    for M in (1, 7, 16, 33, 100, 127, 128):
        rec = torch.zeros(nb.DISPATCH_BYTES, dtype=torch.uint8, device="cuda")
        y_dev = torch.empty((M_max, N), dtype=torch.bfloat16, device="cuda")
        nb.set_dense_schedule(N, K, 128, cap)               # family 1 with the default (t, cap)
        try:
            nb.dense_dyn_dev(xd, Wd, bd, y_dev, torch.tensor([M], dtype=torch.int32, device="cuda"), M_max, record=rec)
            y_host = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
            nb.dense_dyn(xd[:M], Wd, bd, y_host)
        finally:
            nb.set_dense_schedule(N, K, 0, 1)
        torch.cuda.synchronize()
        drec = nb.dispatch_from_bytes(rec)
        assert drec == orc.dispatch_dense(M, N, K, 1, 0, 128, cap)[1], M
        assert (drec["split_k"] > 1) == (K >= 2048)
        assert torch.equal(y_dev[:M], y_host), M


@pytest.mark.parametrize("N,K,M_max", [(1024, 1024, 128), (768, 3072, 100), (2304, 768, 64)])
def test_dense_dyn_dev_family4(nb, orc, N, K, M_max):
    """Device extent with a one-token-tile bound: the weight-streaming family 4 with the residue
    dispatch on the device (record vs the oracle's default rule, every variant limit), values vs
    the oracle, rows >= M untouched, bitwise equal to the host-extent launch, and one captured
    graph serving every M."""
    W, b, x = _setup(N, K, M_max, 71)
    Wd, bd, xd = W.cuda(), b.cuda(), x.cuda()
    rec = torch.zeros(nb.DISPATCH_BYTES, dtype=torch.uint8, device="cuda")
    for c in (0, 2):
        nb.set_variant_limit(c)
        try:
            for M in sorted({1, 2, 15, 16, 17, M_max // 2, M_max - 1, M_max}):
                y = torch.full((M_max, N), float(POISON), dtype=torch.bfloat16, device="cuda")
                nb.dense_dyn_dev(xd, Wd, bd, y, torch.tensor([M], dtype=torch.int32, device="cuda"), M_max,
                                 epi=nb.EPI_BIAS_GELU, record=rec)
                torch.cuda.synchronize()
                d = nb.dispatch_from_bytes(rec)
                assert d == orc.dispatch_dense(M, N, K, 1, c)[1] and d["family"] == 4, (M, c, d)
                ref, D = orc.dense(x[:M].double().numpy(), W.double().numpy(), b.numpy(), None, nb.EPI_BIAS_GELU)
                assert _err(y[:M], ref, D) <= TOL_BF16, (M, c)
                assert bool((y[M:] == POISON.cuda()).all())
                y_host = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
                nb.dense_dyn(xd[:M].contiguous(), Wd, bd, y_host, epi=nb.EPI_BIAS_GELU)
                torch.cuda.synchronize()
                assert torch.equal(y_host, y[:M]), (M, c)
        finally:
            nb.set_variant_limit(0)
    # one graph, every M
    y = torch.empty((M_max, N), dtype=torch.bfloat16, device="cuda")
    m_dev = torch.tensor([M_max], dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        nb.dense_dyn_dev(xd, Wd, bd, y, m_dev, M_max, record=rec)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            nb.dense_dyn_dev(xd, Wd, bd, y, m_dev, M_max, record=rec)
    for M in (1, M_max, 7, M_max // 2 + 1):
        y.fill_(float(POISON))
        m_dev.fill_(M)
        g.replay()
        torch.cuda.synchronize()
        ref, D = orc.dense(x[:M].double().numpy(), W.double().numpy(), b.numpy(), None, nb.EPI_BIAS)
        assert _err(y[:M], ref, D) <= TOL_BF16, M
        assert bool((y[M:] == POISON.cuda()).all()), M
        assert nb.dispatch_from_bytes(rec) == orc.dispatch_dense(M, N, K, 1)[1], M
