"""GPU parity: nimble_dense_dyn / nimble_bmm_dyn (through the C ABI) vs the fp64 oracle.

Gate (BJ:5, reading 17): err = max |y - y*| / D, D = sum |x||W| + |b| + |res|
(the componentwise error-bound denominator the oracle returns):
  fp32 (SIMT8)  err <= 1e-4;   bf16 in / fp32 accumulate   err <= 2e-2.
Integer-valued inputs make every partial sum exact, so those runs are bit-exact.
Every case also checks that the launched dispatch equals the oracle's (bit-exact).
"""
import numpy as np
import pytest
import torch

from paper_2006_03031_b200 import synth
from parity import gate, gate_bf16, gate_f32

pytestmark = pytest.mark.gpu
TOL_F32, TOL_BF16 = 1e-4, 2e-2


@pytest.fixture(scope="module")
def nb():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2006_03031_b200 import nimble
    return nimble


def _err(y, ref, D):
    y = y.double().cpu().numpy()
    return float(np.max(np.abs(y - ref) / np.maximum(D, 1e-30)))


def _dense_gpu(nb, x, W, b, epi, res=None, M=None, ypad=0, poison=True):
    """Run dense_dyn on device with poisoned rows beyond M in x and sentinel rows in y."""
    M = x.shape[0] if M is None else M
    dev = "cuda"
    xd = torch.empty((M + 3, x.shape[1]), dtype=x.dtype, device=dev)
    xd[M:] = float("nan") if poison else 0.0              # rows >= M must never be read
    xd[:M] = x.to(dev)
    N = W.shape[0]
    y = torch.full((M + 3, N + ypad), 7.0, dtype=x.dtype, device=dev)   # rows >= M must stay 7
    resd = res.to(dev) if res is not None else None
    nb.dense_dyn(xd, W.to(dev), b.to(dev) if b is not None else None, y, epi=epi, residual=resd, M=M)
    torch.cuda.synchronize()
    assert torch.all(y[M:] == 7.0), "wrote rows beyond the symbolic extent"
    return y[:M, :N]


# ------------------------------------------------------------------ config 1: fp32 SIMT8
def test_config1_fp32_every_residue(nb, orc):
    for M in range(1, 65):
        x, W, b = synth.config1_dense(M)
        for epi in (nb.EPI_NONE, nb.EPI_BIAS, nb.EPI_BIAS_GELU, nb.EPI_BIAS_RESIDUAL):
            res = synth.uniform((M, 128), -1, 1, 77 + M) if epi == nb.EPI_BIAS_RESIDUAL else None
            y = _dense_gpu(nb, x, W, b, epi, res)
            ref, D = orc.dense(x.numpy(), W.numpy(), b.numpy(), None if res is None else res.numpy(), epi)
            gate_f32(y, ref, D, ("config1", M, epi))
            assert nb.last_dispatch() == orc.dispatch_dense(M, 128, 128, 0)[1]


def test_config1_integer_exact_and_variant_limit(nb, orc):
    for M in (1, 5, 8, 13, 63, 64):
        x = synth.ternary((M, 128), 5 + M, torch.float32)
        W = synth.ternary((128, 128), 6, torch.float32)
        b = synth.ternary((128,), 7, torch.float32)
        ref, _ = orc.dense(x.numpy(), W.numpy(), b.numpy(), None, 1)
        outs = []
        for c in (0, 1, 2, 4, 8):
            nb.set_variant_limit(c)
            try:
                y = _dense_gpu(nb, x, W, b, nb.EPI_BIAS)
                assert nb.last_dispatch() == orc.dispatch_dense(M, 128, 128, 0, c)[1]
            finally:
                nb.set_variant_limit(0)
            assert np.array_equal(y.double().cpu().numpy(), ref), (M, c)
            outs.append(y)
        for y in outs[1:]:
            assert torch.equal(y, outs[0])


def test_fp32_general_shapes(nb, orc):
    for (M, N, K) in ((3, 130, 44), (77, 300, 256), (200, 2600, 652)):
        x = synth.normal((M, K), 1.0, 11, torch.float32)
        W = synth.normal((N, K), 0.05, 12, torch.float32)
        b = synth.normal((N,), 0.1, 13, torch.float32)
        y = _dense_gpu(nb, x, W, b, nb.EPI_BIAS)
        ref, D = orc.dense(x.numpy(), W.numpy(), b.numpy(), None, 1)
        gate_f32(y, ref, D, ("fp32", M, N, K))


# ------------------------------------------------------------------ bf16 tcgen05 dense
BF16_SHAPES = [(128, 64), (384, 768), (1024, 1024), (256, 4096)]
BF16_MS = [1, 7, 16, 17, 100, 128, 200, 255, 256, 257, 300, 511, 512, 513, 777]


@pytest.mark.parametrize("N,K", BF16_SHAPES)
def test_bf16_dense_vs_oracle(nb, orc, N, K):
    W = synth.normal((N, K), 0.05, 21)
    b = synth.normal((N,), 0.1, 22, torch.float32)
    for M in BF16_MS:
        x = synth.normal((M, K), 1.0, 1000 + M)
        for epi in (nb.EPI_BIAS, nb.EPI_BIAS_GELU, nb.EPI_BIAS_RESIDUAL):
            res = synth.normal((M, N), 1.0, 33 + M) if epi == nb.EPI_BIAS_RESIDUAL else None
            y = _dense_gpu(nb, x, W, b, epi, res)
            ref, D = orc.dense(x.double().numpy(), W.double().numpy(), b.numpy(),
                               None if res is None else res.double().numpy(), epi)
            gate_bf16(y, ref, D, ("bf16 dense", N, K, M, epi))
            assert nb.last_dispatch() == orc.dispatch_dense(M, N, K, 1)[1]


@pytest.mark.parametrize("tile_t,split_max", [(32, 8), (64, 1), (64, 8), (128, 1), (256, 2), (256, 8)])
def test_bf16_tuned_schedule_vs_oracle(nb, orc, tile_t, split_max):
    """Every tunable schedule (token tile t, split-K cap) computes the same op: parity with
    the oracle at residues of t (incl. the tail widths 16..t) and the dispatch record equals
    the oracle's schedule-aware dispatch."""
    N, K = 1024, 4096
    W = synth.normal((N, K), 0.05, 71)
    b = synth.normal((N,), 0.1, 72, torch.float32)
    nb.set_dense_schedule(N, K, tile_t, split_max)
    try:
        for M in (1, 15, 17, 31, 33, 64, 65, 100, 129, 200, 255, 257, 513, 1000):
            x = synth.normal((M, K), 1.0, 2000 + M)
            for epi in (nb.EPI_BIAS, nb.EPI_BIAS_RESIDUAL):
                res = synth.normal((M, N), 1.0, 77 + M) if epi == nb.EPI_BIAS_RESIDUAL else None
                y = _dense_gpu(nb, x, W, b, epi, res)
                ref, D = orc.dense(x.double().numpy(), W.double().numpy(), b.numpy(),
                                   None if res is None else res.double().numpy(), epi)
                gate_bf16(y, ref, D, ("tuned", tile_t, split_max, M, epi))
                assert nb.last_dispatch() == orc.dispatch_dense(M, N, K, 1, 0, tile_t, split_max)[1]
    finally:
        nb.set_dense_schedule(N, K, 0, 8)


@pytest.mark.parametrize("N,K", [(256, 256), (1024, 4096), (3072, 1024)])
def test_bf16_integer_exact_bitwise(nb, orc, N, K):
    W = synth.ternary((N, K), 31, torch.bfloat16)
    b = synth.ternary((N,), 32, torch.float32)
    for M in (1, 16, 33, 256, 300, 600):
        x = synth.ternary((M, K), 40 + M, torch.bfloat16, max_nonzero_per_row=200)
        res = synth.ternary((M, N), 50 + M, torch.bfloat16)
        y = _dense_gpu(nb, x, W, b, nb.EPI_BIAS_RESIDUAL, res)
        ref, _ = orc.dense(x.double().numpy(), W.double().numpy(), b.numpy(), res.double().numpy(), 3)
        assert np.array_equal(y.double().cpu().numpy(), ref), (N, K, M)


def test_bf16_variant_limit_same_result(nb, orc):
    N, K = 512, 1024
    W = synth.normal((N, K), 0.05, 61)
    b = synth.normal((N,), 0.1, 62, torch.float32)
    for M in (5, 100, 300, 497):
        x = synth.normal((M, K), 1.0, 63 + M)
        ref, D = orc.dense(x.double().numpy(), W.double().numpy(), b.numpy(), None, 1)
        base = None
        for c in (0, 1, 2, 9, 17):
            nb.set_variant_limit(c)
            try:
                y = _dense_gpu(nb, x, W, b, nb.EPI_BIAS)
                assert nb.last_dispatch() == orc.dispatch_dense(M, N, K, 1, c)[1]
            finally:
                nb.set_variant_limit(0)
            gate_bf16(y, ref, D, ("variant limit", M, c))
            if base is None:
                base = y
            assert torch.equal(y, base), (M, c)         # residue variants compute the same function


def test_bf16_pad_then_slice_bitwise(nb):
    # dynamic M result == pad-to-static (zero rows) then slice, bit for bit (BJ:5 invariant)
    N, K = 384, 768
    W = synth.normal((N, K), 0.05, 71)
    b = synth.normal((N,), 0.1, 72, torch.float32)
    for M in (3, 129, 250, 259):
        x = synth.normal((M, K), 1.0, 73 + M)
        y = _dense_gpu(nb, x, W, b, nb.EPI_BIAS)
        Mp = 128 * ((M + 127) // 128)
        xp = torch.zeros((Mp, K), dtype=torch.bfloat16)
        xp[:M] = x
        yp = _dense_gpu(nb, xp, W, b, nb.EPI_BIAS)
        assert torch.equal(y, yp[:M])


def test_bf16_deterministic(nb):
    N, K = 1024, 4096          # split-K cluster path at small M
    W = synth.normal((N, K), 0.05, 81)
    b = synth.normal((N,), 0.1, 82, torch.float32)
    x = synth.normal((40, K), 1.0, 83)
    y1 = _dense_gpu(nb, x, W, b, nb.EPI_BIAS)
    assert nb.last_dispatch()["split_k"] > 1
    for _ in range(3):
        assert torch.equal(_dense_gpu(nb, x, W, b, nb.EPI_BIAS), y1)


# ------------------------------------------------------------------ bmm_dyn (attention shapes)
def _qkv(L, d, seed):
    return synth.normal((L, 3 * d), 1.0, seed)


@pytest.mark.parametrize("L", [1, 9, 64, 128, 130, 255, 256, 300, 512])
def test_bmm_scores_and_context_vs_oracle(nb, orc, L):
    H, dh = 16, 64
    d = H * dh
    qkv = _qkv(L, d, 90 + L).cuda()
    ldS = 8 * ((L + 7) // 8)
    S = torch.full((H, L, ldS), 7.0, dtype=torch.float32, device="cuda")
    # scores: S_h = Q_h K_h^T / 8, Q_h/K_h are strided views into QKV (batch stride 64 elements)
    base = qkv.data_ptr()
    nb.bmm_dyn(base, 3 * d, dh, base + 2 * d, 3 * d, dh, 0, S, ldS, L * ldS, H, L, L, dh, alpha=0.125)
    torch.cuda.synchronize()
    assert nb.last_dispatch() == orc.dispatch_bmm(H, L, L, dh, 0, 1)[1]
    q = qkv[:, :d].double().cpu().numpy().reshape(L, H, dh).transpose(1, 0, 2)
    k = qkv[:, d:2 * d].double().cpu().numpy().reshape(L, H, dh).transpose(1, 0, 2)
    v = qkv[:, 2 * d:].double().cpu().numpy().reshape(L, H, dh).transpose(1, 0, 2)
    ref, D = orc.bmm(q, k, 0, 0.125)
    Sg = S[:, :, :L].double().cpu().numpy()
    gate(Sg, ref, D, TOL_BF16, ("bmm scores fp32 out", L))
    assert torch.all(S[:, :, 4 * ((L + 3) // 4):] == 7.0)     # TMA may fill the row's last 16-B segment
    # context: C_h = P_h V_h with V_h MN-major (trans_b = 1), P bf16 [H x L x ldP]
    ldP = 8 * ((L + 7) // 8)
    P = synth.normal((H, L, ldP), 0.5, 95 + L).cuda()
    ctx = torch.full((L, d), 7.0, dtype=torch.bfloat16, device="cuda")
    nb.bmm_dyn(P, ldP, L * ldP, base + 4 * d, 3 * d, dh, 1, ctx.data_ptr(), d, dh, H, L, dh, L, alpha=1.0,
               out_dt=nb.BF16)
    torch.cuda.synchronize()
    assert nb.last_dispatch() == orc.dispatch_bmm(H, L, dh, L, 1, 1)[1]
    Pn = P[:, :, :L].double().cpu().numpy()
    refc, Dc = orc.bmm(Pn, v, 1, 1.0)
    cg = ctx.double().cpu().numpy().reshape(L, H, dh).transpose(1, 0, 2)
    gate_bf16(cg, refc, Dc, ("bmm context", L))


def test_bmm_integer_exact(nb, orc):
    H, L, dh = 4, 200, 64
    A = synth.ternary((H * L, dh), 101, torch.bfloat16).reshape(H, L, dh).cuda()
    B = synth.ternary((H * L, dh), 102, torch.bfloat16).reshape(H, L, dh).cuda()
    C = torch.empty((H, L, L), dtype=torch.float32, device="cuda")
    nb.bmm_dyn(A, dh, L * dh, B, dh, L * dh, 0, C, L, L * L, H, L, L, dh)
    ref, _ = orc.bmm(A.double().cpu().numpy(), B.double().cpu().numpy(), 0)
    assert np.array_equal(C.double().cpu().numpy(), ref)
    Bt = synth.ternary((H * L, dh), 103, torch.bfloat16).reshape(H, L, dh).cuda()
    P = synth.ternary((H * L, L), 104, torch.bfloat16).reshape(H, L, L)
    P = torch.nn.functional.pad(P, (0, 8 * ((L + 7) // 8) - L)).contiguous().cuda()
    ldP = P.shape[2]
    C2 = torch.empty((H, L, dh), dtype=torch.float32, device="cuda")
    nb.bmm_dyn(P, ldP, L * ldP, Bt, dh, L * dh, 1, C2, dh, L * dh, H, L, dh, L)
    ref2, _ = orc.bmm(P[:, :, :L].double().cpu().numpy(), Bt.double().cpu().numpy(), 1)
    assert np.array_equal(C2.double().cpu().numpy(), ref2)


# ------------------------------------------------------------------ static twins
def test_static_twin_bitwise_equal(nb, orc):
    # the static-shape instantiation computes exactly what the symbolic kernel computes.  The
    # twins are family-1/3 kernels; where the default rule picks family 4 the symbolic family-1
    # kernel is selected with the default rule's (t, cap) as a schedule.
    for (M, N, K) in ((128, 3072, 1024), (527, 3072, 1024), (513, 1024, 4096), (128, 768, 3072)):
        W = synth.normal((N, K), 0.05, 3 + M)
        b = synth.normal((N,), 0.1, 4 + M, torch.float32)
        x = synth.normal((M, K), 1.0, 5 + M)
        nb.set_dense_schedule(N, K, 128, 8 if K >= 2048 else 1)
        try:
            y1 = _dense_gpu(nb, x, W, b, nb.EPI_BIAS)
            assert nb.last_dispatch()["family"] in (1, 3)
        finally:
            nb.set_dense_schedule(N, K, 0, 8)
        Wd, bd, xd = W.cuda(), b.cuda(), x.cuda()
        y2 = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
        nb.dense_static(xd, Wd, bd, y2)
        torch.cuda.synchronize()
        assert torch.equal(y1, y2), (M, N, K)
    for M in (1, 8, 13, 64):
        x, W, b = synth.config1_dense(M)
        y1 = _dense_gpu(nb, x, W, b, nb.EPI_BIAS)
        y2 = torch.empty((M, 128), dtype=torch.float32, device="cuda")
        nb.dense_static(x.cuda(), W.cuda(), b.cuda(), y2)
        torch.cuda.synchronize()
        assert torch.equal(y1, y2), M
    with pytest.raises(nb.NimbleError):
        nb.dense_static(torch.zeros((77, 1024), dtype=torch.bfloat16, device="cuda"),
                        torch.zeros((3072, 1024), dtype=torch.bfloat16, device="cuda"),
                        torch.zeros((3072,), device="cuda"),
                        torch.zeros((77, 3072), dtype=torch.bfloat16, device="cuda"))


@pytest.mark.parametrize("M", [3713, 3840, 4111, 4300])
def test_bf16_large_m_cta_pairs(nb, orc, M):
    # family 3: 2-CTA pairs (tcgen05 cta_group::2), each CTA loads half of the token tile; at
    # N = 640 the pairs need fewer waves than 128 x 128 tiles from M = 3713 (DISPATCH.md)
    N, K = 640, 256
    W = synth.normal((N, K), 0.05, 91)
    b = synth.normal((N,), 0.1, 92, torch.float32)
    x = synth.normal((M, K), 1.0, 93 + M)
    for epi in (nb.EPI_BIAS, nb.EPI_BIAS_GELU, nb.EPI_BIAS_RESIDUAL):
        res = synth.normal((M, N), 1.0, 94 + M) if epi == nb.EPI_BIAS_RESIDUAL else None
        y = _dense_gpu(nb, x, W, b, epi, res)
        d = nb.last_dispatch()
        assert d == orc.dispatch_dense(M, N, K, 1)[1] and d["cluster"] == (2, 1, 1)
        ref, D = orc.dense(x.double().numpy(), W.double().numpy(), b.numpy(),
                           None if res is None else res.double().numpy(), epi)
        gate_bf16(y, ref, D, ("family 3", M, epi))
    xi = synth.ternary((M, K), 95 + M, torch.bfloat16, max_nonzero_per_row=200)
    Wi = synth.ternary((N, K), 96, torch.bfloat16)
    bi = synth.ternary((N,), 97, torch.float32)
    y = _dense_gpu(nb, xi, Wi, bi, nb.EPI_BIAS)
    ref, _ = orc.dense(xi.double().numpy(), Wi.double().numpy(), bi.numpy(), None, 1)
    assert np.array_equal(y.double().cpu().numpy(), ref)


@pytest.mark.parametrize("M,N", [(77, 200), (300, 72), (2100, 520), (2049, 264)])
def test_bf16_partial_feature_boxes(nb, orc, M, N):
    """N not a multiple of the 64-feature swizzled store box (nor of 128 / 256): the epilogue's
    last store / residual box is clipped by TMA, every epilogue kind, families 1 and 3."""
    K = 192
    W = synth.normal((N, K), 0.05, 500 + N)
    b = synth.normal((N,), 0.1, 501 + N, torch.float32)
    x = synth.normal((M, K), 1.0, 502 + M)
    for epi in (nb.EPI_BIAS, nb.EPI_BIAS_GELU, nb.EPI_BIAS_RESIDUAL):
        res = synth.normal((M, N), 1.0, 503 + M) if epi == nb.EPI_BIAS_RESIDUAL else None
        y = _dense_gpu(nb, x, W, b, epi, res)
        ref, D = orc.dense(x.double().numpy(), W.double().numpy(), b.numpy(),
                           None if res is None else res.double().numpy(), epi)
        gate_bf16(y, ref, D, ("partial feature boxes", M, N, epi))
