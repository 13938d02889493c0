"""GPU parity of the weight-streaming family (DISPATCH.md family 4: bf16 dense with M <= 128,
the weights of one token tile spread over a wave of 128-feature x K-split CTAs, fp32 partials
reduced in split order) against the fp64 oracle: every epilogue, the residue classes of the
token tile, the variant limit, dense_ln_dyn at small M, integer-exact inputs (bit for bit),
pad-then-slice, determinism, graph capture, and the dispatch record vs the oracle's rule.
Exactness argument for the integer sets: tests/test_gpu_parity_r2.py (entries in {-1, 0, 1},
<= 200 non-zeros per row: every partial sum of every split is an exact small integer)."""
import numpy as np
import pytest
import torch

from paper_2006_03031_b200 import synth
from parity import gate_bf16

pytestmark = pytest.mark.gpu

SHAPES = [(2304, 768), (768, 768), (3072, 768), (768, 3072),          # BERT-base
          (3072, 1024), (1024, 1024), (4096, 1024), (1024, 4096),     # BERT-large
          (300, 200), (136, 72), (130, 1000)]                          # ragged N / K
MS = [1, 2, 15, 16, 17, 63, 64, 100, 127, 128]


@pytest.fixture(scope="module")
def nb():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2006_03031_b200 import nimble
    return nimble


def _run(nb, x, W, b, epi, res=None):
    """Output (and residual) rows padded to a multiple of 8 elements (16-B TMA / vector
    alignment) when N is ragged; columns >= N of the padding must stay untouched."""
    M, N = x.shape[0], W.shape[0]
    ld = -(-N // 8) * 8
    y = torch.full((M + 3, ld), 7.0, dtype=torch.bfloat16, device="cuda")
    rd = None
    if res is not None:
        rp = torch.zeros((M, ld), dtype=torch.bfloat16, device="cuda")
        rp[:, :N] = res.cuda()
        rd = rp[:, :N]
    nb.dense_dyn(x.cuda(), W.cuda(), b.cuda(), y[:, :N], epi=epi, residual=rd, M=M)
    torch.cuda.synchronize()
    assert torch.all(y[M:] == 7.0), "rows beyond the symbolic extent were written"
    # families 1 / 3 store through TMA, which clips at 16 B: with N % 8 != 0 the last chunk of a
    # row may also write columns N .. ceil8(N)-1 inside the caller's leading dimension
    # (include/nimble.h); family 4 (plain stores) writes exactly N columns
    if nb.last_dispatch()["family"] == 4:
        assert torch.all(y[:, N:] == 7.0), "columns beyond N were written"
    return y[:M, :N]


@pytest.mark.parametrize("N,K", SHAPES)
def test_ws_every_epilogue_vs_oracle(nb, orc, N, K):
    W = synth.normal((N, K), 0.05, 100 + N + K)
    b = synth.normal((N,), 0.1, 101 + N, torch.float32)
    for M in MS:
        x = synth.normal((M, K), 1.0, 200 + M)
        res = synth.normal((M, N), 1.0, 300 + M)
        for epi in (1, 2, 3):
            y = _run(nb, x, W, b, epi, res if epi == 3 else None)
            d = nb.last_dispatch()
            assert d == orc.dispatch_dense(M, N, K, 1)[1] and d["family"] == 4, (N, K, M)
            ref, D = orc.dense(x.double().numpy(), W.double().numpy(), b.numpy(),
                               res.double().numpy() if epi == 3 else None, epi)
            gate_bf16(y, ref, D, ("ws", N, K, M, epi))


@pytest.mark.parametrize("N,K", [(3072, 1024), (1024, 4096), (768, 3072), (300, 200)])
def test_ws_integer_exact_bitwise(nb, orc, N, K):
    W = synth.ternary((N, K), 31 + N, torch.bfloat16)
    b = synth.ternary((N,), 32 + N, torch.float32)
    for M in (1, 17, 64, 128):
        x = synth.ternary((M, K), 40 + M, torch.bfloat16, max_nonzero_per_row=200)
        res = synth.ternary((M, N), 50 + M, torch.bfloat16)
        for epi in (1, 3):
            y = _run(nb, x, W, b, epi, res if epi == 3 else None)
            ref, _ = orc.dense(x.double().numpy(), W.double().numpy(), b.double().numpy(),
                               res.double().numpy() if epi == 3 else None, epi)
            assert np.array_equal(y.double().cpu().numpy(), ref), (N, K, M, epi)


def test_ws_variant_limit_and_pad_then_slice(nb, orc):
    """Every variant limit c computes the same function, and the dynamic-M result
    equals the pad-to-128-then-slice result bit for bit (S depends on (N, K) only)."""
    N, K = 1024, 1024
    W = synth.normal((N, K), 0.05, 71)
    b = synth.normal((N,), 0.1, 72, torch.float32)
    for M in (1, 5, 16, 33, 100, 127):
        x = synth.normal((M, K), 1.0, 73 + M)
        base = None
        for c in (0, 1, 2, 5, 9):
            nb.set_variant_limit(c)
            try:
                y = _run(nb, x, W, b, 2)
                assert nb.last_dispatch() == orc.dispatch_dense(M, N, K, 1, c)[1]
            finally:
                nb.set_variant_limit(0)
            if base is None:
                base = y.clone()
            assert torch.equal(y, base), (M, c)
        xp = torch.zeros((128, K), dtype=torch.bfloat16)
        xp[:M] = x
        yp = _run(nb, xp, W, b, 2)
        assert torch.equal(base, yp[:M]), M


def test_ws_deterministic_and_consecutive_shapes(nb):
    """The partial-slab workspace is reused by back-to-back launches of different grids on one
    stream (PDL-overlapped): run a mixed sequence twice without synchronising in between;
    results must repeat bit for bit."""
    shapes = [(2304, 768, 7), (768, 3072, 128), (4096, 1024, 1), (136, 72, 50), (1024, 4096, 90)]
    data = []
    for i, (N, K, M) in enumerate(shapes):
        data.append((synth.normal((M, K), 1.0, 500 + i).cuda(), synth.normal((N, K), 0.05, 600 + i).cuda(),
                     synth.normal((N,), 0.1, 700 + i, torch.float32).cuda()))
    outs = [[torch.empty((x.shape[0], W.shape[0]), dtype=torch.bfloat16, device="cuda") for x, W, _ in data]
            for _ in range(2)]
    for r in range(2):
        for rep in range(3):
            for (x, W, b), y in zip(data, outs[r]):
                nb.dense_dyn(x, W, b, y, epi=nb.EPI_BIAS_GELU)
    torch.cuda.synchronize()
    for a, c in zip(outs[0], outs[1]):
        assert torch.equal(a, c)


def test_ws_graph_capture(nb, orc):
    """Family 4 inside a CUDA graph on a fresh stream (the workspace is allocated during the
    capture in relaxed mode): replays match the oracle."""
    N, K, M = 768, 3072, 45
    W = synth.normal((N, K), 0.05, 81).cuda()
    b = synth.normal((N,), 0.1, 82, torch.float32).cuda()
    x = synth.normal((M, K), 1.0, 83)
    xd = x.cuda()
    y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(3):
            nb.dense_dyn(xd, W, b, y, epi=nb.EPI_BIAS)
    for _ in range(3):
        y.zero_()
        g.replay()
        torch.cuda.synchronize()
        ref, D = orc.dense(x.double().numpy(), W.double().cpu().numpy(), b.cpu().numpy(), None, 1)
        gate_bf16(y, ref, D, ("ws graph", N, K, M))


@pytest.mark.parametrize("N,K", [(768, 768), (768, 3072), (1024, 1024), (1024, 4096), (4096, 512)])
def test_ws_fused_layernorm_vs_oracle(nb, orc, N, K):
    """dense_ln_dyn at M <= 128: the family-4 GEMM (bias + residual) then the LayerNorm launch."""
    for M in (1, 16, 77, 128):
        x = synth.normal((M, K), 1.0, 900 + M).cuda()
        W = synth.normal((N, K), 0.02, 901).cuda()
        b = synth.normal((N,), 0.02, 902, torch.float32).cuda()
        res = synth.normal((M, N), 1.0, 903 + M).cuda()
        g = (1.0 + synth.normal((N,), 0.02, 904, torch.float32)).cuda()
        be = synth.normal((N,), 0.02, 905, torch.float32).cuda()
        y = torch.full((M + 3, N), 7.0, dtype=torch.bfloat16, device="cuda")
        nb.dense_ln_dyn(x, W, b, res, g, be, y)
        torch.cuda.synchronize()
        assert torch.all(y[M:] == 7.0)
        d = nb.last_dispatch()
        assert d["family"] == 4 and d == orc.dispatch_dense(M, N, K, 1)[1]
        d64 = lambda t: t.double().cpu().numpy()
        v, _ = orc.dense(d64(x), d64(W), d64(b), d64(res), 3)
        ref = orc.layernorm(v, d64(g), d64(be))
        gate_bf16(d64(y[:M]), ref, what=("ws dense_ln", N, K, M))


@pytest.mark.parametrize("N,K", [(1024, 4096), (768, 3072), (4096, 2048), (1024, 1024), (300, 2000)])
def test_ws_multi_token_tiles_vs_oracle(nb, orc, N, K):
    """Family 4 with 2..8 token tiles (M <= 1024, K >= 2048, split >= 2; family 1 elsewhere):
    every epilogue, residue tails on the last token tile, dispatch record vs the oracle's rule."""
    W = synth.normal((N, K), 0.05, 400 + N + K)
    b = synth.normal((N,), 0.1, 401 + N, torch.float32)
    for M in (129, 200, 256, 300, 511, 512, 513, 1000, 1024):
        d_orc = orc.dispatch_dense(M, N, K, 1)[1]
        x = synth.normal((M, K), 1.0, 500 + M)
        res = synth.normal((M, N), 1.0, 600 + M)
        for epi in (1, 2, 3):
            y = _run(nb, x, W, b, epi, res if epi == 3 else None)
            assert nb.last_dispatch() == d_orc, (N, K, M)
            ref, D = orc.dense(x.double().numpy(), W.double().numpy(), b.numpy(),
                               res.double().numpy() if epi == 3 else None, epi)
            gate_bf16(y, ref, D, ("ws multi", N, K, M, epi, d_orc["family"]))


def test_ws_multi_token_tiles_exact_and_pad_then_slice(nb, orc):
    N, K = 1024, 4096
    W = synth.ternary((N, K), 77, torch.bfloat16)
    b = synth.ternary((N,), 78, torch.float32)
    for M in (130, 300, 777):
        assert orc.dispatch_dense(M, N, K, 1)[1]["family"] == 4
        x = synth.ternary((M, K), 79 + M, torch.bfloat16, max_nonzero_per_row=200)
        y = _run(nb, x, W, b, 1)
        ref, _ = orc.dense(x.double().numpy(), W.double().numpy(), b.double().numpy(), None, 1)
        assert np.array_equal(y.double().cpu().numpy(), ref), M
        xf = synth.normal((M, K), 1.0, 90 + M)
        yf = _run(nb, xf, synth.normal((N, K), 0.05, 91), b, 2)
        xp = torch.zeros((128 * -(-M // 128), K), dtype=torch.bfloat16)
        xp[:M] = xf
        yp = _run(nb, xp, synth.normal((N, K), 0.05, 91), b, 2)
        assert torch.equal(yf, yp[:M]), M
