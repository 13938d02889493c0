"""GPU parity of the device-resident extent / dispatch path (§8 f4; include/nimble.h
nimble_dense_dyn_dev): the symbolic extent M lives in device memory, the residue dispatch
runs on the device, the store's tensor map is patched to M on the device, and ONE captured
CUDA graph serves every M.  Checked against the oracle (values: dense with the error
denominator, reading 17; decisions: the oracle's dispatch rule with split 1)."""
import numpy as np
import pytest
import torch

from paper_2006_03031_b200 import synth

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2


@pytest.fixture(scope="module")
def nb():
    from paper_2006_03031_b200 import nimble
    return nimble


def _err(y, ref, D):
    return float(np.max(np.abs(y.double().cpu().numpy() - ref) / D))


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
