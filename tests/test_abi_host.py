"""CPU tests of the C-ABI boundary (no GPU): the library loads, exports every symbol
include/nimble.h declares, and its host-side shape functions, residue dispatch and
request partition agree BIT-EXACTLY with the independent oracle (BJ:5 "Shape
functions and dispatch choices must match the oracle bit-exact")."""
import itertools
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ANY = -1


@pytest.fixture(scope="module")
def nb():
    from paper_2006_03031_b200 import build
    build.build()
    from paper_2006_03031_b200 import nimble
    return nimble


def test_exports_every_declared_symbol(nb):
    hdr = open(os.path.join(ROOT, "include", "nimble.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)          # drop comments
    declared = set(re.findall(r"\b(nimble_[a-z_0-9]+)\s*\(", hdr))
    assert len(declared) == 32
    for name in declared:
        assert hasattr(nb._lib, name), name
    assert set(nb.EXPORTED) <= declared | {"nimble_last_error", "nimble_version"}
    assert nb.version().startswith("nimble-b200")


def test_shape_dense_matches_oracle(nb, orc):
    dims = [ANY, 0, 1, 2, 3, 768]
    for a0, a1, w0, w1 in itertools.product(dims, repeat=4):
        assert nb.shape_dense_status((a0, a1), (w0, w1)) == orc.shape_dense((a0, a1), (w0, w1)), (a0, a1, w0, w1)


def test_shape_bmm_matches_oracle(nb, orc):
    dims = [ANY, 1, 2, 3]
    for a0, a2, b0, b1, b2 in itertools.product(dims + [0], dims, dims, dims, dims):
        for tb in (0, 1):
            got = nb.shape_bmm_status((a0, 5, a2), (b0, b1, b2), tb)
            assert got == orc.shape_bmm((a0, 5, a2), (b0, b1, b2), tb), (a0, a2, b0, b1, b2, tb)


@pytest.mark.parametrize("c", [0, 1, 2, 3, 8, 9, 16, 17, 18])
def test_dispatch_dense_bit_exact(nb, orc, c):
    nb.set_variant_limit(c)
    try:
        Ms = range(1, 65537) if c in (0, 1) else range(1, 4097)
        for dt in (0, 1):
            for (N, K) in ((128, 128), (1024, 4096)):
                for M in Ms:
                    assert nb.dispatch_dense(M, N, K, dt) == orc.dispatch_dense(M, N, K, dt, c), (M, N, K, dt, c)
    finally:
        nb.set_variant_limit(0)


@pytest.mark.parametrize("c", [0, 1, 2])
def test_dispatch_bmm_bit_exact(nb, orc, c):
    nb.set_variant_limit(c)
    try:
        for L in range(1, 1025):
            for (batch, tb) in ((12, 0), (12, 1), (16, 0), (16, 1), (1, 0)):
                M, N, K = (L, L, 64) if tb == 0 else (L, 64, L)
                assert nb.dispatch_bmm(batch, M, N, K, tb, 1) == orc.dispatch_bmm(batch, M, N, K, tb, 1, c)
        for bad in ((0, 5, 5, 5, 0, 1), (2, 5, 5, 5, 0, 0), (2, 5, 5, 5, 0, 9), (2, 0, 5, 5, 1, 1)):
            assert nb.dispatch_bmm(*bad)[0] == orc.dispatch_bmm(*bad, c)[0]
    finally:
        nb.set_variant_limit(0)


@pytest.mark.parametrize("tile_t,split_max", [(32, 8), (64, 1), (64, 4), (128, 2), (256, 8), (256, 1)])
def test_dispatch_tuned_schedule_bit_exact(nb, orc, tile_t, split_max):
    """A registered schedule changes the residue tile and split cap identically
    in the library and the oracle; other (N, K) keep the default; removal restores it."""
    N, K = 1024, 4096
    nb.set_dense_schedule(N, K, tile_t, split_max)
    try:
        assert nb.get_dense_schedule(N, K) == (tile_t, split_max)
        for c in (0, 2):
            nb.set_variant_limit(c)
            for M in range(1, 2200):
                assert nb.dispatch_dense(M, N, K, 1) == orc.dispatch_dense(M, N, K, 1, c, tile_t, split_max), (M, c)
        nb.set_variant_limit(0)
        for M in (1, 77, 300):
            assert nb.dispatch_dense(M, 128, 128, 1) == orc.dispatch_dense(M, 128, 128, 1)
    finally:
        nb.set_variant_limit(0)
        nb.set_dense_schedule(N, K, 0, 8)
    assert nb.get_dense_schedule(N, K) == (0, 8)
    assert nb.dispatch_dense(100, N, K, 1) == orc.dispatch_dense(100, N, K, 1)


def test_dense_dyn_dev_validation(nb):
    E = nb.NimbleError
    L = nb._lib
    # M_max >= 2048 is family 3: not available with a device extent
    with pytest.raises(E) as ei:
        nb._check(L.nimble_dense_dyn_dev(16, 1024, 16, 1024, 16, None, 0, 16, 1024, 16, 2048, 1024, 1024, 1, None, None))
    assert ei.value.status == -7
    with pytest.raises(E) as ei:     # NULL M_dev
        nb._check(L.nimble_dense_dyn_dev(16, 1024, 16, 1024, 16, None, 0, 16, 1024, None, 100, 1024, 1024, 1, None, None))
    assert ei.value.status == -1
    with pytest.raises(E) as ei:     # K mismatch is impossible here; bad extent
        nb._check(L.nimble_dense_dyn_dev(16, 1024, 16, 1024, 16, None, 0, 16, 1024, 16, 0, 1024, 1024, 1, None, None))
    assert ei.value.status == -4


def test_dense_schedule_validation(nb):
    for bad in ((1024, 4096, 48, 8), (1024, 4096, 128, 3), (0, 4096, 128, 8), (1024, 4096, -1, 8)):
        with pytest.raises(nb.NimbleError):
            nb.set_dense_schedule(*bad)


def test_dispatch_errors_match(nb, orc):
    for args in ((0, 128, 128, 0), (5, 0, 128, 1), (5, 128, 0, 1), (5, 128, 128, 3), (2 ** 31, 128, 128, 0)):
        assert nb.dispatch_dense(*args)[0] == orc.dispatch_dense(*args)[0]
    with pytest.raises(nb.NimbleError):
        nb.set_variant_limit(-1)


def test_partition_bit_exact(nb, orc):
    rs = np.random.default_rng(2)
    for R in (0, 1, 5, 64, 1000):
        lens = rs.integers(1, 513, R)
        for G in (1, 2, 3, 4, 8):
            st, o = orc.partition_lpt(lens, G)
            assert st == 0 and np.array_equal(nb.partition_lpt(lens, G), o)
    for L in (1, 100, 512):
        assert nb.request_cost(L) == orc.request_cost(L)


def test_validation_errors_before_launch(nb):
    # these return before any CUDA call, so they are safe without a GPU
    E = nb.NimbleError
    with pytest.raises(E) as ei:
        nb._check(nb._lib.nimble_dense_dyn(None, 128, None, 128, None, None, 0, None, 128, 0, 128, 128, 0, 1, None))
    assert ei.value.status == -4
    st = nb._lib.nimble_dense_dyn(None, 128, None, 128, None, None, 0, None, 128, 4, 128, 128, 0, 1, None)
    assert st == -1
    st = nb._lib.nimble_dense_dyn(16, 128, 16, 128, 16, None, 0, 16, 128, 4, 128, 128, 5, 1, None)
    assert st == -5
    st = nb._lib.nimble_dense_dyn(8, 128, 16, 128, 16, None, 0, 16, 128, 4, 128, 128, 1, 1, None)
    assert st == -6                                    # bf16 base not 16-B aligned
    st = nb._lib.nimble_bmm_dyn(16, 64, 64, 16, 64, 64, 0, 16, 64, 64, 2, 4, 4, 64, 1.0, 0, 0, None)
    assert st == -7                                    # fp32 bmm not built
    assert nb.lstm_workspace_bytes(650) >= 2 * 650 * 4
