"""Pins for oracle O3 (dense) and O4 (bmm), SURVEY §8(c).

Pinned to: special cases (W = I, one-hot rows) that are exact; brute-force exact
integer arithmetic on small inputs; numpy fp64 matmul (a library routine, not a
retyping); the pad-to-static-then-slice invariant of residue specialisation
(every variant computes the same function as the static kernel);
the 2^e scaling invariant; scipy's erf for the GELU epilogue.
"""
import numpy as np
import pytest
import scipy.special

rng = np.random.default_rng(1234)


def test_identity_weight_exact(orc):
    K = 37
    x = rng.standard_normal((9, K))
    b = rng.standard_normal(K)
    y, _ = orc.dense(x, np.eye(K), b, epi=orc.EPI_BIAS)
    assert np.array_equal(y, x + b)


def test_one_hot_rows_exact(orc):
    N, K = 11, 13
    W = rng.standard_normal((N, K))
    b = rng.standard_normal(N)
    x = np.zeros((K, K))
    x[np.arange(K), np.arange(K)] = 1.0
    y, _ = orc.dense(x, W, b)
    assert np.array_equal(y, W.T + b)


def test_integer_exact_brute_force(orc):
    M, N, K = 7, 5, 19
    x = rng.integers(-1, 2, (M, K))
    W = rng.integers(-1, 2, (N, K))
    b = rng.integers(-1, 2, N)
    res = rng.integers(-3, 4, (M, N))
    y, D = orc.dense(x, W, b, res, epi=orc.EPI_BIAS_RESIDUAL)
    for m in range(M):
        for n in range(N):
            exact = sum(int(x[m, k]) * int(W[n, k]) for k in range(K)) + int(b[n]) + int(res[m, n])
            assert y[m, n] == exact
            assert D[m, n] == sum(abs(int(x[m, k]) * int(W[n, k])) for k in range(K)) + abs(b[n]) + abs(res[m, n])


def test_matches_numpy_fp64(orc):
    for (M, N, K) in [(1, 128, 128), (13, 40, 77), (64, 128, 128)]:
        x = rng.standard_normal((M, K)); W = rng.standard_normal((N, K)); b = rng.standard_normal(N)
        y, D = orc.dense(x, W, b)
        ref = x @ W.T + b
        assert np.max(np.abs(y - ref) / (np.abs(x) @ np.abs(W).T + np.abs(b))) < 1e-13
        assert np.all(D >= np.abs(y) - 1e-12)
        y0, _ = orc.dense(x, W, None, epi=orc.EPI_NONE)
        assert np.max(np.abs(y0 - x @ W.T)) < 1e-11


def test_gelu_epilogue_vs_scipy(orc):
    x = rng.standard_normal((6, 33)); W = rng.standard_normal((21, 33)); b = rng.standard_normal(21)
    y, _ = orc.dense(x, W, b, epi=orc.EPI_BIAS_GELU)
    z = x @ W.T + b
    ref = 0.5 * z * (1.0 + scipy.special.erf(z / np.sqrt(2.0)))
    assert np.max(np.abs(y - ref)) < 1e-10


def test_pad_then_slice_invariant(orc):
    # dynamic-M result == pad-to-static-then-slice result for every residue mod 8 (BJ:5)
    N, K = 16, 24
    W = rng.standard_normal((N, K)); b = rng.standard_normal(N)
    xs = rng.standard_normal((64, K))
    yfull, _ = orc.dense(xs, W, b)
    for M in range(1, 65):
        y, _ = orc.dense(xs[:M], W, b)
        Mp = 8 * ((M + 7) // 8)
        xp = np.zeros((Mp, K)); xp[:M] = xs[:M]
        yp, _ = orc.dense(xp, W, b)
        assert np.array_equal(y, yp[:M])
        assert np.array_equal(y, yfull[:M])


def test_power_of_two_scaling(orc):
    x = rng.standard_normal((5, 17)); W = rng.standard_normal((9, 17)); b = rng.standard_normal(9)
    y, _ = orc.dense(x, W, b)
    y8, _ = orc.dense(x * 8.0, W, b)
    assert np.array_equal(y8 - b, (y - b) * 8.0) or np.max(np.abs((y8 - b) - 8 * (y - b))) < 1e-12


def test_flops_closed_form(orc):
    assert orc.dense_flops(128, 3072, 1024) == 2 * 128 * 3072 * 1024


def test_bmm_reduces_to_dense(orc):
    A = rng.standard_normal((3, 7, 10)); B = rng.standard_normal((3, 5, 10))
    Cm, D = orc.bmm(A, B, 0, alpha=0.125)
    for b in range(3):
        y, Dd = orc.dense(A[b], B[b], None, epi=orc.EPI_NONE)
        assert np.array_equal(Cm[b], 0.125 * y)
        assert np.array_equal(D[b], 0.125 * Dd)


def test_bmm_trans_b_consistency_and_einsum(orc):
    A = rng.standard_normal((4, 6, 9)); Bt = rng.standard_normal((4, 9, 5))
    C1, _ = orc.bmm(A, Bt, 1)
    C2, _ = orc.bmm(A, np.ascontiguousarray(np.swapaxes(Bt, 1, 2)), 0)
    assert np.array_equal(C1, C2)
    assert np.max(np.abs(C1 - np.einsum("bik,bkj->bij", A, Bt))) < 1e-12


def test_bmm_broadcast_batch(orc):
    A = rng.standard_normal((1, 4, 6)); B = rng.standard_normal((3, 5, 6))
    Cm, _ = orc.bmm(A, B, 0)
    for b in range(3):
        assert np.max(np.abs(Cm[b] - A[0] @ B[b].T)) < 1e-12
