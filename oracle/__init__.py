"""oracle — plain CPU fp64 oracle for the Nimble (arXiv 2006.03031) hot path.

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import this
package. The product package ``paper_2006_03031_b200`` never imports it, and the
two share no code: this is a thin ctypes wrapper around ``oracle/oracle.c``
(argument marshalling only; every step of the arithmetic is in the C file, which
cites the PAPER.md passage each function follows).

Inputs are numpy arrays; they are widened to float64 here (the exact bf16/fp32
values the GPU saw). Shape/dispatch functions return plain Python values.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ANY = -1


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (fp64, -O2, no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-fPIC", "-shared",
                               "-fno-fast-math", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


class Dispatch(C.Structure):
    """The oracle's own declaration of the dispatch record (DISPATCH.md)."""
    _fields_ = [("family", C.c_int32), ("tile_t", C.c_int32), ("granule", C.c_int32),
                ("n_classes", C.c_int32), ("residue_class", C.c_int32), ("variant", C.c_int32),
                ("split_k", C.c_int32), ("umma_m", C.c_int32), ("umma_n_full", C.c_int32),
                ("umma_n_tail", C.c_int32), ("k", C.c_int64), ("r", C.c_int64),
                ("grid", C.c_int32 * 3), ("cluster", C.c_int32 * 3)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f not in ("grid", "cluster")}
        d["grid"] = tuple(self.grid)
        d["cluster"] = tuple(self.cluster)
        return d


_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)


def _declare(L):
    L.orc_bcast.argtypes = [C.c_int64, C.c_int64, _i64p]
    L.orc_shape_dense.argtypes = [_i64p, _i64p, _i64p]
    L.orc_shape_bmm.argtypes = [_i64p, _i64p, C.c_int, _i64p]
    L.orc_dispatch_dense.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int, C.POINTER(Dispatch)]
    L.orc_dispatch_dense_sched.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int32, C.c_int32,
                                           C.POINTER(Dispatch)]
    L.orc_dispatch_bmm.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(Dispatch)]
    L.orc_gelu.argtypes = [C.c_double]
    L.orc_gelu.restype = C.c_double
    L.orc_dense.argtypes = [_dp, C.c_int64, C.c_int64, _dp, C.c_int64, _dp, _dp, C.c_int, _dp, _dp]
    L.orc_dense.restype = None
    L.orc_bmm.argtypes = [_dp, C.c_int64, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                          C.c_double, _dp, _dp]
    L.orc_bmm.restype = None
    L.orc_softmax_rows.argtypes = [_dp, C.c_int64, C.c_int64, _dp]
    L.orc_softmax_rows.restype = None
    L.orc_layernorm.argtypes = [_dp, C.c_int64, C.c_int64, _dp, _dp, C.c_double, _dp]
    L.orc_layernorm.restype = None
    L.orc_lstm_layer.argtypes = [_dp, C.c_int64, C.c_int64, C.c_int64, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
    L.orc_lstm_layer.restype = None
    L.orc_treelstm.argtypes = [C.c_int32, _i32p, _i32p, _i32p, _dp, C.c_int64, C.c_int64, _dp, _dp, _dp,
                               _dp, _dp, _dp]
    L.orc_treelstm.restype = None
    L.orc_bert_layer.argtypes = [_dp, C.c_int64, C.c_int64, C.c_int64, C.c_int64] + [_dp] * 12 + [_dp]
    L.orc_bert_layer.restype = None
    L.orc_request_cost.argtypes = [C.c_int64]
    L.orc_request_cost.restype = C.c_int64
    L.orc_partition_lpt.argtypes = [_i64p, C.c_int64, C.c_int32, _i32p]


def _f64(a):
    if a is None:
        return None
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return None if a is None else a.ctypes.data_as(_dp)


# ---------------------------------------------------------------- O1 shape fns
def bcast(a: int, b: int):
    out = C.c_int64(0)
    st = lib().orc_bcast(a, b, C.byref(out))
    return st, (out.value if st == 0 else None)


def shape_dense(x_shape, w_shape):
    x = (C.c_int64 * 2)(*x_shape); w = (C.c_int64 * 2)(*w_shape); o = (C.c_int64 * 2)()
    st = lib().orc_shape_dense(x, w, o)
    return st, (tuple(o) if st == 0 else None)


def shape_bmm(a_shape, b_shape, trans_b=0):
    a = (C.c_int64 * 3)(*a_shape); b = (C.c_int64 * 3)(*b_shape); o = (C.c_int64 * 3)()
    st = lib().orc_shape_bmm(a, b, int(trans_b), o)
    return st, (tuple(o) if st == 0 else None)


# ---------------------------------------------------------------- O2 dispatch
def dispatch_dense(M, N, K, dt, c=0, tile_t=0, split_max=8):
    """tile_t / split_max: a tuned family-1 schedule (DISPATCH.md); 0 = default."""
    d = Dispatch()
    if tile_t:
        st = lib().orc_dispatch_dense_sched(M, N, K, dt, c, tile_t, split_max, C.byref(d))
    else:
        st = lib().orc_dispatch_dense(M, N, K, dt, c, C.byref(d))
    return st, (d.as_dict() if st == 0 else None)


def dispatch_bmm(batch, M, N, K, trans_b, dt, c=0):
    d = Dispatch()
    st = lib().orc_dispatch_bmm(batch, M, N, K, int(trans_b), dt, c, C.byref(d))
    return st, (d.as_dict() if st == 0 else None)


# ---------------------------------------------------------------- O3 / O4
EPI_NONE, EPI_BIAS, EPI_BIAS_GELU, EPI_BIAS_RESIDUAL = 0, 1, 2, 3


def dense(x, W, b=None, res=None, epi=EPI_BIAS):
    """y = ep(x W^T + b) (+res); returns (y, D) in float64."""
    x = _f64(x); W = _f64(W); b = _f64(b); res = _f64(res)
    M, K = x.shape
    N = W.shape[0]
    assert W.shape[1] == K
    y = np.empty((M, N)); D = np.empty((M, N))
    lib().orc_dense(_p(x), M, K, _p(W), N, _p(b), _p(res), epi, _p(y), _p(D))
    return y, D


def bmm(A, B, trans_b=0, alpha=1.0):
    """C[b] = alpha * A[b] @ (B[b]^T if trans_b == 0 else B[b]); returns (C, D)."""
    A = _f64(A); B = _f64(B)
    bA, M, K = A.shape
    if trans_b:
        bB, K2, N = B.shape
    else:
        bB, N, K2 = B.shape
    assert K2 == K
    batch = max(bA, bB)
    Cm = np.empty((batch, M, N)); D = np.empty((batch, M, N))
    lib().orc_bmm(_p(A), bA, _p(B), bB, M, N, K, int(trans_b), float(alpha), _p(Cm), _p(D))
    return Cm, D


# ---------------------------------------------------------------- O5
def gelu(z):
    return np.vectorize(lambda v: lib().orc_gelu(float(v)))(np.asarray(z, dtype=np.float64))


def softmax_rows(S):
    S = _f64(S)
    shp = S.shape
    S2 = S.reshape(-1, shp[-1])
    P = np.empty_like(S2)
    lib().orc_softmax_rows(_p(S2), S2.shape[0], S2.shape[1], _p(P))
    return P.reshape(shp)


def layernorm(X, gamma, beta, eps=1e-12):
    X = _f64(X); gamma = _f64(gamma); beta = _f64(beta)
    Y = np.empty_like(X)
    lib().orc_layernorm(_p(X), X.shape[0], X.shape[1], _p(gamma), _p(beta), eps, _p(Y))
    return Y


# ---------------------------------------------------------------- O6
def lstm_layer(X, W_ih, W_hh, b, h0=None, c0=None):
    X = _f64(X); W_ih = _f64(W_ih); W_hh = _f64(W_hh); b = _f64(b); h0 = _f64(h0); c0 = _f64(c0)
    T, I = X.shape
    H = W_hh.shape[1]
    Hs = np.empty((T, H)); hT = np.empty(H); cT = np.empty(H)
    lib().orc_lstm_layer(_p(X), T, I, H, _p(W_ih), _p(W_hh), _p(b), _p(h0), _p(c0), _p(Hs), _p(hT), _p(cT))
    return Hs, hT, cT


def lstm(X, layers):
    """Stacked LSTM; layers = [(W_ih, W_hh, b), ...]. Returns (H_last_seq, [(hT, cT)...], all Hseq)."""
    seqs, states = [], []
    inp = X
    for (W_ih, W_hh, b) in layers:
        Hs, hT, cT = lstm_layer(inp, W_ih, W_hh, b)
        seqs.append(Hs); states.append((hT, cT))
        inp = Hs
    return inp, states, seqs


# ---------------------------------------------------------------- O7
def treelstm(root, left, right, word, X, W_l, b_l, U, b_u):
    left = np.ascontiguousarray(left, dtype=np.int32)
    right = np.ascontiguousarray(right, dtype=np.int32)
    word = np.ascontiguousarray(word, dtype=np.int32)
    X = _f64(X); W_l = _f64(W_l); b_l = _f64(b_l); U = _f64(U); b_u = _f64(b_u)
    n = left.shape[0]
    I = X.shape[1]
    H = U.shape[1] // 2
    Hn = np.zeros((n, H)); Cn = np.zeros((n, H))
    lib().orc_treelstm(int(root), left.ctypes.data_as(_i32p), right.ctypes.data_as(_i32p),
                       word.ctypes.data_as(_i32p), _p(X), I, H, _p(W_l), _p(b_l), _p(U), _p(b_u),
                       _p(Hn), _p(Cn))
    return Hn, Cn


# ---------------------------------------------------------------- O8
def bert_layer(X, w, nh):
    """w: dict Wqkv,bqkv,Wo,bo,g1,be1,W1,b1,W2,b2,g2,be2 (any array type)."""
    X = _f64(X)
    L, d = X.shape
    f = np.asarray(w["W1"]).shape[0]
    arrs = [_f64(w[k]) for k in ("Wqkv", "bqkv", "Wo", "bo", "g1", "be1", "W1", "b1", "W2", "b2", "g2", "be2")]
    Y = np.empty((L, d))
    lib().orc_bert_layer(_p(X), L, d, nh, f, *[_p(a) for a in arrs], _p(Y))
    return Y


# ---------------------------------------------------------------- O9
def request_cost(L):
    return lib().orc_request_cost(int(L))


def partition_lpt(lens, G):
    lens = np.ascontiguousarray(lens, dtype=np.int64)
    owner = np.full(lens.shape[0], -1, dtype=np.int32)
    st = lib().orc_partition_lpt(lens.ctypes.data_as(_i64p), lens.shape[0], G, owner.ctypes.data_as(_i32p))
    return st, owner


def dense_flops(M, N, K):
    return 2 * M * N * K
