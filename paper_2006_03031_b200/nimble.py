"""Thin Python binding of libnimble.so (include/nimble.h) — argument marshalling only.

Every function here has the C-ABI name without the ``nimble_`` prefix and does
nothing but unpack torch tensors / Python ints into pointers and sizes, pass the
current torch CUDA stream, and raise :class:`NimbleError` on a non-OK status.
All arithmetic runs in the CUDA kernels of libnimble.so; there is no CPU
fallback: if the library cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NIMBLE_LIB") or os.path.join(HERE, "libnimble.so")

ANY = -1
F32, BF16 = 0, 1
EPI_NONE, EPI_BIAS, EPI_BIAS_GELU, EPI_BIAS_RESIDUAL = 0, 1, 2, 3

STATUS = {0: "OK", -1: "E_NULL", -2: "E_RANK", -3: "E_SHAPE", -4: "E_EXTENT", -5: "E_DTYPE",
          -6: "E_ALIGN", -7: "E_UNSUPPORTED", -8: "E_CUDA"}


class NimbleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)} ({status}): {msg}")
        self.status = status


if not os.path.exists(LIB_PATH):
    raise ImportError(f"libnimble.so not built at {LIB_PATH}: run `python -m paper_2006_03031_b200.build` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)


class Dispatch(C.Structure):
    """Mirror of nimble_dispatch (include/nimble.h)."""
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


_i64 = C.c_int64
_vp = C.c_void_p
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)

_SIGS = {
    "nimble_shape_dense": [_i64p, _i64p, _i64p],
    "nimble_shape_bmm": [_i64p, _i64p, C.c_int, _i64p],
    "nimble_dispatch_dense": [_i64, _i64, _i64, C.c_int, C.POINTER(Dispatch)],
    "nimble_dispatch_bmm": [_i64, _i64, _i64, _i64, C.c_int, C.c_int, C.POINTER(Dispatch)],
    "nimble_set_variant_limit": [C.c_int],
    "nimble_set_dense_schedule": [_i64, _i64, C.c_int32, C.c_int32],
    "nimble_get_dense_schedule": [_i64, _i64, _i32p, _i32p],
    "nimble_get_variant_limit": [],
    "nimble_last_dispatch": [C.POINTER(Dispatch)],
    "nimble_dense_dyn": [_vp, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _i64, _i64, _i64, C.c_int, C.c_int, _vp],
    "nimble_dense_dyn_dev": [_vp, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64, C.c_int, _vp,
                             _vp],
    "nimble_dense_static": [_vp, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _i64, _i64, _i64, C.c_int, C.c_int, _vp],
    "nimble_dense_ln_dyn": [_vp, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _vp, C.c_float, _vp, _i64, _i64, _i64, _i64,
                            _vp],
    "nimble_bmm_dyn": [_vp, _i64, _i64, _vp, _i64, _i64, C.c_int, _vp, _i64, _i64, _i64, _i64, _i64, _i64,
                       C.c_float, C.c_int, C.c_int, _vp],
    "nimble_bmm_static": [_vp, _i64, _i64, _vp, _i64, _i64, C.c_int, _vp, _i64, _i64, _i64, _i64, _i64, _i64,
                          C.c_float, C.c_int, C.c_int, _vp],
    "nimble_softmax_rows": [_vp, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _vp],
    "nimble_layernorm": [_vp, _i64, _vp, _vp, C.c_float, _vp, _i64, _i64, _i64, _vp],
    "nimble_lstm_seq": [_vp, _i64, _vp, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _i64, _i64, _vp, _vp],
    "nimble_treelstm_level": [_vp, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _i64, _i64, _i64,
                              _i64, C.c_int, _vp],
    "nimble_treelstm_forest": [_vp, _i64, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp,
                               _i64, _vp, _vp, _i64, _vp, _vp],
    "nimble_partition_lpt": [_i64p, _i64, C.c_int32, _i32p],
    "nimble_debug_trace": [_vp],
    "nimble_lstm2_seq": [_vp, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _i64, _i64, _vp, _vp],
    "nimble_lstm2_forward": [_vp, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp, _vp,
                             _i64, _i64, _vp, _vp],
    "nimble_layernorm_dev": [_vp, _i64, _vp, _vp, C.c_float, _vp, _i64, _vp, _i64, _i64, _vp],
    "nimble_attention_varlen_dev": [_vp, _i64, _i64, _vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_float, _vp,
                                    _i64, _vp],
    "nimble_attention_varlen": [_vp, _i64, _i64, _vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_float, _vp,
                                _i64, _vp],
}
for _name, _args in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = C.c_int
_lib.nimble_last_error.restype = C.c_char_p
_lib.nimble_last_error.argtypes = []
_lib.nimble_version.restype = C.c_char_p
_lib.nimble_lstm_workspace_bytes.restype = C.c_size_t
_lib.nimble_lstm_workspace_bytes.argtypes = [_i64]
_lib.nimble_lstm2_workspace_bytes.restype = C.c_size_t
_lib.nimble_lstm2_workspace_bytes.argtypes = [_i64]
_lib.nimble_request_cost.restype = C.c_int64
_lib.nimble_request_cost.argtypes = [_i64]

EXPORTED = sorted(list(_SIGS) + ["nimble_last_error", "nimble_version", "nimble_lstm_workspace_bytes",
                                 "nimble_lstm2_workspace_bytes", "nimble_request_cost"])


def _check(st: int):
    if st != 0:
        raise NimbleError(st, _lib.nimble_last_error().decode())


def last_error() -> str:
    return _lib.nimble_last_error().decode()


def version() -> str:
    return _lib.nimble_version().decode()


# ------------------------------------------------------------------ host-only
def shape_dense(x_shape, w_shape):
    o = (C.c_int64 * 2)()
    _check(_lib.nimble_shape_dense((C.c_int64 * 2)(*x_shape), (C.c_int64 * 2)(*w_shape), o))
    return tuple(o)


def shape_bmm(a_shape, b_shape, trans_b=0):
    o = (C.c_int64 * 3)()
    _check(_lib.nimble_shape_bmm((C.c_int64 * 3)(*a_shape), (C.c_int64 * 3)(*b_shape), int(trans_b), o))
    return tuple(o)


def shape_dense_status(x_shape, w_shape):
    o = (C.c_int64 * 2)()
    st = _lib.nimble_shape_dense((C.c_int64 * 2)(*x_shape), (C.c_int64 * 2)(*w_shape), o)
    return st, (tuple(o) if st == 0 else None)


def shape_bmm_status(a_shape, b_shape, trans_b=0):
    o = (C.c_int64 * 3)()
    st = _lib.nimble_shape_bmm((C.c_int64 * 3)(*a_shape), (C.c_int64 * 3)(*b_shape), int(trans_b), o)
    return st, (tuple(o) if st == 0 else None)


def dispatch_dense(M, N, K, dt):
    d = Dispatch()
    st = _lib.nimble_dispatch_dense(M, N, K, dt, C.byref(d))
    return st, (d.as_dict() if st == 0 else None)


def dispatch_bmm(batch, M, N, K, trans_b, dt):
    d = Dispatch()
    st = _lib.nimble_dispatch_bmm(batch, M, N, K, int(trans_b), dt, C.byref(d))
    return st, (d.as_dict() if st == 0 else None)


def set_variant_limit(c: int):
    _check(_lib.nimble_set_variant_limit(int(c)))


def get_variant_limit() -> int:
    return _lib.nimble_get_variant_limit()


def set_dense_schedule(N: int, K: int, tile_t: int, split_max: int = 8):
    """Register a tuned family-1 schedule for bf16 dense ops with weight shape (N, K)
    (tile_t = 0 removes it).  See include/nimble.h and scripts/tune_symbolic.py."""
    _check(_lib.nimble_set_dense_schedule(N, K, tile_t, split_max))


def get_dense_schedule(N: int, K: int):
    t, s = C.c_int32(), C.c_int32()
    _check(_lib.nimble_get_dense_schedule(N, K, C.byref(t), C.byref(s)))
    return t.value, s.value


def load_dense_schedules(path: str):
    """Register every schedule of a tuning table written by scripts/tune_symbolic.py."""
    import json
    with open(path) as f:
        table = json.load(f)
    for e in table["schedules"]:
        set_dense_schedule(e["N"], e["K"], e["tile_t"], e["split_max"])
    return table["schedules"]


def last_dispatch():
    d = Dispatch()
    _check(_lib.nimble_last_dispatch(C.byref(d)))
    return d.as_dict()


def request_cost(L: int) -> int:
    return _lib.nimble_request_cost(int(L))


def partition_lpt(lens, G: int):
    import numpy as np
    lens = np.ascontiguousarray(lens, dtype=np.int64)
    owner = np.full(lens.shape[0], -1, dtype=np.int32)
    _check(_lib.nimble_partition_lpt(lens.ctypes.data_as(_i64p), lens.shape[0], int(G), owner.ctypes.data_as(_i32p)))
    return owner


def lstm_workspace_bytes(H: int) -> int:
    return int(_lib.nimble_lstm_workspace_bytes(int(H)))


# ------------------------------------------------------------------ device ops
def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream(stream=None):
    if stream is not None:
        return stream
    import torch
    return torch.cuda.current_stream().cuda_stream


_DT = {"torch.float32": F32, "torch.bfloat16": BF16}


def _dt(t):
    return _DT[str(t.dtype)]


def dense_dyn(x, W, bias, y, epi=EPI_BIAS, residual=None, M=None, stream=None):
    """y[:M] = ep(x[:M] W^T + bias) (+ residual[:M]); x [>=M x K], W [N x K], y [>=M x N]."""
    M = x.shape[0] if M is None else M
    N, K = W.shape
    _check(_lib.nimble_dense_dyn(_ptr(x), x.stride(0), _ptr(W), W.stride(0), _ptr(bias), _ptr(residual),
                                 residual.stride(0) if residual is not None else 0, _ptr(y), y.stride(0),
                                 M, N, K, _dt(x), epi, _stream(stream)))
    return y


def dense_dyn_dev(x, W, bias, y, M_dev, M_max=None, epi=EPI_BIAS, residual=None, record=None, stream=None):
    """y[:M] = ep(x[:M] W^T + bias) (+ residual[:M]) with M = M_dev[0] read ON THE DEVICE (int32
    tensor); buffers sized by the bound M_max (default x.shape[0]).  record: optional device
    tensor of nimble_dispatch size (uint8) receiving the device-side dispatch decision."""
    M_max = x.shape[0] if M_max is None else M_max
    N, K = W.shape
    _check(_lib.nimble_dense_dyn_dev(_ptr(x), x.stride(0), _ptr(W), W.stride(0), _ptr(bias), _ptr(residual),
                                     residual.stride(0) if residual is not None else 0, _ptr(y), y.stride(0),
                                     _ptr(M_dev), M_max, N, K, epi, _ptr(record), _stream(stream)))
    return y


DISPATCH_BYTES = C.sizeof(Dispatch)


def dispatch_from_bytes(buf) -> dict:
    """Decode a device dispatch record (uint8 tensor / bytes of nimble_dispatch) into a dict."""
    raw = bytes(buf.cpu().numpy().tobytes()) if hasattr(buf, "cpu") else bytes(buf)
    return Dispatch.from_buffer_copy(raw[:DISPATCH_BYTES]).as_dict()


def dense_static(x, W, bias, y, epi=EPI_BIAS, residual=None, M=None, stream=None):
    """The static-shape twin of dense_dyn (measurement baseline; compiled shapes only)."""
    M = x.shape[0] if M is None else M
    N, K = W.shape
    _check(_lib.nimble_dense_static(_ptr(x), x.stride(0), _ptr(W), W.stride(0), _ptr(bias), _ptr(residual),
                                    residual.stride(0) if residual is not None else 0, _ptr(y), y.stride(0),
                                    M, N, K, _dt(x), epi, _stream(stream)))
    return y


def dense_dyn_dev_raw(x_ptr, ldx, W_ptr, ldw, bias_ptr, res_ptr, ldr, y_ptr, ldy, m_ptr, M_max, N, K, epi, stream):
    _check(_lib.nimble_dense_dyn_dev(x_ptr, ldx, W_ptr, ldw, bias_ptr, res_ptr, ldr, y_ptr, ldy, m_ptr, M_max, N, K,
                                     epi, None, stream))


def dense_ln_dyn(x, W, bias, residual, gamma, beta, y, eps=1e-12, M=None, stream=None):
    """y[:M] = LayerNorm(x[:M] W^T + bias + residual[:M]) * gamma + beta (bf16; fused in the GEMM
    epilogue where the dispatch allows it)."""
    M = x.shape[0] if M is None else M
    N, K = W.shape
    _check(_lib.nimble_dense_ln_dyn(_ptr(x), x.stride(0), _ptr(W), W.stride(0), _ptr(bias), _ptr(residual),
                                    residual.stride(0), _ptr(gamma), _ptr(beta), eps, _ptr(y), y.stride(0), M, N, K,
                                    _stream(stream)))
    return y


def dense_ln_dyn_raw(x_ptr, ldx, W_ptr, ldw, bias_ptr, res_ptr, ldr, g_ptr, b_ptr, eps, y_ptr, ldy, M, N, K, stream):
    _check(_lib.nimble_dense_ln_dyn(x_ptr, ldx, W_ptr, ldw, bias_ptr, res_ptr, ldr, g_ptr, b_ptr, eps, y_ptr, ldy, M,
                                    N, K, stream))


def dense_dyn_raw(x_ptr, ldx, W_ptr, ldw, bias_ptr, res_ptr, ldr, y_ptr, ldy, M, N, K, dt, epi, stream):
    _check(_lib.nimble_dense_dyn(x_ptr, ldx, W_ptr, ldw, bias_ptr, res_ptr, ldr, y_ptr, ldy, M, N, K, dt, epi,
                                 stream))


def bmm_dyn(A, lda, strideA, B, ldb, strideB, trans_b, Cout, ldc, strideC, batch, M, N, K, alpha=1.0,
            out_dt=None, stream=None):
    """Strided-batch C[b] = alpha A[b] Bhat[b]; A/B/C are tensors (base pointers) or raw ints."""
    a = A if isinstance(A, int) else _ptr(A)
    b = B if isinstance(B, int) else _ptr(B)
    c = Cout if isinstance(Cout, int) else _ptr(Cout)
    if out_dt is None:
        out_dt = _dt(Cout)
    _check(_lib.nimble_bmm_dyn(a, lda, strideA, b, ldb, strideB, int(trans_b), c, ldc, strideC, batch, M, N, K,
                               float(alpha), BF16, out_dt, _stream(stream)))
    return Cout


def bmm_static(A, lda, strideA, B, ldb, strideB, trans_b, Cout, ldc, strideC, batch, M, N, K, alpha=1.0,
               out_dt=None, stream=None):
    """The static-shape twin of bmm_dyn (measurement baseline; compiled score shapes only)."""
    a = A if isinstance(A, int) else _ptr(A)
    b = B if isinstance(B, int) else _ptr(B)
    c = Cout if isinstance(Cout, int) else _ptr(Cout)
    if out_dt is None:
        out_dt = _dt(Cout)
    _check(_lib.nimble_bmm_static(a, lda, strideA, b, ldb, strideB, int(trans_b), c, ldc, strideC, batch, M, N, K,
                                  float(alpha), BF16, out_dt, _stream(stream)))
    return Cout


def attention_varlen(qkv, seq_off, R, max_len, heads, out, T=None, scale=None, head_dim=64, stream=None):
    """Fused softmax(Q K^T * scale) V over token-packed requests; seq_off: device int32 [R+1]."""
    T = qkv.shape[0] if T is None else T
    scale = head_dim ** -0.5 if scale is None else scale
    q = qkv if isinstance(qkv, int) else _ptr(qkv)
    o = out if isinstance(out, int) else _ptr(out)
    ldq = 3 * heads * head_dim if isinstance(qkv, int) else qkv.stride(0)
    ldo = heads * head_dim if isinstance(out, int) else out.stride(0)
    _check(_lib.nimble_attention_varlen(q, ldq, T, _ptr(seq_off), R, max_len, heads, head_dim, float(scale), o, ldo,
                                        _stream(stream)))
    return out


def softmax_rows(S, ldS, strideS, P, ldP, strideP, batch, rows, L, stream=None):
    s = S if isinstance(S, int) else _ptr(S)
    p = P if isinstance(P, int) else _ptr(P)
    _check(_lib.nimble_softmax_rows(s, ldS, strideS, p, ldP, strideP, batch, rows, L, _stream(stream)))


def layernorm_dev(X, gamma, beta, Y, rows_dev, rows_max=None, eps=1e-12, stream=None):
    """LayerNorm over rows [0, rows_dev[0]) with the row count read on the device."""
    rows_max = X.shape[0] if rows_max is None else rows_max
    _check(_lib.nimble_layernorm_dev(_ptr(X), X.stride(0), _ptr(gamma), _ptr(beta), float(eps), _ptr(Y), Y.stride(0),
                                     _ptr(rows_dev), rows_max, X.shape[1], _stream(stream)))
    return Y


def attention_varlen_dev(qkv, seq_off, R, max_len, heads, out, T_max=None, scale=None, head_dim=64, stream=None):
    """attention_varlen with the token count T = seq_off[R] read on the device."""
    T_max = qkv.shape[0] if T_max is None else T_max
    scale = head_dim ** -0.5 if scale is None else scale
    _check(_lib.nimble_attention_varlen_dev(_ptr(qkv), qkv.stride(0), T_max, _ptr(seq_off), R, max_len, heads,
                                            head_dim, float(scale), _ptr(out), out.stride(0), _stream(stream)))
    return out


def layernorm(X, gamma, beta, Y, eps=1e-12, rows=None, stream=None):
    rows = X.shape[0] if rows is None else rows
    _check(_lib.nimble_layernorm(_ptr(X), X.stride(0), _ptr(gamma), _ptr(beta), float(eps), _ptr(Y), Y.stride(0),
                                 rows, X.shape[1], _stream(stream)))
    return Y


def lstm_seq(G, W_hh, H_seq, hT, cT, workspace, T=None, h0=None, c0=None, stream=None):
    T = G.shape[0] if T is None else T
    H = W_hh.shape[1]
    _check(_lib.nimble_lstm_seq(_ptr(G), G.stride(0), _ptr(W_hh), W_hh.stride(0), _ptr(h0), _ptr(c0), _ptr(H_seq),
                                H_seq.stride(0), _ptr(hT), _ptr(cT), T, H, _ptr(workspace), _stream(stream)))


def lstm2_workspace_bytes(H: int) -> int:
    return int(_lib.nimble_lstm2_workspace_bytes(int(H)))


def lstm2_forward(X, I, W_ih1, b1, W_hh1, W_ih2, W_hh2, b2, H1, H2, hT, cT, workspace, T=None, stream=None):
    """Both layers incl. the layer-1 input projection in one launch (nimble_lstm2_forward)."""
    T = X.shape[0] if T is None else T
    H = W_hh1.shape[1]
    _check(_lib.nimble_lstm2_forward(_ptr(X), X.stride(0), I, _ptr(W_ih1), W_ih1.stride(0), _ptr(b1), _ptr(W_hh1),
                                     _ptr(W_ih2), _ptr(W_hh2), W_hh1.stride(0), _ptr(b2), _ptr(H1), _ptr(H2),
                                     H1.stride(0), _ptr(hT), _ptr(cT), T, H, _ptr(workspace), _stream(stream)))


def lstm2_seq(G1, W_hh1, W_ih2, W_hh2, b2, H1, H2, hT, cT, workspace, T=None, stream=None):
    T = G1.shape[0] if T is None else T
    H = W_hh1.shape[1]
    _check(_lib.nimble_lstm2_seq(_ptr(G1), G1.stride(0), _ptr(W_hh1), _ptr(W_ih2), _ptr(W_hh2), W_hh1.stride(0),
                                 _ptr(b2), _ptr(H1), _ptr(H2), H1.stride(0), _ptr(hT), _ptr(cT), T, H,
                                 _ptr(workspace), _stream(stream)))


TREE_WORKSPACE_BYTES = 256


def treelstm_forest(X, W_l, b_l, U, b_u, level_off, n_levels, max_level, nodes, rows, parent_slot, hcat, ccat,
                    h_out, c_out, workspace, stream=None):
    I, H = W_l.shape[1], U.shape[1] // 2
    _check(_lib.nimble_treelstm_forest(_ptr(X), X.stride(0), _ptr(W_l), _ptr(b_l), _ptr(U), _ptr(b_u), I, H,
                                       _ptr(level_off), n_levels, max_level, _ptr(nodes), _ptr(rows),
                                       _ptr(parent_slot), _ptr(hcat), _ptr(ccat), hcat.stride(0), _ptr(h_out),
                                       _ptr(c_out), h_out.stride(0), _ptr(workspace), _stream(stream)))


def treelstm_level(nodes, A, a_rows, W, bias, parent_slot, hcat, ccat, h_out, c_out, M, K, H, is_leaf,
                   stream=None):
    _check(_lib.nimble_treelstm_level(_ptr(nodes), _ptr(A), A.stride(0), _ptr(a_rows), _ptr(W), W.stride(0),
                                      _ptr(bias), _ptr(parent_slot), _ptr(hcat), _ptr(ccat), hcat.stride(0),
                                      _ptr(h_out), _ptr(c_out), h_out.stride(0), M, K, H, int(is_leaf),
                                      _stream(stream)))
