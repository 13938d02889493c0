"""Parity gates shared by the GPU tests (reading 17; BJ:5 "max relative error <= 2e-2
for bf16 inputs with fp32 accumulation and <= 1e-4 for fp32").

Two gates, both asserted for every floating-point output:
  * componentwise-bound gate   max |y - y*| / D <= tol,  D = sum_k |x||W| + |b| + |res|
    (the denominator the oracle returns: it bounds the rounding error of ANY summation order);
  * elementwise gate           |y - y*| <= tol * max(|y*|, rms(y*))   for every element
    (the relative wording of BJ:5; the rms floor keeps it meaningful where y* ~ 0).
The plain elementwise relative error max |y - y*| / |y*| over |y*| >= 1e-3 max|y*| is reported
(not gated) to gpurun_out/parity_report.jsonl, one line per check.
"""
from __future__ import annotations

import json
import os

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REPORT = os.path.join(ROOT, "gpurun_out", "parity_report.jsonl")


def _np(y):
    return y.double().cpu().numpy() if torch.is_tensor(y) else np.asarray(y, dtype=np.float64)


def errors(y, ref, D=None):
    """(D-normalised error, elementwise error against max(|y*|, rms), plain relative error)."""
    y, ref = _np(y), _np(ref)
    diff = np.abs(y - ref)
    if diff.size == 0:
        return 0.0, 0.0, 0.0
    d_err = float(np.max(diff / np.maximum(D, 1e-30))) if D is not None else None
    rms = float(np.sqrt(np.mean(ref * ref)))
    elem = float(np.max(diff / np.maximum(np.maximum(np.abs(ref), rms), 1e-30)))
    big = np.abs(ref) >= 1e-3 * float(np.max(np.abs(ref)))
    rel = float(np.max(diff[big] / np.abs(ref[big]))) if np.any(big) else 0.0
    return d_err, elem, rel


def record(what, **kw):
    try:
        os.makedirs(os.path.dirname(REPORT), exist_ok=True)
        with open(REPORT, "a") as f:
            f.write(json.dumps({"check": str(what), **kw}) + "\n")
    except OSError:
        pass


def gate(y, ref, D=None, tol=2e-2, what=""):
    """Assert both gates (the D gate only when D is given); returns the three errors."""
    d_err, elem, rel = errors(y, ref, D)
    record(what, tol=tol, d_err=d_err, elem_err=elem, rel_err=rel, n=int(np.size(ref)))
    if D is not None:
        assert d_err <= tol, (what, "D-normalised", d_err)
    assert elem <= tol, (what, "elementwise vs max(|y*|, rms)", elem)
    return d_err, elem, rel


def gate_bf16(y, ref, D=None, what=""):
    return gate(y, ref, D, 2e-2, what)


def gate_f32(y, ref, D=None, what=""):
    return gate(y, ref, D, 1e-4, what)
