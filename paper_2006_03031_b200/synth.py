"""Seeded synthetic inputs shaped like the paper's workloads.

This module holds NO arithmetic of the method: it only draws random numbers
(numpy PCG64, generated in fp64, rounded once to the target dtype with RNE) and
random tree structures.  It is the one module shared by the product-side benches
and the oracle-side tests; the oracle never imports the product and vice versa.

Seeds: 0 weights, 1 activations, 2 request lengths / trees; per-case seeds 1000+M.
"""
from __future__ import annotations

import numpy as np
import torch

BERT_BASE = dict(d=768, heads=12, ffn=3072, layers=12)
BERT_LARGE = dict(d=1024, heads=16, ffn=4096, layers=24)


def gen(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def to_dtype(a: np.ndarray, dtype: torch.dtype) -> torch.Tensor:
    """fp64 numpy -> torch CPU tensor of `dtype` (round-to-nearest-even)."""
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dtype)


def normal(shape, std: float, seed: int, dtype=torch.bfloat16) -> torch.Tensor:
    return to_dtype(gen(seed).standard_normal(shape) * std, dtype)


def uniform(shape, lo: float, hi: float, seed: int, dtype=torch.float32) -> torch.Tensor:
    return to_dtype(gen(seed).uniform(lo, hi, shape), dtype)


def ternary(shape, seed: int, dtype, max_nonzero_per_row: int | None = None) -> torch.Tensor:
    """Integer-valued inputs in {-1, 0, 1}; with max_nonzero_per_row every row has at most that
    many non-zeros, so every partial sum is an integer of magnitude <= that bound (exact in
    bf16 up to 256 and in fp32 up to 2^24, whatever the summation order)."""
    g = gen(seed)
    a = g.integers(-1, 2, shape).astype(np.float64)
    if max_nonzero_per_row is not None and a.ndim == 2 and a.shape[1] > max_nonzero_per_row:
        for r in range(a.shape[0]):
            keep = g.choice(a.shape[1], max_nonzero_per_row, replace=False)
            mask = np.zeros(a.shape[1], bool)
            mask[keep] = True
            a[r, ~mask] = 0.0
    return to_dtype(a, dtype)


# ------------------------------------------------------------------ configs
def config1_dense(M: int, seed_w: int = 0):
    """Config 1: y = x W^T + b, K = N = 128, fp32; x ~ U[-1,1), W ~ U(+-1/sqrt(128)), b ~ U[-0.1,0.1)."""
    x = uniform((M, 128), -1.0, 1.0, 1000 + M)
    W = uniform((128, 128), -128 ** -0.5, 128 ** -0.5, seed_w)
    b = uniform((128,), -0.1, 0.1, seed_w + 7)
    return x, W, b


def bert_weights(cfg: dict, seed: int = 0, layers: int | None = None, dtype=torch.bfloat16):
    """BERT encoder weights: W, b ~ N(0, 0.02^2); LN gamma = 1 + N(0, 0.02^2), beta ~ N(0, 0.02^2).
    Per layer a dict Wqkv [3d x d], bqkv, Wo [d x d], bo, g1, be1, W1 [f x d], b1, W2 [d x f], b2, g2, be2."""
    d, f = cfg["d"], cfg["ffn"]
    n = cfg["layers"] if layers is None else layers
    out = []
    for l in range(n):
        s = seed * 100003 + l * 97
        w = {
            "Wqkv": normal((3 * d, d), 0.02, s + 1, dtype), "bqkv": normal((3 * d,), 0.02, s + 2, torch.float32),
            "Wo": normal((d, d), 0.02, s + 3, dtype), "bo": normal((d,), 0.02, s + 4, torch.float32),
            "g1": to_dtype(1.0 + 0.02 * gen(s + 5).standard_normal(d), torch.float32),
            "be1": normal((d,), 0.02, s + 6, torch.float32),
            "W1": normal((f, d), 0.02, s + 7, dtype), "b1": normal((f,), 0.02, s + 8, torch.float32),
            "W2": normal((d, f), 0.02, s + 9, dtype), "b2": normal((d,), 0.02, s + 10, torch.float32),
            "g2": to_dtype(1.0 + 0.02 * gen(s + 11).standard_normal(d), torch.float32),
            "be2": normal((d,), 0.02, s + 12, torch.float32),
        }
        out.append(w)
    return out


def bert_input(L: int, d: int, seed: int) -> torch.Tensor:
    """Synthetic embeddings X ~ N(0, 1) [L x d] bf16 (no tokenizer / embedding table)."""
    return normal((L, d), 1.0, seed, torch.bfloat16)


def request_lengths(R: int, seed: int = 2, lo: int = 1, hi: int = 512) -> np.ndarray:
    """Config 5 request stream: L_i ~ U{lo..hi}."""
    return gen(seed).integers(lo, hi + 1, R).astype(np.int64)


def lstm_weights(I: int, H: int, layers: int = 2, seed: int = 0):
    """PyTorch-default init U(+-1/sqrt(H)); returns [(W_ih [4H x I], W_hh [4H x H], b [4H])] fp32,
    b = b_ih + b_hh drawn separately and summed in fp64 before rounding."""
    out = []
    k = H ** -0.5
    for l in range(layers):
        g = gen(seed * 1009 + l)
        inp = I if l == 0 else H
        W_ih = g.uniform(-k, k, (4 * H, inp))
        W_hh = g.uniform(-k, k, (4 * H, H))
        b = g.uniform(-k, k, 4 * H) + g.uniform(-k, k, 4 * H)
        out.append((to_dtype(W_ih, torch.float32), to_dtype(W_hh, torch.float32), to_dtype(b, torch.float32)))
    return out


def lstm_input(T: int, I: int, seed: int = 1) -> torch.Tensor:
    return normal((T, I), 1.0, seed, torch.float32)


def random_tree(n_leaves: int, g: np.random.Generator, first_word: int = 0):
    """Binary tree by recursive uniform split of n_leaves words.  Returns (root, left, right, word)
    with left/right = -1 for leaves; node ids in post-order."""
    left, right, word = [], [], []

    def build(lo, hi):
        if hi - lo == 1:
            left.append(-1); right.append(-1); word.append(first_word + lo)
            return len(left) - 1
        mid = int(g.integers(lo + 1, hi))
        l = build(lo, mid)
        r = build(mid, hi)
        left.append(l); right.append(r); word.append(-1)
        return len(left) - 1

    root = build(0, n_leaves)
    return root, left, right, word


def random_forest(n_trees: int, seed: int = 2, lo: int = 2, hi: int = 60):
    """Config 4: n_trees trees with n_leaves ~ U{lo..hi}, SST-sentence scale."""
    g = gen(seed)
    trees, words = [], 0
    for _ in range(n_trees):
        n = int(g.integers(lo, hi + 1))
        trees.append(random_tree(n, g, words))
        words += n
    return trees, words


def tree_weights(I: int, H: int, seed: int = 0):
    """W_l [3H x I], b_l [3H], U [5H x 2H], b_u [5H] ~ U(+-1/sqrt(H)), fp32."""
    g = gen(seed * 7919 + 3)
    k = H ** -0.5
    return (to_dtype(g.uniform(-k, k, (3 * H, I)), torch.float32), to_dtype(g.uniform(-k, k, 3 * H), torch.float32),
            to_dtype(g.uniform(-k, k, (5 * H, 2 * H)), torch.float32),
            to_dtype(g.uniform(-k, k, 5 * H), torch.float32))


def bert_weights_device(cfg: dict, seed: int = 0, layers: int | None = None, device="cuda"):
    """Same recipe as bert_weights (N(0, 0.02^2) weights/biases, gamma = 1 + N(0, 0.02^2)) drawn
    with a seeded torch device generator — used by bench.py, where 604 MB of BERT-large
    weights per GPU are too slow to draw on the host."""
    d, f = cfg["d"], cfg["ffn"]
    n = cfg["layers"] if layers is None else layers
    g = torch.Generator(device=device)
    g.manual_seed(seed)

    def rn(shape, dtype=torch.bfloat16, mean=0.0):
        return (torch.randn(shape, generator=g, device=device, dtype=torch.float32) * 0.02 + mean).to(dtype)

    out = []
    for _ in range(n):
        out.append({"Wqkv": rn((3 * d, d)), "bqkv": rn((3 * d,), torch.float32), "Wo": rn((d, d)),
                    "bo": rn((d,), torch.float32), "g1": rn((d,), torch.float32, 1.0),
                    "be1": rn((d,), torch.float32), "W1": rn((f, d)), "b1": rn((f,), torch.float32),
                    "W2": rn((d, f)), "b2": rn((d,), torch.float32), "g2": rn((d,), torch.float32, 1.0),
                    "be2": rn((d,), torch.float32)})
    return out


def device_normal(n_rows: int, d: int, seed: int, device="cuda") -> torch.Tensor:
    """X ~ N(0, 1) [n_rows x d] bf16 drawn on the device (bench request inputs)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.randn((n_rows, d), generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
