"""Pins for oracle O5-O9 (row ops, LSTM, Tree-LSTM, BERT layer, request partition).

Each pin is something other than the oracle's own formula: a closed form, an
invariant, a textbook/library routine in fp64 (torch.nn.LSTM, torch.nn.functional,
scipy), or brute force on tiny inputs.
"""
import itertools

import numpy as np
import pytest
import scipy.special
import torch
import torch.nn.functional as F

rng = np.random.default_rng(99)


# ---------------------------------------------------------------- O5
def test_gelu_closed_forms(orc):
    z = rng.standard_normal(200) * 3
    g = orc.gelu(z)
    assert orc.gelu(np.array([0.0]))[0] == 0.0
    assert np.max(np.abs(g - orc.gelu(-z) - z)) < 1e-14            # Phi(z)+Phi(-z)=1
    assert np.max(np.abs(g - 0.5 * z * (1 + scipy.special.erf(z / np.sqrt(2))))) < 1e-14
    t = torch.tensor(z, dtype=torch.float64)
    assert np.max(np.abs(g - F.gelu(t, approximate="none").numpy())) < 1e-14


def test_softmax_pins(orc):
    P = orc.softmax_rows(np.full((3, 7), 2.5))
    assert np.allclose(P, 1.0 / 7, atol=0, rtol=1e-15)                # constant row -> 1/L
    S = rng.standard_normal((5, 33)) * 4
    P = orc.softmax_rows(S)
    assert np.max(np.abs(P.sum(1) - 1)) < 1e-14
    ref = F.softmax(torch.tensor(S, dtype=torch.float64), dim=-1).numpy()
    assert np.max(np.abs(P - ref)) < 1e-15
    assert np.max(np.abs(orc.softmax_rows(S + 100.0) - P)) < 1e-14    # shift invariance
    assert np.array_equal(orc.softmax_rows(np.array([[3.0]])), np.array([[1.0]]))   # L = 1


def test_layernorm_pins(orc):
    X = rng.standard_normal((6, 64)) * 3 + 1
    Y = orc.layernorm(X, np.ones(64), np.zeros(64))
    var = X.var(1)
    assert np.max(np.abs(Y.mean(1))) < 1e-14
    assert np.max(np.abs(Y.var(1) - var / (var + 1e-12))) < 1e-12
    g = rng.standard_normal(64); b = rng.standard_normal(64)
    Y2 = orc.layernorm(X, g, b)
    ref = F.layer_norm(torch.tensor(X), (64,), torch.tensor(g), torch.tensor(b), eps=1e-12).numpy()
    assert np.max(np.abs(Y2 - ref)) < 1e-12


# ---------------------------------------------------------------- O6
def _sig(z):
    return 1 / (1 + np.exp(-z))


def test_lstm_single_step_closed_form(orc):
    I, H = 5, 4
    W_ih = rng.standard_normal((4 * H, I)); W_hh = rng.standard_normal((4 * H, H)); b = rng.standard_normal(4 * H)
    x = rng.standard_normal((1, I))
    Hs, hT, cT = orc.lstm_layer(x, W_ih, W_hh, b)
    z = W_ih @ x[0] + b
    c1 = _sig(z[:H]) * np.tanh(z[2 * H:3 * H])
    h1 = _sig(z[3 * H:]) * np.tanh(c1)
    assert np.max(np.abs(cT - c1)) < 1e-15 and np.max(np.abs(hT - h1)) < 1e-15
    assert np.array_equal(Hs[0], hT)


def test_lstm_zero_weights_geometric(orc):
    # W = 0 -> gates constant; c_t = s(b_f) c_{t-1} + s(b_i) tanh(b_g) (closed-form sum)
    I, H, T = 3, 6, 9
    b = rng.standard_normal(4 * H)
    Hs, hT, cT = orc.lstm_layer(rng.standard_normal((T, I)), np.zeros((4 * H, I)), np.zeros((4 * H, H)), b)
    fg, ig, gg, og = _sig(b[H:2 * H]), _sig(b[:H]), np.tanh(b[2 * H:3 * H]), _sig(b[3 * H:])
    cT_closed = ig * gg * (1 - fg ** T) / (1 - fg)
    assert np.max(np.abs(cT - cT_closed)) < 1e-13
    assert np.max(np.abs(hT - og * np.tanh(cT_closed))) < 1e-13


def test_lstm_matches_torch_fp64(orc):
    I, H, T = 12, 10, 17
    m = torch.nn.LSTM(I, H, num_layers=2, dtype=torch.float64)
    x = torch.randn(T, 1, I, dtype=torch.float64)
    with torch.no_grad():
        ref, (hn, cn) = m(x)
    layers = []
    for l in range(2):
        layers.append((getattr(m, f"weight_ih_l{l}").detach().numpy(), getattr(m, f"weight_hh_l{l}").detach().numpy(),
                       (getattr(m, f"bias_ih_l{l}") + getattr(m, f"bias_hh_l{l}")).detach().numpy()))
    out, states, _ = orc.lstm(x[:, 0].numpy(), layers)
    assert np.max(np.abs(out - ref[:, 0].numpy())) < 1e-13
    for l in range(2):
        assert np.max(np.abs(states[l][0] - hn[l, 0].numpy())) < 1e-13
        assert np.max(np.abs(states[l][1] - cn[l, 0].numpy())) < 1e-13


# ---------------------------------------------------------------- O7
def _tree_params(I, H):
    return (rng.standard_normal((3 * H, I)) * 0.3, rng.standard_normal(3 * H) * 0.1,
            rng.standard_normal((5 * H, 2 * H)) * 0.3, rng.standard_normal(5 * H) * 0.1)


def test_tree_single_leaf_and_three_nodes(orc):
    I, H = 7, 5
    W_l, b_l, U, b_u = _tree_params(I, H)
    X = rng.standard_normal((2, I))
    Hn, Cn = orc.treelstm(0, [-1], [-1], [1], X, W_l, b_l, U, b_u)
    z = W_l @ X[1] + b_l
    c = _sig(z[:H]) * np.tanh(z[2 * H:])
    assert np.max(np.abs(Cn[0] - c)) < 1e-15
    assert np.max(np.abs(Hn[0] - _sig(z[H:2 * H]) * np.tanh(c))) < 1e-15
    # root 2 with leaves 0 (word 0) and 1 (word 1), expanded by hand
    Hn, Cn = orc.treelstm(2, [-1, -1, 0], [-1, -1, 1], [0, 1, -1], X, W_l, b_l, U, b_u)
    hs, cs = [], []
    for w in (0, 1):
        z = W_l @ X[w] + b_l
        c = _sig(z[:H]) * np.tanh(z[2 * H:]); hs.append(_sig(z[H:2 * H]) * np.tanh(c)); cs.append(c)
    z = U @ np.concatenate(hs) + b_u
    c = _sig(z[:H]) * np.tanh(z[4 * H:]) + _sig(z[H:2 * H]) * cs[0] + _sig(z[2 * H:3 * H]) * cs[1]
    assert np.max(np.abs(Cn[2] - c)) < 1e-14
    assert np.max(np.abs(Hn[2] - _sig(z[3 * H:4 * H]) * np.tanh(c))) < 1e-14


def _random_tree(n_leaves, rs):
    """Uniform recursive split; returns (root, left, right, word) with leaves first."""
    left, right, word = [], [], []

    def build(lo, hi):
        if hi - lo == 1:
            left.append(-1); right.append(-1); word.append(lo)
            return len(left) - 1
        mid = rs.integers(lo + 1, hi)
        l = build(lo, mid); r = build(mid, hi)
        left.append(l); right.append(r); word.append(-1)
        return len(left) - 1
    root = build(0, n_leaves)
    return root, left, right, word


def test_tree_mirror_symmetry(orc):
    I, H = 6, 4
    W_l, b_l, U, b_u = _tree_params(I, H)
    X = rng.standard_normal((9, I))
    root, left, right, word = _random_tree(9, np.random.default_rng(3))
    Hn, Cn = orc.treelstm(root, left, right, word, X, W_l, b_l, U, b_u)
    # mirror: swap children, swap U's h_l/h_r column blocks and f_l/f_r row blocks
    Um = U.copy()
    Um = np.concatenate([Um[:, H:], Um[:, :H]], axis=1)
    Um[[*range(H, 2 * H), *range(2 * H, 3 * H)]] = Um[[*range(2 * H, 3 * H), *range(H, 2 * H)]]
    bm = b_u.copy()
    bm[H:3 * H] = np.concatenate([b_u[2 * H:3 * H], b_u[H:2 * H]])
    Hm, Cm = orc.treelstm(root, right, left, word, X, W_l, b_l, Um, bm)
    assert np.max(np.abs(Hm - Hn)) < 1e-13 and np.max(np.abs(Cm - Cn)) < 1e-13


def test_tree_identical_leaves_complete_tree(orc):
    I, H = 5, 3
    W_l, b_l, U, b_u = _tree_params(I, H)
    X = np.tile(rng.standard_normal((1, I)), (8, 1))
    # complete binary tree over 8 leaves: leaves 0..7, then level nodes
    left = [-1] * 8 + [0, 2, 4, 6, 8, 10, 12]
    right = [-1] * 8 + [1, 3, 5, 7, 9, 11, 13]
    word = list(range(8)) + [-1] * 7
    Hn, _ = orc.treelstm(14, left, right, word, X, W_l, b_l, U, b_u)
    for level in ([0, 8], [8, 12], [12, 14]):
        blk = Hn[level[0]:level[1]]
        assert np.max(np.abs(blk - blk[0])) == 0.0


def test_tree_matches_torch_recursive(orc):
    I, H = 8, 6
    W_l, b_l, U, b_u = _tree_params(I, H)
    X = rng.standard_normal((13, I))
    root, left, right, word = _random_tree(13, np.random.default_rng(11))
    Hn, Cn = orc.treelstm(root, left, right, word, X, W_l, b_l, U, b_u)
    tW, tb, tU, tbu, tX = (torch.tensor(a) for a in (W_l, b_l, U, b_u, X))

    def node(i):
        if left[i] < 0:
            i_, o_, u_ = torch.split(F.linear(tX[word[i]], tW, tb), H)
            c = torch.sigmoid(i_) * torch.tanh(u_)
            return torch.sigmoid(o_) * torch.tanh(c), c
        (hl, cl), (hr, cr) = node(left[i]), node(right[i])
        i_, fl, fr, o_, u_ = torch.split(F.linear(torch.cat([hl, hr]), tU, tbu), H)
        c = torch.sigmoid(i_) * torch.tanh(u_) + torch.sigmoid(fl) * cl + torch.sigmoid(fr) * cr
        return torch.sigmoid(o_) * torch.tanh(c), c
    h, c = node(root)
    assert np.max(np.abs(Hn[root] - h.numpy())) < 1e-13 and np.max(np.abs(Cn[root] - c.numpy())) < 1e-13


# ---------------------------------------------------------------- O8
def test_bert_layer_matches_torch(orc):
    L, d, nh, f = 11, 64, 4, 128
    w = {"Wqkv": rng.standard_normal((3 * d, d)) * 0.1, "bqkv": rng.standard_normal(3 * d) * 0.1,
         "Wo": rng.standard_normal((d, d)) * 0.1, "bo": rng.standard_normal(d) * 0.1,
         "g1": 1 + 0.1 * rng.standard_normal(d), "be1": 0.1 * rng.standard_normal(d),
         "W1": rng.standard_normal((f, d)) * 0.1, "b1": rng.standard_normal(f) * 0.1,
         "W2": rng.standard_normal((d, f)) * 0.1, "b2": rng.standard_normal(d) * 0.1,
         "g2": 1 + 0.1 * rng.standard_normal(d), "be2": 0.1 * rng.standard_normal(d)}
    X = rng.standard_normal((L, d))
    Y = orc.bert_layer(X, w, nh)
    t = {k: torch.tensor(v) for k, v in w.items()}
    x = torch.tensor(X)
    qkv = F.linear(x, t["Wqkv"], t["bqkv"])
    q, k, v = (z.view(L, nh, d // nh).transpose(0, 1) for z in qkv.split(d, -1))
    att = F.softmax(q @ k.transpose(1, 2) / 8.0 if d // nh == 64 else q @ k.transpose(1, 2) / np.sqrt(d // nh), -1)
    ctx = (att @ v).transpose(0, 1).reshape(L, d)
    h1 = F.layer_norm(F.linear(ctx, t["Wo"], t["bo"]) + x, (d,), t["g1"], t["be1"], eps=1e-12)
    o = F.linear(F.gelu(F.linear(h1, t["W1"], t["b1"])), t["W2"], t["b2"]) + h1
    ref = F.layer_norm(o, (d,), t["g2"], t["be2"], eps=1e-12)
    assert np.max(np.abs(Y - ref.numpy())) < 1e-11


# ---------------------------------------------------------------- O9
def test_request_cost_closed_form(orc):
    # BERT-large per-request flops: 24 layers x (24 L d^2 + 4 L^2 d), d = 1024
    for L in (1, 7, 128, 512):
        assert orc.request_cost(L) == 24 * (24 * L * 1024 ** 2 + 4 * L * L * 1024)


def test_partition_worked_example(orc):
    # lens [512, 1, 256, 256] on G = 2: 512 -> rank0, 256 -> rank1, 256 -> rank1, 1 -> rank1
    st, owner = orc.partition_lpt([512, 1, 256, 256], 2)
    assert st == 0 and list(owner) == [0, 1, 1, 1]


def test_partition_lpt_bound_brute_force(orc):
    # LPT makespan <= (4/3 - 1/(3G)) * OPT (Graham 1969); OPT by exhaustive search
    rs = np.random.default_rng(5)
    for trial in range(30):
        R = int(rs.integers(1, 8)); G = int(rs.integers(1, 4))
        lens = rs.integers(1, 513, R)
        st, owner = orc.partition_lpt(lens, G)
        cost = [orc.request_cost(int(L)) for L in lens]
        assert st == 0 and set(owner.tolist()) <= set(range(G)) and len(owner) == R
        loads = [sum(c for c, o in zip(cost, owner) if o == g) for g in range(G)]
        opt = min(max(sum(c for c, a in zip(cost, asg) if a == g) for g in range(G))
                  for asg in itertools.product(range(G), repeat=R))
        assert max(loads) * 3 * G <= (4 * G - 1) * opt


def test_partition_deterministic_and_total(orc):
    lens = np.random.default_rng(2).integers(1, 513, 500)
    for G in (1, 2, 4, 8):
        st1, o1 = orc.partition_lpt(lens, G)
        st2, o2 = orc.partition_lpt(lens, G)
        assert st1 == 0 and np.array_equal(o1, o2) and o1.min() >= 0 and o1.max() < G
