"""Pins for oracle O1 (shape functions) and O2 (dispatch rule).

O1 is pinned to the broadcast rules printed at PAPER.md:230-235 (golden file), to
numpy's broadcasting (the footnote at PAPER.md:228 cites it) by exhaustive
enumeration, and to invariants (symmetry, error iff static mismatch).
O2 is pinned to the paper's residue identity x = t*k + r, the SPEC
worked examples (golden file), and the totality/uniqueness invariants.
"""
import itertools
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ANY = -1


def _read_golden(name):
    rows = []
    for line in open(os.path.join(HERE, "golden", name)):
        line = line.split("#")[0].strip()
        if line:
            rows.append(line.split())
    return rows


def _tok(v):
    return ANY if v == "ANY" else int(v)


def test_broadcast_rel_golden(orc):
    for a, b, e in _read_golden("broadcast_rel.txt"):
        st, out = orc.bcast(_tok(a), _tok(b))
        assert st == 0 and out == _tok(e), (a, b, e, out)


def test_broadcast_static_matches_numpy(orc):
    # brute force over static dims 1..8: the oracle agrees with numpy broadcasting
    for a, b in itertools.product(range(1, 9), repeat=2):
        st, out = orc.bcast(a, b)
        try:
            ref = np.broadcast_shapes((a,), (b,))[0]
            assert st == 0 and out == ref
        except ValueError:
            assert st == -3 and a != b and a > 1 and b > 1


def test_broadcast_symmetric_and_any(orc):
    dims = [ANY] + list(range(1, 9))
    for a, b in itertools.product(dims, repeat=2):
        s1, o1 = orc.bcast(a, b)
        s2, o2 = orc.bcast(b, a)
        assert (s1, o1) == (s2, o2)
        if ANY in (a, b):
            assert s1 == 0          # Any never fails statically (gradual typing)


def test_shape_dense_rules(orc):
    # config 3 QKV: (L,768) x (2304,768) -> (L,2304); Any propagates
    assert orc.shape_dense((37, 768), (2304, 768)) == (0, (37, 2304))
    assert orc.shape_dense((ANY, 768), (2304, 768)) == (0, (ANY, 2304))
    assert orc.shape_dense((5, ANY), (7, 3)) == (0, (5, 7))            # deferred K check
    assert orc.shape_dense((5, 4), (7, 3))[0] == -3                    # runtime K mismatch
    assert orc.shape_dense((0, 4), (7, 4))[0] == -4                    # extent 0
    # exhaustive: error iff both K static and different
    dims = [ANY] + list(range(1, 6))
    for a0, a1, w0, w1 in itertools.product(dims, repeat=4):
        st, out = orc.shape_dense((a0, a1), (w0, w1))
        if a1 != ANY and w1 != ANY and a1 != w1:
            assert st == -3
        else:
            assert st == 0 and out == (a0, w0)


def test_shape_bmm_rules(orc):
    # config 3 scores: (12,L,64) x (12,L,64) -> (12,L,L); context with trans_b
    assert orc.shape_bmm((12, 50, 64), (12, 50, 64), 0) == (0, (12, 50, 50))
    assert orc.shape_bmm((12, 50, 50), (12, 50, 64), 1) == (0, (12, 50, 64))
    assert orc.shape_bmm((12, ANY, 64), (12, ANY, 64), 0) == (0, (12, ANY, ANY))
    assert orc.shape_bmm((1, 5, 3), (4, 6, 3), 0) == (0, (4, 5, 6))    # batch broadcast
    assert orc.shape_bmm((2, 5, 3), (4, 6, 3), 0)[0] == -3
    assert orc.shape_bmm((2, 5, 3), (2, 6, 4), 0)[0] == -3
    dims = [ANY, 1, 2, 3]
    for p0, p2, q0, q1, q2 in itertools.product(dims, repeat=5):
        for tb in (0, 1):
            st, out = orc.shape_bmm((p0, 4, p2), (q0, q1, q2), tb)
            kb = q1 if tb else q2
            kbad = p2 != ANY and kb != ANY and p2 != kb
            bbad = p0 != ANY and q0 != ANY and p0 != q0 and p0 > 1 and q0 > 1
            if kbad or bbad:
                assert st == -3
            else:
                assert st == 0
                assert out[1] == 4 and out[2] == (q2 if tb else q1)


def test_sub_shape_example(orc):
    # Tensor[(128,128)] is a sub-type of Tensor[(Any,128)] -- instantiating Any
    # by 128 in the type relation must give the same output shape as the static one.
    st1, o1 = orc.shape_dense((ANY, 128), (64, 128))
    st2, o2 = orc.shape_dense((128, 128), (64, 128))
    assert st1 == st2 == 0 and o1 == (ANY, 64) and o2 == (128, 64)


def test_dispatch_worked_examples(orc):
    for M, c, k, r, v in _read_golden("residue_examples.txt"):
        st, d = orc.dispatch_dense(int(M), 128, 128, 0, int(c))
        assert st == 0
        assert (d["k"], d["r"], d["variant"]) == (int(k), int(r), int(v)), (M, c, d)


def _pairs(M, N, batch=1):
    """DISPATCH.md "Family 3": CTA pairs exactly when their 256 x 256 tiles need fewer waves
    (74 pairs) than 128 x 128 tiles (148 CTAs)."""
    waves_128 = -(-(-(-N // 128) * -(-M // 128) * batch) // 148)
    waves_256 = -(-(-(-N // 256) * -(-M // 256) * batch) // 74)
    return waves_256 < waves_128


def test_dispatch_pair_rule_examples(orc):
    # the measured crossovers DISPATCH.md cites (profiles/r02e_f1_vs_f3.jsonl): equal waves keep
    # family 1 (2048 x 1024: 1 wave either way), fewer pair waves take family 3 at any M
    for (M, N, K, fam) in [(2048, 1024, 1024, 1), (2304, 1024, 1024, 1), (2433, 1024, 1024, 3),
                           (2560, 1024, 1024, 3), (2048, 1024, 4096, 1), (2560, 1024, 4096, 3),
                           (1024, 3072, 1024, 3), (768, 3072, 1024, 1), (768, 4096, 1024, 3),
                           (3072, 768, 768, 1), (4096, 768, 768, 3), (1536, 2304, 768, 3),
                           (1024, 2304, 768, 1), (17448, 1024, 1024, 3), (2048, 3072, 1024, 3)]:
        st, d = orc.dispatch_dense(M, N, K, 1)
        assert st == 0 and d["family"] == fam and _pairs(M, N) == (fam == 3), (M, N, K, d)
        assert d["cluster"][0] == (2 if fam == 3 else 1) and d["umma_m"] == (256 if fam == 3 else 128)
        # padding M to a multiple of 128 keeps the family (pad-then-slice)
        assert orc.dispatch_dense(128 * -(-M // 128), N, K, 1)[1]["family"] == fam
    # a tuned schedule replaces the rule below M = 2048 only
    assert orc.dispatch_dense(1024, 3072, 1024, 1, 0, 64, 1)[1]["family"] == 1
    assert orc.dispatch_dense(4096, 3072, 1024, 1, 0, 64, 1)[1]["family"] == 3
    assert orc.dispatch_dense(2048, 1024, 1024, 1, 0, 64, 1)[1]["tile_t"] == 128
    # bmm: heads multiply the tile counts
    assert orc.dispatch_bmm(16, 512, 512, 64, 0, 1)[1]["family"] == (3 if _pairs(512, 512, 16) else 1)
    assert orc.dispatch_bmm(16, 2048, 2048, 64, 0, 1)[1]["family"] == 3


@pytest.mark.parametrize("dt", [0, 1])
def test_dispatch_invariants(orc, dt):
    for M in list(range(1, 2049)) + list(range(2400, 2600)) + [4095, 4096, 4097, 65535, 65536]:
        wide = dt == 1 and _pairs(M, 1024)
        t = 8 if dt == 0 else (256 if wide else 128)
        for c in (0, 1, 2, 5, 8, 9, 17):
            st, d = orc.dispatch_dense(M, 1024, 1024, dt, c)
            assert st == 0
            assert d["tile_t"] == t
            assert d["n_classes"] == (8 if dt == 0 else t // 16 + 1)
            assert d["k"] * t + d["r"] == M and 0 <= d["r"] < t           # x = t k + r
            assert d["grid"][1] == d["k"] + (d["r"] > 0)                  # every row covered once
            n = d["n_classes"]
            if c in (0,) or c >= n:
                assert d["variant"] == d["residue_class"]                   # full dispatch
            if c == 1:
                assert d["variant"] == -1                                   # no dispatch
            if dt == 1 and d["r"] > 0:
                # the tail UMMA width covers the residue with < 16 wasted columns when specialised
                if d["variant"] >= 0:
                    assert d["r"] <= d["umma_n_tail"] < d["r"] + 16 and d["umma_n_tail"] % 16 == 0
                else:
                    assert d["umma_n_tail"] == t
            if dt == 1 and M <= 128:
                # family 4 (weight streaming): 8 feature tiles x 1 token tile x S splits of the
                # 16 k-blocks, one wave (8 S <= 148), no cluster record; S does not depend on M
                s = d["split_k"]
                assert d["family"] == 4 and d["umma_m"] == 128 and list(d["cluster"]) == [1, 1, 1]
                assert list(d["grid"]) == [8, 1, s] and s == 8             # min(16 k-blocks, 148 // 8, 8)
            elif dt == 1:
                s = d["split_k"]
                assert s in (1, 2, 4, 8) and d["cluster"] == ((2 if wide else 1), 1, s)
                assert d["umma_m"] == (256 if wide else 128)
                assert (1024 // 64) // s >= 4 or s == 1
                assert d["family"] == (3 if wide else 1)
                if wide:
                    assert s == 1


def test_dispatch_errors(orc):
    assert orc.dispatch_dense(0, 128, 128, 0)[0] == -4
    assert orc.dispatch_dense(5, 0, 128, 0)[0] == -4
    assert orc.dispatch_dense(5, 128, 128, 7)[0] == -5
    assert orc.dispatch_dense(5, 128, 128, 0, -1)[0] == -4
    assert orc.dispatch_bmm(12, 5, 5, 64, 0, 0)[0] == -7
    assert orc.dispatch_bmm(0, 5, 5, 64, 0, 1)[0] == -4


def test_dispatch_bmm_families(orc):
    st, d = orc.dispatch_bmm(16, 300, 300, 64, 0, 1)
    assert st == 0 and d["family"] == 1 and d["grid"][0] == 3 and d["grid"][1] == 3
    st, d = orc.dispatch_bmm(16, 300, 64, 300, 1, 1)
    assert st == 0 and d["family"] == 2 and d["k"] == 2 and d["r"] == 44
    assert d["umma_n_full"] == 64 and d["umma_n_tail"] == 64 and d["grid"][1] == 1


def test_dispatch_weight_streaming_family(orc):
    """Family 4 pins (DISPATCH.md): taken exactly when M <= 128 and the 128-feature tiles fit
    one wave; grid = tiles x S with S = min(k-blocks, 148 // tiles, 8) >= 1 — every CTA owns at
    least one k-block of 64, the grid never exceeds one wave of 148 and a tile's splits fit one
    cluster; S is the same for every M (pad-then-slice invariant); the residue split equals
    family 1's."""
    cases = [(2304, 768, 8), (768, 768, 8), (3072, 768, 6), (768, 3072, 8), (1024, 1024, 8),
             (3072, 1024, 6), (4096, 1024, 4), (1024, 4096, 8), (128, 64, 1), (128, 100000, 8),
             (18944, 512, 1), (300, 200, 4)]
    for N, K, S in cases:
        tiles = -(-N // 128)
        for M in (1, 2, 15, 16, 17, 100, 127, 128):
            st, d = orc.dispatch_dense(M, N, K, 1)
            assert st == 0 and d["family"] == 4 and d["split_k"] == S, (N, K, M, d)
            assert tiles * S <= 148 and S <= -(-K // 64) and S <= 8
            assert list(d["grid"]) == [tiles, 1, S]
            d1 = orc.dispatch_dense(M, N, K, 1, 0, 128, 1)[1]      # family 1 with the same t
            for key in ("k", "r", "residue_class", "variant", "umma_n_full", "umma_n_tail", "n_classes"):
                assert d[key] == d1[key], key
    # several token tiles (M <= 1024): family 4 only at K >= 2048 and while the split stays >= 2
    # (fewer than 75 units), with S = min(k-blocks, 148 // units, 8); the same S for M and M
    # padded to 128 k
    for (N, K, M, fam, S) in [(2304, 768, 129, 1, 1), (3072, 1024, 129, 1, 1), (4096, 2048, 200, 4, 2),
                              (4096, 2048, 300, 1, 1), (1024, 4096, 1024, 4, 2), (1024, 4096, 1025, 1, 1),
                              (1024, 4096, 513, 4, 3), (768, 3072, 1000, 4, 3), (3072, 3072, 384, 4, 2),
                              (3072, 3072, 512, 1, 1), (1024, 1024, 513, 1, 1)]:
        d = orc.dispatch_dense(M, N, K, 1)[1]
        assert d["family"] == fam, (N, K, M, d)
        if fam == 4:
            Mp = 128 * -(-M // 128)
            assert d["split_k"] == S and list(d["grid"]) == [-(-N // 128), -(-M // 128), S]
            assert orc.dispatch_dense(Mp, N, K, 1)[1]["split_k"] == S
    # more feature tiles than one wave: family 1
    assert orc.dispatch_dense(5, 149 * 128, 256, 1)[1]["family"] == 1
    assert orc.dispatch_dense(5, 148 * 128, 256, 1)[1]["family"] == 4
    # fp32 keeps the paper's SIMT8 family
    assert orc.dispatch_dense(5, 1024, 1024, 0)[1]["family"] == 0


@pytest.mark.parametrize("tile_t,split_max", [(32, 8), (64, 2), (128, 8), (256, 4)])
def test_oracle_tuned_schedule_invariants(orc, tile_t, split_max):
    """Pins of the schedule-parameterised dispatch (DISPATCH.md "Tuned schedules"): the
    decomposition x = t k + r with 0 <= r < t, class = ceil(r / 16), t/16 + 1 classes, the
    tail width 16 class, one token tile per t tokens (+1 for a residue), split-K a power of
    two <= split_max that keeps one wave (tiles * 2s <= 148) — and (128, 8) reproduces the
    default schedule exactly; M >= 2048 ignores the schedule."""
    N, K = 1024, 4096
    m_tiles = -(-N // 128)
    for M in list(range(1, 600)) + [1000, 2047]:
        st, d = orc.dispatch_dense(M, N, K, 1, 0, tile_t, split_max)
        assert st == 0 and d["family"] == 1 and d["tile_t"] == tile_t
        assert d["k"] * tile_t + d["r"] == M and 0 <= d["r"] < tile_t
        assert d["residue_class"] == -(-d["r"] // 16) and d["n_classes"] == tile_t // 16 + 1
        assert d["umma_n_full"] == tile_t
        assert d["umma_n_tail"] == (0 if d["r"] == 0 else 16 * d["residue_class"])
        n_tiles = d["k"] + (d["r"] > 0)
        assert list(d["grid"][:2]) == [m_tiles, n_tiles]
        s = d["split_k"]
        assert s in (1, 2, 4, 8) and s <= split_max and (s == 1 or m_tiles * n_tiles * s <= 148)
        assert tile_t <= 128 or s == 1
        assert d["grid"][2] == s and list(d["cluster"]) == [1, 1, s]
        if tile_t == 128 and split_max == (8 if K >= 2048 else 1) and orc.dispatch_dense(M, N, K, 1)[1]["family"] != 4:
            assert d == orc.dispatch_dense(M, N, K, 1)[1]     # the default rule's (t, cap)
    for M in (2048, 5000):
        assert orc.dispatch_dense(M, N, K, 1, 0, tile_t, split_max)[1] == orc.dispatch_dense(M, N, K, 1)[1]
