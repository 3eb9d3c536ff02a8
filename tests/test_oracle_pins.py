"""Pins for the CPU oracle (-m "not gpu").

Each oracle function is checked against something other than itself:
hand-worked examples, constructed closed forms, exact rational arithmetic,
library routines on special cases, an independent algorithm (tuple buckets)
and brute force.  Citations: P:n = PAPER.md line, S:n = SPEC.md line.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import pqsynth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def f32(x):
    return np.array(x, dtype=np.float32)


# ---------------------------------------------------------------- F1 hand instance
def test_spec_hand_instance(orc):
    """SPEC hand instance."""
    g = load("spec_hand_instance.json")
    phi, psi = f32(g["phi"]), f32(g["psi"])
    codes = np.array(g["codes"], np.uint8)
    S64, _ = orc.subscores64(phi, psi)
    assert np.array_equal(S64, np.array(g["S"], np.float64))
    S = S64.astype(np.float32)
    for fn in (orc.scores_alg1, orc.scores_alg2, orc.scores_numpy):
        assert np.array_equal(fn(codes, S[0]), f32(g["scores"]))
    W = orc.reconstruct(codes, psi)
    assert np.array_equal(W[0], f32(g["w0"]))
    for K, key in ((3, "top3"), (2, "top2"), (5, "top5")):
        ids, sc = orc.pq_topk(codes, S, K)
        assert ids[0].tolist() == g[key + "_ids"]
        assert sc[0].tolist() == [float(x) for x in g[key + "_scores"]]
        ids2, sc2 = orc.tuple_topk(codes, S, K)
        assert np.array_equal(ids2, ids) and np.array_equal(sc2, sc)
        ids3, sc3 = orc.recjpq_topk(codes, S, K)
        assert np.array_equal(ids3, ids) and np.array_equal(sc3, sc)
    # dense fp64 scoring (Eq. 3) gives the same numbers exactly here
    assert orc.dense_scores64(codes, psi, phi[0]).tolist() == g["scores"]
    # K = 0: empty result
    ids, sc = orc.pq_topk(codes, S, 0)
    assert ids.shape == (1, 0)


# ---------------------------------------------------------------- F2 order pin
def test_order_pin(orc):
    g = load("order_pin.json")
    S = f32(g["S"])
    codes = np.array(g["codes"], np.uint8)
    for fn in (orc.scores_alg1, orc.scores_alg2, orc.scores_numpy):
        assert fn(codes, S[0]).tolist() == g["scores_k_order"]
    # the alternatives really do differ (the pin is sensitive to the order)
    v = [S[0][k][0] for k in range(4)]
    assert float((v[0] + v[1]) + (v[2] + v[3])) == g["pairwise_item0"]
    assert float(((v[3] + v[2]) + v[1]) + v[0]) == g["reverse_item0"]
    assert sum(Fraction(float(x)) for x in v) == g["exact_item0"]
    ids, sc = orc.pq_topk(codes, S, 5)
    assert ids[0].tolist() == g["top5_ids"] and sc[0].tolist() == g["top5_scores"]


# ---------------------------------------------------------------- F3 -0 pin
def test_negzero_pin(orc):
    g = load("negzero_pin.json")
    S = np.array(g["S"], np.float32)
    assert np.signbit(S[0, 0, 0])
    codes = np.array(g["codes"], np.uint8)
    for fn in (orc.scores_alg1, orc.scores_alg2, orc.scores_numpy):
        r = fn(codes, S[0])
        assert np.signbit(r).astype(int).tolist() == g["scores_signbit"]
    ids, sc = orc.pq_topk(codes, S, 2)
    assert ids[0].tolist() == g["top2_ids"]
    assert not np.signbit(sc).any()


# ---------------------------------------------------------------- F4 all ties
@pytest.mark.parametrize("K", [1, 7, 50, 60])
def test_all_ties(orc, K):
    """b = 1: every item has the same score; top-K = ids 0..K-1."""
    G, P, F = pqsynth.random_instance(11, 50, 3, 1, 6, 2)
    S = orc.subscores(F, P)
    ids, sc = orc.pq_topk(G, S, K, id_base=1000)
    n = min(K, 50)
    for u in range(2):
        expect = float(orc.scores_numpy(G[:1], S[u])[0])
        assert ids[u, :n].tolist() == list(range(1000, 1000 + n))
        assert (sc[u, :n] == np.float32(expect)).all()
        assert (ids[u, n:] == -1).all() and np.isneginf(sc[u, n:]).all()


# ---------------------------------------------------------------- F5 m = 1
def test_m1_is_gather_then_stable_argsort(orc):
    G, P, F = pqsynth.random_instance(12, 3000, 1, 64, 8, 3)
    S = orc.subscores(F, P)
    ids, sc = orc.pq_topk(G, S, 40)
    for u in range(3):
        r = S[u][0][G[:, 0]]                      # m = 1: score = S[1, g_i1]
        order = np.argsort(-r, kind="stable")[:40]
        assert ids[u].tolist() == order.tolist()
        assert np.array_equal(sc[u], r[order])


# ---------------------------------------------------------------- F6 boundaries
def test_k_gt_n_and_empty(orc):
    G, P, F = pqsynth.random_instance(13, 5, 2, 4, 4, 2)
    S = orc.subscores(F, P)
    ids, sc = orc.pq_topk(G, S, 9)
    assert (ids[:, 5:] == -1).all() and np.isneginf(sc[:, 5:]).all()
    assert sorted(ids[0, :5].tolist()) == list(range(5))
    ids, sc = orc.pq_topk(G, S[:0], 3)
    assert ids.shape == (0, 3)


# ---------------------------------------------------------------- F13 Eq. 4 exact
def _round_f32(x: Fraction) -> np.float32:
    """Correctly rounded fp32 of an exact rational (ties to even)."""
    c = np.float32(float(x))
    cands = [np.nextafter(c, np.float32(-np.inf)), c, np.nextafter(c, np.float32(np.inf))]
    best = min(cands, key=lambda y: (abs(Fraction(float(y)) - x),
                                     int(np.float32(y).view(np.uint32)) & 1))
    return np.float32(best)


@pytest.mark.parametrize("seed,m,b,d,B", [(21, 4, 8, 32, 2), (22, 8, 16, 64, 1), (23, 2, 5, 64, 3)])
def test_subscores_exact_rational(orc, seed, m, b, d, B):
    """Eq. 4 against exact rational arithmetic: S64 within the fp64
    recursive-summation bound, and fl32(S64) == correctly rounded exact value."""
    G, P, F = pqsynth.random_instance(seed, 1, m, b, d, B)
    S64, C = orc.subscores64(F, P)
    dm = d // m
    gam = dm * 2.0 ** -53 / (1 - dm * 2.0 ** -53)
    for u in range(B):
        for k in range(m):
            for g in range(b):
                ex = sum(Fraction(float(P[k, g, t])) * Fraction(float(F[u, k * dm + t]))
                         for t in range(dm))
                assert abs(Fraction(S64[u, k, g]) - ex) <= Fraction(gam) * Fraction(C[u, k, g])
                assert np.float32(S64[u, k, g]) == _round_f32(ex)
    # the split of phi is contiguous: permuting phi outside chunk k
    # leaves S[:, k] unchanged
    F2 = F.copy()
    F2[:, dm:] = F2[:, dm:][:, ::-1]
    assert np.array_equal(orc.subscores64(F2, P)[0][:, 0], S64[:, 0])


def test_subscores_zero_cases(orc):
    """Psi = 0 or phi = 0 -> S = 0."""
    G, P, F = pqsynth.random_instance(24, 1, 4, 8, 16, 2)
    assert not orc.subscores64(F, np.zeros_like(P))[0].any()
    assert not orc.subscores64(np.zeros_like(F), P)[0].any()


# ---------------------------------------------------------------- F7 Alg. 1 == Alg. 2
def test_alg1_equals_alg2_bitwise(orc):
    rng = np.random.default_rng(7)
    for it in range(120):
        N = int(rng.integers(1, 400)); m = int(rng.integers(1, 9)); b = int(rng.integers(1, 257))
        G = rng.integers(0, b, size=(N, m)).astype(np.uint8)
        S = (rng.standard_normal((m, b)) * 10.0 ** rng.uniform(-3, 3)).astype(np.float32)
        r1, r2, r3 = orc.scores_alg1(G, S), orc.scores_alg2(G, S), orc.scores_numpy(G, S)
        assert np.array_equal(r1.view(np.uint32), r2.view(np.uint32))
        assert np.array_equal(r1.view(np.uint32), r3.view(np.uint32))


# ---------------------------------------------------------------- F8 dense vs PQ
@pytest.mark.parametrize("seed,N,m,b,d,scale", [(31, 20000, 8, 256, 64, 1.0),
                                                (32, 20000, 8, 256, 512, 0.02),
                                                (33, 8000, 16, 256, 512, 1.0),
                                                (34, 20000, 4, 16, 64, 1.0)])
def test_dense_fp64_vs_pq_fp32(orc, seed, N, m, b, d, scale):
    """Eq. 2-3 (dense, fp64) vs Eq. 5 (PQ, fp32) within the closed-form bound;
    top-K id sets agree whenever the K-th/(K+1)-th gap exceeds twice it."""
    G, P, F = pqsynth.random_instance(seed, N, m, b, d, 2, scale=scale)
    S64, C = orc.subscores64(F, P)
    S = S64.astype(np.float32)
    W = orc.reconstruct(G, P)
    for u in range(2):
        r64 = orc.dense_scores64(G, P, F[u])
        assert np.allclose(r64, W.astype(np.float64) @ F[u].astype(np.float64), rtol=0, atol=1e-9)
        rpq = orc.scores_alg1(G, S[u])
        bound = orc.dense_error_bound(S[u], S64[u], G, C[u], d)
        assert (np.abs(rpq.astype(np.float64) - r64) <= bound).all()
        K = 10
        ids64, s64 = orc.topk_sort64(r64, K + 1)
        ids, _ = orc.pq_topk(G, S[u:u + 1], K)
        gap = s64[K - 1] - s64[K]
        if gap > 2 * bound.max():
            assert set(ids[0].tolist()) == set(ids64[:K].tolist())


# ---------------------------------------------------------------- F9 brute force
@pytest.mark.parametrize("dist", ["uniform", "zipf", "few"])
def test_pq_topk_vs_bruteforce_sort(orc, dist):
    rng = np.random.default_rng({"uniform": 1, "zipf": 2, "few": 3}[dist])
    for it in range(25):
        N = int(rng.integers(1, 10001)); m = int(rng.choice([1, 2, 4, 8, 16]))
        b = int(rng.choice([1, 2, 16, 256])); K = int(rng.choice([1, 10, 100, 1000]))
        G, P, F = pqsynth.random_instance(1000 + it, N, m, b, m * 2, 2, code_dist=dist)
        S = orc.subscores(F, P)
        ids, sc = orc.pq_topk(G, S, K, id_base=77)
        for u in range(2):
            r = orc.scores_numpy(G, S[u])
            ids_b, sc_b = orc.topk_numpy(r, K, id_base=77)
            assert np.array_equal(ids[u], ids_b), (it, N, m, b, K)
            assert np.array_equal(sc[u].view(np.uint32), sc_b.view(np.uint32))
            ids_s, sc_s = orc.topk_sort(r, K, id_base=77)
            assert np.array_equal(ids_s, ids_b)


# ---------------------------------------------------------------- F10 tuple buckets
def test_tuple_bucket_equals_bruteforce_c5_shape(orc):
    """C5-shaped (m=4, b=16): independent tuple-bucket algorithm == Alg. 1."""
    G, P, F = pqsynth.random_instance(41, 200_000, 4, 16, 64, 3)
    S = orc.subscores(F, P)
    a = orc.pq_topk(G, S, 1000, id_base=5)
    t = orc.tuple_topk(G, S, 1000, id_base=5)
    assert np.array_equal(a[0], t[0]) and np.array_equal(a[1], t[1])


def test_tuple_structure_massive_ties(orc):
    """When the best tuple holds >= K items, every top-K score equals that tuple's
    fp32 sum and the ids are the smallest ids carrying an equal-score tuple."""
    G, P, F = pqsynth.random_instance(42, 200_000, 2, 16, 16, 2)
    S = orc.subscores(F, P)
    K = 500
    ids, sc = orc.pq_topk(G, S, K)
    for u in range(2):
        assert (sc[u] == sc[u, 0]).all()
        assert (np.diff(ids[u]) > 0).all()
        best = float(sc[u, 0])
        has = np.zeros(G.shape[0], bool)
        for g0 in range(16):
            for g1 in range(16):
                if float(np.float32(np.float32(0) + S[u, 0, g0]) + S[u, 1, g1]) == best:
                    has |= (G[:, 0] == g0) & (G[:, 1] == g1)
        assert ids[u].tolist() == np.flatnonzero(has)[:K].tolist()


# ---------------------------------------------------------------- fp environment
def test_fpenv_is_ieee(orc):
    assert orc.lib().orc_check_fpenv() == 0


def test_thread_count_invariance(orc):
    import subprocess, sys, json as js
    code = ("import sys, json, numpy as np; sys.path.insert(0, %r); import oracle, pqsynth;"
            "G,P,F=pqsynth.random_instance(51,30000,8,256,64,2); S=oracle.subscores(F,P);"
            "i,s=oracle.pq_topk(G,S,100); print(json.dumps(i.tolist()))") % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for nt in ("1", "3", "8"):
        env = dict(os.environ, OMP_NUM_THREADS=nt)
        outs.append(subprocess.check_output([sys.executable, "-c", code], env=env, cwd=os.path.dirname(GOLD)))
    assert outs[0] == outs[1] == outs[2]
