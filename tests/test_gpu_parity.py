"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star):
  * S (K1) within 1e-5 relative of the fp64 oracle S64 (mixed 1e-5*C fallback
    only where |S64| < 1e-6*C, reading R5); the number of entries with
    S_gpu != fl32(S64) is reported and expected to be 0;
  * given the GPU's S, top-K ids and scores are BIT-EXACT against the oracle's
    Algorithm 1 (ties: score desc, id asc).
Sizes span several CTA tiles / item chunks and ragged tails.
"""
import json
import os

import numpy as np
import pytest

import pqsynth

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def pq():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2408_09992_b200 as pq
    pq.load_library()
    return pq


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


def cuda(torch, x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def run_pq(pq, torch, G, P, F, K, b=None, id_base=0, tuning=None):
    """K1 + K2 + K3 through the ABI; returns (S_gpu, ids, scores) as numpy."""
    b = P.shape[1] if b is None else b
    idx = pq.pq_create(G, b=b, id_base=id_base)
    if tuning:
        idx.set_tuning(**tuning)
    S = pq.pq_subscores(cuda(torch, F), cuda(torch, P))
    ids, sc = pq.pq_score_topk(idx, S, K)
    torch.cuda.synchronize()
    return S.cpu().numpy(), ids.cpu().numpy(), sc.cpu().numpy(), idx


def assert_same(a_ids, a_sc, b_ids, b_sc, msg=""):
    assert np.array_equal(a_ids, b_ids), msg
    assert np.array_equal(a_sc.view(np.uint32), b_sc.view(np.uint32)), msg


def check_S(orc, F, P, S_gpu):
    S64, C = orc.subscores64(F, P)
    err = np.abs(S_gpu.astype(np.float64) - S64)
    strict = err <= 1e-5 * np.abs(S64)
    small = np.abs(S64) < 1e-6 * C
    mixed = err <= 1e-5 * C
    assert (strict | (small & mixed)).all(), float((err / np.maximum(np.abs(S64), 1e-300)).max())
    return int((S_gpu != S64.astype(np.float32)).sum())


# ------------------------------------------------------------------ fixtures
def test_spec_hand_instance_gpu(pq, torch, orc):
    g = json.load(open(os.path.join(GOLD, "spec_hand_instance.json")))
    P = np.array(g["psi"], np.float32)
    F = np.array(g["phi"], np.float32)
    G = np.array(g["codes"], np.uint8)
    S, ids, sc, idx = run_pq(pq, torch, G, P, F, 3)
    assert S.tolist() == g["S"]
    assert ids[0].tolist() == g["top3_ids"] and sc[0].tolist() == g["top3_scores"]
    S_t = cuda(torch, S)
    for K, key in ((2, "top2"), (5, "top5")):
        i2, s2 = pq.pq_score_topk(idx, S_t, K)
        assert i2.cpu().numpy()[0].tolist() == g[key + "_ids"]
        assert s2.cpu().numpy()[0].tolist() == [float(x) for x in g[key + "_scores"]]
    W = pq.pq_reconstruct(idx, cuda(torch, P)).cpu().numpy()
    assert W[0].tolist() == g["w0"]


def test_order_pin_gpu(pq, torch):
    g = json.load(open(os.path.join(GOLD, "order_pin.json")))
    S = cuda(torch, np.array(g["S"], np.float32))
    idx = pq.pq_create(np.array(g["codes"], np.uint8), b=2)
    ids, sc = pq.pq_score_topk(idx, S, 5)
    assert ids.cpu().numpy()[0].tolist() == g["top5_ids"]
    assert sc.cpu().numpy()[0].tolist() == g["top5_scores"]


def test_negzero_pin_gpu(pq, torch):
    g = json.load(open(os.path.join(GOLD, "negzero_pin.json")))
    S = cuda(torch, np.array(g["S"], np.float32))
    idx = pq.pq_create(np.array(g["codes"], np.uint8), b=2)
    ids, sc = pq.pq_score_topk(idx, S, 2)
    assert ids.cpu().numpy()[0].tolist() == g["top2_ids"]
    assert not np.signbit(sc.cpu().numpy()).any()


def test_all_ties_gpu(pq, torch, orc):
    G, P, F = pqsynth.random_instance(11, 5000, 3, 1, 6, 5)
    S, ids, sc, _ = run_pq(pq, torch, G, P, F, 100, id_base=1000)
    for u in range(5):
        assert ids[u].tolist() == list(range(1000, 1100))
        assert (sc[u] == sc[u, 0]).all()


def test_boundaries_gpu(pq, torch, orc):
    G, P, F = pqsynth.random_instance(13, 5, 2, 4, 4, 3)
    S, ids, sc, idx = run_pq(pq, torch, G, P, F, 9)
    ref = orc.pq_topk(G, S, 9)
    assert_same(ids, sc, *ref)
    assert (ids[:, 5:] == -1).all() and np.isneginf(sc[:, 5:]).all()
    # K = 0 and B = 0: no-ops
    e_ids, e_sc = pq.pq_score_topk(idx, cuda(torch, S), 0)
    assert e_ids.shape == (3, 0)
    e_ids, e_sc = pq.pq_score_topk(idx, cuda(torch, S[:0]), 4)
    assert e_ids.shape == (0, 4)
    with pytest.raises(pq.PQError):
        pq.pq_score_topk(idx, cuda(torch, S), 5000)


def test_code_range_error(pq):
    G = np.zeros((10, 3), np.uint8)
    G[7, 2] = 9
    with pytest.raises(pq.PQError) as e:
        pq.pq_create(G, b=9)
    assert e.value.name == "PQ_ERR_CODE_RANGE" and "item 7 split 2" in str(e.value)


# ------------------------------------------------------------------ random shapes
CASES = [
    # seed, N, m, b, d, B, K, dist
    (101, 1, 8, 256, 64, 1, 10, "uniform"),
    (102, 31, 4, 16, 16, 3, 7, "uniform"),
    (103, 10_000, 8, 256, 64, 1, 10, "uniform"),            # C1 shape
    (104, 100_003, 8, 256, 64, 17, 100, "uniform"),
    (105, 77_777, 16, 256, 512, 40, 100, "uniform"),        # C4-like split count
    (106, 200_001, 4, 16, 64, 33, 1000, "uniform"),         # C5-like ties
    (107, 150_000, 8, 256, 512, 64, 100, "zipf"),           # C3-like
    (108, 60_000, 1, 64, 8, 5, 50, "uniform"),              # m = 1
    (109, 50_000, 3, 256, 24, 9, 20, "uniform"),            # generic m path
    (110, 40_000, 6, 100, 48, 70, 64, "few"),               # generic m, ties
    (111, 300_000, 16, 256, 512, 2, 4096, "uniform"),       # max K
    (112, 120_000, 2, 4, 8, 130, 33, "few"),                # massive ties, many users
]


@pytest.mark.parametrize("case", CASES, ids=[str(c[0]) for c in CASES])
def test_random_parity(pq, torch, orc, case):
    seed, N, m, b, d, B, K, dist = case
    G, P, F = pqsynth.random_instance(seed, N, m, b, d, B, code_dist=dist)
    S, ids, sc, idx = run_pq(pq, torch, G, P, F, K, id_base=seed)
    nmis = check_S(orc, F, P, S)
    assert nmis == 0, f"{nmis} S entries differ from fl32(S64)"
    ref_ids, ref_sc = orc.pq_topk(G, S, K, id_base=seed)
    assert_same(ids, sc, ref_ids, ref_sc, str(case))


@pytest.mark.parametrize("tuning", [dict(users_per_row=4), dict(users_per_row=32, warps=4),
                                    dict(ctas=7, chunks=13), dict(warps=16, chunks=3),
                                    dict(users_per_row=1)])
def test_geometry_invariance(pq, torch, orc, tuning):
    """F12: different launch geometries give identical bits."""
    G, P, F = pqsynth.random_instance(120, 90_001, 8, 256, 64, 21, code_dist="few")
    S, ids0, sc0, idx = run_pq(pq, torch, G, P, F, 77)
    _, ids1, sc1, _ = run_pq(pq, torch, G, P, F, 77, tuning=tuning)
    assert_same(ids0, sc0, ids1, sc1)
    assert_same(ids0, sc0, *orc.pq_topk(G, S, 77))


def test_sharded_merge_equals_unsharded(pq, torch, orc):
    """Item sharding (id_base) + pq_merge_topk == unsharded, bit for bit (F12)."""
    G, P, F = pqsynth.random_instance(130, 123_457, 4, 16, 32, 19, code_dist="uniform")
    K = 300
    S_t = pq.pq_subscores(cuda(torch, F), cuda(torch, P))
    full = pq.pq_score_topk(pq.pq_create(G, b=16), S_t, K)
    for nsh in (2, 3, 8):
        cuts = np.linspace(0, G.shape[0], nsh + 1).astype(int)
        parts_i, parts_s = [], []
        for s in range(nsh):
            idx = pq.pq_create(G[cuts[s]:cuts[s + 1]], b=16, id_base=int(cuts[s]))
            i, sc = pq.pq_score_topk(idx, S_t, K)
            parts_i.append(i); parts_s.append(sc)
        mi, ms = pq.pq_merge_topk(torch.stack(parts_i), torch.stack(parts_s))
        assert_same(mi.cpu().numpy(), ms.cpu().numpy(), full[0].cpu().numpy(), full[1].cpu().numpy())
    assert_same(full[0].cpu().numpy(), full[1].cpu().numpy(), *orc.pq_topk(G, S_t.cpu().numpy(), K))


def test_merge_large_p(pq, torch, orc):
    """P*K above one K3 segment (multi-level merge)."""
    G, P, F = pqsynth.random_instance(131, 40_000, 4, 16, 32, 3)
    K = 1000
    S_t = pq.pq_subscores(cuda(torch, F), cuda(torch, P))
    cuts = np.linspace(0, G.shape[0], 21).astype(int)
    pi, ps = [], []
    for s in range(20):
        i, sc = pq.pq_score_topk(pq.pq_create(G[cuts[s]:cuts[s + 1]], b=16, id_base=int(cuts[s])), S_t, K)
        pi.append(i); ps.append(sc)
    mi, ms = pq.pq_merge_topk(torch.stack(pi), torch.stack(ps))
    assert_same(mi.cpu().numpy(), ms.cpu().numpy(), *orc.pq_topk(G, S_t.cpu().numpy(), K))


def test_recjpq_gpu_bitwise(pq, torch, orc):
    """Alg. 2 (RecJPQScore) on the GPU == the oracle's Alg. 2 AND
    Alg. 1 given the same S, bit for bit (equivalence A)."""
    for seed, N, m, b, B, K, dist in ((140, 70_001, 8, 256, 9, 50, "uniform"),
                                      (141, 33_333, 4, 16, 3, 700, "uniform"),   # ties
                                      (142, 3_000, 3, 64, 2, 4_000, "zipf")):    # K > N
        G, P, F = pqsynth.random_instance(seed, N, m, b, 4 * m, B, code_dist=dist)
        idx = pq.pq_create(G, b=b, id_base=7)
        S_t = pq.pq_subscores(cuda(torch, F), cuda(torch, P))
        ri, rs = pq.pq_recjpq_topk(idx, S_t, K)
        S_h = S_t.cpu().numpy()
        oi, os_ = orc.recjpq_topk(G, S_h, K, id_base=7)
        assert_same(ri.cpu().numpy(), rs.cpu().numpy(), oi, os_, str(seed))
        assert_same(oi, os_, *orc.pq_topk(G, S_h, K, id_base=7), str(seed))


def test_dense_path(pq, torch, orc):
    """Eq. 2 reconstruction (exact copy) and r = W phi + top-K vs the fp64 oracle."""
    G, P, F = pqsynth.random_instance(150, 50_000, 8, 256, 64, 4)
    idx = pq.pq_create(G, b=256, id_base=10)
    W = pq.pq_reconstruct(idx, cuda(torch, P))
    assert np.array_equal(W.cpu().numpy(), orc.reconstruct(G, P))
    K = 20
    ids, sc = pq.pq_dense_topk(W, cuda(torch, F), K, id_base=10)
    ids, sc = ids.cpu().numpy(), sc.cpu().numpy()
    S64, C = orc.subscores64(F, P)
    for u in range(4):
        r64 = orc.dense_scores64(G, P, F[u])
        # fp32 GEMM error bound: gamma_d * sum |w_i * phi|
        gam = 64 * 2.0 ** -24 / (1 - 64 * 2.0 ** -24)
        cab = np.zeros(G.shape[0])
        for k in range(8):
            cab += C[u, k][G[:, k]]
        assert (np.abs(sc[u].astype(np.float64) - r64[ids[u] - 10]) <= gam * cab[ids[u] - 10] + 1e-30).all()
        order = np.argsort(-r64, kind="stable")
        gap = r64[order[K - 1]] - r64[order[K]]
        if gap > 2 * gam * cab.max():
            assert set((ids[u] - 10).tolist()) == set(order[:K].tolist())
        assert (np.diff(sc[u]) <= 0).all()


def test_search_host_buffers(pq, torch, orc):
    """pq_search with host (pinned) inputs/outputs -- the call bench.py's e2e
    times -- and with device buffers, both against the oracle given the S the
    library computes (and the multi-kernel host-staging path: B = 12 > 4)."""
    for seed, N, B, K in ((160, 80_000, 12, 30), (161, 50_001, 3, 10), (162, 20_011, 40, 100)):
        G, P, F = pqsynth.random_instance(seed, N, 8, 256, 64, B)
        idx = pq.pq_create(G, b=256)
        Fh = torch.from_numpy(F).pin_memory()
        Ph = torch.from_numpy(P).pin_memory()
        oi = torch.empty((B, K), dtype=torch.int32).pin_memory()
        os_ = torch.empty((B, K), dtype=torch.float32).pin_memory()
        S_t = torch.empty((B, 8, 256), dtype=torch.float32, device="cuda")
        pq.pq_search(idx, Fh, Ph, K, ids=oi, scores=os_, S_out=S_t)
        torch.cuda.synchronize()
        S_h = S_t.cpu().numpy()
        assert check_S(orc, F, P, S_h) == 0
        ref = orc.pq_topk(G, S_h, K)
        assert_same(oi.numpy(), os_.numpy(), *ref, str(seed))
        di, ds = pq.pq_search(idx, cuda(torch, F), cuda(torch, P), K)
        assert_same(di.cpu().numpy(), ds.cpu().numpy(), *ref, str(seed))


def test_packed_merge_equals_oracle(pq, torch, orc):
    """The multi-GPU exchange layout: shard results written into packed
    [2][B][K] buffers (dist.alloc_local), stacked as ONE all-gather would
    deliver them ([P][2][B][K]) and merged by pq_merge_topk_packed == the
    oracle over the whole catalogue; includes an empty (padding) shard."""
    from paper_2408_09992_b200.dist import alloc_local, fill_empty, shard_range
    G, P, F = pqsynth.random_instance(133, 90_001, 8, 256, 64, 24)
    K = 100
    S_t = pq.pq_subscores(cuda(torch, F), cuda(torch, P))
    for world in (2, 5):
        bufs = []
        for r in range(world):
            lo, hi = shard_range(G.shape[0], world, r)
            packed, li, ls = alloc_local(24, K, S_t.device)
            pq.pq_score_topk(pq.pq_create(G[lo:hi], b=256, id_base=lo), S_t, K, ids=li, scores=ls)
            bufs.append(packed)
        e, _, _ = alloc_local(24, K, S_t.device)
        fill_empty(e)
        bufs.append(e)
        mi, ms = pq.pq_merge_topk_packed(torch.stack(bufs))
        assert_same(mi.cpu().numpy(), ms.cpu().numpy(), *orc.pq_topk(G, S_t.cpu().numpy(), K), str(world))


def test_invariants_and_launch_count(pq, torch, orc):
    """F11 on a mid-size instance: sorted rows, unique ids, scores recompute
    bit-exactly from codes + S; and the library really launched kernels."""
    G, P, F = pqsynth.random_instance(170, 500_000, 16, 256, 512, 50)
    n0 = pq.launch_count()
    S, ids, sc, idx = run_pq(pq, torch, G, P, F, 100)
    assert pq.launch_count() - n0 >= 3
    for u in range(50):
        assert len(set(ids[u].tolist())) == 100
        key = [(-float(s), int(i)) for s, i in zip(sc[u], ids[u])]
        assert key == sorted(key)
        assert np.array_equal(orc.scores_numpy(G[ids[u]], S[u]).view(np.uint32), sc[u].view(np.uint32))


@pytest.mark.parametrize("m,B,dist", [(8, 48, "uniform"), (16, 33, "uniform"), (8, 20, "zipf"), (4, 64, "few")])
def test_paired_layout_matches_generic(pq, torch, orc, m, B, dist):
    """K2 v3 on the colour-paired layout == K2 v1 (item order) == oracle, bit
    for bit, over several launch geometries."""
    N = 1_500_001 if m == 16 else 150_001         # m = 16: 65,536 colour classes
    G, P, F = pqsynth.random_instance(200 + m, N, m, 256, 4 * m, B, code_dist=dist)
    idx = pq.pq_create(G, b=256, id_base=3)
    lay = idx.layout()
    assert lay["paired"] == (0 if m == 4 else 1) and lay["tmem_splits"] == 0   # m = 4: 32-user item-order tables
    assert idx.variants() == {1, 3, 4}
    if dist == "uniform":
        assert lay["leftover_items"] < 0.2 * G.shape[0]
    S_t = pq.pq_subscores(cuda(torch, F), cuda(torch, P))
    K = 64
    outs = []
    assert idx.plan(B, K)["variant"] == 3
    for tun in (dict(), dict(variant=1), dict(variant=1, ctas=5, chunks=11),
                dict(variant=3, warps=8, ctas=5, chunks=11), dict(variant=3, chunks=1),
                dict(variant=3, ctas=3)):
        idx.set_tuning(**tun)
        i, s = pq.pq_score_topk(idx, S_t, K)
        outs.append((i.cpu().numpy(), s.cpu().numpy()))
    for o in outs[1:]:
        assert_same(*outs[0], *o)
    assert_same(*outs[0], *orc.pq_topk(G, S_t.cpu().numpy(), K, id_base=3))
    # dense reconstruction must use the ORIGINAL codes (cmap), not the stored ones
    W = pq.pq_reconstruct(idx, cuda(torch, P)).cpu().numpy()
    assert np.array_equal(W, orc.reconstruct(G, P))


def test_paired_sparse_classes(pq, torch, orc):
    """m = 16 with few items: most signature classes have no complement, so
    nearly every item is a leftover (pairing must still cover every item)."""
    G, P, F = pqsynth.random_instance(230, 20_011, 16, 256, 64, 17)
    S, ids, sc, idx = run_pq(pq, torch, G, P, F, 50)
    assert idx.layout()["paired"] == 1
    assert_same(ids, sc, *orc.pq_topk(G, S, 50))


TILED_CASES = [
    # seed, N, m, b, B, K, dist — ragged tiles, padding users, many units
    (300, 9_000, 16, 256, 16, 10, "uniform"),
    (301, 250_001, 16, 256, 37, 100, "uniform"),
    (302, 123_457, 8, 256, 20, 64, "zipf"),
    (303, 70_001, 4, 256, 64, 300, "few"),           # R = 32, item order
    (304, 40_000, 8, 256, 17, 1000, "uniform"),
    (305, 1_000, 16, 256, 48, 2000, "uniform"),      # K > N
    (306, 300_001, 4, 16, 70, 1000, "uniform"),      # C5-like: massive exact ties, R = 32
    (307, 90_001, 8, 16, 33, 50, "uniform"),
    (308, 5_003, 4, 16, 40, 3000, "uniform"),        # K close to N, ties
    (309, 60_001, 64, 256, 40, 100, "uniform"),      # m = 64 (Fig. 2b): R = 32, 32 phases of 2 splits
    (310, 30_011, 32, 256, 33, 500, "zipf"),         # m = 32
    # all-ties stress of the shrink protocol's capacity (cap >= wm + 3 TR):
    # 2^m distinct tuples, K = 4000, every tile floods the buffers at the threshold
    (311, 400_003, 8, 256, 16, 4000, "few"),
    (312, 200_003, 16, 256, 16, 4000, "few"),        # m = 16: TMEM phases
    # small K on single-phase tables: small lists per unit, seeded thresholds, first-tile shrink (the
    # C2 regime)
    (314, 123_457, 8, 256, 20, 10, "zipf"),
    (315, 90_001, 8, 16, 33, 16, "few"),             # ties
    (316, 200_001, 4, 256, 40, 32, "uniform"),
]


@pytest.mark.parametrize("case", TILED_CASES, ids=[str(c[0]) for c in TILED_CASES])
def test_tiled_parity(pq, torch, orc, case):
    """K2 v3 (4 users per lane, TMA-staged tables, TMEM partial sums for
    m = 16, CTA-wide candidate buffers) is bit-exact against the oracle given
    S, in two launch geometries."""
    seed, N, m, b, B, K, dist = case
    G, P, F = pqsynth.random_instance(seed, N, m, b, 4 * m, B, code_dist=dist)
    idx = pq.pq_create(G, b=b, id_base=seed)
    assert 3 in idx.variants()
    S_t = pq.pq_subscores(cuda(torch, F), cuda(torch, P))
    ref = orc.pq_topk(G, S_t.cpu().numpy(), K, id_base=seed)
    for tun in (dict(variant=3), dict(variant=3, warps=8, ctas=3, chunks=5),
                dict(variant=3, ctas=7, shrink_watermark=1)):       # shrink after almost every tile
        idx.set_tuning(**tun)
        assert idx.plan(B, K)["variant"] == 3
        i, s = pq.pq_score_topk(idx, S_t, K)
        assert_same(i.cpu().numpy(), s.cpu().numpy(), *ref, str(tun))


BALANCED_CASES = [
    # seed, N, m, b, B, K, dist, ctas -- single-phase tables; CTA ranges of the (group, tile)
    # sequence that start mid-group, hold whole groups and end mid-group
    (320, 50_001, 8, 256, 100, 10, "uniform", 5),     # 7 groups x 13 tiles over 5 CTAs
    (321, 50_001, 8, 256, 100, 100, "zipf", 13),
    (322, 150_001, 4, 16, 200, 1000, "uniform", 6),   # C5-shaped ties, R = 32, union floors off (few lists)
    (323, 150_001, 4, 16, 130, 300, "few", 40),
    (324, 600_001, 8, 256, 40, 10, "uniform", 0),     # default grid: 3 groups x 147 tiles over 148 CTAs
    (325, 300_001, 8, 256, 20, 10, "few", 20),        # heavy ties
    (326, 300_001, 8, 256, 70, 3, "uniform", 37),
]


@pytest.mark.parametrize("case", BALANCED_CASES, ids=[str(c[0]) for c in BALANCED_CASES])
def test_tiled_balanced_partition(pq, torch, orc, case):
    """K2 v3 balanced partition (single-phase tables): each CTA scores one
    contiguous range of the group-major (group, tile) sequence, a unit per
    group it touches; a user's lists = the CTAs touching its group.  Bit-exact
    against the oracle, and identical to the legacy chunk x group units."""
    seed, N, m, b, B, K, dist, ctas = case
    G, P, F = pqsynth.random_instance(seed, N, m, b, 4 * m, B, code_dist=dist)
    idx = pq.pq_create(G, b=b, id_base=seed)
    S_t = pq.pq_subscores(cuda(torch, F), cuda(torch, P))
    ref = orc.pq_topk(G, S_t.cpu().numpy(), K, id_base=seed)
    idx.set_tuning(variant=3, ctas=ctas)
    plan = idx.plan(B, K)
    R = plan["users_per_row"]
    n_groups = -(-B // R)
    assert plan["variant"] == 3
    # fewer lists per user than any legacy plan filling the grid could give
    assert plan["chunks"] <= -(-plan["ctas"] // n_groups) + 1, plan
    i, s = pq.pq_score_topk(idx, S_t, K)
    assert_same(i.cpu().numpy(), s.cpu().numpy(), *ref, str(plan))
    idx.set_tuning(variant=3, ctas=ctas, shrink_watermark=1)
    i, s = pq.pq_score_topk(idx, S_t, K)
    assert_same(i.cpu().numpy(), s.cpu().numpy(), *ref, "shrink_watermark=1")


@pytest.mark.parametrize("dist,chunks", [("uniform", 37), ("few", 11)])
def test_union_floors_many_chunks(pq, torch, orc, dist, chunks):
    """Union floors (K >= 256, single-phase tables, 3..64 chunks): a unit starts
    from the largest key that c finished chunks of the user vouch for with their
    rank-ceil(K/c) keys, and writes its list unpadded (K3 reads per-list
    counts).  C5-shaped (m = 4, b = 16: exact score ties across tuples), many
    chunks per user, bit-exact against the oracle."""
    G, P, F = pqsynth.random_instance(313, 1_200_007, 4, 16, 16, 70, code_dist=dist)
    idx = pq.pq_create(G, b=16, id_base=5)
    S_t = pq.pq_subscores(cuda(torch, F), cuda(torch, P))
    ref = orc.pq_topk(G, S_t.cpu().numpy(), 1000, id_base=5)
    for tun in (dict(variant=3, chunks=chunks), dict(variant=3, chunks=chunks, ctas=9)):
        idx.set_tuning(**tun)
        assert idx.plan(70, 1000)["chunks"] == chunks
        i, s = pq.pq_score_topk(idx, S_t, 1000)
        assert_same(i.cpu().numpy(), s.cpu().numpy(), *ref, str(tun))


LATENCY_CASES = [
    # seed, N, m, b, B, K, dist — the serving case (B <= 4)
    (500, 10_000, 8, 256, 1, 10, "uniform"),        # C1 shape
    (501, 1_280_000, 8, 256, 1, 10, "uniform"),     # C2a shape
    (502, 70_001, 16, 256, 3, 100, "uniform"),
    (503, 50_000, 4, 16, 2, 512, "uniform"),        # heavy exact ties
    (504, 7, 8, 256, 4, 10, "uniform"),             # K > N
    (505, 40_000, 8, 256, 1, 1, "few"),
]


@pytest.mark.parametrize("case", LATENCY_CASES, ids=[str(c[0]) for c in LATENCY_CASES])
def test_latency_parity(pq, torch, orc, case):
    """K2 v4 (small-batch, lane = item, CTA-wide exact selection) is bit-exact
    against the oracle given S, in two launch geometries."""
    seed, N, m, b, B, K, dist = case
    G, P, F = pqsynth.random_instance(seed, N, m, b, 4 * m, B, code_dist=dist)
    idx = pq.pq_create(G, b=b, id_base=seed)
    S_t = pq.pq_subscores(cuda(torch, F), cuda(torch, P))
    ref = orc.pq_topk(G, S_t.cpu().numpy(), K, id_base=seed)
    assert idx.plan(B, K)["variant"] == 4
    for tun in (dict(), dict(variant=4, chunks=3, ctas=2)):
        idx.set_tuning(**tun)
        i, s = pq.pq_score_topk(idx, S_t, K)
        assert_same(i.cpu().numpy(), s.cpu().numpy(), *ref, str(tun))


FUSED_CASES = [
    # seed, N, m, b, d, B, K, dist — pq_search's single-launch K6 path (B <= 4)
    (520, 10_000, 8, 256, 64, 1, 10, "uniform"),       # C1 shape
    (521, 1_280_000, 8, 256, 512, 1, 10, "uniform"),   # C2a shape (d/m = 64)
    (522, 70_001, 16, 256, 48, 3, 100, "uniform"),     # d/m = 3: scalar Psi loads
    (523, 50_000, 4, 16, 64, 2, 512, "uniform"),       # heavy exact ties, K = 512
    (524, 7, 8, 256, 32, 4, 10, "uniform"),            # K > N: padding
    (525, 40_000, 8, 256, 40, 1, 1, "few"),            # ties, K = 1
    (526, 300_007, 16, 200, 128, 4, 64, "zipf"),       # b not a power of 2, ragged tail
    (527, 2_000_003, 16, 256, 64, 4, 100, "uniform"),  # many chunks per user, 8 table copies
    (528, 900_001, 8, 256, 256, 2, 50, "zipf"),        # skewed codes, d/m = 32
    (529, 20_000_003, 8, 256, 64, 1, 10, "uniform"),   # long chunks (thousands of rounds per CTA)
    (530, 500_001, 8, 128, 64, 2, 20, "zipf"),         # b = 128
    (531, 3_000_001, 4, 256, 64, 3, 100, "uniform"),   # m = 4
    # K7 (chunk-resident codes) shapes
    (532, 1_700_001, 8, 256, 64, 1, 10, "uniform"),    # near K7's chunk capacity, ragged tail
    (533, 600_001, 16, 256, 64, 1, 50, "zipf"),        # m = 16: 8 table copies
    (534, 300_000, 8, 256, 64, 4, 30, "few"),          # 4 users, heavy ties
    (535, 100_000, 4, 16, 64, 1, 300, "uniform"),      # K = 300 ties: radix-selected floor / cuts
    (536, 10_000_019, 8, 256, 64, 2, 50, "zipf"),      # K6 on colour-paired rows (long stream), skewed codes
    (537, 60_000, 8, 256, 64, 3, 20, "few"),           # K7 cluster mode: 3 users x 8-CTA clusters, ties
    (538, 30_001, 4, 256, 32, 2, 64, "zipf"),          # K7 cluster mode, m = 4, 4-CTA clusters (cl * K <= 256)
]


@pytest.mark.parametrize("case", FUSED_CASES, ids=[str(c[0]) for c in FUSED_CASES])
def test_fused_query_parity(pq, torch, orc, case):
    """K6 (K1 + K2 + K3 in one launch) is bit-exact: its S equals pq_subscores'
    S bit for bit (and meets the 1e-5 bound vs fp64), and its ids/scores equal
    the oracle given that S — in several cluster / chunk geometries."""
    seed, N, m, b, d, B, K, dist = case
    G, P, F = pqsynth.random_instance(seed, N, m, b, d, B, code_dist=dist)
    idx = pq.pq_create(G, b=b, id_base=seed)
    Fd, Pd = cuda(torch, F), cuda(torch, P)
    S_ref = pq.pq_subscores(Fd, Pd).cpu().numpy()
    check_S(orc, F, P, S_ref)
    ref = orc.pq_topk(G, S_ref, K, id_base=seed)
    assert idx.search_plan(B, d, K)["variant"] in (5, 7)
    for tun in (dict(), dict(cluster=1), dict(cluster=2, chunks=6), dict(cluster=8), dict(variant=5, chunks=1),
                dict(chunks=3), dict(users_per_row=8, chunks=4), dict(variant=5), dict(variant=5, chunks=3),
                dict(variant=7, chunks=2), dict(variant=7, users_per_row=8)):
        idx.set_tuning(**tun)
        S_out = torch.full((B, m, b), float("nan"), device="cuda")
        i, s = pq.pq_search(idx, Fd, Pd, K, S_out=S_out)
        assert np.array_equal(S_out.cpu().numpy().view(np.uint32), S_ref.view(np.uint32)), str(tun)
        assert_same(i.cpu().numpy(), s.cpu().numpy(), *ref, str(tun))
    idx.set_tuning()
    i2, s2 = pq.pq_search(idx, Fd, Pd, K, fused=False)           # the multi-kernel path agrees
    assert_same(i2.cpu().numpy(), s2.cpu().numpy(), *ref, "fused=False")


def test_fused_query_graph_replay_and_host_buffers(pq, torch, orc):
    """K6's per-user completion counters are reset every call: repeated calls,
    CUDA-graph replays and the host-buffer (e2e) path all return the same bits."""
    G, P, F = pqsynth.random_instance(530, 200_000, 8, 256, 64, 2)
    idx = pq.pq_create(G, b=256)
    Fd, Pd = cuda(torch, F), cuda(torch, P)
    S = pq.pq_subscores(Fd, Pd)
    ref = orc.pq_topk(G, S.cpu().numpy(), 20)
    ids = torch.empty((2, 20), dtype=torch.int32, device="cuda")
    sc = torch.empty((2, 20), dtype=torch.float32, device="cuda")
    ws = torch.empty(pq.load_library().pq_search_workspace_bytes(idx.handle, 2, 64, 20),
                     dtype=torch.uint8, device="cuda")
    for _ in range(3):
        pq.pq_search(idx, Fd, Pd, 20, ws=ws, ids=ids, scores=sc)
        assert_same(ids.cpu().numpy(), sc.cpu().numpy(), *ref)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        pq.pq_search(idx, Fd, Pd, 20, ws=ws, ids=ids, scores=sc)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        pq.pq_search(idx, Fd, Pd, 20, ws=ws, ids=ids, scores=sc)
    for _ in range(3):
        ids.fill_(-7)
        g.replay()
        torch.cuda.synchronize()
        assert_same(ids.cpu().numpy(), sc.cpu().numpy(), *ref, "graph replay")
    oi = torch.empty((2, 20), dtype=torch.int32).pin_memory()
    os_ = torch.empty((2, 20), dtype=torch.float32).pin_memory()
    pq.pq_search(idx, torch.from_numpy(F).pin_memory(), torch.from_numpy(P).pin_memory(), 20, ids=oi, scores=os_)
    assert_same(oi.numpy(), os_.numpy(), *ref, "host buffers")


@pytest.mark.gpu
def test_search_host_buffers_zero_copy(pq, torch, orc):
    """pq_search through K7 with pinned host ids / scores (written in place by the
    kernel), with pageable host buffers (staged copies) and mixed host / device
    buffers: the same bits as the oracle every time."""
    G, P, F = pqsynth.random_instance(541, 700_001, 8, 256, 64, 2)
    idx = pq.pq_create(G, b=256)
    assert idx.search_plan(2, 64, 10)["variant"] == 7
    Pd = cuda(torch, P)
    S = pq.pq_subscores(cuda(torch, F), Pd)
    ref = orc.pq_topk(G, S.cpu().numpy(), 10)
    Fp = torch.from_numpy(F).pin_memory()
    for pin_out in (True, False):
        oi = torch.full((2, 10), -7, dtype=torch.int32)
        os_ = torch.full((2, 10), float("nan"), dtype=torch.float32)
        if pin_out:
            oi, os_ = oi.pin_memory(), os_.pin_memory()
        for phi in (Fp, torch.from_numpy(F.copy())):
            oi.fill_(-7)
            pq.pq_search(idx, phi, Pd, 10, ids=oi, scores=os_)
            assert_same(oi.numpy(), os_.numpy(), *ref, f"pin_out={pin_out} pinned_phi={phi.is_pinned()}")
    di, ds = pq.pq_search(idx, Fp, Pd, 10)                  # pinned phi, device outputs
    assert_same(di.cpu().numpy(), ds.cpu().numpy(), *ref, "device outputs")


SUBSET_CASES = [
    # seed, N, m, b, B, K, nV, dist
    (600, 100_000, 8, 256, 3, 10, 5_000, "uniform"),      # small batch (v4 + row map)
    (601, 80_001, 16, 256, 20, 100, 30_011, "uniform"),   # batched (v1 + row map)
    (602, 50_000, 4, 16, 7, 300, 777, "few"),             # ties, K close to nV
    (603, 20_000, 8, 256, 2, 50, 17, "uniform"),          # K > nV: padding
]


@pytest.mark.parametrize("case", SUBSET_CASES, ids=[str(c[0]) for c in SUBSET_CASES])
def test_subset_parity(pq, torch, orc, case):
    """Alg. 1 with an explicit item subset V: equals the oracle over
    V, i.e. the full ranking restricted to V ("subset consistency")."""
    seed, N, m, b, B, K, nV, dist = case
    G, P, F = pqsynth.random_instance(seed, N, m, b, 4 * m, B, code_dist=dist)
    rng = np.random.default_rng(seed)
    V = np.sort(rng.choice(N, nV, replace=False)).astype(np.int32)
    base = 1000 + seed
    idx = pq.pq_create(G, b=b, id_base=base)
    S_t = pq.pq_subscores(cuda(torch, F), cuda(torch, P))
    ids, sc = pq.pq_score_topk_subset(idx, S_t, K, torch.from_numpy(V).cuda())
    ri, rs = orc.pq_topk(G[V], S_t.cpu().numpy(), K)          # V ascending: row order = id order
    ri = np.where(ri >= 0, V[np.clip(ri, 0, None)] + base, -1).astype(np.int32)
    assert_same(ids.cpu().numpy(), sc.cpu().numpy(), ri, rs)
    with pytest.raises(pq.PQError):                            # V must be strictly increasing (validated call)
        pq.pq_score_topk_subset(idx, S_t, K, torch.from_numpy(V[::-1].copy()).cuda(), validate=True)
    # the asynchronous call is graph-capturable and equals the validated one
    vi, vs = pq.pq_score_topk_subset(idx, S_t, K, torch.from_numpy(V).cuda(), validate=True)
    assert_same(vi.cpu().numpy(), vs.cpu().numpy(), ri, rs)
    Vd = torch.from_numpy(V).cuda()
    ws = torch.empty(max(1, int(pq.load_library().pq_subset_workspace_bytes(idx.handle, len(V), B, K))),
                     dtype=torch.uint8, device="cuda")
    gi = torch.empty((B, K), dtype=torch.int32, device="cuda")
    gs = torch.empty((B, K), dtype=torch.float32, device="cuda")
    pq.pq_score_topk_subset(idx, S_t, K, Vd, ws=ws, ids=gi, scores=gs)      # warm (plans, attributes)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        pq.pq_score_topk_subset(idx, S_t, K, Vd, ws=ws, ids=gi, scores=gs)
    gi.fill_(7); gs.fill_(0.0)
    g.replay()
    torch.cuda.synchronize()
    assert_same(gi.cpu().numpy(), gs.cpu().numpy(), ri, rs)


@pytest.mark.parametrize("B,K,dist", [(2, 10, "uniform"), (24, 100, "uniform"), (5, 64, "few")])
def test_exclude_parity(pq, torch, orc, B, K, dist):
    """V_u = I minus user u's exclusion list: equals the oracle over V_u."""
    N, m, b = 60_007, 8, 256
    G, P, F = pqsynth.random_instance(700 + B, N, m, b, 32, B, code_dist=dist)
    idx = pq.pq_create(G, b=b, id_base=11)
    S_t = pq.pq_subscores(cuda(torch, F), cuda(torch, P))
    S_h = S_t.cpu().numpy()
    full_i, _ = orc.pq_topk(G, S_h, 2 * K, id_base=11)
    rng = np.random.default_rng(B)
    excl = []
    for u in range(B):        # drop some of the user's own best items plus random ones
        own = full_i[u][rng.random(2 * K) < 0.4]
        excl.append(np.concatenate([own, rng.integers(11, 11 + N, 20)]))
    ids, sc = pq.pq_score_topk_exclude(idx, S_t, K, excl)
    for u in range(B):
        keep = np.setdiff1d(np.arange(N), np.asarray(excl[u]) - 11).astype(np.int32)
        ri, rs = orc.pq_topk(G[keep], S_h[u:u + 1], K)
        ri = np.where(ri >= 0, keep[np.clip(ri, 0, None)] + 11, -1).astype(np.int32)
        assert_same(ids.cpu().numpy()[u:u + 1], sc.cpu().numpy()[u:u + 1], ri, rs, str(u))


def test_create_destroy_frees_device_memory(pq, torch):
    """pq_destroy (and a failed pq_create) release every device buffer of the
    index, including the tiled (v3) layout's row map and colour map."""
    G, P, F = pqsynth.random_instance(700, 1_000_000, 8, 256, 64, 1)
    idx = pq.pq_create(G, b=256)                       # warm-up: allocator / context state
    idx.close()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(4):
        idx = pq.pq_create(G, b=256)
        assert idx.layout()["paired"] == 1
        idx.close()
    bad = G.copy()
    bad[123, 3] = 255
    for _ in range(2):
        with pytest.raises(pq.PQError):
            pq.pq_create(bad, b=200)                   # code out of range: nothing may leak
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < (8 << 20), (free0, free1)


def test_search_plan_and_flags(pq, torch):
    """pq_search_plan_info reports the fused kernel for B <= 4 and the batched
    K2 plan otherwise; unknown pq_search_ex flags are rejected."""
    import ctypes
    G, P, F = pqsynth.random_instance(710, 100_000, 8, 256, 64, 8)
    idx = pq.pq_create(G, b=256)
    assert idx.search_plan(1, 64, 10)["variant"] == 5
    assert idx.search_plan(8, 64, 10)["variant"] == idx.plan(8, 10)["variant"]
    idx.set_tuning(variant=4)                          # K2 v4 forced: pq_search runs K1 + v4 + K3
    assert idx.search_plan(1, 64, 10)["variant"] == 4
    idx.set_tuning()
    L = pq.load_library()
    Fd, Pd = cuda(torch, F[:1]), cuda(torch, P)
    ids = torch.empty((1, 10), dtype=torch.int32, device="cuda")
    sc = torch.empty((1, 10), dtype=torch.float32, device="cuda")
    nb = int(L.pq_search_workspace_bytes(idx.handle, 1, 64, 10))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    st = L.pq_search_ex(idx.handle, ctypes.c_void_p(Fd.data_ptr()), ctypes.c_void_p(Pd.data_ptr()), 1, 64, 10,
                        0x100, ctypes.c_void_p(ws.data_ptr()), nb, ctypes.c_void_p(ids.data_ptr()),
                        ctypes.c_void_p(sc.data_ptr()), None, None)
    assert st != 0 and b"flags" in L.pq_last_error()


@pytest.mark.parametrize("N,m,b,dist", [(1_500_001, 16, 256, "uniform"), (150_001, 8, 256, "zipf"),
                                        (300_001, 4, 16, "uniform"), (60_001, 64, 256, "uniform"),
                                        (9_000, 16, 256, "few"), (3, 8, 256, "uniform")])
def test_gpu_layout_builder(pq, torch, orc, N, m, b, dist):
    """a0 on the GPU (k0_layout.cu): the K2 v3 layout built from the device
    code rows has the same pairing statistics as the host builder (the counts
    are deterministic; the order inside a class is not), and both indexes give
    the oracle's answer bit for bit (Eq. 1; results independent of the
    layout, R4)."""
    G, P, F = pqsynth.random_instance(880 + m, N, m, b, 4 * m, 20, code_dist=dist)
    S_t = pq.pq_subscores(cuda(torch, F), cuda(torch, P))
    ref = orc.pq_topk(G, S_t.cpu().numpy(), 50, id_base=5)
    gpu_idx = pq.pq_create(cuda(torch, G), b=b, id_base=5)    # device codes
    os.environ["PQTOPK_HOST_LAYOUT"] = "1"
    try:
        host_idx = pq.pq_create(G, b=b, id_base=5)
    finally:
        del os.environ["PQTOPK_HOST_LAYOUT"]
    assert gpu_idx.layout() == host_idx.layout()
    for idx in (gpu_idx, host_idx):
        if 3 in idx.variants():
            assert idx.plan(20, 50)["variant"] == 3
        i, s = pq.pq_score_topk(idx, S_t, 50)
        assert_same(i.cpu().numpy(), s.cpu().numpy(), *ref)
        W = pq.pq_reconstruct(idx, cuda(torch, P)).cpu().numpy()
        assert np.array_equal(W, orc.reconstruct(G, P))
