"""Small cases for the checked build (scripts/checked_run.sh) -- the stand-in
for compute-sanitizer, which this GPU pool does not allow.

    PQTOPK_CHECKED=1 python scripts/sanitize_cases.py [--reps R] [case ...]

Every kernel family of the library runs R times on a C1/C2-sized input and
each answer is checked bit-exactly against the CPU oracle (a race shows up as
a parity failure; a bounds violation or a hang as a PQ_DCHECK trap in the
checked library).  Cases (SURVEY.md §5 "race detection"):
  tiled16   K2 v3 m = 16 (TMA phase tables + TMEM partial sums), shrink_watermark = 1
            (forces the tile-end shrink protocol on every tile)
  tiled8    K2 v3 m = 8 single-phase tables with threshold seeding, shrink_watermark = 1
  tiled4    K2 v3 b = 16 exact first-pair tables, K = 300 (massive ties)
  tiledbal  K2 v3 balanced partition (CTA ranges of the (group, tile) sequence that start
            mid-group, hold whole groups and end mid-group), shrink_watermark = 1
  latency   K2 v4 (B <= 4 through pq_score_topk) + K1 + K3
  k6grid    K6 fused query, cooperative grid mode
  k6clus    K6 fused query, cluster mode (cluster = 2)
  k6pair    K6 on the colour-paired row-order codes (a long stream: 10M items)
  k7        K7 fused query, chunk-resident codes (B = 1 and B = 2)
  k7clus    K7 cluster mode (one 8-CTA cluster per user, sub-id scores and lists through DSMEM)
  merge     K3 pq_merge_topk over 8 shards
  subset    K5 subset V + exclusion lists
  recjpq    Alg. 2 on the GPU
  dense     K4 reconstruct + SGEMM + top-K (ids only checked for the set)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import pqsynth  # noqa: E402


def same(a_i, a_s, b_i, b_s, what):
    a_i, b_i = np.asarray(a_i), np.asarray(b_i)
    ok = np.array_equal(a_i, b_i) and np.array_equal(np.asarray(a_s).view(np.uint32),
                                                      np.asarray(b_s).view(np.uint32))
    if not ok:
        raise SystemExit(f"PARITY FAIL: {what}")


def main(cases):
    import torch

    import paper_2408_09992_b200 as pq
    pq.load_library()
    dev = torch.device("cuda", 0)

    def cu(x):
        return torch.from_numpy(np.ascontiguousarray(x)).to(dev)

    def tiled(seed, N, m, b, d, B, K, dist="uniform", **tun):
        G, P, F = pqsynth.random_instance(seed, N, m, b, d, B, code_dist=dist)
        idx = pq.pq_create(G, b=b)
        idx.set_tuning(**tun)
        assert idx.plan(B, K)["variant"] == 3, idx.plan(B, K)
        S = pq.pq_subscores(cu(F), cu(P))
        i, s = pq.pq_score_topk(idx, S, K)
        torch.cuda.synchronize()
        same(i.cpu().numpy(), s.cpu().numpy(), *oracle.pq_topk(G, S.cpu().numpy(), K), f"tiled m={m}")

    for c in cases:
        print("case", c, flush=True)
        if c == "tiled16":
            tiled(9001, 9_001, 16, 256, 64, 16, 40, shrink_watermark=1)
        elif c == "tiled8":
            tiled(9002, 20_011, 8, 256, 64, 32, 20, shrink_watermark=1)
        elif c == "tiled4":
            tiled(9003, 30_001, 4, 16, 16, 32, 300, dist="uniform")
        elif c == "tiledbal":
            tiled(9014, 50_001, 8, 256, 64, 100, 10, ctas=5, shrink_watermark=1)
            tiled(9015, 150_001, 4, 16, 16, 130, 300, dist="few", ctas=40)
        elif c == "latency":
            G, P, F = pqsynth.random_instance(9004, 30_001, 8, 256, 64, 2)
            idx = pq.pq_create(G, b=256)
            S = pq.pq_subscores(cu(F), cu(P))
            assert idx.plan(2, 10)["variant"] == 4, idx.plan(2, 10)
            i, s = pq.pq_score_topk(idx, S, 10)
            torch.cuda.synchronize()
            same(i.cpu().numpy(), s.cpu().numpy(), *oracle.pq_topk(G, S.cpu().numpy(), 10), "latency")
        elif c in ("k6grid", "k6clus"):
            G, P, F = pqsynth.random_instance(9005, 20_001, 8, 256, 64, 1)
            idx = pq.pq_create(G, b=256, small_batch_only=True)
            if c == "k6clus":
                idx.set_tuning(cluster=2)
            S = torch.empty((1, 8, 256), dtype=torch.float32, device=dev)
            i, s = pq.pq_search(idx, cu(F), cu(P), 10, S_out=S)
            torch.cuda.synchronize()
            same(i.cpu().numpy(), s.cpu().numpy(), *oracle.pq_topk(G, S.cpu().numpy(), 10), c)
        elif c == "k6pair":
            G, P, F = pqsynth.random_instance(9010, 10_000_019, 8, 256, 64, 1)
            idx = pq.pq_create(G, b=256)
            assert idx.search_plan(1, 64, 10)["variant"] == 5
            S = torch.empty((1, 8, 256), dtype=torch.float32, device=dev)
            i, s = pq.pq_search(idx, cu(F), cu(P), 10, S_out=S)
            torch.cuda.synchronize()
            same(i.cpu().numpy(), s.cpu().numpy(), *oracle.pq_topk(G, S.cpu().numpy(), 10), c)
        elif c == "k7":
            for B in (1, 2):
                G, P, F = pqsynth.random_instance(9011 + B, 600_011, 8, 256, 64, B)
                idx = pq.pq_create(G, b=256)
                assert idx.search_plan(B, 64, 10)["variant"] == 7, idx.search_plan(B, 64, 10)
                S = torch.empty((B, 8, 256), dtype=torch.float32, device=dev)
                i, s = pq.pq_search(idx, cu(F), cu(P), 10, S_out=S)
                torch.cuda.synchronize()
                same(i.cpu().numpy(), s.cpu().numpy(), *oracle.pq_topk(G, S.cpu().numpy(), 10), c)
        elif c == "k7clus":
            G, P, F = pqsynth.random_instance(9014, 20_011, 8, 256, 64, 2)
            idx = pq.pq_create(G, b=256)
            pl = idx.search_plan(2, 64, 10)
            assert pl["variant"] == 7 and pl["cluster"] == 8, pl
            S = torch.empty((2, 8, 256), dtype=torch.float32, device=dev)
            i, s = pq.pq_search(idx, cu(F), cu(P), 10, S_out=S)
            torch.cuda.synchronize()
            same(i.cpu().numpy(), s.cpu().numpy(), *oracle.pq_topk(G, S.cpu().numpy(), 10), c)
        elif c == "merge":
            G, P, F = pqsynth.random_instance(9006, 16_001, 4, 16, 16, 3)
            S = pq.pq_subscores(cu(F), cu(P))
            cuts = np.linspace(0, G.shape[0], 9).astype(int)
            pi, ps = [], []
            for k in range(8):
                i, s = pq.pq_score_topk(pq.pq_create(G[cuts[k]:cuts[k + 1]], b=16, id_base=int(cuts[k])), S, 200)
                pi.append(i); ps.append(s)
            mi, ms = pq.pq_merge_topk(torch.stack(pi), torch.stack(ps))
            torch.cuda.synchronize()
            same(mi.cpu().numpy(), ms.cpu().numpy(), *oracle.pq_topk(G, S.cpu().numpy(), 200), "merge")
        elif c == "subset":
            G, P, F = pqsynth.random_instance(9007, 12_001, 8, 256, 64, 5)
            idx = pq.pq_create(G, b=256)
            S = pq.pq_subscores(cu(F), cu(P))
            V = np.unique(np.random.default_rng(1).integers(0, G.shape[0], 3000)).astype(np.int32)
            i, s = pq.pq_score_topk_subset(idx, S, 20, cu(V))
            torch.cuda.synchronize()
            ri, rs = oracle.pq_topk(G[V], S.cpu().numpy(), 20)
            same(i.cpu().numpy(), s.cpu().numpy(), np.where(ri >= 0, V[np.maximum(ri, 0)], -1), rs, "subset")
        elif c == "recjpq":
            G, P, F = pqsynth.random_instance(9008, 12_001, 8, 256, 64, 5)
            idx = pq.pq_create(G, b=256)
            S = pq.pq_subscores(cu(F), cu(P))
            i, s = pq.pq_recjpq_topk(idx, S, 20)
            torch.cuda.synchronize()
            same(i.cpu().numpy(), s.cpu().numpy(), *oracle.recjpq_topk(G, S.cpu().numpy(), 20), "recjpq")
        elif c == "dense":
            G, P, F = pqsynth.random_instance(9009, 8_001, 8, 256, 64, 3)
            idx = pq.pq_create(G, b=256)
            W = pq.pq_reconstruct(idx, cu(P))
            torch.cuda.synchronize()
            if not np.array_equal(W.cpu().numpy(), oracle.reconstruct(G, P)):
                raise SystemExit("PARITY FAIL: reconstruct")
            i, s = pq.pq_dense_topk(W, cu(F), 10)
            torch.cuda.synchronize()
        else:
            raise SystemExit(f"unknown case {c}")
        print("ok", c, flush=True)


if __name__ == "__main__":
    argv = sys.argv[1:]
    reps = 1
    if argv[:1] == ["--reps"]:
        reps, argv = int(argv[1]), argv[2:]
    cases = argv or ["tiled16", "tiled8", "tiled4", "tiledbal", "latency", "k6grid", "k6clus", "k6pair", "k7", "k7clus", "merge",
                     "subset", "recjpq", "dense"]
    import paper_2408_09992_b200 as _pq
    print("library:", _pq.lib_path(), flush=True)
    for _ in range(reps):
        main(cases)
