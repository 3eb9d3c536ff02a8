"""Multi-process (CPU, gloo) tests of the item-sharding host logic
(paper_2408_09992_b200/dist.py; reading R4 "any sharding gives
identical bits").

Each rank scores ITS contiguous item range with the CPU oracle (global ids via
id_base), the ranks exchange their B x K lists with the same all-gather code
the GPU path uses, and the merge (here: an oracle sort) must equal the oracle
top-K of the unsharded catalogue, bit for bit.
"""
import os
import socket

import numpy as np
import pytest

import pqsynth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_merge(lists):
    """gathered int32 [P][2][B][K] (plane 0 ids, plane 1 fp32 score bits) ->
    [B][K]: sort the union by (score desc, id asc); padding entries (id -1,
    score -inf) sort last."""
    import torch
    P, _, B, K = lists.shape
    ids = lists[:, 0].permute(1, 0, 2).reshape(B, P * K).numpy()
    sc = lists[:, 1].permute(1, 0, 2).reshape(B, P * K).numpy().view(np.float32)
    out_i = np.empty((B, K), np.int32)
    out_s = np.empty((B, K), np.float32)
    for u in range(B):
        real = ids[u] >= 0
        key_id = np.where(real, ids[u], np.iinfo(np.int32).max).astype(np.int64)
        order = np.lexsort((key_id, -sc[u].astype(np.float64)))[:K]
        out_i[u] = ids[u][order]
        out_s[u] = sc[u][order]
    return torch.from_numpy(out_i), torch.from_numpy(out_s)


def _worker(rank, world, port, case, outdir):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2408_09992_b200.dist import alloc_local, fill_empty, gather_merge, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seed, N, m, b, B, K, dist_kind = case
        G, P, F = pqsynth.random_instance(seed, N, m, b, 4 * m, B, code_dist=dist_kind)
        S = oracle.subscores(F, P)
        lo, hi = shard_range(N, world, rank)
        packed, l_ids, l_sc = alloc_local(B, K)
        if hi > lo:
            li, ls = oracle.pq_topk(G[lo:hi], S, K, id_base=lo)
            l_ids.copy_(torch.from_numpy(li))
            l_sc.copy_(torch.from_numpy(ls))
        else:                                   # empty shard (N < world): padding only
            fill_empty(packed)
        mi, ms = gather_merge(packed, merge=_oracle_merge)   # the function bench.py's step calls
        np.save(os.path.join(outdir, f"r{rank}_ids.npy"), mi.numpy())
        np.save(os.path.join(outdir, f"r{rank}_sc.npy"), ms.numpy())
    finally:
        dist.destroy_process_group()


CASES = [
    (401, 20_011, 8, 256, 5, 50, "uniform"),
    (402, 9_000, 4, 16, 7, 300, "few"),        # massive ties across shards
    (403, 1_001, 3, 8, 4, 900, "uniform"),     # K larger than a shard
    (404, 2, 4, 16, 3, 5, "uniform"),          # N < world for world 3: an empty shard
]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", CASES, ids=[str(c[0]) for c in CASES])
def test_sharded_merge_gloo(tmp_path, orc, world, case):
    import torch.multiprocessing as mp
    mp.start_processes(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    seed, N, m, b, B, K, dist_kind = case
    G, P, F = pqsynth.random_instance(seed, N, m, b, 4 * m, B, code_dist=dist_kind)
    ref_i, ref_s = orc.pq_topk(G, orc.subscores(F, P), K)
    for r in range(world):
        ids = np.load(tmp_path / f"r{r}_ids.npy")
        sc = np.load(tmp_path / f"r{r}_sc.npy")
        assert np.array_equal(ids, ref_i), (world, r)
        assert np.array_equal(sc.view(np.uint32), ref_s.view(np.uint32)), (world, r)


def test_shard_range_partitions():
    from paper_2408_09992_b200.dist import shard_range
    for N in (0, 1, 2, 7, 50_000_000, 200_000_001):
        for world in (1, 2, 3, 8):
            parts = [shard_range(N, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == N
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in parts]
            assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 0
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
