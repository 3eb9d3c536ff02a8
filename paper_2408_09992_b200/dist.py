"""Item-sharded PQTopK across the GPUs of one node.

Items are scored independently (Alg. 1 loops over items; "can be
efficiently parallelised"), so the catalogue is split into contiguous
item ranges, one per rank.  Each rank builds its shard's index with
``id_base = lo`` (global ids), scores it with the fused kernels, and the B x K
local results are exchanged with ONE all-gather over the process group (NCCL
over NVLink on a B200 node) and merged by ``pq_merge_topk``.  Under the total
order of reading R3 (score desc, id asc) the global top-K is a subset of the
union of the local top-Ks, so the result is bit-identical for any number of
shards.

The exchange and merge are plain host logic around the library calls; the
``merge`` argument exists so the same code is exercised by the CPU (gloo) tests
with the oracle as the merge (tests/test_dist_gloo.py).
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple


def shard_range(N: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous item range [lo, hi) of `rank`; the last rank takes the remainder."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    n = N // world
    lo = rank * n
    hi = N if rank == world - 1 else lo + n
    return lo, hi


def gather_merge(ids, scores, group=None, merge: Optional[Callable] = None, out=None):
    """All-gather the [B][K] local (ids, scores) of every rank and merge them
    into the global [B][K] top-K (every rank gets the result).

    ids int32 [B][K], scores fp32 [B][K] on the group's device.  `merge` maps
    ([P][B][K] ids, [P][B][K] scores) -> ([B][K], [B][K]); default: the
    library's pq_merge_topk (CUDA)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    B, K = (int(x) for x in ids.shape)
    # concatenated [world * B][K] output (accepted by both NCCL and gloo), viewed as [world][B][K]
    g_ids = torch.empty((world * B, K), dtype=ids.dtype, device=ids.device)
    g_sc = torch.empty((world * B, K), dtype=scores.dtype, device=scores.device)
    dist.all_gather_into_tensor(g_ids, ids.contiguous(), group=group)
    dist.all_gather_into_tensor(g_sc, scores.contiguous(), group=group)
    g_ids, g_sc = g_ids.view(world, B, K), g_sc.view(world, B, K)
    if merge is None:
        from .binding import pq_merge_topk
        if out is not None:
            return pq_merge_topk(g_ids, g_sc, out_ids=out[0], out_scores=out[1])
        return pq_merge_topk(g_ids, g_sc)
    return merge(g_ids, g_sc)


class ShardedIndex:
    """One rank's shard of an item-sharded catalogue.

    codes: uint8 [N_local][m] of THIS rank's items [lo, hi) (host or device),
    lo: the global id of the first local item."""

    def __init__(self, codes, b: int, lo: int, group=None):
        from .binding import pq_create
        self.group = group
        self.lo = int(lo)
        self.index = pq_create(codes, b=b, id_base=self.lo)

    @classmethod
    def from_full(cls, full_codes, b: int, group=None):
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        lo, hi = shard_range(int(full_codes.shape[0]), world, rank)
        return cls(full_codes[lo:hi], b, lo, group)

    def search(self, seq_emb, subitem_emb, K: int):
        """Global top-K of the whole catalogue for every user: local fused
        PQTopK (K1 + K2 + K3 through pq_search) + all-gather + merge."""
        from .binding import pq_search
        ids, scores = pq_search(self.index, seq_emb, subitem_emb, K)
        return gather_merge(ids, scores, self.group)
