"""Item-sharded PQTopK across the GPUs of one node.

Items are scored independently (Alg. 1 loops over items; "can be
efficiently parallelised"), so the catalogue is split into contiguous
item ranges, one per rank.  Each rank builds its shard's index with
``id_base = lo`` (global ids), scores it with the fused kernels into ONE packed
int32 buffer [2][B][K] (plane 0 ids, plane 1 fp32 score bits), and the ranks
exchange those buffers with ONE all-gather over the process group (NCCL over
NVLink/NVSwitch on a B200 node: B*K*8 bytes per rank); ``pq_merge_topk_packed``
merges the gathered [P][2][B][K] lists in place (no unpacking copy).  Under the
total order of reading R3 (score desc, id asc) the global top-K is a subset of
the union of the local top-Ks, so the result is bit-identical for any number of
shards.

The exchange and merge are plain host logic around the library calls; the
``merge`` argument exists so the SAME function (``gather_merge``) is exercised
by the CPU (gloo) tests with the oracle as the merge (tests/test_dist_gloo.py).
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple


def shard_range(N: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous item range [lo, hi) of `rank`: floor(rank*N/world) ..
    floor((rank+1)*N/world), so shard sizes differ by at most one item.  When
    N < world some ranks get an EMPTY range; they contribute padding only."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    if N < 0:
        raise ValueError(f"bad N {N}")
    return (rank * N) // world, ((rank + 1) * N) // world


def alloc_local(B: int, K: int, device=None):
    """The packed local-result buffer: (packed int32 [2][B][K], ids view int32
    [B][K], scores view fp32 [B][K]).  The scoring call writes ids/scores
    straight into the two planes, so the all-gather sends one tensor."""
    import torch
    packed = torch.empty((2, B, K), dtype=torch.int32, device=device)
    return packed, packed[0], packed[1].view(torch.float32)


def fill_empty(packed) -> None:
    """An empty shard's result: every entry is padding (id -1, score -inf)."""
    import torch
    packed[0].fill_(-1)
    packed[1].view(torch.float32).fill_(float("-inf"))


def gather_merge(packed, group=None, merge: Optional[Callable] = None, out=None, ws=None,
                 gathered=None):
    """All-gather every rank's packed [2][B][K] local result (ONE collective)
    and merge into the global [B][K] top-K (every rank gets the result).

    `merge` maps the gathered int32 [P][2][B][K] -> ([B][K] ids, [B][K]
    scores); default: the library's pq_merge_topk_packed (CUDA), writing into
    `out` = (ids, scores) when given.  `gathered` may pass a preallocated
    [P*2][B][K] int32 receive buffer (no allocation on the hot path)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    two, B, K = (int(x) for x in packed.shape)
    assert two == 2 and packed.dtype == torch.int32 and packed.is_contiguous()
    if gathered is None:
        gathered = torch.empty((world * 2, B, K), dtype=torch.int32, device=packed.device)
    dist.all_gather_into_tensor(gathered, packed, group=group)
    lists = gathered.view(world, 2, B, K)
    if merge is None:
        from .binding import pq_merge_topk_packed
        if out is not None:
            return pq_merge_topk_packed(lists, ws=ws, out_ids=out[0], out_scores=out[1])
        return pq_merge_topk_packed(lists, ws=ws)
    return merge(lists)


class ShardedIndex:
    """One rank's shard of an item-sharded catalogue.

    codes: uint8 [N_local][m] of THIS rank's items [lo, hi) (host or device;
    may be empty when the catalogue has fewer items than ranks),
    lo: the global id of the first local item."""

    def __init__(self, codes, b: int, lo: int, group=None):
        from .binding import pq_create
        self.group = group
        self.lo = int(lo)
        self.n_local = int(codes.shape[0])
        self.index = pq_create(codes, b=b, id_base=self.lo) if self.n_local > 0 else None

    @classmethod
    def from_full(cls, full_codes, b: int, group=None):
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        lo, hi = shard_range(int(full_codes.shape[0]), world, rank)
        return cls(full_codes[lo:hi], b, lo, group)

    def search(self, seq_emb, subitem_emb, K: int):
        """Global top-K of the whole catalogue for every user: local fused
        PQTopK (K1 + K2 + K3 through pq_search) + one all-gather + merge."""
        from .binding import pq_search
        B = int(seq_emb.shape[0])
        packed, ids, scores = alloc_local(B, K, seq_emb.device)
        if self.index is None:
            fill_empty(packed)
        else:
            pq_search(self.index, seq_emb, subitem_emb, K, ids=ids, scores=scores)
        return gather_merge(packed, self.group)
