"""B200-native PQTopK: fused sub-id scoring + exact top-K (arXiv 2408.09992).

Thin Python binding over the C ABI in include/pqtopk.h (libpqtopk.so, built
in-tree for sm_100a).  Every step of the hot path runs in the library's CUDA
kernels; this module only marshals pointers, sizes and streams.  There is no
CPU fallback: if the library cannot be loaded, or no CUDA device is present
when a compute call is made, it raises.

    from paper_2408_09992_b200 import pq_create, pq_subscores, pq_score_topk
"""
from .binding import (  # noqa: F401
    PQError,
    PQIndex,
    Tuning,
    abi_version,
    launch_count,
    lib_path,
    load_library,
    pq_create,
    pq_dense_topk,
    pq_merge_topk,
    pq_merge_topk_packed,
    pq_recjpq_topk,
    pq_reconstruct,
    pq_score_topk,
    pq_score_topk_exclude,
    pq_score_topk_subset,
    pq_search,
    pq_subscores,
)

from . import dist  # noqa: F401,E402  (item sharding across GPUs)

__all__ = [
    "PQError", "PQIndex", "Tuning", "abi_version", "launch_count", "lib_path", "load_library",
    "pq_create", "pq_subscores", "pq_score_topk", "pq_score_topk_subset", "pq_score_topk_exclude", "pq_search", "pq_merge_topk", "pq_merge_topk_packed",
    "pq_reconstruct", "pq_dense_topk", "pq_recjpq_topk",
]
