"""ctypes binding of libpqtopk.so (include/pqtopk.h).  Argument marshalling only.

Tensors: torch tensors on the current CUDA device (device buffers) or CPU
tensors / numpy arrays (host buffers, only where the C ABI accepts host
memory: pq_create's codes and pq_search's inputs/outputs).  Streams default to
torch's current stream.  Workspaces are caller-owned uint8 device tensors;
when one is not passed, the binding allocates it with torch (outside the
library, which never allocates on the hot path).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# PQTOPK_CHECKED=1 loads the checked diagnostics build (device-side bounds
# checks, bounded waits: `python -m paper_2408_09992_b200.build --checked`)
_LIB_PATH = os.path.join(HERE, "libpqtopk_checked.so" if os.environ.get("PQTOPK_CHECKED") == "1"
                         else "libpqtopk.so")
_lib = None

PQ_STATUS = {0: "PQ_OK", 1: "PQ_ERR_INVALID_ARG", 2: "PQ_ERR_CODE_RANGE", 3: "PQ_ERR_NONFINITE",
             4: "PQ_ERR_CUDA", 5: "PQ_ERR_OUT_OF_MEMORY", 6: "PQ_ERR_UNSUPPORTED",
             7: "PQ_ERR_WORKSPACE"}
MAX_K = 4096

EXPORTS = ["pq_abi_version", "pq_last_error", "pq_launch_count", "pq_create", "pq_create_ex", "pq_destroy",
           "pq_index_info", "pq_index_layout", "pq_index_variants", "pq_plan_info", "pq_set_tuning", "pq_subscores", "pq_topk_workspace_bytes",
           "pq_score_topk", "pq_search_workspace_bytes", "pq_search", "pq_search_ex", "pq_search_plan_info", "pq_merge_workspace_bytes",
           "pq_merge_topk", "pq_merge_topk_packed", "pq_reconstruct", "pq_dense_workspace_bytes", "pq_dense_topk",
           "pq_recjpq_workspace_bytes", "pq_recjpq_topk", "pq_timing_enable", "pq_timing_read",
           "pq_subset_workspace_bytes", "pq_score_topk_subset", "pq_score_topk_subset_ex", "pq_exclude_workspace_bytes",
           "pq_score_topk_exclude"]


class PQError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{PQ_STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = PQ_STATUS.get(status, str(status))


class Tuning(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int32), ("ctas", ctypes.c_int32), ("warps", ctypes.c_int32),
                ("chunks", ctypes.c_int32), ("users_per_row", ctypes.c_int32),
                ("shrink_watermark", ctypes.c_int32), ("cluster", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 1)]


def lib_path() -> str:
    return _LIB_PATH


def load_library():
    """Load libpqtopk.so; raise if it is missing (no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is not built; run `python -m paper_2408_09992_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(_LIB_PATH)
    P, I32, I64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    st = ctypes.c_int
    sig = {
        "pq_abi_version": (I32, []),
        "pq_last_error": (ctypes.c_char_p, []),
        "pq_launch_count": (I64, []),
        "pq_create": (st, [P, I64, I32, I32, I64, P, ctypes.POINTER(P)]),
        "pq_create_ex": (st, [P, I64, I32, I32, I64, I32, P, ctypes.POINTER(P)]),
        "pq_destroy": (st, [P]),
        "pq_index_info": (st, [P, ctypes.POINTER(I64), ctypes.POINTER(I32), ctypes.POINTER(I32),
                               ctypes.POINTER(I64)]),
        "pq_set_tuning": (st, [P, ctypes.POINTER(Tuning)]),
        "pq_plan_info": (st, [P, I32, I32, ctypes.POINTER(I64)]),
        "pq_index_layout": (st, [P, ctypes.POINTER(I32), ctypes.POINTER(I32), ctypes.POINTER(I64),
                                 ctypes.POINTER(I64)]),
        "pq_index_variants": (st, [P, ctypes.POINTER(I32)]),
        "pq_subscores": (st, [P, P, I32, I32, I32, I32, P, P]),
        "pq_topk_workspace_bytes": (SZ, [P, I32, I32]),
        "pq_score_topk": (st, [P, P, I32, I32, P, SZ, P, P, P]),
        "pq_subset_workspace_bytes": (SZ, [P, I64, I32, I32]),
        "pq_score_topk_subset": (st, [P, P, I32, I32, P, I64, P, SZ, P, P, P]),
        "pq_score_topk_subset_ex": (st, [P, P, I32, I32, P, I64, I32, P, SZ, P, P, P]),
        "pq_exclude_workspace_bytes": (SZ, [P, I32, I32, I32]),
        "pq_score_topk_exclude": (st, [P, P, I32, I32, P, P, I32, P, SZ, P, P, P]),
        "pq_search_workspace_bytes": (SZ, [P, I32, I32, I32]),
        "pq_search": (st, [P, P, P, I32, I32, I32, P, SZ, P, P, P]),
        "pq_search_ex": (st, [P, P, P, I32, I32, I32, I32, P, SZ, P, P, P, P]),
        "pq_search_plan_info": (st, [P, I32, I32, I32, ctypes.POINTER(I64)]),
        "pq_merge_workspace_bytes": (SZ, [I32, I32, I32]),
        "pq_merge_topk": (st, [P, P, I32, I32, I32, P, SZ, P, P, P]),
        "pq_merge_topk_packed": (st, [P, I32, I32, I32, P, SZ, P, P, P]),
        "pq_reconstruct": (st, [P, P, I32, P, P]),
        "pq_dense_workspace_bytes": (SZ, [I64, I32, I32]),
        "pq_dense_topk": (st, [P, I64, I32, P, I32, I32, I64, P, SZ, P, P, P]),
        "pq_recjpq_workspace_bytes": (SZ, [P, I32, I32]),
        "pq_recjpq_topk": (st, [P, P, I32, I32, P, SZ, P, P, P]),
        "pq_timing_enable": (st, [P, I32]),
        "pq_timing_read": (st, [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(I64)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    if L.pq_abi_version() != 2:
        raise ImportError("libpqtopk ABI version mismatch")
    _lib = L
    return L


def abi_version() -> int:
    return load_library().pq_abi_version()


def launch_count() -> int:
    """Kernels the library has launched in this process."""
    return load_library().pq_launch_count()


def _check(status: int):
    if status != 0:
        msg = load_library().pq_last_error().decode(errors="replace")
        raise PQError(status, msg)


def _torch():
    import torch
    return torch


def _stream(stream) -> int:
    torch = _torch()
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _ptr(x) -> int:
    """Device or host address of a contiguous torch tensor / numpy array."""
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data
    assert x.is_contiguous(), "tensor must be contiguous"
    return x.data_ptr()


def _need_cuda(t, name):
    if not (hasattr(t, "is_cuda") and t.is_cuda):
        raise ValueError(f"{name} must be a CUDA tensor")


def _ws(nbytes: int, ws, device):
    torch = _torch()
    if nbytes == 0:
        return None, 0
    if ws is None or ws.numel() < nbytes:
        if device is None:
            device = ws.device if ws is not None else torch.device("cuda", torch.cuda.current_device())
        ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
    return ws, ws.numel()


class PQIndex:
    """Owns a pq_index handle (immutable catalogue of codes on the GPU)."""

    def __init__(self, handle: int, N: int, m: int, b: int, id_base: int):
        self._h = ctypes.c_void_p(handle)
        self.N, self.m, self.b, self.id_base = N, m, b, id_base
        self._search_ws = {}                     # (B, d, K) -> pq_search workspace bytes (per tuning)

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h and self._h.value:
            _check(load_library().pq_destroy(self._h))
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self):
        L = load_library()
        N, m, b, ib = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
        _check(L.pq_index_info(self._h, ctypes.byref(N), ctypes.byref(m), ctypes.byref(b), ctypes.byref(ib)))
        return N.value, m.value, b.value, ib.value

    def layout(self):
        """dict(paired, tmem_splits, pairs_matched, leftover_items)."""
        p, t, mp, lo = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
        _check(load_library().pq_index_layout(self._h, ctypes.byref(p), ctypes.byref(t), ctypes.byref(mp),
                                              ctypes.byref(lo)))
        return {"paired": p.value, "tmem_splits": t.value, "pairs_matched": mp.value,
                "leftover_items": lo.value}

    def variants(self):
        """Set of K2 scoring variants this index supports (1 generic, 3 tiled,
        4 small-batch latency)."""
        m = ctypes.c_int32()
        _check(load_library().pq_index_variants(self._h, ctypes.byref(m)))
        return {v for v in (1, 2, 3, 4) if m.value >> v & 1}

    def plan(self, B: int, K: int):
        """The K2 launch plan for (B, K) as a dict (diagnostics)."""
        out = (ctypes.c_int64 * 8)()
        _check(load_library().pq_plan_info(self._h, B, K, out))
        keys = ["variant", "users_per_row", "users_per_group", "warps", "ctas", "chunks",
                "tmem_splits", "smem_bytes"]
        return dict(zip(keys, [int(x) for x in out]))

    def search_plan(self, B: int, d: int, K: int) -> dict:
        """The plan pq_search uses for (B, d, K): variant 5 = the fused K6 kernel, 7 = the
        fused K7 kernel ("cluster" = CTAs per user cluster in its cluster mode, 0 = grid)."""
        out = (ctypes.c_int64 * 8)()
        _check(load_library().pq_search_plan_info(self._h, B, d, K, out))
        v = [int(x) for x in out]
        if v[0] in (5, 7):
            keys = ["variant", "table_copies", "cluster", "warps", "ctas", "chunks", "tmem_splits", "smem_bytes"]
        else:
            keys = ["variant", "users_per_row", "users_per_group", "warps", "ctas", "chunks",
                    "tmem_splits", "smem_bytes"]
        return dict(zip(keys, v))

    def set_tuning(self, variant=0, ctas=0, warps=0, chunks=0, users_per_row=0, shrink_watermark=0,
                   cluster=0):
        t = Tuning(variant, ctas, warps, chunks, users_per_row, shrink_watermark, cluster)
        _check(load_library().pq_set_tuning(self._h, ctypes.byref(t)))
        self._search_ws.clear()                  # the plans (and their workspaces) depend on it

    def timing_enable(self, on: bool = True):
        _check(load_library().pq_timing_enable(self._h, 1 if on else 0))

    def timing_read(self):
        """(k2_ms_total, k3_ms_total, launches) since the last read (synchronises)."""
        a, b, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        _check(load_library().pq_timing_read(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(n)))
        return a.value, b.value, n.value

    def topk_workspace_bytes(self, B: int, K: int) -> int:
        return int(load_library().pq_topk_workspace_bytes(self._h, B, K))

    def search_workspace_bytes(self, B: int, d: int, K: int) -> int:
        return int(load_library().pq_search_workspace_bytes(self._h, B, d, K))

    def recjpq_workspace_bytes(self, B: int, K: int) -> int:
        return int(load_library().pq_recjpq_workspace_bytes(self._h, B, K))


SMALL_BATCH_ONLY = 1


def pq_create(codes, b: int, id_base: int = 0, stream=None, small_batch_only: bool = False) -> PQIndex:
    """Build an index from codes uint8 [N][m] (numpy / CPU tensor / CUDA tensor).
    small_batch_only: skip the batched layouts (B <= 4 serving / huge catalogues)."""
    L = load_library()
    if isinstance(codes, np.ndarray):
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
    else:
        codes = codes.contiguous()
    N, m = int(codes.shape[0]), int(codes.shape[1])
    h = ctypes.c_void_p()
    _check(L.pq_create_ex(ctypes.c_void_p(_ptr(codes)), N, m, int(b), int(id_base),
                          SMALL_BATCH_ONLY if small_batch_only else 0,
                          ctypes.c_void_p(_stream(stream)), ctypes.byref(h)))
    return PQIndex(h.value, N, m, int(b), int(id_base))


def pq_subscores(seq_emb, subitem_emb, S=None, stream=None):
    """S[B][m][b] = fp64-accumulated psi_{k,g} . phi_k  (Eq. 4)."""
    torch = _torch()
    _need_cuda(seq_emb, "seq_emb"); _need_cuda(subitem_emb, "subitem_emb")
    B, d = seq_emb.shape
    m, b, dm = subitem_emb.shape
    if S is None:
        S = torch.empty((B, m, b), dtype=torch.float32, device=seq_emb.device)
    _check(load_library().pq_subscores(ctypes.c_void_p(_ptr(seq_emb)), ctypes.c_void_p(_ptr(subitem_emb)),
                                       B, d, m, b, ctypes.c_void_p(_ptr(S)), ctypes.c_void_p(_stream(stream))))
    return S


def pq_score_topk(index: PQIndex, S, K: int, ws=None, ids=None, scores=None, stream=None
                  ) -> Tuple["torch.Tensor", "torch.Tensor"]:
    """Fused PQTopK (Alg. 1): ids int32 [B][K], scores fp32 [B][K]."""
    torch = _torch()
    _need_cuda(S, "S")
    B = int(S.shape[0])
    dev = S.device
    if ids is None:
        ids = torch.empty((B, K), dtype=torch.int32, device=dev)
    if scores is None:
        scores = torch.empty((B, K), dtype=torch.float32, device=dev)
    L = load_library()
    nb = int(L.pq_topk_workspace_bytes(index.handle, B, K)) if B > 0 and 0 < K <= MAX_K else 0
    ws, wsb = _ws(nb, ws, dev)
    _check(L.pq_score_topk(index.handle, ctypes.c_void_p(_ptr(S)), B, K,
                           ctypes.c_void_p(_ptr(ws) if ws is not None else 0), wsb,
                           ctypes.c_void_p(_ptr(ids)), ctypes.c_void_p(_ptr(scores)),
                           ctypes.c_void_p(_stream(stream))))
    return ids, scores


def pq_score_topk_subset(index: PQIndex, S, K: int, V, ws=None, ids=None, scores=None, stream=None,
                         validate: bool = False):
    """PQTopK over the item subset V (Alg. 1 input V): V = sorted unique
    LOCAL item ids (int32 CUDA tensor), shared by the batch.  Asynchronous;
    validate=True checks V on the device first (synchronises, raises PQError)."""
    torch = _torch()
    _need_cuda(S, "S")
    B = int(S.shape[0])
    dev = S.device
    V = V.to(device=dev, dtype=torch.int32).contiguous()
    nV = int(V.numel())
    if ids is None:
        ids = torch.empty((B, K), dtype=torch.int32, device=dev)
    if scores is None:
        scores = torch.empty((B, K), dtype=torch.float32, device=dev)
    L = load_library()
    nb = int(L.pq_subset_workspace_bytes(index.handle, nV, B, K)) if B > 0 and 0 < K <= MAX_K and nV > 0 else 0
    ws, wsb = _ws(nb, ws, dev)
    _check(L.pq_score_topk_subset_ex(index.handle, ctypes.c_void_p(_ptr(S)), B, K,
                                     ctypes.c_void_p(_ptr(V) if nV else 0), nV, 1 if validate else 0,
                                     ctypes.c_void_p(_ptr(ws) if ws is not None else 0), wsb,
                                  ctypes.c_void_p(_ptr(ids)), ctypes.c_void_p(_ptr(scores)),
                                  ctypes.c_void_p(_stream(stream))))
    return ids, scores


def pq_score_topk_exclude(index: PQIndex, S, K: int, excluded, ws=None, ids=None, scores=None,
                          stream=None):
    """PQTopK over I minus a per-user exclusion list.  `excluded`: a sequence of
    B arrays of GLOBAL item ids (any order; duplicates allowed), or a tuple
    (excl int32 CUDA tensor sorted per user, excl_off int64 CUDA tensor [B+1])."""
    torch = _torch()
    _need_cuda(S, "S")
    B = int(S.shape[0])
    dev = S.device
    if isinstance(excluded, tuple):
        excl, off = excluded
        off_h = off.cpu().numpy()
    else:
        lists = [np.unique(np.asarray(e, dtype=np.int64)).astype(np.int32) for e in excluded]
        if len(lists) != B:
            raise ValueError("one exclusion list per user")
        off_h = np.zeros(B + 1, np.int64)
        off_h[1:] = np.cumsum([len(x) for x in lists])
        excl = torch.from_numpy(np.concatenate(lists) if off_h[-1] else np.zeros(1, np.int32)).to(dev)
        off = torch.from_numpy(off_h).to(dev)
    max_excl = int(np.max(np.diff(off_h))) if B > 0 else 0
    if ids is None:
        ids = torch.empty((B, K), dtype=torch.int32, device=dev)
    if scores is None:
        scores = torch.empty((B, K), dtype=torch.float32, device=dev)
    L = load_library()
    nb = int(L.pq_exclude_workspace_bytes(index.handle, B, K, max_excl)) if B > 0 and K > 0 else 0
    ws, wsb = _ws(nb, ws, dev)
    _check(L.pq_score_topk_exclude(index.handle, ctypes.c_void_p(_ptr(S)), B, K,
                                   ctypes.c_void_p(_ptr(excl)), ctypes.c_void_p(_ptr(off)), max_excl,
                                   ctypes.c_void_p(_ptr(ws) if ws is not None else 0), wsb,
                                   ctypes.c_void_p(_ptr(ids)), ctypes.c_void_p(_ptr(scores)),
                                   ctypes.c_void_p(_stream(stream))))
    return ids, scores


SEARCH_NO_FUSED = 1


def pq_search(index: PQIndex, seq_emb, subitem_emb, K: int, ws=None, ids=None, scores=None,
              stream=None, S_out=None, fused: bool = True):
    """The whole hot path: K1 + K2 + K3, or the fused single-launch K6 kernel
    for B <= 4 (``fused=False`` forces the multi-kernel path).  Inputs/outputs
    may be host buffers (pinned CPU tensors / numpy) or CUDA tensors; S_out
    (optional CUDA fp32 [B][m][b]) receives the sub-id scores."""
    torch = _torch()
    B, d = int(seq_emb.shape[0]), int(seq_emb.shape[1])
    dev = None
    if ids is None or scores is None or ws is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    if ids is None:
        ids = torch.empty((B, K), dtype=torch.int32, device=dev)
    if scores is None:
        scores = torch.empty((B, K), dtype=torch.float32, device=dev)
    if S_out is not None:
        _need_cuda(S_out, "S_out")
    L = load_library()
    nb = index._search_ws.get((B, d, K))       # (a serving loop asks for the same shape every call)
    if nb is None:
        nb = int(L.pq_search_workspace_bytes(index.handle, B, d, K)) if B > 0 and 0 < K <= MAX_K else 0
        index._search_ws[(B, d, K)] = nb
    ws, wsb = _ws(nb, ws, dev)
    _check(L.pq_search_ex(index.handle, ctypes.c_void_p(_ptr(seq_emb)), ctypes.c_void_p(_ptr(subitem_emb)),
                          B, d, K, 0 if fused else SEARCH_NO_FUSED,
                          ctypes.c_void_p(_ptr(ws) if ws is not None else 0), wsb,
                          ctypes.c_void_p(_ptr(ids)), ctypes.c_void_p(_ptr(scores)),
                          ctypes.c_void_p(_ptr(S_out) if S_out is not None else 0),
                          ctypes.c_void_p(_stream(stream))))
    return ids, scores


def pq_merge_topk(ids, scores, ws=None, out_ids=None, out_scores=None, stream=None):
    """Merge [P][B][K] partial lists (e.g. allgathered shards) into [B][K]."""
    torch = _torch()
    _need_cuda(ids, "ids"); _need_cuda(scores, "scores")
    P, B, K = (int(x) for x in ids.shape)
    dev = ids.device
    if out_ids is None:
        out_ids = torch.empty((B, K), dtype=torch.int32, device=dev)
    if out_scores is None:
        out_scores = torch.empty((B, K), dtype=torch.float32, device=dev)
    L = load_library()
    nb = int(L.pq_merge_workspace_bytes(P, B, K))
    ws, wsb = _ws(nb, ws, dev)
    _check(L.pq_merge_topk(ctypes.c_void_p(_ptr(ids)), ctypes.c_void_p(_ptr(scores)), P, B, K,
                           ctypes.c_void_p(_ptr(ws) if ws is not None else 0), wsb,
                           ctypes.c_void_p(_ptr(out_ids)), ctypes.c_void_p(_ptr(out_scores)),
                           ctypes.c_void_p(_stream(stream))))
    return out_ids, out_scores


def pq_merge_topk_packed(lists, ws=None, out_ids=None, out_scores=None, stream=None):
    """Merge the packed int32 [P][2][B][K] lists (plane 0 ids, plane 1 fp32
    score bits) that ONE all-gather of the shards' results produces into [B][K]."""
    torch = _torch()
    _need_cuda(lists, "lists")
    if lists.dtype != torch.int32 or lists.dim() != 4 or int(lists.shape[1]) != 2:
        raise ValueError("lists must be int32 [P][2][B][K]")
    P, _, B, K = (int(x) for x in lists.shape)
    dev = lists.device
    if out_ids is None:
        out_ids = torch.empty((B, K), dtype=torch.int32, device=dev)
    if out_scores is None:
        out_scores = torch.empty((B, K), dtype=torch.float32, device=dev)
    L = load_library()
    nb = int(L.pq_merge_workspace_bytes(P, B, K))
    ws, wsb = _ws(nb, ws, dev)
    _check(L.pq_merge_topk_packed(ctypes.c_void_p(_ptr(lists)), P, B, K,
                                  ctypes.c_void_p(_ptr(ws) if ws is not None else 0), wsb,
                                  ctypes.c_void_p(_ptr(out_ids)), ctypes.c_void_p(_ptr(out_scores)),
                                  ctypes.c_void_p(_stream(stream))))
    return out_ids, out_scores


def pq_reconstruct(index: PQIndex, subitem_emb, W=None, stream=None):
    """W[N][d] with w_i = psi_{1,g_i1} || ... || psi_{m,g_im}  (Eq. 2)."""
    torch = _torch()
    _need_cuda(subitem_emb, "subitem_emb")
    m, b, dm = subitem_emb.shape
    d = m * dm
    if W is None:
        W = torch.empty((index.N, d), dtype=torch.float32, device=subitem_emb.device)
    _check(load_library().pq_reconstruct(index.handle, ctypes.c_void_p(_ptr(subitem_emb)), d,
                                         ctypes.c_void_p(_ptr(W)), ctypes.c_void_p(_stream(stream))))
    return W


def pq_dense_topk(W, seq_emb, K: int, id_base: int = 0, ws=None, ids=None, scores=None, stream=None):
    """Dense baseline r = W phi (fp32 SGEMM) + top-K."""
    torch = _torch()
    _need_cuda(W, "W"); _need_cuda(seq_emb, "seq_emb")
    N, d = int(W.shape[0]), int(W.shape[1])
    B = int(seq_emb.shape[0])
    dev = W.device
    if ids is None:
        ids = torch.empty((B, K), dtype=torch.int32, device=dev)
    if scores is None:
        scores = torch.empty((B, K), dtype=torch.float32, device=dev)
    L = load_library()
    nb = int(L.pq_dense_workspace_bytes(N, B, K))
    ws, wsb = _ws(nb, ws, dev)
    _check(L.pq_dense_topk(ctypes.c_void_p(_ptr(W)), N, d, ctypes.c_void_p(_ptr(seq_emb)), B, K,
                           int(id_base), ctypes.c_void_p(_ptr(ws) if ws is not None else 0), wsb,
                           ctypes.c_void_p(_ptr(ids)), ctypes.c_void_p(_ptr(scores)),
                           ctypes.c_void_p(_stream(stream))))
    return ids, scores


def pq_recjpq_topk(index: PQIndex, S, K: int, ws=None, ids=None, scores=None, stream=None):
    """RecJPQScore (Alg. 2) on the GPU; bitwise equal to pq_score_topk."""
    torch = _torch()
    _need_cuda(S, "S")
    B = int(S.shape[0])
    dev = S.device
    if ids is None:
        ids = torch.empty((B, K), dtype=torch.int32, device=dev)
    if scores is None:
        scores = torch.empty((B, K), dtype=torch.float32, device=dev)
    L = load_library()
    nb = int(L.pq_recjpq_workspace_bytes(index.handle, B, K)) if B > 0 and 0 < K <= MAX_K else 0
    ws, wsb = _ws(nb, ws, dev)
    _check(L.pq_recjpq_topk(index.handle, ctypes.c_void_p(_ptr(S)), B, K,
                            ctypes.c_void_p(_ptr(ws) if ws is not None else 0), wsb,
                            ctypes.c_void_p(_ptr(ids)), ctypes.c_void_p(_ptr(scores)),
                            ctypes.c_void_p(_stream(stream))))
    return ids, scores
