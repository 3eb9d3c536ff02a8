"""CPU oracle for the PQTopK hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(paper_2408_09992_b200) never imports it, and it never imports the product
package: the two share no code.  The only shared module is ``pqsynth`` (seeded
random inputs, no arithmetic of the method).

Functions follow PAPER.md (P:n) line by line; see pq_oracle.c for the C
bodies and DESIGN.md for the readings R1..R18 where the paper is silent.

Pins (tests/test_oracle_pins.py): every function below is pinned by at least
one check that does not re-run its own formula — exact rational arithmetic
(subscores64), hand-worked examples (SPEC hand instance), constructed closed
forms (order pin, -0 pin, all-ties), the independent tuple-bucket algorithm,
dense fp64 scoring with a closed-form error bound, and brute-force sort.
No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pq_oracle.c")
_LIB = os.path.join(_HERE, "libpq_oracle.so")
CFLAGS = ["-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off", "-fopenmp",
          "-fPIC", "-shared", "-Wall"]

_lib = None


def build(force: bool = False) -> str:
    """Compile pq_oracle.c (plain C + OpenMP) into libpq_oracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.orc_check_fpenv.restype = ctypes.c_int
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_set_threads.argtypes = [ctypes.c_int]
        L.orc_subscores64.argtypes = [P, P, I64, I32, I32, I32, P, P]
        L.orc_scores_alg1.argtypes = [P, I64, I32, I32, P, P]
        L.orc_scores_alg2.argtypes = [P, I64, I32, I32, P, P]
        L.orc_topk_sort.argtypes = [P, I64, I64, I64, P, P]
        L.orc_topk_sort.restype = I64
        L.orc_topk_sort64.argtypes = [P, I64, I64, I64, P, P]
        L.orc_topk_sort64.restype = I64
        L.orc_pq_topk.argtypes = [P, I64, I32, I32, P, I64, I64, I64, P, P]
        L.orc_pq_topk.restype = ctypes.c_int
        L.orc_reconstruct.argtypes = [P, I64, I32, I32, P, I32, P]
        L.orc_dense_scores64.argtypes = [P, I64, I32, I32, P, I32, P, P]
        L.orc_tuple_topk.argtypes = [P, I64, I32, I32, P, I64, I64, I64, P, P]
        L.orc_tuple_topk.restype = ctypes.c_int
        _lib = L
    fp = _lib.orc_check_fpenv()
    if fp:
        raise RuntimeError(f"oracle: MXCSR has FTZ/DAZ set (0x{fp:x}); IEEE denormals required (R7)")
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def max_threads() -> int:
    return int(lib().orc_max_threads())


def set_threads(n: int) -> None:
    """OpenMP thread count for later calls (results are thread-count invariant)."""
    lib().orc_set_threads(int(n))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# Eq. 4
# ---------------------------------------------------------------------------
def subscores64(phi: np.ndarray, psi: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """S64[u][k][g] = psi_{k,g} . phi_k in fp64, and C = sum |psi*phi| (R5)."""
    phi = _c(np.atleast_2d(phi), np.float32)
    psi = _c(psi, np.float32)
    m, b, dm = psi.shape
    B, d = phi.shape
    assert d == m * dm
    S64 = np.empty((B, m, b), np.float64)
    C = np.empty((B, m, b), np.float64)
    lib().orc_subscores64(_p(phi), _p(psi), B, d, m, b, _p(S64), _p(C))
    return S64, C


def subscores(phi, psi) -> np.ndarray:
    """S_ref = fl32(S64) (R5)."""
    return subscores64(phi, psi)[0].astype(np.float32)


# ---------------------------------------------------------------------------
# Eq. 5; Alg. 1; Alg. 2
# ---------------------------------------------------------------------------
def scores_alg1(codes: np.ndarray, S_user: np.ndarray) -> np.ndarray:
    codes = _c(codes, np.uint8)
    S_user = _c(S_user, np.float32)
    N, m = codes.shape
    b = S_user.shape[1]
    r = np.empty(N, np.float32)
    lib().orc_scores_alg1(_p(codes), N, m, b, _p(S_user), _p(r))
    return r


def scores_alg2(codes: np.ndarray, S_user: np.ndarray) -> np.ndarray:
    codes = _c(codes, np.uint8)
    S_user = _c(S_user, np.float32)
    N, m = codes.shape
    b = S_user.shape[1]
    r = np.empty(N, np.float32)
    lib().orc_scores_alg2(_p(codes), N, m, b, _p(S_user), _p(r))
    return r


def scores_numpy(codes: np.ndarray, S_user: np.ndarray) -> np.ndarray:
    """Alg. 2 in numpy: acc = 0 (fp32); for k: acc = acc + S[k][G[:, k]].
    Bit-exact with the k-ordered fp32 sum (elementwise adds, no reduction)."""
    acc = np.zeros(codes.shape[0], np.float32)
    for k in range(codes.shape[1]):
        acc = acc + S_user[k][codes[:, k]]
    return acc


# ---------------------------------------------------------------------------
# TopK (R3, R11)
# ---------------------------------------------------------------------------
def topk_sort(r: np.ndarray, K: int, id_base: int = 0):
    r = _c(r, np.float32)
    ids = np.empty(K, np.int32)
    sc = np.empty(K, np.float32)
    n = lib().orc_topk_sort(_p(r), r.shape[0], K, id_base, _p(ids), _p(sc))
    if n < 0:
        raise MemoryError
    return ids, sc


def topk_numpy(r: np.ndarray, K: int, id_base: int = 0):
    """Library-routine form: stable argsort of -r keeps ids ascending on ties."""
    order = np.argsort(-r.astype(np.float64), kind="stable")[:K]
    n = order.shape[0]
    ids = np.full(K, -1, np.int32)
    sc = np.full(K, -np.inf, np.float32)
    ids[:n] = order + id_base
    sc[:n] = r[order]
    return ids, sc


def topk_sort64(r64: np.ndarray, K: int, id_base: int = 0):
    r64 = _c(r64, np.float64)
    ids = np.empty(K, np.int32)
    sc = np.empty(K, np.float64)
    lib().orc_topk_sort64(_p(r64), r64.shape[0], K, id_base, _p(ids), _p(sc))
    return ids, sc


def pq_topk(codes: np.ndarray, S: np.ndarray, K: int, id_base: int = 0):
    """Algorithm 1 for a batch: S [B][m][b] fp32 -> ids, scores [B][K]."""
    codes = _c(codes, np.uint8)
    S = _c(np.asarray(S, np.float32).reshape(-1, *np.shape(S)[-2:]), np.float32)
    N, m = codes.shape
    B, m2, b = S.shape
    assert m2 == m
    ids = np.empty((B, K), np.int32)
    sc = np.empty((B, K), np.float32)
    if K > 0 and B > 0:
        rc = lib().orc_pq_topk(_p(codes), N, m, b, _p(S), B, K, id_base, _p(ids), _p(sc))
        if rc:
            raise MemoryError
    return ids, sc


def recjpq_topk(codes: np.ndarray, S: np.ndarray, K: int, id_base: int = 0):
    """Algorithm 2: per user, N-length accumulator, then TopK."""
    S = np.asarray(S, np.float32).reshape(-1, *np.shape(S)[-2:])
    ids = np.empty((S.shape[0], K), np.int32)
    sc = np.empty((S.shape[0], K), np.float32)
    for u in range(S.shape[0]):
        ids[u], sc[u] = topk_sort(scores_alg2(codes, S[u]), K, id_base)
    return ids, sc


def tuple_topk(codes: np.ndarray, S: np.ndarray, K: int, id_base: int = 0):
    """Independent tuple-bucket algorithm; b^m <= 2^24."""
    codes = _c(codes, np.uint8)
    S = _c(np.asarray(S, np.float32).reshape(-1, *np.shape(S)[-2:]), np.float32)
    N, m = codes.shape
    B, _, b = S.shape
    ids = np.empty((B, K), np.int32)
    sc = np.empty((B, K), np.float32)
    rc = lib().orc_tuple_topk(_p(codes), N, m, b, _p(S), B, K, id_base, _p(ids), _p(sc))
    if rc:
        raise ValueError(f"tuple_topk rc={rc}")
    return ids, sc


# ---------------------------------------------------------------------------
# Dense baseline (Eq. 2; Eq. 3)
# ---------------------------------------------------------------------------
def reconstruct(codes: np.ndarray, psi: np.ndarray) -> np.ndarray:
    codes = _c(codes, np.uint8)
    psi = _c(psi, np.float32)
    N, m = codes.shape
    _, b, dm = psi.shape
    W = np.empty((N, m * dm), np.float32)
    lib().orc_reconstruct(_p(codes), N, m, b, _p(psi), m * dm, _p(W))
    return W


def dense_scores64(codes: np.ndarray, psi: np.ndarray, phi_u: np.ndarray) -> np.ndarray:
    codes = _c(codes, np.uint8)
    psi = _c(psi, np.float32)
    phi_u = _c(phi_u, np.float32)
    N, m = codes.shape
    _, b, dm = psi.shape
    r = np.empty(N, np.float64)
    lib().orc_dense_scores64(_p(codes), N, m, b, _p(psi), m * dm, _p(phi_u), _p(r))
    return r


def dense_error_bound(S: np.ndarray, S64: np.ndarray, codes: np.ndarray,
                      C: np.ndarray, d: int) -> np.ndarray:
    """Bound on |r_pq - r64| for one user:
        sum_k |S - S64|              (rounding S64 to fp32)
      + gamma_m * sum_k |S|          (fp32 recursive summation, Higham Thm 4.4,
                                      gamma_m = m u/(1 - m u), u = 2^-24)
      + 2 gamma64_d * sum_k C        (fp64 rounding inside S64 and r64,
                                      gamma64_d = d v/(1 - d v), v = 2^-53)."""
    m = codes.shape[1]
    u, v = 2.0 ** -24, 2.0 ** -53
    gam = m * u / (1 - m * u)
    gam64 = d * v / (1 - d * v)
    dS = np.abs(S.astype(np.float64) - S64)
    aS = np.abs(S.astype(np.float64))
    e = np.zeros(codes.shape[0])
    a = np.zeros(codes.shape[0])
    c = np.zeros(codes.shape[0])
    for k in range(m):
        e += dS[k][codes[:, k]]
        a += aS[k][codes[:, k]]
        c += C[k][codes[:, k]]
    return e + gam * a + 2 * gam64 * c
