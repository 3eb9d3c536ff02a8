"""Seeded synthetic inputs for the PQTopK hot path.

This module is the ONLY code shared by the CUDA path (tests / bench) and the
CPU oracle.  It draws random numbers and nothing else: it holds none of the
method's arithmetic (no sub-id scores, no sums, no selection).

Workload recipe:
  * the paper simulates "a random model output" phi and "a random sub-id
    embedding matrix Psi" (RQ2) and uses m = 8 splits, d = 512
    (PAPER.md:187); the five configs are the ones BASELINE.json names;
  * codes  G[N][m]  uint8  — uniform in [0, b), or truncated Zipf(s) over the
    sub-ids with P(g) ∝ (g+1)^-s (BASELINE.json config 3; reading R15);
  * Psi    [m][b][d/m] float32 — standard normal × sigma (sigma = 0.02 for the
    Gowalla-shaped config, reading R14);
  * phi    [B][d] float32 — standard normal.
Every stream is a PCG64 generator keyed by
SeedSequence([240809992, cfg_id, stream, chunk]); codes are drawn in fixed
chunks of 2**20 items, so any item shard [lo, hi) regenerates bit-identically
regardless of how many GPUs the catalogue is split over.
"""
from __future__ import annotations

import dataclasses
import hashlib
from typing import Optional

import numpy as np

ROOT_SEED = 240809992            # arXiv 2408.09992
CODE_CHUNK = 1 << 20             # items per code-generation chunk
STREAM_CODES, STREAM_PSI, STREAM_PHI = 0, 1, 2


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    cfg_id: int
    N: int          # catalogue size |I|
    m: int          # splits
    b: int          # sub-ids per split
    d: int          # embedding dim
    B: int          # users per batch
    K: int          # results per user
    codes: str = "uniform"      # "uniform" | "zipf"
    zipf_s: float = 1.1
    psi_sigma: float = 1.0
    gpus: tuple = (1,)
    note: str = ""

    @property
    def dm(self) -> int:
        return self.d // self.m


# BASELINE.json "configs", in order.
CONFIGS = {
    "c1": Config("c1", 1, 10_000, 8, 256, 64, 1, 10,
                 note="latency regime (PAPER.md:259 elbow)"),
    "c2": Config("c2", 2, 1_280_000, 8, 256, 512, 128, 10, psi_sigma=0.02,
                 note="Gowalla-shaped (PAPER.md:173); B=1 is row 0 of B=128"),
    "c2a": Config("c2a", 2, 1_280_000, 8, 256, 512, 1, 10, psi_sigma=0.02,
                  note="Gowalla-shaped single user: row 0 of c2 (same cfg_id -> same codes/Psi)"),
    "c3": Config("c3", 3, 10_000_000, 8, 256, 512, 256, 100, codes="zipf",
                 note="Zipf(1.1) codes per split"),
    "c4": Config("c4", 4, 50_000_000, 16, 256, 512, 1024, 100, gpus=(1, 2, 4, 8),
                 note="graded: 50M items, item-sharded 1/2/4/8 GPUs"),
    "c6": Config("c6", 6, 10_000_000, 64, 256, 512, 256, 100,
                 note="next row f2: m = 64 splits (Fig. 2b, PAPER.md:257), not a BASELINE config"),
    "c7": Config("c7", 7, 1_000_000_000, 8, 256, 512, 1, 10,
                 note="next row f2: 10^9 items (RQ2, PAPER.md:255), single user; not a BASELINE config"),
    "c7b": Config("c7b", 7, 1_000_000_000, 8, 256, 512, 128, 10,
                  note="10^9 items (RQ2, PAPER.md:255) for a BATCH of 128 users (same codes as c7): the "
                       "batched layout built on the GPU; not a BASELINE config"),
    "c5": Config("c5", 5, 200_000_000, 4, 16, 64, 4096, 1000, gpus=(8,),
                 note="tie stress: 65,536 code tuples"),
}


def _rng(cfg_id: int, stream: int, chunk: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(
        np.random.SeedSequence([ROOT_SEED, cfg_id, stream, chunk])))


def zipf_probs(b: int, s: float) -> np.ndarray:
    """Truncated Zipf over sub-ids 0..b-1: P(g) ∝ (g+1)^-s (reading R15)."""
    w = np.arange(1, b + 1, dtype=np.float64) ** (-s)
    return w / w.sum()


def _draw_codes_chunk(cfg: Config, chunk: int, n: int) -> np.ndarray:
    rng = _rng(cfg.cfg_id, STREAM_CODES, chunk)
    if cfg.codes == "uniform":
        return rng.integers(0, cfg.b, size=(n, cfg.m), dtype=np.uint8)
    if cfg.codes == "zipf":
        cdf = np.cumsum(zipf_probs(cfg.b, cfg.zipf_s))
        cdf[-1] = 1.0
        u = rng.random((n, cfg.m))
        g = np.searchsorted(cdf, u, side="right")
        return np.minimum(g, cfg.b - 1).astype(np.uint8)
    raise ValueError(cfg.codes)


def codes(cfg: Config, lo: int = 0, hi: Optional[int] = None,
          out: Optional[np.ndarray] = None) -> np.ndarray:
    """Codes G[lo:hi] (uint8 [hi-lo][m]); identical for any shard split."""
    hi = cfg.N if hi is None else hi
    assert 0 <= lo <= hi <= cfg.N
    n = hi - lo
    if out is None:
        out = np.empty((n, cfg.m), dtype=np.uint8)
    c0, c1 = lo // CODE_CHUNK, (hi + CODE_CHUNK - 1) // CODE_CHUNK
    for c in range(c0, c1):
        a = c * CODE_CHUNK
        z = min(cfg.N, a + CODE_CHUNK)
        blk = _draw_codes_chunk(cfg, c, z - a)
        s, e = max(a, lo), min(z, hi)
        if s < e:
            out[s - lo:e - lo] = blk[s - a:e - a]
    return out


def psi(cfg: Config) -> np.ndarray:
    """Sub-item embeddings Psi [m][b][d/m] float32."""
    x = _rng(cfg.cfg_id, STREAM_PSI).standard_normal(
        (cfg.m, cfg.b, cfg.dm), dtype=np.float32)
    if cfg.psi_sigma != 1.0:
        x *= np.float32(cfg.psi_sigma)
    return x


def phi(cfg: Config, B: Optional[int] = None) -> np.ndarray:
    """Sequence embeddings phi [B][d] float32. Row u does
    not depend on B, so a smaller batch is a prefix of a larger one."""
    B = cfg.B if B is None else B
    return _rng(cfg.cfg_id, STREAM_PHI).standard_normal(
        (max(B, 1), cfg.d), dtype=np.float32)[:B].copy()


def instance(cfg: Config, B: Optional[int] = None, lo: int = 0, hi: Optional[int] = None):
    return codes(cfg, lo, hi), psi(cfg), phi(cfg, B)


def random_instance(seed: int, N: int, m: int, b: int, d: int, B: int,
                    code_dist: str = "uniform", scale: float = 1.0):
    """Small ad-hoc instance for tests: (codes uint8 [N][m], Psi f32 [m][b][d/m],
    phi f32 [B][d])."""
    assert d % m == 0
    rng = _rng(900 + (seed & 0xFFFF), seed >> 16 & 0xFFFF, seed)
    if code_dist == "uniform":
        G = rng.integers(0, b, size=(N, m), dtype=np.uint8) if N else np.zeros((0, m), np.uint8)
    elif code_dist == "zipf":
        cdf = np.cumsum(zipf_probs(b, 1.1)); cdf[-1] = 1.0
        G = np.minimum(np.searchsorted(cdf, rng.random((N, m)), side="right"), b - 1).astype(np.uint8)
    elif code_dist == "few":      # very few distinct tuples -> many exact ties
        G = rng.integers(0, min(b, 2), size=(N, m), dtype=np.uint8)
    else:
        raise ValueError(code_dist)
    P = rng.standard_normal((m, b, d // m), dtype=np.float32) * np.float32(scale)
    F = rng.standard_normal((B, d), dtype=np.float32)
    return G, P, F


def sha256(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()
