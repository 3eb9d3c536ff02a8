"""Seeded input generator (pqsynth): determinism, shard invariance, recipe."""
import numpy as np

import pqsynth


def test_codes_shard_invariance():
    cfg = pqsynth.Config("t", 99, 3 * pqsynth.CODE_CHUNK + 12345, 4, 16, 64, 3, 5)
    full = pqsynth.codes(cfg)
    for G in (2, 4, 8):
        n = cfg.N // G
        parts = [pqsynth.codes(cfg, g * n, cfg.N if g == G - 1 else (g + 1) * n) for g in range(G)]
        assert np.array_equal(np.concatenate(parts), full)
    assert full.max() < 16


def test_determinism_and_prefix():
    cfg = pqsynth.CONFIGS["c1"]
    a = pqsynth.instance(cfg)
    b = pqsynth.instance(cfg)
    for x, y in zip(a, b):
        assert pqsynth.sha256(x) == pqsynth.sha256(y)
    c2 = pqsynth.CONFIGS["c2"]
    assert np.array_equal(pqsynth.phi(c2, 1)[0], pqsynth.phi(c2)[0])   # B=1 is row 0 of B=128


def test_zipf_closed_form():
    p = pqsynth.zipf_probs(256, 1.1)
    H = sum((g + 1) ** -1.1 for g in range(256))
    assert abs(p[0] - 1.0 / H) < 1e-15
    assert abs(p[0] - 0.2065) < 5e-4
    cfg = pqsynth.Config("z", 98, 400_000, 2, 256, 16, 1, 1, codes="zipf")
    G = pqsynth.codes(cfg)
    freq = np.bincount(G[:, 0], minlength=256) / G.shape[0]
    assert abs(freq[0] - p[0]) < 5 * np.sqrt(p[0] * (1 - p[0]) / G.shape[0])


def test_psi_sigma():
    c2 = pqsynth.CONFIGS["c2"]
    P = pqsynth.psi(c2)
    assert P.shape == (8, 256, 64) and P.dtype == np.float32
    assert abs(P.std() - 0.02) < 0.001
