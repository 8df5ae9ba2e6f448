"""Size-independent fingerprints of long vectors for the full-config fixtures.

TEST INFRASTRUCTURE ONLY (used by oracle/full_config.py and tests/).  A
CountSketch with a seeded hash h: [n] -> [K] and seeded signs s: [n] -> {+-1}
is linear, so sketch(a) - sketch(b) = sketch(a - b), and
E |sketch(v)|^2 = |v|^2 with relative spread about sqrt(2/K): the relative L2
distance between the GPU vector and the oracle's can be estimated to a few
percent from K numbers per vector (4096 here) instead of the vector itself.
"""
import numpy as np

K = 4096


def _hash(n, seed):
    rng = np.random.default_rng([seed, n])
    return rng.integers(0, K, n), rng.choice((-1.0, 1.0), n)


def count_sketch(v, seed=20260, k=K):
    v = np.asarray(v, dtype=np.float64).ravel()
    h, s = _hash(len(v), seed)
    assert k == K
    return np.bincount(h, weights=s * v, minlength=K)


def sample_idx(n, m=4096, seed=7):
    """Seeded sample of entry indices (sorted, distinct)."""
    rng = np.random.default_rng([seed, n])
    return np.sort(rng.choice(n, size=min(m, n), replace=False))
