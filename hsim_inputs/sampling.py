"""Seeded index samplers (splitmix64) — shared input plumbing, no method arithmetic.

Seed 0x5EED2508 is the parity-sample seed named in SURVEY.md §8(d).
"""
import numpy as np

PARITY_SEED = 0x5EED2508
_MASK = (1 << 64) - 1


class SplitMix64:
    """Counter-based splitmix64 (Steele et al.); pure-Python, deterministic."""

    def __init__(self, seed):
        self.state = seed & _MASK

    def next(self):
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def below(self, n):
        return self.next() % n


def sample_indices(n_space, count, seed=PARITY_SEED, extra=()):
    """Sorted unique int64 indices: ``count`` seeded uniform draws from
    [0, n_space) plus the given extra indices (e.g. template first/last)."""
    if n_space <= 0:
        return np.zeros(0, dtype=np.int64)
    rng = SplitMix64(seed)
    idx = {rng.below(n_space) for _ in range(count)}
    idx.update(int(e) for e in extra if 0 <= int(e) < n_space)
    return np.array(sorted(idx), dtype=np.int64)
