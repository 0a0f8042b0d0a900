"""Shared, seeded, synthetic inputs for the product and the oracle.

Holds presets (data), the five BASELINE workloads, tiny random workloads and
seeded index samplers.  It contains none of the method's arithmetic, so both
sides may import it without sharing any computation (task rule ③).
"""
from . import presets, configs, sampling  # noqa: F401
from .configs import get, tiny_random, deep_tiny, four_types_tiny, with_changes, with_mem_check, with_sync_overlap, with_interleave, with_ep_dp, variant_tiny  # noqa: F401
from .sampling import sample_indices, PARITY_SEED, SplitMix64  # noqa: F401
