"""The oracle's two modes agree ("It runs in two modes ...
The two modes must agree"; C.11 "Equivalences to test").

literal: every replica simulated, stage time = sum over the stage's layers of
the layer-op chain, every ring collective simulated send by send.
compact: one pipeline per sub-class of replicas with equal p2p vectors (m =
their largest m), stage time = l x chain, ring = steps x slowest edge.

The literal == compact identity rests on three facts, each pinned elsewhere:
the async ring finishes at steps x max tau (test_oracle_pins.py, random
heterogeneous rings), T_pipe is non-decreasing in m
(test_1f1b_monotone_in_microbatches), and integer sums equal products.  Here
the two whole simulators are compared candidate by candidate, int64-equal.
CPU only; the exhaustive config-2 comparison is marked slow.
"""
import os

import numpy as np
import pytest

import hsim_inputs as H

THREADS = os.cpu_count() or 4


def _pair(oracle_mod, cfg):
    return oracle_mod.Oracle(cfg), oracle_mod.Oracle(cfg, compact=True)


def _check(lit, cmp_, idx):
    a = lit.eval_many(idx, threads=THREADS)
    b = cmp_.eval_many(idx, threads=THREADS)
    bad = np.nonzero(a != b)[0]
    assert bad.size == 0, f"{bad.size} differ, first i={idx[bad[0]]}: literal {a[bad[0]]} compact {b[bad[0]]}"
    return a


def test_config1(oracle_mod):
    lit, cmp_ = _pair(oracle_mod, H.get(1))
    assert lit.eval(0) == cmp_.eval(0) > 0


@pytest.mark.parametrize("n,count", [(2, 20000), (3, 10000), (4, 10000), (5, 10000)])
def test_sampled_configs(oracle_mod, n, count):
    """1e4 seeded samples of configs 3-5, 2e4 of config 2, plus
    the first and last candidate of 300 templates."""
    lit, cmp_ = _pair(oracle_mod, H.get(n))
    pre = lit.template_prefix()
    ks = np.unique(np.linspace(0, len(pre) - 2, 300).astype(int))
    idx = H.sample_indices(lit.space_size(), count, seed=H.PARITY_SEED + 40 + n,
                           extra=np.concatenate([pre[ks], pre[ks + 1] - 1]))
    a = _check(lit, cmp_, idx)
    assert (a >= 0).mean() > 0.5


@pytest.mark.parametrize("seed", range(100, 112))
def test_tiny_spaces_full(oracle_mod, seed):
    cfg = H.tiny_random(seed)
    lit, cmp_ = _pair(oracle_mod, cfg)
    N = lit.space_size()
    _check(lit, cmp_, np.arange(N, dtype=np.int64))


@pytest.mark.parametrize("variant", ["mem_check", "sync_overlap"])
@pytest.mark.parametrize("n", [2, 4])
def test_rows_f1_f2(oracle_mod, variant, n):
    cfg = H.with_mem_check(H.get(n)) if variant == "mem_check" else H.with_sync_overlap(H.get(n))
    lit, cmp_ = _pair(oracle_mod, cfg)
    idx = H.sample_indices(lit.space_size(), 4000, seed=H.PARITY_SEED + 60 + n)
    _check(lit, cmp_, idx)


@pytest.mark.slow
@pytest.mark.skipif(os.environ.get("HSIM_FULL") != "1", reason="exhaustive: set HSIM_FULL=1")
def test_config2_exhaustive(oracle_mod):
    lit, cmp_ = _pair(oracle_mod, H.get(2))
    _check(lit, cmp_, np.arange(lit.space_size(), dtype=np.int64))
