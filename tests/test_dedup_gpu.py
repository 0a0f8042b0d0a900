"""GPU: the pipeline dedupe (hsim_set_dedup) is exact.

With the dedupe on (the default) a batch runs the 1F1B recurrence once per
distinct (template, class, boundary digits, sub-class micro-batch vector)
through a device hash table; off, once per (candidate, class).  Both must give
the same int64 results for every candidate -- and the oracle's (every other
GPU parity test runs with the dedupe on, this file adds the on/off
equivalence, table reuse across calls and the cases it does not apply to).
"""
import numpy as np
import pytest

import hsim_inputs as H

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_05370_b200 import build
    build.build()
    return torch


def both(sim, fn):
    sim.set_dedup(True)
    a = fn()
    sim.set_dedup(False)
    b = fn()
    sim.set_dedup(True)
    return a, b


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


CFGS = {
    "c2": lambda: H.get(2),
    "c3": lambda: H.get(3),
    "c4": lambda: H.get(4),
    "c5": lambda: H.get(5),
    "c2-mixtp": lambda: H.with_changes(H.get(2), search__mixtp=1),
    "c4-epdp": lambda: H.with_ep_dp(H.get(4)),
    "c2-buckets": lambda: H.with_changes(H.get(2), search__sync_buckets=2),
    "c2-mem": lambda: H.with_mem_check(H.get(2)),
    "deep": lambda: H.deep_tiny(0),
    "four": lambda: H.four_types_tiny(),
}


@pytest.mark.parametrize("name", list(CFGS))
def test_on_off_equal_range(torch_cuda, name):
    """Every candidate of a contiguous range (the whole space up to 4M):
    dedupe on == off, int64-equal, and the dedupe is active."""
    from paper_2508_05370_b200 import Sim
    sim = Sim(CFGS[name]())
    assert sim.dedup_active()
    N = sim.space_size()
    n = min(N, 4_000_000)
    first = (N - n) // 3
    a, b = both(sim, lambda: _np(sim.eval_batch(n=n, first=first)))
    bad = np.nonzero(a != b)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first at {first + bad[0]}: on={a[bad[0]]} off={b[bad[0]]}"
    assert (a >= 0).any()


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_on_off_equal_explicit_lists(torch_cuda, name):
    """Explicit index lists in random order with repeats (lanes of a warp from
    different templates, equal keys across warps): on == off."""
    from paper_2508_05370_b200 import Sim
    torch = torch_cuda
    sim = Sim(CFGS[name]())
    N = sim.space_size()
    rng = np.random.default_rng(0x5EED)
    idx = rng.integers(0, N, size=300_000)
    idx = np.concatenate([idx, idx[:50_000], np.arange(min(N, 20_000))])
    rng.shuffle(idx)
    t = torch.as_tensor(idx, device="cuda")
    a, b = both(sim, lambda: _np(sim.eval_batch(idx=t)))
    assert np.array_equal(a, b)


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c2-mixtp"])
def test_on_off_equal_topk(torch_cuda, name):
    from paper_2508_05370_b200 import Sim
    sim = Sim(CFGS[name]())
    n = min(sim.space_size(), 6_000_000)
    for k in (1, 16, 32, 100):
        (ta, ia), (tb, ib) = both(sim, lambda: sim.topk(k, n=n))
        assert np.array_equal(_np(ta), _np(tb)) and np.array_equal(_np(ia), _np(ib))


def test_table_reuse_across_calls(torch_cuda):
    """The table is emptied by each call's final kernel: a sequence of calls of
    different sizes and modes on one handle equals fresh-handle results."""
    from paper_2508_05370_b200 import Sim
    cfg = H.get(3)
    sim = Sim(cfg)
    N = sim.space_size()
    calls = [(0, 3_000_000), (1_000_000, 5000), (N - 40_000, 40_000), (0, 3_000_000), (17, 1)]
    got = []
    for first, n in calls:
        got.append(_np(sim.eval_batch(n=n, first=first)))
        sim.topk(16, n=n, first=first)  # interleave top-k calls (pruned K_final clears too)
        sim.count_cells(first=first, n=min(n, 100_000))  # count mode clears its table itself
    for (first, n), g in zip(calls, got):
        fresh = Sim(cfg)
        fresh.set_dedup(False)
        assert np.array_equal(g, _np(fresh.eval_batch(n=n, first=first))), (first, n)
        fresh.close()


def test_block_cyclic_shards(torch_cuda):
    from paper_2508_05370_b200 import Sim
    sim = Sim(H.get(2))
    N = sim.space_size()
    for r, W in ((0, 2), (1, 2), (3, 8)):
        n = (N // (W * 4096)) * 4096
        a, b = both(sim, lambda: _np(sim.eval_batch(n=n, first=r * 4096, block=4096, stride=W * 4096)))
        assert np.array_equal(a, b)


def test_cells_drop_with_dedupe(torch_cuda):
    """The dedupe runs fewer 1F1B cells (the count reports what executes)."""
    from paper_2508_05370_b200 import Sim
    sim = Sim(H.get(2))
    on, off = both(sim, lambda: sim.count_cells())
    assert 0 < on < off


@pytest.mark.parametrize("mk", [lambda: H.with_sync_overlap(H.get(2)), lambda: H.with_interleave(H.variant_tiny(3))])
def test_not_active_for_overlap_and_interleave(torch_cuda, mk):
    from paper_2508_05370_b200 import Sim
    sim = Sim(mk())
    assert not sim.dedup_active()
    sim.set_dedup(False)
    assert not sim.dedup_active()
