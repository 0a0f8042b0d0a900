"""GPU parity of the overlapped gradient-sync row (SURVEY.md §8(f) f1,
DESIGN.md S.1): the CUDA path (1F1B kernels export every stage's last-backward
end, K_sync_overlap schedules the segments) vs the oracle's event engine,
int64-equal, on sampled BASELINE configs (template first / last indices
included), a contiguous range with a ragged tail, full tiny spaces, top-k,
and combined with the memory check."""
import os

import numpy as np
import pytest

import hsim_inputs as H

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 8


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_05370_b200 import build
    build.build()
    return torch


def _sim(cfg):
    from paper_2508_05370_b200 import Sim
    return Sim(cfg)


def _check(idx, got, want):
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first: i={idx[bad[0]]} gpu={got[bad[0]]} oracle={want[bad[0]]}"


@pytest.mark.parametrize("n,count", [(1, 1), (2, 5000), (3, 1200), (4, 3000), (5, 1200)])
def test_overlap_sampled_parity(torch_cuda, oracle_mod, n, count):
    cfg = H.with_sync_overlap(H.get(n))
    sim, o = _sim(cfg), oracle_mod.Oracle(cfg)
    N = o.space_size()
    pre = o.template_prefix()
    ks = np.unique(np.linspace(0, len(pre) - 2, 300).astype(int))
    extra = np.concatenate([pre[ks], pre[ks + 1] - 1])
    idx = H.sample_indices(N, min(count, N), seed=H.PARITY_SEED + 50 + n, extra=extra)
    got = sim.eval_batch(idx=torch_cuda.as_tensor(idx, device="cuda")).cpu().numpy()
    want = o.eval_many(idx, threads=THREADS)
    _check(idx, got, want)


def test_overlap_range_topk_and_memcheck_config2(torch_cuda, oracle_mod):
    for cfg in (H.with_sync_overlap(H.get(2)), H.with_mem_check(H.with_sync_overlap(H.get(2)))):
        sim, o = _sim(cfg), oracle_mod.Oracle(cfg)
        first, n = 150000, 12345
        got = sim.eval_batch(n=n, first=first).cpu().numpy()
        want = o.eval_many(first=first, n=n, threads=THREADS)
        _check(np.arange(first, first + n), got, want)
        ok = np.nonzero(want >= 0)[0]
        order = np.lexsort((ok, want[ok]))
        t, i = sim.topk(16, n=n, first=first)
        t, i = t.cpu().numpy(), i.cpu().numpy()
        nv = min(16, ok.size)
        assert np.array_equal(t[:nv], want[ok][order[:nv]])
        assert np.array_equal(i[:nv], ok[order[:nv]] + first)
        assert np.all(t[nv:] == np.iinfo(np.int64).max) and np.all(i[nv:] == -1)


@pytest.mark.parametrize("seed", [300, 301, 302, 303, 304, 305])
def test_overlap_tiny_full(torch_cuda, oracle_mod, seed):
    cfg = H.with_sync_overlap(H.tiny_random(seed))
    sim, o = _sim(cfg), oracle_mod.Oracle(cfg)
    N = o.space_size()
    got = sim.eval_batch(n=N).cpu().numpy()
    want = o.eval_many(first=0, n=N, threads=THREADS)
    _check(np.arange(N), got, want)
