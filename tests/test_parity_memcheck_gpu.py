"""GPU parity of the memory-feasibility row (DESIGN.md M.1):
with mem_check on, the CUDA path (through the C ABI) and the oracle agree
int64-exactly -- -3 for candidates over capacity, unchanged times otherwise --
on sampled BASELINE configs, contiguous ranges, full tiny spaces with
capacities around the median need, and the top-k (which skips -3)."""
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


@pytest.mark.parametrize("n,count", [(2, 5000), (3, 1200), (4, 3000), (5, 1200)])
def test_memcheck_sampled_parity(torch_cuda, oracle_mod, n, count):
    cfg = H.with_mem_check(H.get(n))
    sim, o = _sim(cfg), oracle_mod.Oracle(cfg)
    idx = H.sample_indices(o.space_size(), count, seed=H.PARITY_SEED + 30 + n)
    t = torch_cuda.as_tensor(idx, device="cuda")
    got = sim.eval_batch(idx=t).cpu().numpy()
    want = o.eval_many(idx, threads=THREADS)
    _check(idx, got, want)
    assert (want == -3).any()
    if n in (2, 4):  # GPT-3 175B / Llama-3 70B at s = 8192 rarely fit without ZeRO / recomputation
        assert (want >= 0).any()


def test_memcheck_range_and_topk_config2(torch_cuda, oracle_mod):
    cfg = H.with_mem_check(H.get(2))
    sim, o = _sim(cfg), oracle_mod.Oracle(cfg)
    first, n = 150000, 20000
    got = sim.eval_batch(n=n, first=first).cpu().numpy()
    want = o.eval_many(first=first, n=n, threads=THREADS)
    _check(np.arange(first, first + n), got, want)
    ok = np.nonzero(want >= 0)[0]
    order = np.lexsort((ok, want[ok]))
    for k in (1, 16, 300):
        t, i = sim.topk(k, n=n, first=first)
        assert np.array_equal(t.cpu().numpy(), want[ok][order[:k]])
        assert np.array_equal(i.cpu().numpy(), ok[order[:k]] + first)


@pytest.mark.parametrize("seed", [200, 201, 202, 203])
def test_memcheck_tiny_full(torch_cuda, oracle_mod, seed):
    base = H.tiny_random(seed)
    o0 = oracle_mod.Oracle(base)
    N = o0.space_size()
    needs = []
    for i in range(N):
        d = o0.describe(i)
        if d["status"] == 0:
            for c in d["classes"]:
                P = len(c["stages"])
                for s, (ty, tp) in enumerate(c["stages"]):
                    needs.append(o0.device_bytes(ty, tp, P, s, c["layers"][s], max(c["mb"]), d["b"]))
    cfg = H.with_mem_check(base, [int(np.median(needs))] * len(base["cluster"]["types"]))
    sim, o = _sim(cfg), oracle_mod.Oracle(cfg)
    got = sim.eval_batch(n=N).cpu().numpy()
    want = o.eval_many(first=0, n=N, threads=THREADS)
    _check(np.arange(N), got, want)
    assert (want == -3).any()
