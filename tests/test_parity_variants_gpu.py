"""GPU parity of the SURVEY §8(f) f4 variants (DESIGN.md V.2, V.3) through the
C-ABI (hsim_eval_batch / hsim_topk), int64-equal to the oracle:

* V.2 interleaved 1F1B (K_ilv, K_sync_ilv): every candidate of tiny spaces
  with v = 2, 3, 4, and with the S.1 overlapped sync; the whole config-2
  space (v = 2) against the compact oracle; config 3 / 4 / 5 samples plus
  template endpoints; the deep tiny spaces (17..64 stages: two stages per
  lane, the largest shared-memory rings); top-k against brute force.
* V.3 expert parallelism across the replicas: tiny MoE spaces in full, config
  4 in full (compact oracle) and its top-k.
* both variants together, and the ABI's rejections.
"""
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


def assert_equal(idx, got, want):
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first: i={idx[bad[0]]} gpu={got[bad[0]]} oracle={want[bad[0]]}"


def full_space(cfg, oracle_mod, compact=False, topk=8):
    from paper_2508_05370_b200 import Sim
    sim, o = Sim(cfg), oracle_mod.Oracle(cfg, compact=compact)
    N = o.space_size()
    assert sim.space_size() == N
    got = sim.eval_batch(n=N).cpu().numpy()
    want = o.eval_many(first=0, n=N, threads=THREADS)
    assert_equal(np.arange(N), got, want)
    assert not (got == -5).any()
    if topk:
        t, i = sim.topk(topk)
        ok = np.nonzero(want >= 0)[0]
        order = np.lexsort((ok, want[ok]))[:topk]
        assert np.array_equal(t.cpu().numpy()[:len(order)], want[ok][order])
        assert np.array_equal(i.cpu().numpy()[:len(order)], ok[order])
    return want


def sampled(cfg, oracle_mod, n, seed, compact=True):
    import torch
    from paper_2508_05370_b200 import Sim
    sim, o = Sim(cfg), oracle_mod.Oracle(cfg, compact=compact)
    pre = o.template_prefix()
    k = np.linspace(0, len(pre) - 2, min(len(pre) - 1, 400)).astype(np.int64)
    idx = H.sample_indices(o.space_size(), n, seed=seed, extra=np.concatenate([pre[k], pre[k + 1] - 1]))
    got = sim.eval_batch(idx=torch.as_tensor(idx, device="cuda")).cpu().numpy()
    want = o.eval_many(idx, threads=THREADS)
    assert_equal(idx, got, want)
    return want


@pytest.mark.parametrize("seed", [100, 101, 103, 105, 107, 110])
@pytest.mark.parametrize("v", [2, 3, 4])
def test_interleave_tiny_full(torch_cuda, oracle_mod, seed, v):
    want = full_space(H.with_interleave(H.variant_tiny(seed), v), oracle_mod)
    assert (want >= 0).any()


@pytest.mark.parametrize("seed", [101, 105, 110])
def test_interleave_overlap_tiny_full(torch_cuda, oracle_mod, seed):
    full_space(H.with_sync_overlap(H.with_interleave(H.variant_tiny(seed), 2)), oracle_mod)


@pytest.mark.parametrize("variant", [0, 1])
def test_interleave_deep_tiny_full(torch_cuda, oracle_mod, variant):
    """17..64-stage interleaved pipelines (stages 32..63 on the lanes' second
    slot; rings of 32 / 64 entries)."""
    cfg = H.with_interleave(H.with_changes(H.deep_tiny(variant), model__global_batch=7680, model__layers=192), 2)
    want = full_space(cfg, oracle_mod, compact=True)
    assert (want >= 0).sum() > 10


def test_interleave_config2_full(torch_cuda, oracle_mod):
    want = full_space(H.with_interleave(H.get(2), 2), oracle_mod, compact=True, topk=16)
    assert (want >= 0).sum() > 1000


@pytest.mark.parametrize("n,v", [(3, 2), (4, 2), (4, 4), (5, 2)])
def test_interleave_configs_sampled(torch_cuda, oracle_mod, n, v):
    want = sampled(H.with_interleave(H.get(n), v), oracle_mod, 4000, seed=H.PARITY_SEED + n)
    assert (want >= 0).sum() > 10


def test_interleave_overlap_config2_sampled(torch_cuda, oracle_mod):
    sampled(H.with_sync_overlap(H.with_interleave(H.get(2), 2)), oracle_mod, 6000, seed=3)


@pytest.mark.parametrize("seed", [100, 102, 104, 106, 108])
def test_ep_dp_tiny_full(torch_cuda, oracle_mod, seed):
    full_space(H.with_ep_dp(H.variant_tiny(seed, moe=True)), oracle_mod)


def test_ep_dp_config4_full(torch_cuda, oracle_mod):
    want = full_space(H.with_ep_dp(H.get(4)), oracle_mod, compact=True, topk=16)
    assert (want >= 0).sum() > 1000


def test_both_variants(torch_cuda, oracle_mod):
    full_space(H.with_ep_dp(H.with_interleave(H.variant_tiny(104, moe=True), 2)), oracle_mod)
    sampled(H.with_sync_overlap(H.with_ep_dp(H.with_interleave(H.get(4), 2))), oracle_mod, 4000, seed=5)


def test_variant_rejections(torch_cuda):
    import torch
    from paper_2508_05370_b200 import Sim
    with pytest.raises(Exception):
        Sim(H.with_mem_check(H.with_interleave(H.get(2), 2)))
    with pytest.raises(Exception):
        Sim(H.with_mem_check(H.with_ep_dp(H.get(4))))
    sim = Sim(H.with_interleave(H.get(2), 2))
    with pytest.raises(Exception):
        sim.flow_resim(torch.tensor([0], device="cuda"))


# ----------------------------------------------------------------------------
# V.1 mixed-type TP groups (the MIXTP family)
# ----------------------------------------------------------------------------
def mixtp_range(cfg, oracle_mod):
    """Every candidate of the MIXTP family (appended after each micro-batch
    size's MIXED templates: compared over the whole space's MIXTP templates)."""
    from paper_2508_05370_b200 import Sim
    sim, o = Sim(cfg), oracle_mod.Oracle(cfg, compact=True)
    pre = o.template_prefix()
    idx = []
    for k in range(o.n_templates()):
        st = o.describe(int(pre[k]))["classes"][0]["stages"][0]
        if len(st) == 3:
            idx.append(np.arange(pre[k], pre[k + 1]))
    idx = np.concatenate(idx)
    import torch
    got = sim.eval_batch(idx=torch.as_tensor(idx, device="cuda")).cpu().numpy()
    want = o.eval_many(idx, threads=THREADS)
    assert_equal(idx, got, want)
    return want


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_mixtp_family_full(torch_cuda, oracle_mod, n):
    want = mixtp_range(H.with_changes(H.get(n), search__mixtp=1), oracle_mod)
    assert (want >= 0).sum() > 10


@pytest.mark.parametrize("mode", ["interleave", "overlap"])
def test_mixtp_with_schedule_variants(torch_cuda, oracle_mod, mode):
    cfg = H.with_changes(H.get(2), search__mixtp=1)
    cfg = H.with_interleave(cfg, 2) if mode == "interleave" else H.with_sync_overlap(cfg)
    mixtp_range(cfg, oracle_mod)


@pytest.mark.parametrize("seed", [101, 105, 110])
def test_mixtp_tiny_full(torch_cuda, oracle_mod, seed):
    full_space(H.with_changes(H.variant_tiny(seed), search__mixtp=1), oracle_mod)


def test_mixtp_config2_topk(torch_cuda, oracle_mod):
    full_space(H.with_changes(H.get(2), search__mixtp=1), oracle_mod, compact=True, topk=16)


# ----------------------------------------------------------------------------
# B.1 two gradient buckets per stage group (f1, Table 1 "DP frequency 2")
# ----------------------------------------------------------------------------
def with_buckets(cfg):
    return H.with_changes(cfg, search__sync_buckets=2)


@pytest.mark.parametrize("overlap", [False, True])
def test_buckets_config2_full(torch_cuda, oracle_mod, overlap):
    cfg = with_buckets(H.with_sync_overlap(H.get(2)) if overlap else H.get(2))
    want = full_space(cfg, oracle_mod, compact=True, topk=16)
    assert (want >= 0).sum() > 1000


@pytest.mark.parametrize("n,overlap", [(3, True), (4, False), (4, True), (5, True)])
def test_buckets_configs_sampled(torch_cuda, oracle_mod, n, overlap):
    cfg = with_buckets(H.with_sync_overlap(H.get(n)) if overlap else H.get(n))
    sampled(cfg, oracle_mod, 4000, seed=H.PARITY_SEED + 7 * n)


@pytest.mark.parametrize("seed", [101, 105, 110])
def test_buckets_tiny_full(torch_cuda, oracle_mod, seed):
    full_space(with_buckets(H.with_sync_overlap(H.variant_tiny(seed))), oracle_mod)
    full_space(with_buckets(H.variant_tiny(seed)), oracle_mod)


def test_buckets_with_mixtp_and_ep(torch_cuda, oracle_mod):
    mixtp_range(with_buckets(H.with_sync_overlap(H.with_changes(H.get(2), search__mixtp=1))), oracle_mod)
    sampled(with_buckets(H.with_sync_overlap(H.with_ep_dp(H.get(4)))), oracle_mod, 4000, seed=13)
