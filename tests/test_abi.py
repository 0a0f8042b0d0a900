"""C-ABI library: loads, exports every symbol include/hsim.h declares, validates
descriptors, and its host-side decode agrees with the oracle (CPU only; no
compute call is made without a GPU)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import hsim_inputs as H
from paper_2508_05370_b200 import build as pbuild
from paper_2508_05370_b200 import hsim

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    pbuild.build()
    return hsim.lib()


def test_exports_every_declared_symbol(L):
    hdr = open(os.path.join(ROOT, "include", "hsim.h")).read()
    declared = set(re.findall(r"\b(hsim_[a-z_]+)\s*\(", hdr))
    assert declared == set(hsim.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name


def _create(cfg):
    cd, md, keep = hsim.descriptors(cfg)
    h = C.c_void_p()
    rc = hsim.lib().hsim_create(C.byref(cd), C.byref(md), C.byref(h))
    return rc, h, hsim.lib().hsim_last_error().decode()


@pytest.mark.parametrize("mutate,code,kind", [
    (lambda c: c["model"].update(hidden=4097), hsim.HSIM_EINVAL, "DivisibilityViolation"),
    (lambda c: c["model"].update(layers=0), hsim.HSIM_EINVAL, "InvalidValue"),
    (lambda c: c["cluster"]["types"][0].update(gpus_per_node=3), hsim.HSIM_EINVAL, "RailMismatch"),
    (lambda c: c["cluster"].update(nodes=[0, 7]), hsim.HSIM_EINVAL, "UnknownGpuType"),
    (lambda c: c["cluster"]["types"][0].update(nic_gbps=0.0), hsim.HSIM_EINVAL, "NonPositiveBandwidth"),
    (lambda c: c["cluster"]["types"][1]["link_kinds"][0][0].update(gbps=-1.0), hsim.HSIM_EINVAL, "NonPositiveBandwidth"),
    (lambda c: c["model"].update(seq=1 << 20, vocab=1 << 20), hsim.HSIM_ERANGE, "2^53"),
    (lambda c: (c["search"].update(mem_check=1), c["cluster"]["types"][0].update(mem_bytes=0)),
     hsim.HSIM_EINVAL, "mem_bytes"),
])
def test_validation_errors(L, mutate, code, kind):
    cfg = H.get(1)
    mutate(cfg)
    rc, h, msg = _create(cfg)
    assert rc == code and kind in msg and not h.value


def test_null_arguments(L):
    assert L.hsim_create(None, None, None) == hsim.HSIM_EINVAL
    assert L.hsim_space_size(None) == -1
    L.hsim_destroy(None)
    assert L.hsim_eval_batch(None, None, 0, None, None) == hsim.HSIM_ESTATE
    buf = C.create_string_buffer(64)
    assert L.hsim_decode(None, 0, buf, 64) == hsim.HSIM_ESTATE


def test_decode_range_and_buffer(L):
    s = hsim.Sim(H.get(1), host_only=True)
    buf = C.create_string_buffer(8)
    assert L.hsim_decode(s.h, 0, buf, 8) == hsim.HSIM_ERANGE
    assert L.hsim_decode(s.h, 1, buf, 8) == hsim.HSIM_ERANGE
    assert s.decode(0)["classes"][0]["layers"] == [3, 9]


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_space_and_templates_match_oracle(oracle_mod, L, n):
    cfg = H.get(n)
    s = hsim.Sim(cfg, host_only=True)
    o = oracle_mod.Oracle(cfg)
    assert s.space_size() == o.space_size()
    assert s.n_templates() == o.n_templates()
    pre = o.template_prefix()
    ks = np.unique(np.linspace(0, len(pre) - 1, 200).astype(int))
    assert all(s.template_first(int(k)) == pre[k] for k in ks)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_host_decode_matches_oracle_plan(oracle_mod, L, n):
    """Step 1 (partition) and placement, host side of the product vs oracle."""
    cfg = H.get(n)
    s = hsim.Sim(cfg, host_only=True)
    o = oracle_mod.Oracle(cfg)
    idx = H.sample_indices(o.space_size(), 150 if n != 3 else 40, seed=n)
    for i in idx:
        a, b = s.decode(int(i)), o.describe(int(i))
        assert a["b"] == b["b"] and a["status"] == b["status"], (i, a, b)
        for ca, cb in zip(a["classes"], b["classes"]):
            assert ca["D"] == cb["D"] and ca["stages"] == cb["stages"]
            assert ca["place"] == cb["place"]
            if b["status"] != -1:
                assert ca["layers"] == cb["layers"], (i, ca, cb)
            if b["status"] == 0:
                assert ca["mb"] == cb["mb"], (i, ca, cb)


def test_eval_without_gpu_fails_loudly(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    s = hsim.Sim(H.get(1), host_only=True)
    c = hsim.hsim_cands()
    rc = L.hsim_eval_batch(s.h, C.byref(c), 1, None, None)
    assert rc == hsim.HSIM_ECUDA
    with pytest.raises(RuntimeError):
        hsim.Sim(H.get(1))


@pytest.mark.parametrize("n", [2, 4, 5])
def test_host_decode_memcheck_status_matches_oracle(oracle_mod, L, n):
    """With mem_check on (DESIGN.md M.1) the product's host-side split (the same
    HD code the kernels run) and the oracle agree on every sampled status."""
    cfg = H.with_mem_check(H.get(n))
    s = hsim.Sim(cfg, host_only=True)
    o = oracle_mod.Oracle(cfg)
    idx = H.sample_indices(s.space_size(), 300, seed=H.PARITY_SEED + 60 + n)
    got = [s.decode(int(i))["status"] for i in idx]
    want = [o.describe(int(i))["status"] for i in idx]
    assert got == want and -3 in got


@pytest.mark.parametrize("cfg_name", ["ilv2-c2", "ilv3-c4", "ilv2-c5", "ep-c4", "ep-ilv-tiny"])
def test_host_decode_variants_match_oracle(oracle_mod, L, cfg_name):
    """SURVEY §8(f) f4 (DESIGN.md V.2, V.3): the product's host-side split (the
    HD partition the kernels run: -1 for a stage with fewer layers than chunks,
    -2 for a micro-batch count that is not a multiple of the depth; V.3's
    expert-sharded partition weights) agrees with the oracle's plan."""
    cfg = {"ilv2-c2": lambda: H.with_interleave(H.get(2), 2),
           "ilv3-c4": lambda: H.with_interleave(H.get(4), 3),
           "ilv2-c5": lambda: H.with_interleave(H.get(5), 2),
           "ep-c4": lambda: H.with_ep_dp(H.get(4)),
           "ep-ilv-tiny": lambda: H.with_ep_dp(H.with_interleave(H.variant_tiny(104, moe=True), 2))}[cfg_name]()
    s = hsim.Sim(cfg, host_only=True)
    o = oracle_mod.Oracle(cfg)
    assert s.space_size() == o.space_size()
    idx = H.sample_indices(o.space_size(), 400, seed=17)
    seen = set()
    for i in idx:
        a, b = s.decode(int(i)), o.describe(int(i))
        assert a["status"] == b["status"], (i, a, b)
        seen.add(b["status"])
        for ca, cb in zip(a["classes"], b["classes"]):
            if b["status"] != -1:
                assert ca["layers"] == cb["layers"], (i, ca, cb)
            if b["status"] == 0:
                assert ca["mb"] == cb["mb"], (i, ca, cb)
    assert 0 in seen


def test_variant_validation(L):
    """interleave outside 0..8, ep_dp outside {0, 1}, and mem_check with either
    variant are HSIM_EINVAL (include/hsim.h)."""
    for cfg in (H.with_interleave(H.get(2), 9), H.with_mem_check(H.with_interleave(H.get(2), 2)),
                H.with_mem_check(H.with_ep_dp(H.get(4))), H.with_changes(H.with_ep_dp(H.get(4)), search__ep_dp=2)):
        with pytest.raises(hsim.HsimError) as e:
            hsim.Sim(cfg, host_only=True)
        assert e.value.code == hsim.HSIM_EINVAL


@pytest.mark.parametrize("n", [2, 4, 5])
def test_host_decode_mixtp_matches_oracle(oracle_mod, L, n):
    """V.1: the MIXTP family's size, order, placement (two nodes
    per group), layer and micro-batch splits agree with the oracle."""
    cfg = H.with_changes(H.get(n), search__mixtp=1)
    s = hsim.Sim(cfg, host_only=True)
    o = oracle_mod.Oracle(cfg)
    base = oracle_mod.Oracle(H.get(n)).space_size()
    assert s.space_size() == o.space_size() > base
    idx = np.unique(np.concatenate([H.sample_indices(s.space_size(), 100, seed=3),
                                    [s.template_first(k) for k in range(s.n_templates() - 40, s.n_templates())]]))
    mixed = 0
    for i in idx:
        a, b = s.decode(int(i)), o.describe(int(i))
        assert a["status"] == b["status"], (i, a, b)
        for ca, cb in zip(a["classes"], b["classes"]):
            assert ca["stages"] == cb["stages"] and ca["place"] == cb["place"], (i, ca, cb)
            mixed += len(ca["stages"][0]) == 3
            if b["status"] != -1:
                assert ca["layers"] == cb["layers"], (i, ca, cb)
            if b["status"] == 0:
                assert ca["mb"] == cb["mb"], (i, ca, cb)
    assert mixed > 0


def test_mixtp_validation(L):
    for cfg in (H.with_mem_check(H.with_changes(H.get(2), search__mixtp=1)),
                H.with_ep_dp(H.with_changes(H.get(4), search__mixtp=1)),
                H.with_changes(H.get(2), search__mixtp=2)):
        with pytest.raises(hsim.HsimError) as e:
            hsim.Sim(cfg, host_only=True)
        assert e.value.code == hsim.HSIM_EINVAL


def test_buckets_validation_and_decode(oracle_mod, L):
    """B.1: sync_buckets outside 0..2 or 2 with interleave are HSIM_EINVAL; the
    knob leaves the candidate space and the splits unchanged."""
    for cfg in (H.with_changes(H.get(2), search__sync_buckets=3),
                H.with_interleave(H.with_changes(H.get(2), search__sync_buckets=2), 2)):
        with pytest.raises(hsim.HsimError) as e:
            hsim.Sim(cfg, host_only=True)
        assert e.value.code == hsim.HSIM_EINVAL
    s = hsim.Sim(H.with_changes(H.get(4), search__sync_buckets=2), host_only=True)
    assert s.space_size() == oracle_mod.Oracle(H.get(4)).space_size()


def test_dedup_knob_host(L):
    """hsim_set_dedup / hsim_dedup_active (DESIGN.md §5 pipeline dedupe): on by
    default for every BASELINE config (the key fits 63 bits), off with S.1 or
    V.2 whatever the knob says, and switchable per handle."""
    for n in (1, 2, 3, 4, 5):
        s = hsim.Sim(H.get(n), host_only=True)
        assert s.dedup_active(), n
        s.set_dedup(False)
        assert not s.dedup_active()
        s.set_dedup(True)
        assert s.dedup_active()
    assert not hsim.Sim(H.with_sync_overlap(H.get(2)), host_only=True).dedup_active()
    assert not hsim.Sim(H.with_interleave(H.variant_tiny(3)), host_only=True).dedup_active()
    assert L.hsim_dedup_active(None) == -1
    assert L.hsim_set_dedup(None, 1) == hsim.HSIM_ESTATE
