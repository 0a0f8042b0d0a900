"""Pins of the memory-feasibility row (DESIGN.md M.1) in
the CPU oracle.  The paper never gates on memory; M.1 is a
reading, pinned here by what fixes its parts independently: public parameter
counts (tests/golden/paper_examples.json), the 34 s b h bytes-per-layer
activation figure and its TP form s b h (10 + 24/t) (Korthikanti et al. 2022,
selective recomputation), 1F1B's in-flight depth counted from the schedule
itself, SPEC.md:93's GPT-13B-on-40-GB example, and invariants.  CPU only."""
import json
import os

import numpy as np
import pytest

import hsim_inputs as H

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _parts(o, type_idx, tp, P, s, L, b):
    """(static bytes, per-layer per-micro-batch activation bytes) from device_bytes."""
    one = o.device_bytes(type_idx, tp, P, s, L, 1, b)
    if P - s >= 2:
        act_l = o.device_bytes(type_idx, tp, P, s, L, 2, b) - one
        return one - act_l, act_l // L
    # last stage holds one micro-batch whatever m: compare with a deeper stage shape
    return None, None


@pytest.mark.parametrize("name,n", [("llama2_7b", 2), ("gpt3", 3), ("mixtral", 4), ("llama3_70b", 5)])
def test_static_bytes_are_public_param_count_times_18(oracle_mod, name, n):
    """One stage holding the whole model at t = 1: static bytes = parameters x
    (2 B weights + 4 B fp32 gradients (A7) + 12 B Adam state) = 18 B/param."""
    cfg = H.get(n)
    o = oracle_mod.Oracle(cfg)
    L = cfg["model"]["layers"]
    # P = 2 shape so in-flight depth can be varied; s = 0 owns the embedding,
    # so add the head by evaluating the P = 1 stage and removing its activations
    stat0, act_l = _parts(o, 0, 1, 2, 0, L, 1)
    whole = o.device_bytes(0, 1, 1, 0, L, 1, 1) - L * act_l  # P = 1: emb + head + all layers
    want = json.load(open(os.path.join(GOLD, "paper_examples.json")))["public_param_counts"]["billions"][name] * 1e9
    assert abs(whole / 18 - want) / want < 0.01, whole / 18
    assert whole % 18 == 0 and stat0 % 18 == 0


@pytest.mark.parametrize("b", [1, 2, 4])
def test_activation_bytes_34sbh_and_tp_form(oracle_mod, b):
    """t = 1: 34 s b h bytes per layer and micro-batch; t: s b h (10 + 24/t)."""
    cfg = H.get(2)
    o = oracle_mod.Oracle(cfg)
    m = cfg["model"]
    sbh = m["seq"] * b * m["hidden"]
    _, act1 = _parts(o, 1, 1, 4, 0, 8, b)
    assert act1 == 34 * sbh
    for t in (2, 4, 8):
        _, act_t = _parts(o, 1, t, 4, 0, 8, b)
        assert act_t == sbh * 10 + (sbh * 24 + t - 1) // t


def _inflight_from_schedule(P, s, m):
    """Peak #micro-batches whose forward is done and backward is not, on stage
    s, walking its 1F1B op order (C.7) -- counted, not a formula."""
    w = min(P - 1 - s, m)
    order = [("F", j) for j in range(w)]
    for i in range(m - w):
        order += [("F", w + i), ("B", i)]
    order += [("B", j) for j in range(m - w, m)]
    live = peak = 0
    for op, _ in order:
        live += 1 if op == "F" else -1
        peak = max(peak, live)
    return peak


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_inflight_depth_is_1f1b_peak(oracle_mod, P):
    cfg = H.get(2)
    o = oracle_mod.Oracle(cfg)
    l, b = 3, 1
    act_l = None
    for s in range(P):
        for m in (1, 2, 3, P, P + 5):
            need = o.device_bytes(1, 1, P, s, l, m, b)
            base = o.device_bytes(1, 1, P, s, l, 0, b)  # m = 0: static only
            if act_l is None and need > base:
                act_l = (need - base) // (l * _inflight_from_schedule(P, s, m))
            assert need - base == l * act_l * _inflight_from_schedule(P, s, m), (P, s, m)


def test_spec_gpt13b_on_one_40gb_gpu_is_infeasible(oracle_mod):
    """GPT-13B entirely on one 40 GB GPU does not fit (13e9 x 2 B
    of weights alone exceed 40 GB); on a 1 TB device it does."""
    cl = {"frame_bytes": 9200, "rail_alpha_ns": 0, "rail_gbps": 200.0,
          "types": [H.presets.a100_sxm(1)], "nodes": [0]}
    md = dict(layers=40, hidden=5120, heads=40, kv_heads=40, ffn=20480, mlp_mats=2, seq=2048, vocab=50257,
              tied=1, moe_experts=1, moe_topk=1, bpe_act=2, bpe_grad=4, global_batch=1)
    se = dict(bset=[1], tpset=[[1]], pset=[1], homo=1, mixed=0, use_all=1, r_layer=0, pmax_perturb=0, r_batch=0)
    cfg = {"name": "gpt13b-1xA100", "cluster": cl, "model": md, "search": se}
    assert oracle_mod.Oracle(cfg).space_size() == 1
    assert oracle_mod.Oracle(cfg).eval(0) > 0
    assert oracle_mod.Oracle(H.with_mem_check(cfg)).eval(0) == -3
    assert oracle_mod.Oracle(H.with_mem_check(cfg, [1 << 40])).eval(0) > 0


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_mem_check_only_adds_infeasible_codes(oracle_mod, n):
    """Times of feasible candidates are unchanged; -1 / -2 keep precedence; with
    huge capacities nothing is pruned; more capacity never prunes more."""
    cfg = H.get(n)
    o = oracle_mod.Oracle(cfg)
    N = o.space_size()
    idx = H.sample_indices(N, 600, seed=H.PARITY_SEED + n)
    base = o.eval_many(idx)
    mc = oracle_mod.Oracle(H.with_mem_check(cfg)).eval_many(idx)
    keep = mc != -3
    assert np.array_equal(base[keep], mc[keep])
    assert np.all(base[~keep] >= 0)
    big = oracle_mod.Oracle(H.with_mem_check(cfg, [1 << 50] * len(cfg["cluster"]["types"]))).eval_many(idx)
    assert np.array_equal(big, base)
    caps = [t["mem_bytes"] * 2 for t in cfg["cluster"]["types"]]
    mc2 = oracle_mod.Oracle(H.with_mem_check(cfg, caps)).eval_many(idx)
    assert np.all((mc2 == -3) <= (mc == -3))


@pytest.mark.parametrize("seed", range(6))
def test_tiny_memcheck_matches_per_device_enumeration(oracle_mod, seed):
    """Brute force over a tiny space: -3 exactly when some device of some
    replica of some stage (from the oracle's own plan) exceeds its type's
    capacity -- capacities drawn around the median need so both outcomes occur."""
    cfg = H.tiny_random(seed)
    o = oracle_mod.Oracle(cfg)
    N = o.space_size()
    needs = []
    plans = [o.describe(i) for i in range(N)]
    for d in plans:
        if d["status"] != 0:
            continue
        for c in d["classes"]:
            P = len(c["stages"])
            for s, (ty, tp) in enumerate(c["stages"]):
                needs.append(o.device_bytes(ty, tp, P, s, c["layers"][s], max(c["mb"]), d["b"]))
    cap = int(np.median(needs))
    mc = oracle_mod.Oracle(H.with_mem_check(cfg, [cap] * len(cfg["cluster"]["types"])))
    got = mc.eval_many(first=0, n=N)
    base = o.eval_many(first=0, n=N)
    for i, d in enumerate(plans):
        if d["status"] != 0:
            assert got[i] == d["status"]
            continue
        over = any(o.device_bytes(ty, tp, len(c["stages"]), s, c["layers"][s], mb, d["b"]) > cap
                   for c in d["classes"] for mb in c["mb"] for s, (ty, tp) in enumerate(c["stages"]))
        assert (got[i] == -3) == over, i
        if not over:
            assert got[i] == base[i]
