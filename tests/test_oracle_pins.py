"""Pins of the CPU oracle against things other than itself (task rule ③).

Each test names what fixes the expected value: a number printed in the paper
(tests/golden/*.json, cited), a closed form, an invariant, an independent
algorithm (DAG longest path vs the event engine), or brute-force counting.
CPU only (``-m "not gpu"``).
"""
import itertools
import json
import math
import os
import random

import numpy as np
import pytest

import hsim_inputs as H

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# --------------------------------------------------------------------------
# Links: Table 4 + the delay formula
# --------------------------------------------------------------------------
def test_table4_delays(oracle_mod):
    g = gold("table4_delays.json")
    for row in g["rows"]:
        d = oracle_mod.hop_delay_exact(row["gbps"], row["bidir"], g["frame_bytes"])
        # printed values are truncated to 2 decimals
        assert row["printed_ns"] <= d < row["printed_ns"] + 0.01, row


def test_table4_needs_bidirectional_halving(oracle_mod):
    # Only the bidirectional reading reproduces 30.66 (DESIGN A9): reading
    # 4800 as uni-directional would give 15.33 ns.
    assert abs(oracle_mod.hop_delay_exact(4800, False) - 15.333) < 1e-2
    assert abs(oracle_mod.hop_delay_exact(4800, True) - 30.666) < 1e-2


def test_rail_path_composition(oracle_mod):
    """Fig 2 case (b) on config 1 (A100 node0 -> H100 node1, same rank):
    GPU->PCIe x2 (2*ceil(287.5)) + NIC 368 + rail 0 + NIC 368 + PCIe x2
    (2*ceil(143.75)); beta = slowest hop = NIC 200 Gbps = 25 B/ns.  Intra-node
    NVSwitch pair = 2 NVLink hops = 2*ceil(30.67); 4800/2/8 = 300 B/ns.
    Case (c) prepends the source node's intra hop."""
    o = oracle_mod.Oracle(H.get(1))
    assert o.link(0, 0, 1, 0) == (2 * 288 + 368 + 0 + 368 + 2 * 144, 25.0)
    assert o.link(0, 0, 0, 1) == (2 * 31, 300.0)
    assert o.link(1, 1, 1, 0) == (2 * 21, 450.0)
    assert o.link(0, 0, 1, 1) == (62 + 1600, 25.0)


# --------------------------------------------------------------------------
# Ring all-reduce closed forms (BASELINE north_star)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("n", [2, 3, 4, 5, 8])
def test_ring_allreduce_uniform_closed_form(oracle_mod, n):
    # alpha = 0, n | S, beta | S/n: T = 2(n-1)/n * S/B
    B = 25
    S = n * B * 1000
    tau = S // n // B
    assert oracle_mod.ring_sim([tau] * n, 2 * (n - 1)) == 2 * (n - 1) * S // (n * B)


def test_ring_per_rank_volume_spec_example():
    # n=4, S=4096 B -> each rank transmits 2*3/4*4096 = 6144 B
    n, S = 4, 4096
    assert 2 * (n - 1) * (S // n) == 6144


def test_ring_heterogeneous_is_steps_times_slowest(oracle_mod):
    # Async ring with send(r,k).start = max(send(r,k-1).end, send(r-1,k-1).end):
    # the longest path stays on the slowest edge for every step.
    rng = random.Random(1)
    for _ in range(300):
        n = rng.randint(1, 9)
        taus = [rng.randint(0, 10 ** 6) for _ in range(n)]
        steps = rng.randint(0, 2 * n)
        assert oracle_mod.ring_sim(taus, steps) == steps * max(taus)


# --------------------------------------------------------------------------
# 1F1B (DESIGN C.7): closed form and an independent DAG longest path
# --------------------------------------------------------------------------
@pytest.mark.parametrize("P,m", [(p, m) for p in range(1, 7) for m in range(1, 9)])
def test_1f1b_uniform_closed_form(oracle_mod, P, m):
    f, g = 1000, 2000
    T = oracle_mod.pipeline([f] * P, [g] * P, [0] * (P - 1), m)
    assert T == (m + P - 1) * (f + g)
    bubble = 1 - m * (f + g) / T
    assert abs(bubble - (P - 1) / (m + P - 1)) < 1e-12


def _op_order(P, s, m):
    w = min(P - 1 - s, m)
    o = [("F", j) for j in range(w)]
    for i in range(m - w):
        o += [("F", w + i), ("B", i)]
    o += [("B", j) for j in range(m - w, m)]
    return o


def _dag_longest_path(f, g, c, m):
    """Explicit DAG of the non-interleaved 1F1B schedule, longest path by
    memoised recursion over predecessors (not an event simulation)."""
    P = len(f)
    preds = {}
    for s in range(P):
        order = _op_order(P, s, m)
        for k, op in enumerate(order):
            preds.setdefault((s,) + op, [])
            if k:
                preds[(s,) + op].append(((s,) + order[k - 1], 0))
    for s in range(P):
        for j in range(m):
            if s > 0:
                preds[(s, "F", j)].append(((s - 1, "F", j), c[s - 1]))
            if s < P - 1:
                preds[(s, "B", j)].append(((s + 1, "B", j), c[s]))
            else:
                preds[(s, "B", j)].append(((s, "F", j), 0))
    memo = {}

    def end(v):
        if v not in memo:
            st = max([end(u) + d for u, d in preds[v]], default=0)
            memo[v] = st + (f[v[0]] if v[1] == "F" else g[v[0]])
        return memo[v]
    return max(end(v) for v in preds)


def test_1f1b_matches_dag_longest_path(oracle_mod):
    rng = random.Random(7)
    for _ in range(250):
        P = rng.randint(1, 7)
        m = rng.randint(1, 10)
        f = [rng.randint(1, 5000) for _ in range(P)]
        g = [rng.randint(1, 9000) for _ in range(P)]
        c = [rng.randint(0, 4000) for _ in range(P - 1)]
        assert oracle_mod.pipeline(f, g, c, m) == _dag_longest_path(f, g, c, m)


def test_1f1b_monotone_in_microbatches(oracle_mod):
    # Exactness of "simulate the max-m replica" (DESIGN A13) rests on this.
    rng = random.Random(11)
    for _ in range(200):
        P = rng.randint(1, 6)
        f = [rng.randint(1, 5000) for _ in range(P)]
        g = [rng.randint(1, 9000) for _ in range(P)]
        c = [rng.randint(0, 4000) for _ in range(P - 1)]
        ts = [oracle_mod.pipeline(f, g, c, m) for m in range(1, 12)]
        assert all(a <= b for a, b in zip(ts, ts[1:]))


# --------------------------------------------------------------------------
# Partition (Fig 3)
# --------------------------------------------------------------------------
def test_fig3_batch_shares(oracle_mod):
    g = gold("paper_examples.json")["fig3_batch_split"]
    assert list(oracle_mod.hamilton(g["n"], g["weights"])) == g["expected"]


def test_hamilton_uniform_and_conservation(oracle_mod):
    rng = random.Random(3)
    assert list(oracle_mod.hamilton(10, [5, 5, 5, 5])) == [3, 3, 2, 2]   # ties -> lower index
    for _ in range(200):
        k = rng.randint(1, 8)
        w = [rng.randint(1, 1 << 40) for _ in range(k)]
        n = rng.randint(0, 3000)
        q = oracle_mod.hamilton(n, w)
        assert q.sum() == n
        for i in range(k):  # quota property of largest remainder
            exact = n * w[i] / sum(w)
            assert math.floor(exact) <= q[i] <= math.floor(exact) + 1


def _single_type(cfg, t):
    c = H.with_changes(cfg)
    cl = c["cluster"]
    cl["types"] = [cl["types"][t]]
    cl["nodes"] = [0 for n in cl["nodes"] if n == t]
    c["search"]["tpset"] = [c["search"]["tpset"][t]]
    c["search"]["mixed"] = 0
    c["search"]["r_layer"] = 0
    c["search"]["r_batch"] = 0
    return c


def test_homogeneous_cluster_gives_uniform_split(oracle_mod):
    """BASELINE north_star: homogeneous clusters reduce to the uniform partition."""
    o = oracle_mod.Oracle(_single_type(H.get(2), 1))
    pre = o.template_prefix()
    for k in range(0, len(pre) - 1, 7):
        d = o.describe(int(pre[k]))
        for c in d["classes"]:
            L, P = 32, len(c["layers"])
            base = L // P
            assert c["layers"] == [base + (1 if s < L - base * P else 0) for s in range(P)]
            mb = c["mb"]
            assert max(mb) - min(mb) <= 1 and mb == sorted(mb, reverse=True)


def test_faster_type_gets_more_layers(oracle_mod):
    """PAPER.md:186 (1): more layers on high-compute GPUs.  Config 1: the H100
    stage gets more layers than the A100 stage."""
    d = oracle_mod.Oracle(H.get(1)).describe(0)
    (cls,) = d["classes"]
    assert cls["stages"] == [[0, 1], [1, 1]]
    assert cls["layers"][1] > cls["layers"][0] and sum(cls["layers"]) == 12
    assert cls["mb"] == [4, 4]          # "DP=2 PP=2, 4 micro-batches" (BASELINE config 1)


# --------------------------------------------------------------------------
# FLOPs / bytes (DESIGN C.5, A3): brute-force matmul dimension counting
# --------------------------------------------------------------------------
def _matmul_flops(model, b):
    s, h = model["seq"], model["hidden"]
    hkv = model["kv_heads"] * h // model["heads"]
    T = b * s
    mm = lambda m, k, n: 2 * m * k * n  # noqa: E731
    attn = mm(T, h, h) + 2 * mm(T, h, hkv) + mm(T, h, h)            # Q, K, V, O projections
    d = h // model["heads"]
    attn += b * model["heads"] * (mm(s, d, s) + mm(s, s, d))         # scores and weighted values
    mlp = model["mlp_mats"] * mm(T, h, model["ffn"])
    head = mm(T, h, model["vocab"])
    return attn, mlp, head


@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_layer_flops_by_dimension_counting(oracle_mod, n):
    cfg = H.get(n)
    o = oracle_mod.Oracle(cfg)
    for b in cfg["search"]["bset"]:
        attn, mlp, head = _matmul_flops(cfg["model"], b)
        assert o.op(0, "attn", 0, 1, b)[0] == attn
        assert o.op(0, "mlp", 0, 1, b)[0] == mlp
        assert o.op(0, "head", 0, 1, b)[0] == head
        assert o.op(0, "emb", 0, 1, b)[0] == 0
        for tp in (2, 4):  # work conservation across a TP group
            for k in ("attn", "mlp", "head"):
                assert o.op(0, k, 0, tp, b)[0] * tp == o.op(0, k, 0, 1, b)[0]
            assert o.op(0, "mlp", 1, tp, b)[0] == 2 * o.op(0, "mlp", 0, tp, b)[0]


def test_moe_flops_topk_times_dense(oracle_mod):
    # top-2 MoE = 2x a single-expert MLP at equal ffn
    o = oracle_mod.Oracle(H.get(4))
    assert o.op(0, "moe", 0, 1, 1)[0] == 2 * o.op(0, "mlp", 0, 1, 1)[0]


def test_roofline_duration(oracle_mod):
    o = oracle_mod.Oracle(H.get(2))
    for t in (0, 1):
        ty = H.get(2)["cluster"]["types"][t]
        for kind in ("attn", "mlp", "emb", "head"):
            for bwd in (0, 1):
                fl, by, d = o.op(t, kind, bwd, 2, 2)
                rf = ty["peak_flop_per_ns"] * 0.5
                assert d == max(math.ceil(fl / rf), math.ceil(by / ty["hbm_bytes_per_ns"]))


# --------------------------------------------------------------------------
# Table 1 and parameter counts
# --------------------------------------------------------------------------
def _cfg_with_model(model):
    c = H.get(2)
    c["model"].update(model)
    return c


def test_table1_dp_payload_and_message_size(oracle_mod):
    g = gold("paper_examples.json")["table1_llama2_70b"]
    o = oracle_mod.Oracle(_cfg_with_model(g["model"]))
    per_stage_layers = g["model"]["layers"] // g["pp"]
    mid = o.segment_bytes(per_stage_layers, 0, 0) / g["tp"]
    first = o.segment_bytes(per_stage_layers, 1, 0) / g["tp"]
    # 4.4 GB per collective (printed, rounded): fp32 main grads (A7)
    assert abs(mid / 1e9 - g["dp_bytes_printed_gb"]) / g["dp_bytes_printed_gb"] < 0.05
    assert abs(first / 1e9 - g["dp_bytes_printed_gb"]) / g["dp_bytes_printed_gb"] < 0.05
    # "67KB" TP/PP message = b*s*h*2 B = 67.1 MB (A5)
    assert round(o.act_bytes(1) / 1e6) == g["act_bytes_printed_mb"]


@pytest.mark.parametrize("name,n,override", [
    ("gpt2s", 1, None), ("llama2_7b", 2, None), ("gpt3", 3, None), ("mixtral", 4, None),
    ("llama3_70b", 5, None),
    ("llama2_70b", 2, "table1"),
])
def test_param_counts(oracle_mod, name, n, override):
    g = gold("paper_examples.json")
    cfg = H.get(n) if override is None else _cfg_with_model(g["table1_llama2_70b"]["model"])
    o = oracle_mod.Oracle(cfg)
    L = cfg["model"]["layers"]
    params = o.segment_bytes(L, 1, 1) / cfg["model"]["bpe_grad"]
    want = g["public_param_counts"]["billions"][name]
    assert abs(params / 1e9 - want) / want < 0.01, params


# --------------------------------------------------------------------------
# Whole-candidate closed forms and invariants
# --------------------------------------------------------------------------
def _find(o, pred, limit=None):
    pre = o.template_prefix()
    for k in range(len(pre) - 1):
        d = o.describe(int(pre[k]))
        if pred(d):
            return int(pre[k]), d
    raise AssertionError("no such template")


def test_single_device_group_closed_form(oracle_mod):
    """D=1, P=1, tp=1: no communication; T = M*(f+g) with f = L*(attn_f+mlp_f)
    + emb_f + head_f (1F1B with one stage is sequential)."""
    cfg = _single_type(H.get(2), 0)
    o = oracle_mod.Oracle(cfg)
    i, d = _find(o, lambda d: len(d["classes"]) == 1 and d["classes"][0]["D"] == 1
                 and d["classes"][0]["stages"] == [[0, 1]])
    b = d["b"]
    L = cfg["model"]["layers"]
    f = L * (o.op(0, "attn", 0, 1, b)[2] + o.op(0, "mlp", 0, 1, b)[2]) + o.op(0, "emb", 0, 1, b)[2] + o.op(0, "head", 0, 1, b)[2]
    g = L * (o.op(0, "attn", 1, 1, b)[2] + o.op(0, "mlp", 1, 1, b)[2]) + o.op(0, "emb", 1, 1, b)[2] + o.op(0, "head", 1, 1, b)[2]
    M = cfg["model"]["global_batch"] // b
    assert o.eval(i) == M * (f + g)


def test_two_replica_sync_closed_form(oracle_mod):
    """D=2, P=1, tp=1 on one NVSwitch node: T = m*(f+g) + 2(D-1)*tau(chunk),
    chunk = ceil(S/D), tau = alpha + ceil(chunk/beta) (one segment, no reshard)."""
    cfg = _single_type(H.get(2), 0)
    o = oracle_mod.Oracle(cfg)
    i, d = _find(o, lambda d: len(d["classes"]) == 1 and d["classes"][0]["D"] == 2
                 and d["classes"][0]["stages"] == [[0, 1]])
    b = d["b"]
    L = cfg["model"]["layers"]
    f = L * (o.op(0, "attn", 0, 1, b)[2] + o.op(0, "mlp", 0, 1, b)[2]) + o.op(0, "emb", 0, 1, b)[2] + o.op(0, "head", 0, 1, b)[2]
    g = L * (o.op(0, "attn", 1, 1, b)[2] + o.op(0, "mlp", 1, 1, b)[2]) + o.op(0, "emb", 1, 1, b)[2] + o.op(0, "head", 1, 1, b)[2]
    m = max(d["classes"][0]["mb"])
    S = o.segment_bytes(L, 1, 1)
    chunk = -(-S // 2)
    alpha, beta = o.link(0, 0, 0, 1)
    assert (alpha, beta) == (62, 300.0)
    assert o.eval(i) == m * (f + g) + 2 * (alpha + math.ceil(chunk / beta))


def _bandwidth_scaled(cfg, factor):
    c = H.with_changes(cfg)
    for t in c["cluster"]["types"]:
        for kind in t["link_kinds"]:
            for hop in kind:
                hop["gbps"] *= factor
        for hop in t["gpu_nic"]:
            hop["gbps"] *= factor
        t["nic_gbps"] *= factor
    c["cluster"]["rail_gbps"] *= factor
    return c


@pytest.mark.parametrize("seed", range(4))
def test_monotone_in_bandwidth_and_latency(oracle_mod, seed):
    """BASELINE north_star: time is monotone in link bandwidth (and latency)."""
    cfg = H.tiny_random(100 + seed)
    base = oracle_mod.Oracle(cfg)
    N = base.space_size()
    idx = H.sample_indices(N, 300, seed=seed)
    t0 = base.eval_many(idx, threads=4)
    faster = oracle_mod.Oracle(_bandwidth_scaled(cfg, 1.5)).eval_many(idx, threads=4)
    slower_lat = oracle_mod.Oracle(H.with_changes(cfg, cluster__frame_bytes=20000)).eval_many(idx, threads=4)
    ok = t0 >= 0
    assert np.all((faster >= 0) == ok)
    assert np.all(faster[ok] <= t0[ok])
    assert np.all(slower_lat[ok] >= t0[ok])


def test_deterministic(oracle_mod):
    o = oracle_mod.Oracle(H.get(4))
    idx = H.sample_indices(o.space_size(), 200)
    a = o.eval_many(idx, threads=3)
    b = o.eval_many(idx, threads=1)
    assert np.array_equal(a, b)


def test_space_sizes_frozen(oracle_mod):
    """The generator's post-filter N per config (SURVEY.md §8(a) estimates:
    1, 8.7e5, 6.2e7, 1.1e7, 1.2e9) frozen so any grammar change is loud."""
    want = {1: 1, 2: 873192, 3: 62232390, 4: 11122050, 5: 1203928800}
    for n, N in want.items():
        assert oracle_mod.Oracle(H.get(n)).space_size() == N


def test_invalid_codes_are_reported(oracle_mod):
    """Layer deltas that empty a stage give -1; M < D is filtered out of the
    space, batch deltas that empty a replica give -2."""
    o = oracle_mod.Oracle(H.get(2))
    r = o.eval_many(first=0, n=20000, threads=4)
    assert set(np.unique(r[r < 0])) <= {-1, -2}
    assert (r >= 0).sum() > 0
