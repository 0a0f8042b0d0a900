"""Pins of the oracle's f3 row (DESIGN.md F.1): the
flow-level contention re-simulation of a candidate's gradient sync.

Fixed against things other than the oracle's code (SPEC.md:358-373 and its
acceptance criteria 5 and 6):
* max-min fairness: an independent exact water-filling (fractions.Fraction,
  raise every unfrozen flow's rate together until a link saturates or a flow
  reaches its own cap) on 200 random instances (<= 10 flows, <= 6 links),
  within 1e-9 relative; capacity conservation; the bottleneck property that
  characterises max-min fairness;
* the fluid engine: a single flow's FCT = alpha + ceil(bytes / beta) (the
  alpha-beta tau) on 100 random scenarios; a zero-byte flow -> FCT = alpha;
  two identical flows on one link drain at half rate; a staggered pair by a
  hand-computed piecewise schedule;
* whole candidates: the alpha-beta schedule of the steps equals the C.8 sync
  the oracle's main evaluation produces (T_iter - T0); contention only ever
  slows (sync_flow >= sync_ab); uncontended candidates reduce exactly to the
  alpha-beta values, flow by flow; the flow count is the step structure's.
"""
import math
import random
from fractions import Fraction

import numpy as np
import pytest

import hsim_inputs as H


def waterfill(linkcap, flows, caps):
    """Exact max-min by water-filling: all unfrozen flows rise together."""
    n = len(flows)
    rate = [Fraction(0)] * n
    frozen = [False] * n
    cap = [Fraction(c) for c in linkcap]
    fc = [Fraction(c) for c in caps]
    while not all(frozen):
        # largest common increment before some link saturates or a flow caps
        inc = None
        for e in range(len(cap)):
            users = [f for f in range(n) if e in flows[f] and not frozen[f]]
            if users:
                used = sum(rate[f] for f in range(n) if e in flows[f])
                x = (cap[e] - used) / len(users)
                inc = x if inc is None else min(inc, x)
        for f in range(n):
            if not frozen[f]:
                x = fc[f] - rate[f]
                inc = x if inc is None else min(inc, x)
        for f in range(n):
            if not frozen[f]:
                rate[f] += inc
        for f in range(n):
            if frozen[f]:
                continue
            if rate[f] == fc[f]:
                frozen[f] = True
            for e in flows[f]:
                if sum(rate[g] for g in range(n) if e in flows[g]) == cap[e]:
                    frozen[f] = True
    return rate


def test_maxmin_matches_waterfilling(oracle_mod):
    rng = random.Random(2508)
    for _ in range(200):
        nl = rng.randint(1, 6)
        nf = rng.randint(1, 10)
        linkcap = [rng.choice([12.5, 25.0, 32.0, 50.0, 64.0, 300.0, 450.0, rng.uniform(1, 500)]) for _ in range(nl)]
        flows = [sorted(rng.sample(range(nl), rng.randint(1, nl))) for _ in range(nf)]
        caps = [rng.choice([25.0, 300.0, 1e6, rng.uniform(1, 400)]) for _ in range(nf)]
        got = oracle_mod.maxmin(linkcap, flows, caps)
        want = waterfill(linkcap, flows, caps)
        for f in range(nf):
            assert abs(got[f] - float(want[f])) <= 1e-9 * float(want[f]), (f, got, want)
        # capacity conservation and the bottleneck property
        for e in range(nl):
            assert sum(got[f] for f in range(nf) if e in flows[f]) <= linkcap[e] * (1 + 1e-12)
        for f in range(nf):
            if abs(got[f] - caps[f]) <= 1e-9 * caps[f]:
                continue
            assert any(sum(got[g] for g in range(nf) if e in flows[g]) >= linkcap[e] * (1 - 1e-9)
                       and got[f] >= max(got[g] for g in range(nf) if e in flows[g]) * (1 - 1e-9)
                       for e in flows[f]), f


def test_two_flows_share_one_link(oracle_mod):
    # two identical flows on one 200 Gbps (25 B/ns) link -> 12.5 each
    assert list(oracle_mod.maxmin([25.0], [[0], [0]], [1e9, 1e9])) == [12.5, 12.5]


@pytest.fixture(scope="module")
def o2(oracle_mod):
    return oracle_mod.Oracle(H.get(2))


def test_single_flow_closed_form(o2):
    """SPEC acceptance 5: 100 random single-flow scenarios: completion =
    arrival + alpha + ceil(bytes / min(cap, links))."""
    rng = random.Random(7)
    for _ in range(100):
        nl = rng.randint(1, 6)
        linkcap = [rng.uniform(5, 500) for _ in range(nl)]
        links = sorted(rng.sample(range(nl), rng.randint(1, nl)))
        f = dict(links=links, arrive=rng.randint(0, 10 ** 6), bytes=rng.randint(0, 10 ** 9),
                 alpha=rng.randint(0, 2000), cap=rng.uniform(5, 500))
        beta = min([f["cap"]] + [linkcap[e] for e in links])
        drain = math.ceil(f["bytes"] / beta) if f["bytes"] else 0
        assert o2.flow_sim(linkcap, [f])[0] == f["arrive"] + f["alpha"] + drain


def test_identical_and_staggered_pairs(o2):
    cap = 25.0
    a = dict(links=[0], arrive=0, bytes=1000, alpha=100, cap=1e9)
    b = dict(links=[0], arrive=0, bytes=1000, alpha=100, cap=1e9)
    # both at 12.5 B/ns: 1000 / 12.5 = 80 ns
    assert list(o2.flow_sim([cap], [a, b])) == [180, 180]
    # b arrives at 20: a alone drains 500 B (20 ns at 25), then both at 12.5:
    # a's 500 B take 40 ns (t = 60); b has 500 left at 60, alone at 25: 20 ns
    b["arrive"] = 20
    assert list(o2.flow_sim([cap], [a, b])) == [60 + 100, 80 + 100]
    # a zero-byte flow completes after its latency alone
    z = dict(links=[0], arrive=5, bytes=0, alpha=100, cap=1e9)
    assert o2.flow_sim([cap], [z])[0] == 105


def _expected_flows(o, i):
    """Flow count from the step structure: per segment, one flow per TP-ring
    edge of every group with tp != t* (if any) plus 2(D-1) ring steps of t* x D
    flows."""
    d = o.describe(i)
    D = sum(c["D"] for c in d["classes"])
    if D == 1:
        return 0
    n = 0
    for sg in o.segments(i):
        rs = 0
        for c in d["classes"]:
            acc, s = 0, 0
            for k, l in enumerate(c["layers"]):
                if acc <= sg["a"]:
                    s = k
                acc += l
            tp = c["stages"][s][1]
            if tp != sg["tstar"]:
                rs += c["D"] * tp
        n += rs + 2 * (D - 1) * sg["tstar"] * D
    return n


@pytest.mark.parametrize("cfg", ["tiny-101", "tiny-105", "tiny-110", "c2", "c4"])
def test_candidates_flow_vs_alpha_beta(oracle_mod, cfg):
    cf = H.tiny_random(int(cfg[5:])) if cfg.startswith("tiny") else H.get(int(cfg[1:]))
    o = oracle_mod.Oracle(cf)
    idx = H.sample_indices(o.space_size(), 60, seed=11)
    seen = 0
    for i in idx:
        r = o.flow_resim(int(i), fct_cap=1 << 20)
        if r["status"]:
            assert r["status"] in (-1, -2)
            continue
        seen += 1
        assert r["sync_ab"] == r["T_iter"] - r["T0"]
        assert r["sync_flow"] >= r["sync_ab"]
        assert r["n_flows"] == _expected_flows(o, int(i))
        if r["sync_flow"] == r["sync_ab"] and r["n_flows"]:
            assert r["fct"].min() > 0
    assert seen > 0


def test_uncontended_candidate_flow_by_flow(oracle_mod):
    """One class, P = 1, tp = 1, D = 2 on one NVSwitch node: every step is the
    two flows 0 -> 1 and 1 -> 0 on disjoint ports, so each FCT is the
    alpha-beta tau of the chunk and the sync lasts 2 (D - 1) taus."""
    cfg = H.with_changes(H.get(2))
    o = oracle_mod.Oracle(cfg)
    pre = o.template_prefix()
    for k in range(len(pre) - 1):
        d = o.describe(int(pre[k]))
        if len(d["classes"]) == 1 and d["classes"][0]["D"] == 2 and d["classes"][0]["stages"] == [[0, 1]]:
            i = int(pre[k])
            break
    r = o.flow_resim(i, fct_cap=64)
    S = o.segment_bytes(cfg["model"]["layers"], 1, 1)
    alpha, beta = o.link(0, 0, 0, 1)
    t = alpha + math.ceil(-(-S // 2) / beta)
    assert r["n_flows"] == 4 and list(r["fct"]) == [t] * 4
    assert r["sync_flow"] == r["sync_ab"] == 2 * t


def test_contention_example(oracle_mod):
    """A candidate whose ring crosses nodes through a peer GPU's NIC (Fig 2
    case (c)) while that GPU's own flow uses the same NIC: the flow level is
    strictly slower.  Found by search over config 4 samples (the property,
    not a stored value)."""
    o = oracle_mod.Oracle(H.get(4))
    idx = H.sample_indices(o.space_size(), 400, seed=5)
    slower = [int(i) for i in idx if (lambda r: r["status"] == 0 and r["sync_flow"] > r["sync_ab"])(o.flow_resim(int(i)))]
    assert slower
