"""Pins of the overlapped gradient-sync row (DESIGN.md
S.1) in the CPU oracle: no barrier -- a gradient segment is synchronised as
soon as every stage group holding its layers has ended its last backward
(Table 1: DP sync is exposed in the backward pass),
segments issued in descending layer order, FIFO per group.  Pinned by a
two-stage closed form built from independent pieces (per-stage ends from an
explicit DAG longest path, ring all-reduce closed form over the oracle's link
table), the single-stage reduction to C.8, and invariants.  CPU only."""
import math

import numpy as np
import pytest

import hsim_inputs as H
from test_oracle_pins import _op_order, _single_type


def _dag_stage_ends(f, g, c, m):
    """End of the last op (the last backward) of every stage of a non-
    interleaved 1F1B pipeline: explicit DAG, longest path by recursion."""
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

    def end(root):  # longest path to the end of `root`, iterative post-order DFS
        stack = [root]
        while stack:
            v = stack[-1]
            todo = [u for u, _ in preds[v] if u not in memo]
            if todo:
                stack.extend(todo)
                continue
            stack.pop()
            if v not in memo:
                st = max([memo[u] + d for u, d in preds[v]], default=0)
                memo[v] = st + (f[v[0]] if v[1] == "F" else g[v[0]])
        return memo[root]
    return [end((s,) + _op_order(P, s, m)[-1]) for s in range(P)]


def _find_all(o, pred, limit=40):
    pre = o.template_prefix()
    out = []
    for k in range(len(pre) - 1):
        d = o.describe(int(pre[k]))
        if pred(d):
            out.append((int(pre[k]), d))
            if len(out) >= limit:
                break
    return out


def test_overlap_two_stage_two_replica_closed_form(oracle_mod):
    """One class, P = 2, D = 2, tp = 1 (one device type):
    T = max(T0 + AR_0, ready_1 + AR_1) with ready_s = max over replicas of the
    end of stage s's last backward, AR_j = 2 (D - 1) max_edge tau(ceil(S_j / D))."""
    cfg = _single_type(H.get(2), 1)
    o = oracle_mod.Oracle(cfg)
    ov = oracle_mod.Oracle(H.with_sync_overlap(cfg))
    found = _find_all(o, lambda d: d["status"] == 0 and len(d["classes"]) == 1 and d["classes"][0]["D"] == 2
                      and d["classes"][0]["stages"] == [[0, 1], [0, 1]], limit=6)
    assert found
    L = cfg["model"]["layers"]
    for i, d in found:
        b, cls = d["b"], d["classes"][0]
        A = o.act_bytes(b)
        ends = []
        for r in range(2):
            l = cls["layers"]
            f = [l[s] * (o.op(0, "attn", 0, 1, b)[2] + o.op(0, "mlp", 0, 1, b)[2]) for s in range(2)]
            g = [l[s] * (o.op(0, "attn", 1, 1, b)[2] + o.op(0, "mlp", 1, 1, b)[2]) for s in range(2)]
            f[0] += o.op(0, "emb", 0, 1, b)[2]
            g[0] += o.op(0, "emb", 1, 1, b)[2]
            f[1] += o.op(0, "head", 0, 1, b)[2]
            g[1] += o.op(0, "head", 1, 1, b)[2]
            (n1, r1), (n2, r2) = cls["place"][r]
            a, be = o.link(n1, r1, n2, r2)
            c = [a + math.ceil(A / be)]
            ends.append(_dag_stage_ends(f, g, c, cls["mb"][r]))
        T0 = max(e[0] for e in ends)
        ready1 = max(e[1] for e in ends)
        S = [o.segment_bytes(cls["layers"][0], 1, 0), o.segment_bytes(cls["layers"][1], 0, 1)]
        AR = []
        for s in range(2):
            (na, ra), (nb, rb) = cls["place"][0][s], cls["place"][1][s]
            chunk = -(-S[s] // 2)
            taus = []
            for (x1, y1, x2, y2) in ((na, ra, nb, rb), (nb, rb, na, ra)):
                a, be = o.link(x1, y1, x2, y2)
                taus.append(a + math.ceil(chunk / be))
            AR.append(2 * max(taus))
        assert ov.eval(i) == max(T0 + AR[0], ready1 + AR[1]), i
        # the barrier schedule (C.8) of the same candidate: both from T0
        assert o.eval(i) == T0 + max(AR)


@pytest.mark.parametrize("n", [2, 4])
def test_overlap_equals_barrier_for_single_stage_pipelines(oracle_mod, n):
    """Every class with P = 1: each group's last backward ends at its
    pipeline's end, all segments share every group -> same chain as C.8."""
    cfg = H.get(n)
    o, ov = oracle_mod.Oracle(cfg), oracle_mod.Oracle(H.with_sync_overlap(cfg))
    found = _find_all(o, lambda d: d["status"] == 0 and all(len(c["stages"]) == 1 for c in d["classes"])
                      and sum(c["D"] for c in d["classes"]) > 1, limit=60)
    assert found
    for i, _ in found:
        assert ov.eval(i) == o.eval(i)


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_overlap_never_slower_and_keeps_status(oracle_mod, n):
    cfg = H.get(n)
    o, ov = oracle_mod.Oracle(cfg), oracle_mod.Oracle(H.with_sync_overlap(cfg))
    idx = H.sample_indices(o.space_size(), 500, seed=H.PARITY_SEED + 40 + n)
    a, b = o.eval_many(idx), ov.eval_many(idx)
    assert np.array_equal(a < 0, b < 0) and np.array_equal(a[a < 0], b[a < 0])
    ok = a >= 0
    assert np.all(b[ok] <= a[ok])
    assert (b[ok] < a[ok]).mean() > 0.5


@pytest.mark.parametrize("seed", range(6))
def test_overlap_tiny_never_slower_d1_equal(oracle_mod, seed):
    cfg = H.tiny_random(300 + seed)
    o, ov = oracle_mod.Oracle(cfg), oracle_mod.Oracle(H.with_sync_overlap(cfg))
    N = o.space_size()
    a, b = o.eval_many(first=0, n=N), ov.eval_many(first=0, n=N)
    ok = a >= 0
    assert np.all(b[ok] <= a[ok])
    for i in range(0, N, max(1, N // 50)):
        d = o.describe(i)
        if d["status"] == 0 and sum(c["D"] for c in d["classes"]) == 1:
            assert a[i] == b[i]  # D = 1: no gradient sync at all
