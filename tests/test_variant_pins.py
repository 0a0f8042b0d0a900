"""Pins of the oracle's SURVEY §8(f) f4 variants (DESIGN.md V.2, V.3).

V.2 interleaved 1F1B (v model chunks per stage, Megatron-LM's virtual
pipeline, Narayanan et al. 2021):
* the textbook closed form: with every chunk taking a forward / b backward
  and free communication, T = (m v + P - 1)(a + b) for m a multiple of P
  (the interleaved bubble (P - 1)/(m v) of the Megatron paper);
* the op lists against the schedule table written out here (groups of P
  micro-batches, chunks ascending for forwards / descending for backwards,
  warm-up 2(P-1-s) + (v-1)P), every op exactly once, F(k, j) before B(k, j);
* deadlock freedom for every P <= 12, v <= 4, m in {P, 2P, 3P};
* an explicit-DAG longest path (not an event engine) on random durations
  and p2p / wrap costs;
* whole candidates: ``py_eval_v`` (below) -- the independent evaluator of
  tests/test_oracle_pins_r2.py extended with chunks, the wrap boundary and
  virtual-stage sync segments -- equals the oracle on tiny spaces;
  the -1 / -2 rules (a stage with fewer layers than chunks; m mod P != 0).

V.3 expert parallelism across the DP replicas:
* the all-to-all over one group is A17's (the round-robin schedule);
* over two groups on two nodes, a hand-computed round-robin over the rail
  (Table 4 link delays);
* with one replica the variant changes nothing (every candidate equal);
* the dense gradient bytes against Mixtral 8x7B's public parameter split
  (46.7 B total, 32 x 8 experts x 3 x 4096 x 14336 expert weights);
* whole candidates against ``py_eval_v`` (lockstep replicas, g = D tp).
"""
import math
import os

import numpy as np
import pytest

import hsim_inputs as H
from test_oracle_pins_r2 import act_bytes, cdiv, model_dims, tau, tp_allreduce_ref, tp_ring_edges

THREADS = os.cpu_count() or 4


# ----------------------------------------------------------------------------
# V.2 schedule, written out from the Megatron-LM description
# ----------------------------------------------------------------------------
def megatron_tables(P, v, m):
    """Forward / backward tables: micro-batches in groups of P; per group the
    chunks 0..v-1 (forward) or v-1..0 (backward), the group's micro-batches in
    order within a chunk."""
    fw, bw = [], []
    for g0 in range(0, m, P):
        grp = list(range(g0, min(g0 + P, m)))
        fw += [(k, j) for k in range(v) for j in grp]
        bw += [(k, j) for k in reversed(range(v)) for j in grp]
    return fw, bw


def megatron_order(P, s, m, v):
    """v = 1 is the non-interleaved 1F1B (C.7, warm-up min(P-1-s, m))."""
    fw, bw = megatron_tables(P, v, m)
    n = m * v
    w = min((P - 1 - s) * 2 + (v - 1) * P, n) if v > 1 else min(P - 1 - s, m)
    out = [("F",) + x for x in fw[:w]]
    for i in range(n - w):
        out += [("F",) + fw[w + i], ("B",) + bw[i]]
    out += [("B",) + x for x in bw[n - w:]]
    return out


def ilv_dag(f, g, c, cw, m):
    """Interleaved 1F1B as an explicit DAG, longest path by Kahn's order.
    f, g: [P][v]; c: boundary costs; cw: wrap cost.  Returns (T, per-stage end
    of its last op)."""
    P, v = len(f), len(f[0])
    preds = {}
    last_op = {}
    for s in range(P):
        prev = None
        for op in megatron_order(P, s, m, v):
            node = (s,) + op
            preds[node] = [(prev, 0)] if prev else []
            prev = node
        last_op[s] = prev
    for s in range(P):
        for k in range(v):
            for j in range(m):
                if s > 0:
                    preds[(s, "F", k, j)].append(((s - 1, "F", k, j), c[s - 1]))
                elif k > 0:
                    preds[(s, "F", k, j)].append(((P - 1, "F", k - 1, j), cw))
                if s < P - 1:
                    preds[(s, "B", k, j)].append(((s + 1, "B", k, j), c[s]))
                elif k < v - 1:
                    preds[(s, "B", k, j)].append(((0, "B", k + 1, j), cw))
                else:
                    preds[(s, "B", k, j)].append(((s, "F", k, j), 0))
    succ = {x: [] for x in preds}
    indeg = {x: len(p) for x, p in preds.items()}
    for x, ps in preds.items():
        for u, _ in ps:
            succ[u].append(x)
    ready = [x for x, d in indeg.items() if d == 0]
    end = {}
    while ready:
        x = ready.pop()
        st = max([end[u] + d for u, d in preds[x]], default=0)
        s, kind, k, _ = x
        end[x] = st + (f[s][k] if kind == "F" else g[s][k])
        for y in succ[x]:
            indeg[y] -= 1
            if indeg[y] == 0:
                ready.append(y)
    assert len(end) == len(preds), "cycle: the schedule deadlocks"
    return max(end.values()), [end[last_op[s]] for s in range(P)]


def test_ilv_uniform_closed_form(oracle_mod):
    for P in range(2, 9):
        for v in (2, 3, 4):
            for m in (P, 2 * P, 3 * P):
                for a, b in ((1, 2), (3, 5), (7, 7)):
                    T = oracle_mod.pipeline_ilv([[a] * v] * P, [[b] * v] * P, [0] * (P - 1), 0, m)
                    assert T == (m * v + P - 1) * (a + b), (P, v, m, a, b)


def test_ilv_op_order_against_table(oracle_mod):
    for P in (2, 3, 4, 5, 8):
        for v in (2, 3, 4):
            for m in (P, 2 * P, 4 * P):
                for s in range(P):
                    got = oracle_mod.op_order(P, s, m, v)
                    want = [(1 if o[0] == "F" else 0, o[1], o[2]) for o in megatron_order(P, s, m, v)]
                    assert got == want, (P, v, m, s)
                    assert sorted(got) == sorted((d, k, j) for d in (0, 1) for k in range(v) for j in range(m))
                    pos = {x: n for n, x in enumerate(got)}
                    assert all(pos[(1, k, j)] < pos[(0, k, j)] for k in range(v) for j in range(m))


def test_ilv_no_deadlock(oracle_mod):
    """The event engine aborts on a deadlock; every (P, v, m) with m mod P = 0
    completes, and equals the uniform closed form."""
    for P in range(2, 13):
        for v in range(2, 5):
            for m in (P, 2 * P, 3 * P):
                assert oracle_mod.pipeline_ilv([[2] * v] * P, [[3] * v] * P, [1] * (P - 1), 1, m) > 0


def test_ilv_dag_random(oracle_mod):
    rng = np.random.default_rng(2508)
    for _ in range(250):
        P, v = int(rng.integers(2, 7)), int(rng.integers(2, 5))
        m = P * int(rng.integers(1, 4))
        f = rng.integers(1, 60, size=(P, v)).tolist()
        g = rng.integers(1, 120, size=(P, v)).tolist()
        c = rng.integers(0, 40, size=P - 1).tolist()
        cw = int(rng.integers(0, 80))
        T, _ = ilv_dag(f, g, c, cw, m)
        assert oracle_mod.pipeline_ilv(f, g, c, cw, m) == T, (P, v, m)


# ----------------------------------------------------------------------------
# V.3 all-to-all
# ----------------------------------------------------------------------------
def a2a_groups_ref(o, cfg, groups, t, b, round_robin=False):
    """All-to-all over the union of the groups' devices (g = n t): each TP
    group's A bytes of routed tokens (k routes per token) leave its t devices
    evenly and spread over the g expert devices, ceil(A k / (t g)) bytes per
    ordered pair, in g - 1 rounds.  DESIGN A17: a round lasts as long as the
    slowest pair of the whole group.  round_robin=True instead ends round r
    (device x -> x + r mod g) with its own slowest pair (a lower bound, equal
    on uniform links)."""
    dev = [(n, b0 + q) for n, b0 in groups for q in range(t)]
    g = len(dev)
    if g == 1:
        return 0
    per = cdiv(act_bytes(cfg, b) * cfg["model"]["moe_topk"], t * g)
    if round_robin:
        return sum(max(tau(o.link(*dev[x], *dev[(x + r) % g]), per) for x in range(g)) for r in range(1, g))
    return (g - 1) * max(tau(o.link(*dev[x], *dev[y]), per) for x in range(g) for y in range(g) if x != y)


@pytest.mark.parametrize("t", [1, 2, 4, 8])
def test_ep_one_group_is_a17(oracle_mod, t):
    cfg = H.get(4)
    o = oracle_mod.Oracle(cfg)
    for b in (1, 2, 4):
        assert o.ep_alltoall_groups([(0, 0)], t, b) == o.ep_alltoall(0, 0, t, b)


@pytest.mark.parametrize("groups,t", [([(0, 0), (1, 0)], 1), ([(0, 0), (1, 0)], 2), ([(0, 0), (0, 4), (1, 0)], 4),
                                      ([(8, 0), (9, 2), (10, 4), (11, 6)], 2)])
def test_ep_groups_round_robin(oracle_mod, groups, t):
    cfg = H.get(4)
    o = oracle_mod.Oracle(cfg)
    for b in (1, 2):
        got = o.ep_alltoall_groups(groups, t, b)
        assert got == a2a_groups_ref(o, cfg, groups, t, b)
        rr = a2a_groups_ref(o, cfg, groups, t, b, round_robin=True)
        assert rr <= got
        if t == 1 and len({n for n, _ in groups}) == len(groups) and len({b0 for _, b0 in groups}) == 1:
            assert rr == got  # every pair on the same rail: uniform links


def test_ep_two_h100_nodes_by_hand(oracle_mod):
    """Two H100 nodes (config 4's nodes 8 and 9), one GPU each (t = 1): g = 2,
    one round over the rail: 1 x tau(rail, ceil(A k / 2)).  Rail path (Table 4,
    PAPER.md:329-333): GPU->NIC PCIe 1024 Gbps bidirectional (2 hops, 143.75 ->
    144 ns each, A9), NIC 368 ns + 200 Gbps, rail 0 ns, NIC 368 ns, PCIe 2 x 144
    ns: alpha = 4 x 144 + 2 x 368 = 1312 ns, beta = 200/8 = 25 B/ns."""
    cfg = H.get(4)
    o = oracle_mod.Oracle(cfg)
    a, beta = o.link(8, 0, 9, 0)
    assert (a, beta) == (1312, 25.0)
    A = 2 * 2048 * 4096 * 2  # b = 2, s = 2048, h = 4096, bf16
    assert o.ep_alltoall_groups([(8, 0), (9, 0)], 1, 2) == 1312 + math.ceil(cdiv(A * 2, 2) / 25.0)


def test_ep_dense_gradient_bytes_mixtral(oracle_mod):
    """Mixtral 8x7B: 46.7 B parameters, of which 32 layers x 8 experts x 3 x
    4096 x 14336 = 45.1 B are expert MLP weights.  With V.3 a single-class
    template synchronises only the rest (plus the router): total segment bytes
    / bpe_grad within 2 % of 46.7e9 - 45.1e9."""
    cfg = H.with_ep_dp(H.get(4))
    o = oracle_mod.Oracle(cfg)
    d = None
    for k in range(o.n_templates()):
        i = int(o.template_prefix()[k]) if d is None else None
        dd = o.describe(i)
        if len(dd["classes"]) == 1 and sum(c["D"] for c in dd["classes"]) > 1 and o.eval(i) >= 0:
            d = dd
            break
    assert d is not None
    S = sum(sg["S"] for sg in o.segments(i)) / cfg["model"]["bpe_grad"]
    expert = 32 * 8 * 3 * 4096 * 14336
    assert abs(S - (46.7e9 - expert)) / (46.7e9 - expert) < 0.02, S
    off = oracle_mod.Oracle(H.get(4))
    S_full = sum(sg["S"] for sg in off.segments(i)) / cfg["model"]["bpe_grad"]
    assert S_full - S == expert


# ----------------------------------------------------------------------------
# whole candidates: an independent evaluator with both variants
# ----------------------------------------------------------------------------
def gdev(place, t, q):
    """Device q of a stage group: [node, base] holds GPUs base..base+t-1; a V.1
    mixed group [node, base, node2] holds q < t/2 on node, the rest at the
    same base on node2."""
    if len(place) == 2:
        return place[0], place[1] + q
    h = t // 2
    return (place[0], place[1] + q) if q < h else (place[2], place[1] + q - h)


def glink(o, p1, t1, q1, p2, t2, q2):
    return o.link(*gdev(p1, t1, q1), *gdev(p2, t2, q2))


def op_max(o, stage, kind, bwd, b):
    """V.1 (PAPER.md:280 C4): a mixed group's op lasts as long as on its slower
    device type; stage = [type, tp] or [type, tp, type2]."""
    d = o.op(stage[0], kind, bwd, stage[1], b)[2]
    if len(stage) == 3:
        d = max(d, o.op(stage[2], kind, bwd, stage[1], b)[2])
    return d


def ring_ar(o, cfg, place, t, b):
    """TP ring all-reduce over devices 0..t-1 of the group (ring law)."""
    if t == 1:
        return 0
    A = cdiv(act_bytes(cfg, b), t)
    return 2 * (t - 1) * max(tau(glink(o, place, t, q, place, t, (q + 1) % t), A) for q in range(t))


def pair_a2a(o, cfg, place, t, b):
    """A17 all-to-all inside one group: t - 1 rounds at its slowest ordered pair."""
    if t == 1:
        return 0
    per = cdiv(act_bytes(cfg, b) * cfg["model"]["moe_topk"], t * t)
    return (t - 1) * max(tau(glink(o, place, t, x, place, t, y), per) for x in range(t) for y in range(t) if x != y)


def py_eval_v(o, cfg, i, overlap=False):
    """Independent evaluator of candidate i under V.2 (cfg search.interleave)
    and V.3 (search.ep_dp).  Chunk k of a stage with l layers has
    l // v + [k < l % v] layers; the embedding rides with chunk 0 of stage 0,
    the head with chunk v-1 of stage P-1; sync segments refine the classes'
    virtual-stage boundaries (virtual stage k P + s = chunk k of stage s)."""
    d = o.describe(i)
    if d["status"]:
        return d["status"]
    se = cfg["search"]
    vset = se.get("interleave", 1)
    m_ = model_dims(cfg)
    b = d["b"]
    A = act_bytes(cfg, b)
    moe = m_["E"] > 1
    ep = bool(se.get("ep_dp", 0)) and moe and len(d["classes"]) == 1
    T0, lastB, lowb = 0, {}, {}
    two = se.get("sync_buckets", 1) == 2  # B.1: lower ceil(l/2) layers (+ embedding) and the rest
    vstarts = []  # per class: [(first layer, stage)] in layer order
    bcut = []     # per class: {stage: first layer of its upper bucket}
    for c, cl in enumerate(d["classes"]):
        P, D = len(cl["stages"]), cl["D"]
        v = vset if P >= 2 else 1
        lay = [[l // v + (1 if k < l % v else 0) for k in range(v)] for l in cl["layers"]]
        acc, st = 0, []
        for k in range(v):
            for s in range(P):
                st.append((acc, s))
                acc += lay[s][k]
        vstarts.append(st)
        bcut.append({s0: a0 + (cl["layers"][s0] + 1) // 2 for a0, s0 in st} if two else {})

        def p2p(r, s1, s2):
            t1, t2 = cl["stages"][s1][1], cl["stages"][s2][1]
            return max(tau(glink(o, cl["place"][r][s1], t1, q, cl["place"][r][s2], t2, q), A) for q in range(min(t1, t2)))

        cc = [[p2p(r, s, s + 1) for s in range(P - 1)] for r in range(D)]
        cw = [p2p(r, P - 1, 0) if v > 1 else 0 for r in range(D)]
        mb = list(cl["mb"])
        if ep:  # lockstep: the slowest boundary of any replica, the largest m
            cc = [[max(x[s] for x in cc) for s in range(P - 1)]] * D
            cw = [max(cw)] * D
            mb = [max(mb)] * D
        for r in range(D):
            f, g = [], []
            for s, stage in enumerate(cl["stages"]):
                ty, tp = stage[0], stage[1]
                pl = cl["place"][r][s]
                ar = ring_ar(o, cfg, pl, tp, b)
                kind = "moe" if moe else "mlp"
                if ep:
                    groups = [tuple(cl["place"][rr][s]) for rr in range(D)]
                    a2a = a2a_groups_ref(o, cfg, groups, tp, b)
                    gexp = D * tp
                else:
                    a2a = pair_a2a(o, cfg, pl, tp, b) if moe else 0
                    gexp = tp
                ch = []
                for bwd in (0, 1):
                    x = op_max(o, stage, "attn", bwd, b) + ar
                    if moe:
                        mo = moe_dur(o, cfg, ty, bwd, tp, b, gexp)
                        if len(stage) == 3:
                            mo = max(mo, moe_dur(o, cfg, stage[2], bwd, tp, b, gexp))
                        x += a2a + mo + a2a
                    else:
                        x += op_max(o, stage, kind, bwd, b) + ar
                    ch.append(x)
                fs = [lay[s][k] * ch[0] for k in range(v)]
                gs = [lay[s][k] * ch[1] for k in range(v)]
                if s == 0:
                    fs[0] += op_max(o, stage, "emb", 0, b)
                    gs[0] += op_max(o, stage, "emb", 1, b)
                if s == P - 1:
                    fs[v - 1] += op_max(o, stage, "head", 0, b)
                    gs[v - 1] += op_max(o, stage, "head", 1, b)
                f.append(fs)
                g.append(gs)
                # the last backward runs head, layers top-down, embedding: the
                # lower bucket's gradients take its last ceil(l/2) layers + emb
                lowb[(c, r, s)] = (cl["layers"][s] + 1) // 2 * ch[1] + (op_max(o, stage, "emb", 1, b) if s == 0 else 0)
            T, last = ilv_dag(f, g, cc[r], cw[r], mb[r])
            T0 = max(T0, T)
            for s in range(P):
                lastB[(c, r, s)] = last[s]
    D = sum(cl["D"] for cl in d["classes"])
    if D == 1:
        return T0
    cuts = sorted(set([0, m_["L"]] + [a for st in vstarts for a, _ in st] +
                      [x for bc in bcut for x in bc.values() if 0 < x < m_["L"]]))
    segs = []
    for a, z in zip(cuts, cuts[1:]):
        sc = [max(st, key=lambda x: (x[0] <= a, x[0]))[1] for st in vstarts]
        bk = [1 if two and a >= bcut[c][sc[c]] else 0 for c in range(len(sc))]
        tps = [cl["stages"][sc[c]][1] for c, cl in enumerate(d["classes"])]
        tstar = min(tps)
        S = seg_bytes_v(cfg, a, z, ep)
        RS = 0
        for c, cl in enumerate(d["classes"]):
            if tps[c] != tstar:
                for r in range(cl["D"]):
                    pl, t = cl["place"][r][sc[c]], tps[c]
                    RS = max([RS] + [tau(glink(o, pl, t, q, pl, t, (q + 1) % t), cdiv(S, tstar)) for q in range(t)])
        ring = [(cl["place"][r][sc[c]], tps[c]) for c, cl in enumerate(d["classes"]) for r in range(cl["D"])]
        chunk = cdiv(cdiv(S, tstar), D)
        slow = max(tau(glink(o, u[0], u[1], q, w[0], w[1], q), chunk)
                   for q in range(tstar) for u, w in zip(ring, ring[1:] + ring[:1]))
        segs.append((sc, RS + 2 * (D - 1) * slow, bk))
    free = {}
    T = T0
    for j in (range(len(segs) - 1, -1, -1) if overlap else range(len(segs))):
        sc, cost, bk = segs[j]
        groups = [(c, r, sc[c]) for c, cl in enumerate(d["classes"]) for r in range(cl["D"])]
        if overlap:
            start = max(max(lastB[x] - (lowb[x] if bk[x[0]] else 0), free.get(x, 0)) for x in groups)
        else:
            start = max(free.get(x, T0) for x in groups)
        for x in groups:
            free[x] = start + cost
        T = max(T, start + cost)
    return T


def moe_dur(o, cfg, ty, bwd, t, b, g):
    """MoE op duration with the expert weights sharded over g devices: the
    roofline of (FLOP of the TP-sharded op, bytes with the weight term / g);
    g = t is the oracle's own op (A17)."""
    if g == t:
        return o.op(ty, "moe", bwd, t, b)[2]
    m = model_dims(cfg)
    T = b * m["s"]
    flop = cdiv(2 * T * m["k"] * m["nm"] * m["h"] * m["f"], t)
    byts = cdiv(m["bpe"] * m["E"] * m["nm"] * m["h"] * m["f"], g) + 2 * T * m["h"] * m["bpe"]
    tyd = cfg["cluster"]["types"][ty]
    mul = 2 if bwd else 1
    rf = tyd["peak_flop_per_ns"] * tyd["eff_flop"][2]
    rm = tyd["hbm_bytes_per_ns"] * tyd["eff_mem"][2]
    return max(math.ceil(mul * flop / rf) if flop else 0, math.ceil(mul * byts / rm))


def seg_bytes_v(cfg, a, z, ep):
    from test_oracle_pins_r2 import segment_bytes_ref
    S = segment_bytes_ref(cfg, a, z)
    if ep:
        m = model_dims(cfg)
        S -= (z - a) * m["nm"] * m["h"] * m["f"] * m["E"] * m["bg"]
    return S


def _check_space(oracle_mod, cfg, n, seed, overlap=False, need_valid=10):
    o = oracle_mod.Oracle(cfg)
    N = o.space_size()
    idx = np.arange(N) if N <= n else H.sample_indices(N, n, seed=seed)
    want = o.eval_many(idx, threads=THREADS)
    for k, i in enumerate(idx):
        assert py_eval_v(o, cfg, int(i), overlap) == want[k], int(i)
    assert (want >= 0).sum() >= need_valid
    return want


@pytest.mark.parametrize("seed", [100, 101, 103, 105, 107, 110])
@pytest.mark.parametrize("v", [2, 3])
def test_py_eval_interleave_tiny(oracle_mod, seed, v):
    _check_space(oracle_mod, H.with_interleave(H.variant_tiny(seed), v), 200, seed, need_valid=3)


@pytest.mark.parametrize("seed", [101, 105])
def test_py_eval_interleave_overlap(oracle_mod, seed):
    _check_space(oracle_mod, H.with_sync_overlap(H.with_interleave(H.variant_tiny(seed), 2)), 150, seed + 1,
                 overlap=True, need_valid=3)


@pytest.mark.parametrize("seed", [100, 102, 104, 106, 108])
def test_py_eval_ep_dp_tiny(oracle_mod, seed):
    _check_space(oracle_mod, H.with_ep_dp(H.variant_tiny(seed, moe=True)), 200, seed)


def test_py_eval_both_variants(oracle_mod):
    _check_space(oracle_mod, H.with_ep_dp(H.with_interleave(H.variant_tiny(104, moe=True), 2)), 200, 7,
                 need_valid=3)


def test_ilv_status_rules(oracle_mod):
    """-1 when a stage holds fewer layers than chunks; -2 when some replica's
    micro-batch count is not a multiple of its depth; P = 1 classes and
    non-variant candidates are untouched."""
    base = H.variant_tiny(101)
    cfg = H.with_interleave(base, 3)
    o, o0 = oracle_mod.Oracle(cfg), oracle_mod.Oracle(base)
    N = o.space_size()
    assert N == o0.space_size()
    idx = np.arange(N) if N <= 3000 else H.sample_indices(N, 3000, seed=5)
    got, ref = o.eval_many(idx, threads=THREADS), o0.eval_many(idx, threads=THREADS)
    seen = set()
    for k, i in enumerate(idx):
        d0 = o0.describe(int(i))
        cls = d0["classes"]
        deep = [c for c in cls if len(c["stages"]) >= 2]
        if ref[k] < 0:  # -1 (a stage with fewer layers than chunks) takes precedence over -2
            short = ref[k] == -2 and any(min(c["layers"]) < 3 for c in deep)
            assert got[k] == (-1 if short else ref[k])
            continue
        if not deep:
            assert got[k] == ref[k]
            seen.add("flat")
        elif any(min(c["layers"]) < 3 for c in deep):
            assert got[k] == -1
            seen.add(-1)
        elif any(mm % len(c["stages"]) for c in deep for mm in c["mb"]):
            assert got[k] == -2
            seen.add(-2)
        else:
            assert got[k] >= 0
            seen.add("ok")
    assert {"flat", -1, -2} <= seen


def test_ep_single_replica_unchanged(oracle_mod):
    """With D = 1 the EP group is the TP group: V.3 equals A17 on every
    single-replica candidate (and on every multi-class one)."""
    base = H.variant_tiny(102, moe=True)
    o, o0 = oracle_mod.Oracle(H.with_ep_dp(base)), oracle_mod.Oracle(base)
    N = o.space_size()
    idx = np.arange(N) if N <= 3000 else H.sample_indices(N, 3000, seed=9)
    got, ref = o.eval_many(idx, threads=THREADS), o0.eval_many(idx, threads=THREADS)
    single = 0
    for k, i in enumerate(idx):
        d0 = o0.describe(int(i))
        if len(d0["classes"]) > 1 or (d0["status"] == 0 and d0["classes"][0]["D"] == 1):
            assert got[k] == ref[k], int(i)
            single += 1
    assert single > 10


def test_variants_literal_equals_compact(oracle_mod):
    for cfg in (H.with_interleave(H.variant_tiny(105), 2), H.with_ep_dp(H.variant_tiny(106, moe=True)),
                H.with_ep_dp(H.with_interleave(H.get(4), 2))):
        lit, cmp_ = oracle_mod.Oracle(cfg), oracle_mod.Oracle(cfg, compact=True)
        idx = H.sample_indices(lit.space_size(), 300, seed=11)
        assert np.array_equal(lit.eval_many(idx, threads=THREADS), cmp_.eval_many(idx, threads=THREADS))


# ----------------------------------------------------------------------------
# V.1 mixed-type TP groups
# ----------------------------------------------------------------------------
def with_mixtp(cfg):
    return H.with_changes(cfg, search__mixtp=1)


def count_mixtp(cfg):
    """Candidates of the MIXTP family, counted from DESIGN V.1's grammar
    (written out independently of the oracle's enumeration)."""
    cl, md, se = cfg["cluster"], cfg["model"], cfg["search"]
    nt = len(cl["types"])
    n_of = [sum(t["gpus_per_node"] for n, t in ((n, cl["types"][n]) for n in cl["nodes"]) if n == k) for k in range(nt)]
    n_of = [cl["nodes"].count(k) * cl["types"][k]["gpus_per_node"] for k in range(nt)]
    rl, rb = 2 * se["r_layer"] + 1, 2 * se["r_batch"] + 1
    total = 0
    for b in sorted(se["bset"]):
        if md["global_batch"] % b:
            continue
        M = md["global_batch"] // b
        for a in range(nt):
            for a2 in range(a + 1, nt):
                for tp in sorted(set(se["tpset"][a]) & set(se["tpset"][a2])):
                    if tp < 2 or md["heads"] % tp or md["kv_heads"] % tp:
                        continue
                    if any(cl["types"][x]["gpus_per_node"] % (tp // 2) for x in (a, a2)):
                        continue
                    for P in sorted(set(se["pset"])):
                        if P > md["layers"]:
                            continue
                        D = 1
                        while D * P * (tp // 2) <= min(n_of[a], n_of[a2]):
                            full = D * P * (tp // 2) == n_of[a] == n_of[a2]
                            if (not se["use_all"] or full) and M >= D:
                                total += rl ** (P - 1) if P <= se["pmax_perturb"] else 1
                            D += 1
    return total


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_mixtp_space_size(oracle_mod, n):
    base = oracle_mod.Oracle(H.get(n)).space_size()
    assert oracle_mod.Oracle(with_mixtp(H.get(n))).space_size() == base + count_mixtp(H.get(n))


def test_mixtp_placement_by_hand(oracle_mod):
    """Config 2 (nodes 0-1 A100, 2-3 H100, 8 GPUs each), tp = 4 mixed groups
    (2 A100 + 2 H100), P = 2, D = 2: groups fill the 2-GPU blocks of node 0
    and node 2 in order -- (0, 0 | 2), (0, 2 | 2), then replica 1 (0, 4 | 2),
    (0, 6 | 2)."""
    o = oracle_mod.Oracle(with_mixtp(H.get(2)))
    pre = o.template_prefix()
    for k in range(o.n_templates()):
        d = o.describe(int(pre[k]))
        cl = d["classes"][0]
        if len(cl["stages"][0]) == 3 and cl["stages"] == [[0, 4, 1]] * 2 and cl["D"] == 2:
            assert cl["place"] == [[[0, 0, 2], [0, 2, 2]], [[0, 4, 2], [0, 6, 2]]]
            return
    raise AssertionError("template not found")


def test_mixtp_single_group_closed_form(oracle_mod):
    """One mixed A100/H100 group of tp = 2 (one GPU on node 0, one on node 2),
    P = 1, D = 1, b = 4: T = M (f + g), each op the slower type's (the
    bottleneck device), each layer with two TP all-reduces over the group's
    two rail edges: 2 (t-1) x tau(rail, ceil(A / 2)).  Rail (Table 4): A100
    PCIe 512 Gbps bidirectional = 2 x ceil(73600 / 256) = 2 x 288 ns, NIC 368 +
    200 Gbps, H100 PCIe 1024 -> 2 x 144 ns, NIC 368: alpha = 576 + 368 + 368 +
    288 = 1600 ns, beta = 25 B/ns."""
    cfg = with_mixtp(H.get(2))
    o = oracle_mod.Oracle(cfg)
    a, beta = o.link(0, 0, 2, 0)
    assert (a, beta) == (1600, 25.0)
    pre = o.template_prefix()
    for k in range(o.n_templates()):
        d = o.describe(int(pre[k]))
        if d["b"] == 4 and d["classes"][0]["stages"] == [[0, 2, 1]] and d["classes"][0]["D"] == 1:
            break
    else:
        raise AssertionError("template not found")
    b, L, M = 4, cfg["model"]["layers"], cfg["model"]["global_batch"] // 4
    A = b * 4096 * 4096 * 2
    ar = 2 * 1 * (1600 + math.ceil(cdiv(A, 2) / 25.0))
    mx = lambda kind, bwd: max(o.op(0, kind, bwd, 2, b)[2], o.op(1, kind, bwd, 2, b)[2])
    fg = [L * (mx("attn", bwd) + ar + mx("mlp", bwd) + ar) + mx("emb", bwd) + mx("head", bwd) for bwd in (0, 1)]
    assert o.eval(int(pre[k])) == M * sum(fg)
    assert mx("mlp", 0) == o.op(0, "mlp", 0, 2, b)[2] > o.op(1, "mlp", 0, 2, b)[2]  # the A100 half bounds it


@pytest.mark.parametrize("cfgf", ["c2", "c4", "tiny101", "tiny105", "c2-ilv", "c4-overlap"])
def test_py_eval_mixtp(oracle_mod, cfgf):
    cfg = {"c2": lambda: with_mixtp(H.get(2)), "c4": lambda: with_mixtp(H.get(4)),
           "tiny101": lambda: with_mixtp(H.variant_tiny(101)), "tiny105": lambda: with_mixtp(H.variant_tiny(105)),
           "c2-ilv": lambda: H.with_interleave(with_mixtp(H.get(2)), 2),
           "c4-overlap": lambda: H.with_sync_overlap(with_mixtp(H.get(4)))}[cfgf]()
    o = oracle_mod.Oracle(cfg)
    base = oracle_mod.Oracle(H.with_changes(cfg, search__mixtp=0)).space_size()
    N = o.space_size()
    assert N > base
    idx = np.arange(base, N) if N - base <= 300 else np.unique(np.concatenate(
        [H.sample_indices(N - base, 250, seed=3) + base, [base, N - 1]]))
    want = o.eval_many(idx, threads=THREADS)
    for k, i in enumerate(idx):
        assert py_eval_v(o, cfg, int(i), overlap=bool(cfg["search"].get("sync_overlap", 0))) == want[k], int(i)
    assert (want >= 0).sum() >= 3


def test_mixtp_literal_equals_compact(oracle_mod):
    cfg = with_mixtp(H.get(2))
    lit, cmp_ = oracle_mod.Oracle(cfg), oracle_mod.Oracle(cfg, compact=True)
    base = oracle_mod.Oracle(H.get(2)).space_size()
    idx = np.arange(base, lit.space_size())
    assert np.array_equal(lit.eval_many(idx, threads=THREADS), cmp_.eval_many(idx, threads=THREADS))


# ----------------------------------------------------------------------------
# B.1 two gradient buckets per stage group (Table 1 "DP frequency 2")
# ----------------------------------------------------------------------------
def with_buckets(cfg):
    return H.with_changes(cfg, search__sync_buckets=2)


@pytest.mark.parametrize("cfgf,overlap", [("c2", False), ("c2", True), ("c4", True), ("tiny105", True),
                                          ("tiny110", False), ("c2-mixtp", True), ("c4-ep", True)])
def test_py_eval_buckets(oracle_mod, cfgf, overlap):
    cfg = {"c2": lambda: H.get(2), "c4": lambda: H.get(4), "tiny105": lambda: H.variant_tiny(105),
           "tiny110": lambda: H.variant_tiny(110), "c2-mixtp": lambda: with_mixtp(H.get(2)),
           "c4-ep": lambda: H.with_ep_dp(H.get(4))}[cfgf]()
    cfg = with_buckets(H.with_sync_overlap(cfg) if overlap else cfg)
    o = oracle_mod.Oracle(cfg)
    N = o.space_size()
    idx = np.arange(N) if N <= 300 else H.sample_indices(N, 250, seed=29)
    want = o.eval_many(idx, threads=THREADS)
    for k, i in enumerate(idx):
        assert py_eval_v(o, cfg, int(i), overlap=overlap) == want[k], int(i)
    assert (want >= 0).sum() >= 10


def test_buckets_table1_frequency_two(oracle_mod):
    """Table 1: DP frequency 2 per iteration.  A single-class
    candidate whose stages hold >= 2 layers each all-reduces every stage
    group's gradient in exactly 2 collectives (segments), and the segment
    bytes of a stage add up to its one-bucket segment."""
    cfg = H.get(2)
    o1, o2 = oracle_mod.Oracle(cfg), oracle_mod.Oracle(with_buckets(cfg))
    pre = o1.template_prefix()
    seen = 0
    for k in range(0, o1.n_templates(), 37):
        i = int(pre[k])
        d = o1.describe(i)
        if d["status"] or len(d["classes"]) != 1 or d["classes"][0]["D"] < 2 or min(d["classes"][0]["layers"]) < 2:
            continue
        s1, s2 = o1.segments(i), o2.segments(i)
        assert len(s2) == 2 * len(s1)
        for j, sg in enumerate(s1):
            lo, hi = s2[2 * j], s2[2 * j + 1]
            assert (lo["a"], hi["z"]) == (sg["a"], sg["z"]) and lo["z"] == hi["a"] == sg["a"] + (sg["z"] - sg["a"] + 1) // 2
            assert lo["S"] + hi["S"] == sg["S"]
        seen += 1
    assert seen > 5


def test_buckets_d1_and_p1_invariants(oracle_mod):
    """One replica: no sync, buckets change nothing.  C.8 with one stage of one
    layer: a single bucket, unchanged."""
    cfg = H.variant_tiny(105)
    o1, o2 = oracle_mod.Oracle(cfg), oracle_mod.Oracle(with_buckets(cfg))
    idx = np.arange(o1.space_size())
    a, b = o1.eval_many(idx, threads=THREADS), o2.eval_many(idx, threads=THREADS)
    for k, i in enumerate(idx):
        d = o1.describe(int(i))
        if d["status"] == 0 and sum(c["D"] for c in d["classes"]) == 1:
            assert a[k] == b[k]
