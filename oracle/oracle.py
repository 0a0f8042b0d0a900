"""ctypes binding of the C++ oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module.  The product package never does.

The binding only copies fields of a shared workload dict (hsim_inputs/) into
the oracle's own input struct (defined in oracle.cpp); it holds none of the
method's arithmetic.
"""
import ctypes as C
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.cpp")
LIB = os.path.join(HERE, "liboracle.so")

KIND = {"attn": 0, "mlp": 1, "moe": 2, "emb": 3, "head": 4}


def build(force=False):
    """Compile oracle.cpp -> liboracle.so (plain g++, IEEE double, no FMA)."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off",
           "-fno-fast-math", "-pthread", SRC, "-o", LIB]
    subprocess.check_call(cmd)
    return LIB


class _Hop(C.Structure):
    _fields_ = [("gbps", C.c_double), ("bidir", C.c_int32), ("pad", C.c_int32)]


class _Path(C.Structure):
    _fields_ = [("n", C.c_int32), ("pad", C.c_int32), ("hop", _Hop * 4)]


class _Type(C.Structure):
    _fields_ = [("peak_flop_per_ns", C.c_double), ("hbm_bytes_per_ns", C.c_double),
                ("eff_flop", C.c_double * 5), ("eff_mem", C.c_double * 5),
                ("mem_bytes", C.c_int64),
                ("gpus_per_node", C.c_int32), ("n_link_kinds", C.c_int32),
                ("link_kind", _Path * 4),
                ("intra_kind", (C.c_int32 * 8) * 8),
                ("gpu_nic", _Path),
                ("nic_gbps", C.c_double),
                ("nic_delay_ns", C.c_int64)]


class _Input(C.Structure):
    _fields_ = [("n_types", C.c_int32), ("n_nodes", C.c_int32),
                ("types", C.POINTER(_Type)), ("node_type", C.POINTER(C.c_int32)),
                ("rail_alpha_ns", C.c_int64), ("rail_gbps", C.c_double), ("frame_bytes", C.c_int64)] + \
               [(k, C.c_int64) for k in ("L", "h", "heads", "kv_heads", "ffn", "nm", "seq", "V",
                                         "tied", "E", "topk", "bpe_act", "bpe_grad", "B")] + \
               [("n_b", C.c_int32), ("bset", C.c_int32 * 8),
                ("n_tp", C.c_int32 * 8), ("tpset", (C.c_int32 * 8) * 8),
                ("n_p", C.c_int32), ("pset", C.c_int32 * 16),
                ("homo", C.c_int32), ("mixed", C.c_int32), ("use_all", C.c_int32),
                ("r_layer", C.c_int32), ("pmax", C.c_int32), ("r_batch", C.c_int32),
                ("mem_check", C.c_int32), ("sync_overlap", C.c_int32),
                ("interleave", C.c_int32), ("ep_dp", C.c_int32), ("mixtp", C.c_int32),
                ("sync_buckets", C.c_int32)]


def _path(hops):
    p = _Path()
    p.n = len(hops)
    for k, hp in enumerate(hops):
        p.hop[k].gbps = hp["gbps"]
        p.hop[k].bidir = hp["bidir"]
    return p


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [C.POINTER(_Input)]
        L.orc_destroy.argtypes = [C.c_void_p]
        for f in ("orc_space_size", "orc_n_templates"):
            getattr(L, f).restype = C.c_int64
            getattr(L, f).argtypes = [C.c_void_p]
        L.orc_template_prefix.restype = C.c_int64
        L.orc_template_prefix.argtypes = [C.c_void_p, C.c_int64]
        L.orc_eval.restype = C.c_int64
        L.orc_eval.argtypes = [C.c_void_p, C.c_int64]
        L.orc_eval_many.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int]
        L.orc_describe.restype = C.c_int
        L.orc_describe.argtypes = [C.c_void_p, C.c_int64, C.c_char_p, C.c_int]
        L.orc_hop_delay_exact.restype = C.c_double
        L.orc_hop_delay_exact.argtypes = [C.c_double, C.c_int, C.c_int64]
        L.orc_ring_sim.restype = C.c_int64
        L.orc_ring_sim.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.orc_pipeline.restype = C.c_int64
        L.orc_pipeline.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_hamilton.argtypes = [C.c_int64, C.c_void_p, C.c_int, C.c_void_p]
        L.orc_op.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                             C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.orc_link.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                               C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        L.orc_last_error.restype = C.c_char_p
        L.orc_segment_bytes.restype = C.c_int64
        L.orc_segment_bytes.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int]
        L.orc_act_bytes.restype = C.c_int64
        L.orc_act_bytes.argtypes = [C.c_void_p, C.c_int]
        L.orc_set_compact.argtypes = [C.c_void_p, C.c_int]
        for f in ("orc_tp_allreduce", "orc_ep_alltoall"):
            getattr(L, f).restype = C.c_int64
            getattr(L, f).argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]
        L.orc_segments.restype = C.c_int
        L.orc_segments.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int]
        L.orc_needs_reshard.restype = C.c_int
        L.orc_needs_reshard.argtypes = [C.c_int] * 5
        L.orc_flow_resim.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64]
        L.orc_flow_sim.argtypes = [C.c_void_p, C.c_int] + [C.c_void_p] * 3 + [C.c_int] + [C.c_void_p] * 5
        L.orc_maxmin.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_pipeline_ilv.restype = C.c_int64
        L.orc_pipeline_ilv.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
        L.orc_op_order.restype = C.c_int
        L.orc_op_order.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int]
        L.orc_ep_alltoall_groups.restype = C.c_int64
        L.orc_ep_alltoall_groups.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int]
        L.orc_device_bytes.restype = C.c_int64
        L.orc_device_bytes.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int]
    return _lib


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


class Oracle:
    """The reference simulator for one workload dict (hsim_inputs.configs)."""

    def __init__(self, cfg, compact=False):
        """compact=True selects the oracle's compact mode (one pipeline per
        sub-class, closed-form ring steps; oracle.cpp header) -- equal to the
        literal mode by tests/test_oracle_compact.py."""
        self.cfg = cfg
        cl, md, se = cfg["cluster"], cfg["model"], cfg["search"]
        nt = len(cl["types"])
        self._types = (_Type * nt)()
        for k, t in enumerate(cl["types"]):
            T = self._types[k]
            T.peak_flop_per_ns = t["peak_flop_per_ns"]
            T.hbm_bytes_per_ns = t["hbm_bytes_per_ns"]
            for q in range(5):
                T.eff_flop[q] = t["eff_flop"][q]
                T.eff_mem[q] = t["eff_mem"][q]
            T.mem_bytes = t["mem_bytes"]
            T.gpus_per_node = t["gpus_per_node"]
            T.n_link_kinds = len(t["link_kinds"])
            for q, hops in enumerate(t["link_kinds"]):
                T.link_kind[q] = _path(hops)
            for i, row in enumerate(t["intra_kind"]):
                for j, v in enumerate(row):
                    T.intra_kind[i][j] = v
            T.gpu_nic = _path(t["gpu_nic"])
            T.nic_gbps = t["nic_gbps"]
            T.nic_delay_ns = t["nic_delay_ns"]
        self._nodes = (C.c_int32 * len(cl["nodes"]))(*cl["nodes"])
        I = _Input()
        I.n_types, I.n_nodes = nt, len(cl["nodes"])
        I.types = self._types
        I.node_type = self._nodes
        I.rail_alpha_ns, I.rail_gbps, I.frame_bytes = cl["rail_alpha_ns"], cl["rail_gbps"], cl["frame_bytes"]
        for k, key in (("L", "layers"), ("h", "hidden"), ("heads", "heads"), ("kv_heads", "kv_heads"),
                       ("ffn", "ffn"), ("nm", "mlp_mats"), ("seq", "seq"), ("V", "vocab"), ("tied", "tied"),
                       ("E", "moe_experts"), ("topk", "moe_topk"), ("bpe_act", "bpe_act"),
                       ("bpe_grad", "bpe_grad"), ("B", "global_batch")):
            setattr(I, k, md[key])
        I.n_b = len(se["bset"])
        for q, v in enumerate(se["bset"]):
            I.bset[q] = v
        for t, tps in enumerate(se["tpset"]):
            I.n_tp[t] = len(tps)
            for q, v in enumerate(tps):
                I.tpset[t][q] = v
        I.n_p = len(se["pset"])
        for q, v in enumerate(se["pset"]):
            I.pset[q] = v
        I.homo, I.mixed, I.use_all = se["homo"], se["mixed"], se["use_all"]
        I.r_layer, I.pmax, I.r_batch = se["r_layer"], se["pmax_perturb"], se["r_batch"]
        I.mem_check = int(se.get("mem_check", 0))
        I.sync_overlap = int(se.get("sync_overlap", 0))
        I.interleave = int(se.get("interleave", 1))
        I.ep_dp = int(se.get("ep_dp", 0))
        I.mixtp = int(se.get("mixtp", 0))
        I.sync_buckets = int(se.get("sync_buckets", 1))
        self._in = I
        self.h = lib().orc_create(C.byref(I))
        if not self.h:
            raise ValueError(lib().orc_last_error().decode())
        lib().orc_set_compact(self.h, int(compact))
        self.compact = bool(compact)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_destroy(self.h)
            self.h = None

    def space_size(self):
        return lib().orc_space_size(self.h)

    def n_templates(self):
        return lib().orc_n_templates(self.h)

    def template_prefix(self):
        n = self.n_templates()
        return np.array([lib().orc_template_prefix(self.h, k) for k in range(n + 1)], dtype=np.int64)

    def eval(self, i):
        return lib().orc_eval(self.h, int(i))

    def eval_many(self, idx=None, first=0, n=None, threads=None):
        threads = threads or os.cpu_count() or 1
        if idx is not None:
            idx = _i64(idx)
            out = np.empty(len(idx), dtype=np.int64)
            lib().orc_eval_many(self.h, idx.ctypes.data, 0, len(idx), out.ctypes.data, threads)
        else:
            out = np.empty(n, dtype=np.int64)
            lib().orc_eval_many(self.h, None, first, n, out.ctypes.data, threads)
        return out

    def topk(self, k, threads=None):
        """Brute force: evaluate every candidate, keep the k smallest (T, i)."""
        n = self.space_size()
        t = self.eval_many(first=0, n=n, threads=threads)
        ok = np.nonzero(t >= 0)[0]
        order = np.lexsort((ok, t[ok]))[:k]
        return t[ok][order], ok[order].astype(np.int64)

    def describe(self, i):
        buf = C.create_string_buffer(1 << 20)
        rc = lib().orc_describe(self.h, int(i), buf, len(buf))
        if rc != 0:
            raise IndexError(i)
        return json.loads(buf.value.decode())

    def op(self, type_idx, kind, bwd, tp, b):
        f, by, d = C.c_int64(), C.c_int64(), C.c_int64()
        lib().orc_op(self.h, type_idx, KIND.get(kind, kind), int(bwd), tp, b, C.byref(f), C.byref(by), C.byref(d))
        return f.value, by.value, d.value

    def segment_bytes(self, n_layers, has_first, has_last):
        return lib().orc_segment_bytes(self.h, n_layers, int(has_first), int(has_last))

    def device_bytes(self, type_idx, tp, P, s, layers, mb, b):
        """DESIGN M.1: bytes one device of stage s (of P) needs (f2 memory check)."""
        return lib().orc_device_bytes(self.h, type_idx, tp, P, s, layers, mb, b)

    def ep_alltoall_groups(self, groups, tp, b):
        """DESIGN V.3: all-to-all over the union of the (node, base) TP groups."""
        nodes = np.array([g[0] for g in groups], dtype=np.int32)
        bases = np.array([g[1] for g in groups], dtype=np.int32)
        return lib().orc_ep_alltoall_groups(self.h, nodes.ctypes.data, bases.ctypes.data, len(groups), tp, b)

    def tp_allreduce(self, node, base, tp, b):
        return lib().orc_tp_allreduce(self.h, node, base, tp, b)

    def ep_alltoall(self, node, base, tp, b):
        return lib().orc_ep_alltoall(self.h, node, base, tp, b)

    def segments(self, i):
        """Gradient-sync segments of candidate i: list of dicts a, z, S, tstar, RS, AR."""
        buf = np.zeros(6 * 256, dtype=np.int64)
        J = lib().orc_segments(self.h, int(i), buf.ctypes.data, 256)
        if J < 0:
            raise ValueError(f"candidate {i}: status {J}")
        keys = ("a", "z", "S", "tstar", "RS", "AR")
        return [dict(zip(keys, (int(x) for x in buf[6 * j:6 * j + 6]))) for j in range(J)]

    def flow_resim(self, i, fct_cap=0):
        """f3 (DESIGN F.1): dict(status, sync_ab, sync_flow, n_flows, T0, T_iter[, fct]);
        T0 / T_iter from the compact mode's C.8 evaluation of the same candidate."""
        out = np.zeros(6, dtype=np.int64)
        fct = np.zeros(max(fct_cap, 1), dtype=np.int64)
        lib().orc_flow_resim(self.h, int(i), out.ctypes.data, fct.ctypes.data if fct_cap else None, fct_cap)
        r = dict(zip(("status", "sync_ab", "sync_flow", "n_flows", "T0", "T_iter"), (int(x) for x in out)))
        if fct_cap:
            r["fct"] = fct[:min(fct_cap, r["n_flows"])].copy()
        return r

    def flow_sim(self, linkcap, flows):
        """The f3 fluid engine on independent flows: flows = list of dicts
        (links, arrive, bytes, alpha, cap); returns completion times."""
        nf = len(flows)
        maxl = max([len(f["links"]) for f in flows] + [1])
        inc = np.full(nf * maxl, -1, dtype=np.int32)
        for k, f in enumerate(flows):
            inc[k * maxl:k * maxl + len(f["links"])] = f["links"]
        nfl = np.array([len(f["links"]) for f in flows], dtype=np.int32)
        lc = np.asarray(linkcap, dtype=np.float64)
        arr = _i64([f["arrive"] for f in flows])
        by = _i64([f["bytes"] for f in flows])
        al = _i64([f["alpha"] for f in flows])
        cp = np.asarray([f["cap"] for f in flows], dtype=np.float64)
        done = np.zeros(nf, dtype=np.int64)
        lib().orc_flow_sim(self.h, nf, lc.ctypes.data, nfl.ctypes.data, inc.ctypes.data, maxl, arr.ctypes.data,
                           by.ctypes.data, al.ctypes.data, cp.ctypes.data, done.ctypes.data)
        return done

    def act_bytes(self, b):
        return lib().orc_act_bytes(self.h, b)

    def link(self, n1, r1, n2, r2):
        a, b = C.c_int64(), C.c_double()
        lib().orc_link(self.h, n1, r1, n2, r2, C.byref(a), C.byref(b))
        return a.value, b.value


def hop_delay_exact(gbps, bidir, frame=9200):
    return lib().orc_hop_delay_exact(gbps, int(bidir), frame)


def ring_sim(taus, steps):
    a = _i64(taus)
    return lib().orc_ring_sim(a.ctypes.data, len(a), steps)


def pipeline(f, g, c, m):
    f, g = _i64(f), _i64(g)
    P = len(f)
    c = _i64(list(c) + [0]) if P > 1 else _i64([0])
    return lib().orc_pipeline(P, m, f.ctypes.data, g.ctypes.data, c.ctypes.data)


def pipeline_ilv(f, g, c, cw, m):
    """DESIGN V.2: interleaved 1F1B; f, g = [P][v] chunk durations, c = P-1 boundary
    costs, cw = wrap cost."""
    f, g = np.ascontiguousarray(f, dtype=np.int64), np.ascontiguousarray(g, dtype=np.int64)
    P, v = f.shape
    c = _i64(list(c) + [0])
    return lib().orc_pipeline_ilv(P, v, m, f.ctypes.data, g.ctypes.data, c.ctypes.data, cw)


def op_order(P, s, m, v):
    """The op list of stage s: [(fwd, chunk, micro-batch)]."""
    buf = np.zeros(3 * 2 * m * v + 3, dtype=np.int32)
    n = lib().orc_op_order(P, s, m, v, buf.ctypes.data, 2 * m * v + 1)
    return [tuple(int(x) for x in buf[3 * k:3 * k + 3]) for k in range(n)]


def maxmin(linkcap, flows, caps):
    """Progressive-filling max-min rates (the oracle's f3 building block):
    flows = list of link-index lists, caps = per-flow private caps."""
    nf, nl = len(flows), len(linkcap)
    maxl = max([len(f) for f in flows] + [1])
    inc = np.full(nf * maxl, -1, dtype=np.int32)
    for k, f in enumerate(flows):
        inc[k * maxl:k * maxl + len(f)] = f
    nfl = np.array([len(f) for f in flows], dtype=np.int32)
    lc = np.asarray(linkcap, dtype=np.float64)
    cp = np.asarray(caps, dtype=np.float64)
    rate = np.zeros(nf, dtype=np.float64)
    lib().orc_maxmin(nf, nl, lc.ctypes.data, nfl.ctypes.data, inc.ctypes.data, maxl, cp.ctypes.data, rate.ctypes.data)
    return rate


def needs_reshard(src_tp, src_mb, dst_tp, dst_mb, pp_only=False):
    return bool(lib().orc_needs_reshard(src_tp, src_mb, dst_tp, dst_mb, int(pp_only)))


def hamilton(n, w):
    w = _i64(w)
    out = np.zeros(len(w), dtype=np.int64)
    lib().orc_hamilton(n, w.ctypes.data, len(w), out.ctypes.data)
    return out
