"""Thin Python binding of libhsim (include/hsim.h) — argument marshalling only.

The names mirror the C ABI: ``hsim_create``, ``hsim_destroy``,
``hsim_space_size``, ``hsim_decode``, ``hsim_eval_batch``, ``hsim_topk``.
Every step of the hot path runs in the CUDA kernels behind the C ABI; this
module only packs the workload dict (hsim_inputs/) into the C descriptors and
passes torch device pointers / streams through.  There is no CPU fallback:
loading fails loudly if the library or a CUDA device is missing.
"""
import ctypes as C
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HSIM_LIB", os.path.join(HERE, "libhsim.so"))  # override: kernel-variant experiments

HSIM_OK, HSIM_EINVAL, HSIM_ENOMEM, HSIM_ECUDA, HSIM_ERANGE, HSIM_ESTATE = range(6)
STATUS = {1: "HSIM_EINVAL", 2: "HSIM_ENOMEM", 3: "HSIM_ECUDA", 4: "HSIM_ERANGE", 5: "HSIM_ESTATE"}

# symbols include/hsim.h declares (checked by tests/test_abi.py)
EXPORTS = ("hsim_create", "hsim_destroy", "hsim_space_size", "hsim_n_templates", "hsim_template_first",
           "hsim_decode", "hsim_eval_batch", "hsim_topk", "hsim_last_launch_count", "hsim_count_cells",
           "hsim_last_error", "hsim_merge_topk", "hsim_flow_resim", "hsim_last_sync_units", "hsim_set_prune",
           "hsim_set_dedup", "hsim_dedup_active")


class HsimError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class hsim_hop(C.Structure):
    _fields_ = [("gbps", C.c_double), ("bidir", C.c_int32), ("_pad", C.c_int32)]


class hsim_path(C.Structure):
    _fields_ = [("n_hops", C.c_int32), ("_pad", C.c_int32), ("hops", hsim_hop * 4)]


class hsim_device_type(C.Structure):
    _fields_ = [("name", C.c_char * 16),
                ("peak_flop_per_ns", C.c_double), ("hbm_bytes_per_ns", C.c_double),
                ("eff_flop", C.c_double * 5), ("eff_mem", C.c_double * 5),
                ("mem_bytes", C.c_int64),
                ("gpus_per_node", C.c_int32), ("n_link_kinds", C.c_int32),
                ("link_kinds", hsim_path * 4),
                ("intra_kind", (C.c_int8 * 8) * 8),
                ("gpu_nic", hsim_path),
                ("nic_gbps", C.c_double),
                ("nic_delay_ns", C.c_int64)]


class hsim_cluster_desc(C.Structure):
    _fields_ = [("n_device_types", C.c_int32), ("n_nodes", C.c_int32),
                ("device_types", C.POINTER(hsim_device_type)),
                ("node_type_of", C.POINTER(C.c_int32)),
                ("rail_alpha_ns", C.c_int64), ("rail_gbps", C.c_double), ("frame_bytes", C.c_int64)]


class hsim_model_desc(C.Structure):
    _fields_ = [(k, C.c_int32) for k in ("layers", "hidden", "heads", "kv_heads", "ffn", "mlp_mats", "seq",
                                         "vocab", "tied", "moe_experts", "moe_topk", "bpe_act", "bpe_grad")] + \
               [("global_batch", C.c_int64),
                ("n_bset", C.c_int32), ("bset", C.c_int32 * 8),
                ("tpset_mask", C.c_int32 * 4),
                ("n_pset", C.c_int32), ("pset", C.c_int32 * 16),
                ("homo", C.c_int32), ("mixed", C.c_int32), ("use_all", C.c_int32),
                ("r_layer", C.c_int32), ("pmax_perturb", C.c_int32), ("r_batch", C.c_int32),
                ("mem_check", C.c_int32), ("sync_overlap", C.c_int32),
                ("interleave", C.c_int32), ("ep_dp", C.c_int32), ("mixtp", C.c_int32),
                ("sync_buckets", C.c_int32)]


class hsim_cands(C.Structure):
    _fields_ = [("idx", C.c_void_p), ("first", C.c_int64), ("block", C.c_int64), ("stride", C.c_int64)]


_lib = None


def lib():
    """Loads libhsim.so; raises if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_2508_05370_b200/build.py (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.hsim_create.restype = C.c_int
        L.hsim_create.argtypes = [C.POINTER(hsim_cluster_desc), C.POINTER(hsim_model_desc), C.POINTER(C.c_void_p)]
        L.hsim_destroy.argtypes = [C.c_void_p]
        for f in ("hsim_space_size", "hsim_n_templates"):
            getattr(L, f).restype = C.c_int64
            getattr(L, f).argtypes = [C.c_void_p]
        L.hsim_template_first.restype = C.c_int64
        L.hsim_template_first.argtypes = [C.c_void_p, C.c_int64]
        L.hsim_decode.restype = C.c_int
        L.hsim_decode.argtypes = [C.c_void_p, C.c_int64, C.c_char_p, C.c_size_t]
        L.hsim_eval_batch.restype = C.c_int
        L.hsim_eval_batch.argtypes = [C.c_void_p, C.POINTER(hsim_cands), C.c_int64, C.c_void_p, C.c_void_p]
        L.hsim_topk.restype = C.c_int
        L.hsim_topk.argtypes = [C.c_void_p, C.POINTER(hsim_cands), C.c_int64, C.c_int32,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.hsim_last_launch_count.restype = C.c_int32
        L.hsim_last_launch_count.argtypes = [C.c_void_p]
        L.hsim_set_prune.restype = C.c_int
        L.hsim_set_prune.argtypes = [C.c_void_p, C.c_int]
        L.hsim_set_dedup.restype = C.c_int
        L.hsim_set_dedup.argtypes = [C.c_void_p, C.c_int]
        L.hsim_dedup_active.restype = C.c_int
        L.hsim_dedup_active.argtypes = [C.c_void_p]
        L.hsim_last_sync_units.restype = C.c_int64
        L.hsim_last_sync_units.argtypes = [C.c_void_p]
        L.hsim_count_cells.restype = C.c_int64
        L.hsim_count_cells.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
        L.hsim_last_error.restype = C.c_char_p
        L.hsim_flow_resim.restype = C.c_int
        L.hsim_flow_resim.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        L.hsim_merge_topk.restype = C.c_int
        L.hsim_merge_topk.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


def _err(code):
    raise HsimError(code, lib().hsim_last_error().decode())


def _path(hops):
    p = hsim_path()
    p.n_hops = len(hops)
    for k, hp in enumerate(hops):
        p.hops[k].gbps = hp["gbps"]
        p.hops[k].bidir = hp["bidir"]
    return p


def descriptors(cfg):
    """Packs a workload dict into (hsim_cluster_desc, hsim_model_desc, keepalive)."""
    cl, md, se = cfg["cluster"], cfg["model"], cfg["search"]
    nt = len(cl["types"])
    types = (hsim_device_type * max(nt, 1))()
    for k, t in enumerate(cl["types"]):
        T = types[k]
        T.name = t["name"].encode()[:15]
        T.peak_flop_per_ns = t["peak_flop_per_ns"]
        T.hbm_bytes_per_ns = t["hbm_bytes_per_ns"]
        for q in range(5):
            T.eff_flop[q] = t["eff_flop"][q]
            T.eff_mem[q] = t["eff_mem"][q]
        T.mem_bytes = t["mem_bytes"]
        T.gpus_per_node = t["gpus_per_node"]
        T.n_link_kinds = len(t["link_kinds"])
        for q, hops in enumerate(t["link_kinds"]):
            T.link_kinds[q] = _path(hops)
        for i, row in enumerate(t["intra_kind"]):
            for j, v in enumerate(row):
                T.intra_kind[i][j] = v
        T.gpu_nic = _path(t["gpu_nic"])
        T.nic_gbps = t["nic_gbps"]
        T.nic_delay_ns = t["nic_delay_ns"]
    nodes = (C.c_int32 * max(len(cl["nodes"]), 1))(*cl["nodes"])
    cd = hsim_cluster_desc(nt, len(cl["nodes"]), types, nodes, cl["rail_alpha_ns"], cl["rail_gbps"], cl["frame_bytes"])
    m = hsim_model_desc()
    for k in ("layers", "hidden", "heads", "kv_heads", "ffn", "mlp_mats", "seq", "vocab", "tied",
              "moe_experts", "moe_topk", "bpe_act", "bpe_grad", "global_batch"):
        setattr(m, k, md[k])
    m.n_bset = len(se["bset"])
    for q, v in enumerate(se["bset"]):
        m.bset[q] = v
    for t, tps in enumerate(se["tpset"]):
        m.tpset_mask[t] = sum(1 << (v.bit_length() - 1) for v in tps)
    m.n_pset = len(se["pset"])
    for q, v in enumerate(se["pset"]):
        m.pset[q] = v
    for k in ("homo", "mixed", "use_all", "r_layer", "pmax_perturb", "r_batch"):
        setattr(m, k, se[k])
    m.mem_check = int(se.get("mem_check", 0))
    m.sync_overlap = int(se.get("sync_overlap", 0))
    m.interleave = int(se.get("interleave", 1))
    m.ep_dp = int(se.get("ep_dp", 0))
    m.mixtp = int(se.get("mixtp", 0))
    m.sync_buckets = int(se.get("sync_buckets", 1))
    return cd, m, (types, nodes)


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


class Sim:
    """One (cluster, model, search space): the handle of hsim_create."""

    def __init__(self, cfg, host_only=False):
        """host_only=True builds the host-side tables without a GPU (space
        size, templates, decode); evaluation then fails with HSIM_ECUDA."""
        if not host_only:
            import torch
            if not torch.cuda.is_available():
                raise RuntimeError("hsim needs a CUDA device (B200); there is no CPU path")
            torch.cuda.init()
        cd, md, keep = descriptors(cfg)
        h = C.c_void_p()
        rc = lib().hsim_create(C.byref(cd), C.byref(md), C.byref(h))
        if rc:
            _err(rc)
        self.h = h
        self.cfg = cfg

    def close(self):
        if getattr(self, "h", None):
            lib().hsim_destroy(self.h)
            self.h = None

    __del__ = close

    def space_size(self):
        return lib().hsim_space_size(self.h)

    def n_templates(self):
        return lib().hsim_n_templates(self.h)

    def template_first(self, k):
        return lib().hsim_template_first(self.h, k)

    def decode(self, i):
        buf = C.create_string_buffer(1 << 22)
        rc = lib().hsim_decode(self.h, int(i), buf, len(buf))
        if rc:
            _err(rc)
        return json.loads(buf.value.decode())

    @staticmethod
    def _cands(first, idx, block, stride):
        c = hsim_cands()
        c.idx = idx.data_ptr() if idx is not None else None
        c.first, c.block, c.stride = first, block, stride
        return c

    def eval_batch(self, n=None, first=0, idx=None, out=None, block=0, stride=0, stream=None):
        """Evaluates candidates [first, first+n) (or the device tensor idx);
        returns the int64 device tensor of iteration times (negative = invalid)."""
        import torch
        if idx is not None:
            assert idx.is_cuda and idx.dtype == torch.int64 and idx.is_contiguous()
            n = idx.numel()
        if n is None:
            n = self.space_size() - first
        if out is None:
            out = torch.empty(n, dtype=torch.int64, device="cuda")
        c = self._cands(first, idx, block, stride)
        rc = lib().hsim_eval_batch(self.h, C.byref(c), n, C.c_void_p(out.data_ptr() if n else 0), _stream(stream))
        if rc:
            _err(rc)
        return out

    def eval_host(self, idx_host, out_host, chunks=2, stream=None):
        """End-to-end evaluation of an index list in pinned host memory into a
        pinned host result buffer (the same hsim_eval_batch calls, chunked):
        the H2D copy of chunk c+1 and the D2H copy of chunk c-1 overlap the
        evaluation of chunk c (two copy streams + events).  On return the
        caller's stream has every copy queued before its next work."""
        import torch
        n = idx_host.numel()
        assert idx_host.dtype == torch.int64 and out_host.dtype == torch.int64 and out_host.numel() >= n
        comp = stream or torch.cuda.current_stream()
        if getattr(self, "_host_buf", None) is None or self._host_buf[0].numel() < n:
            self._host_buf = (torch.empty(n, dtype=torch.int64, device="cuda"),
                              torch.empty(n, dtype=torch.int64, device="cuda"),
                              torch.cuda.Stream(), torch.cuda.Stream())
        idx_dev, out_dev, s_in, s_out = self._host_buf
        s_in.wait_stream(comp)   # buffers free: earlier work on the caller's stream is done
        s_out.wait_stream(comp)
        step = max(1, -(-n // max(1, chunks)))
        for c0 in range(0, n, step):
            c1 = min(n, c0 + step)
            with torch.cuda.stream(s_in):
                idx_dev[c0:c1].copy_(idx_host[c0:c1], non_blocking=True)
            comp.wait_stream(s_in)
            self.eval_batch(idx=idx_dev[c0:c1], out=out_dev[c0:c1], stream=comp)
            s_out.wait_stream(comp)
            with torch.cuda.stream(s_out):
                out_host[c0:c1].copy_(out_dev[c0:c1], non_blocking=True)
        comp.wait_stream(s_out)
        return out_host

    def topk(self, k, n=None, first=0, idx=None, block=0, stride=0, out_ns=None, stream=None, out=None):
        """Top-k (time asc, index asc) over the candidates; returns device tensors (t_ns, idx)."""
        import torch
        if idx is not None:
            n = idx.numel()
        if n is None:
            n = self.space_size() - first
        if out is None:
            out = (torch.empty(k, dtype=torch.int64, device="cuda"), torch.empty(k, dtype=torch.int64, device="cuda"))
        t, i = out
        c = self._cands(first, idx, block, stride)
        rc = lib().hsim_topk(self.h, C.byref(c), n, k, C.c_void_p(t.data_ptr()), C.c_void_p(i.data_ptr()),
                             C.c_void_p(out_ns.data_ptr() if out_ns is not None else 0), _stream(stream))
        if rc:
            _err(rc)
        return t, i

    FLOW_FIELDS = ("status", "sync_ab", "sync_flow", "n_flows", "fct_p50", "fct_p99", "fct_p999", "fct_max")

    def flow_resim(self, idx, fct_cap=0, stream=None):
        """SURVEY 8(f) f3 (hsim_flow_resim): flow-level re-simulation of the
        gradient sync of the candidates in the device tensor idx.  Returns the
        (k, 8) int64 device tensor (FLOW_FIELDS) and, if fct_cap > 0, the
        (k, fct_cap) tensor of flow completion times (unordered, -1 padded)."""
        import torch
        assert idx.is_cuda and idx.dtype == torch.int64 and idx.is_contiguous()
        k = idx.numel()
        out = torch.empty((k, 8), dtype=torch.int64, device=idx.device)
        fct = torch.full((k, fct_cap), -1, dtype=torch.int64, device=idx.device) if fct_cap else None
        rc = lib().hsim_flow_resim(self.h, C.c_void_p(idx.data_ptr() if k else 0), k,
                                   C.c_void_p(out.data_ptr() if k else 0),
                                   C.c_void_p(fct.data_ptr() if fct is not None else 0), fct_cap, _stream(stream))
        if rc:
            _err(rc)
        return (out, fct) if fct_cap else out

    def last_launch_count(self):
        return lib().hsim_last_launch_count(self.h)

    def set_prune(self, on):
        """Pruned sync in top-k sweeps (default on; exact either way)."""
        rc = lib().hsim_set_prune(self.h, int(bool(on)))
        if rc:
            _err(rc)

    def set_dedup(self, on):
        """One 1F1B run per distinct class pipeline (default on; exact either way)."""
        rc = lib().hsim_set_dedup(self.h, int(bool(on)))
        if rc:
            _err(rc)

    def dedup_active(self):
        """Whether calls on this handle use the pipeline dedupe."""
        return lib().hsim_dedup_active(self.h) == 1

    def last_sync_units(self):
        """Sum over the candidates whose gradient sync the last pruned top-k call
        computed of J = sum P - C + 1 (-1: the call did not prune)."""
        return lib().hsim_last_sync_units(self.h)

    def count_cells(self, first=0, n=None):
        n = self.space_size() - first if n is None else n
        v = lib().hsim_count_cells(self.h, first, n)
        if v < 0:
            _err(HSIM_ERANGE)
        return v


def hsim_merge_topk(lists, k, out=None, stream=None):
    """Merges a device tensor of shape (nlists, 2k) = [times | indices] per
    sorted list (the all_gather layout) into the global top-k."""
    import torch
    assert lists.is_cuda and lists.dtype == torch.int64 and lists.is_contiguous() and lists.shape[-1] == 2 * k
    if out is None:
        out = (torch.empty(k, dtype=torch.int64, device="cuda"), torch.empty(k, dtype=torch.int64, device="cuda"))
    nl = lists.numel() // (2 * k)
    rc = lib().hsim_merge_topk(C.c_void_p(lists.data_ptr() if nl else 0), nl, k, C.c_void_p(out[0].data_ptr()),
                               C.c_void_p(out[1].data_ptr()), _stream(stream))
    if rc:
        _err(rc)
    return out


# C-ABI-named functional surface ------------------------------------------------
def hsim_create(cfg):
    return Sim(cfg)


def hsim_destroy(sim):
    sim.close()


def hsim_space_size(sim):
    return sim.space_size()


def hsim_decode(sim, i):
    return sim.decode(i)


def hsim_eval_batch(sim, **kw):
    return sim.eval_batch(**kw)


def hsim_topk(sim, k, **kw):
    return sim.topk(k, **kw)
