"""The five BASELINE.json workloads and seeded tiny workloads — plain DATA.

Shared input plumbing (see presets.py): no arithmetic of the method lives here.
A workload is a dict with three parts, mirroring the paper's three input
descriptions ("Input Description [A1, A2]"):

* ``cluster``: device types (Table 4 style rows, presets.py), the node list
  (device-type index per node; node id order = placement order), the rail
  switch hop and the jumbo frame size;
* ``model``: Table 5 style row plus GQA / SwiGLU / MoE /
  precision fields (reading A3);
* ``search``: the framework description as a *search space* (PAPER.md:183,
  "generate all possible combinations") — micro-batch sizes, TP degrees per
  device type, pipeline depths, families, perturbation radii (DESIGN.md C.2).

Knobs follow SURVEY.md §8(d).
"""
import copy

from . import presets
from .sampling import SplitMix64


def _cluster(types, counts, rail_gbps, gpus_per_node=None):
    """types: list of preset dicts; counts: number of nodes of each type."""
    nodes = []
    for t, n in enumerate(counts):
        nodes += [t] * n
    return {
        "frame_bytes": 9200,
        "rail_alpha_ns": 0,
        "rail_gbps": float(rail_gbps),
        "types": types,
        "nodes": nodes,
    }


def _model(layers, hidden, heads, kv_heads, ffn, mlp_mats, seq, vocab, tied,
           global_batch, experts=1, topk=1, bpe_act=2, bpe_grad=4):
    return dict(layers=layers, hidden=hidden, heads=heads, kv_heads=kv_heads,
                ffn=ffn, mlp_mats=mlp_mats, seq=seq, vocab=vocab, tied=int(tied),
                moe_experts=experts, moe_topk=topk, bpe_act=bpe_act,
                bpe_grad=bpe_grad, global_batch=global_batch)


def _search(bset, tpset, pset, homo, mixed, use_all, r_layer, pmax, r_batch):
    return dict(bset=list(bset), tpset=[list(t) for t in tpset], pset=list(pset),
                homo=int(homo), mixed=int(mixed), use_all=int(use_all),
                r_layer=r_layer, pmax_perturb=pmax, r_batch=r_batch)


def config1():
    """BASELINE config 1: GPT-2 small on 2xA100 + 2xH100 (2 GPUs per node),
    DP=2 PP=2, 4 micro-batches: exactly one candidate."""
    cl = _cluster([presets.a100_sxm(2), presets.h100_sxm(2)], [1, 1], 200)
    md = _model(12, 768, 12, 12, 3072, 2, 1024, 50257, True, 32)
    se = _search([4], [[1], [1]], [1], homo=0, mixed=1, use_all=1,
                 r_layer=0, pmax=0, r_batch=0)
    return {"name": "config1-gpt2s-2A100-2H100", "cluster": cl, "model": md, "search": se}


def config2():
    """BASELINE config 2 (the metric's sweep): Llama-2 7B on 16xA100 +
    16xH100, NVSwitch intra-node, 200 Gb rails; exhaustive TP/PP/DP + layer
    and batch split sweep."""
    cl = _cluster([presets.a100_sxm(), presets.h100_sxm()], [2, 2], 200)
    md = _model(32, 4096, 32, 32, 11008, 3, 4096, 32000, False, 1024)
    tp = [1, 2, 4, 8]
    se = _search([1, 2, 4, 8], [tp, tp], [1, 2, 4, 8, 16], homo=1, mixed=1,
                 use_all=0, r_layer=1, pmax=4, r_batch=1)
    return {"name": "config2-llama2-7b-16A100-16H100", "cluster": cl, "model": md, "search": se}


def config3():
    """BASELINE config 3: GPT-3 175B on 1024 GPUs = 48 V100 (DGX-1-like) +
    48 A100-PCIe (bridged) + 32 H100-SXM nodes."""
    cl = _cluster([presets.v100_dgx1(), presets.a100_pcie(), presets.h100_sxm()],
                  [48, 48, 32], 200)
    md = _model(96, 12288, 96, 96, 49152, 2, 2048, 50257, True, 1536)
    tp = [1, 2, 4, 8]
    se = _search([1, 2, 4], [tp, tp, tp], [1, 2, 4, 8, 16], homo=1, mixed=1,
                 use_all=1, r_layer=1, pmax=4, r_batch=1)
    return {"name": "config3-gpt3-175b-1024-V100-A100P-H100", "cluster": cl, "model": md, "search": se}


def config4():
    """BASELINE config 4: Mixtral 8x7B (Table 5 row + kv8, E=8, top-2) on
    8x8 B200 + 8x8 H100; DP groups with differing TP degree (reshard)."""
    cl = _cluster([presets.b200(), presets.h100_sxm()], [8, 8], 400)
    md = _model(32, 4096, 32, 8, 14336, 3, 2048, 32000, False, 1152,
                experts=8, topk=2)
    tp = [1, 2, 4, 8]
    se = _search([1, 2, 4], [tp, tp], [1, 2, 4], homo=1, mixed=1,
                 use_all=0, r_layer=1, pmax=4, r_batch=1)
    return {"name": "config4-mixtral-8x7b-64B200-64H100", "cluster": cl, "model": md, "search": se}


def config5():
    """BASELINE config 5: Llama-3 70B on 64 GH200 + 64 GH200e quad nodes."""
    cl = _cluster([presets.gh200_quad(), presets.gh200e_quad()], [64, 64], 200)
    md = _model(80, 8192, 64, 8, 28672, 3, 8192, 128256, False, 2048)
    tp = [1, 2, 4]
    se = _search([1, 2], [tp, tp], [2, 4, 5, 8, 10, 16, 20], homo=1, mixed=1,
                 use_all=0, r_layer=1, pmax=5, r_batch=2)
    return {"name": "config5-llama3-70b-512-GH200", "cluster": cl, "model": md, "search": se}


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def get(n):
    return CONFIGS[n]()


def tiny_random(seed):
    """A seeded tiny workload for brute-force tests: <= 2
    device types, <= 4 GPUs per type, few layers, tiny batch, every family
    and non-zero perturbation radii.  Values are drawn, not computed."""
    rng = SplitMix64(seed)
    pool = [presets.a100_sxm, presets.h100_sxm, presets.b200, presets.a100_pcie]
    ntypes = 1 + rng.below(2)
    picks = []
    while len(picks) < ntypes:
        f = pool[rng.below(len(pool))]
        if f not in picks:
            picks.append(f)
    gpn = [2, 4][rng.below(2)]
    types = [f(gpn) for f in picks]
    counts = [1 + rng.below(2) if gpn == 2 else 1 for _ in picks]
    cl = _cluster(types, counts, 200)
    layers = 2 + rng.below(5)
    heads = [2, 4][rng.below(2)]
    hidden = heads * [64, 128][rng.below(2)]
    moe = rng.below(3) == 0
    md = _model(layers, hidden, heads, heads if rng.below(2) else heads // 2,
                hidden * [2, 4][rng.below(2)], 2 + rng.below(2),
                [128, 256][rng.below(2)], 1000 + rng.below(5000), rng.below(2) == 1,
                [4, 6, 8][rng.below(3)],
                experts=4 if moe else 1, topk=2 if moe else 1)
    tp = [[1, 2], [1, 2, 4]][rng.below(2)]
    se = _search([1, 2], [tp] * ntypes, [1, 2, 3], homo=1, mixed=1 if ntypes > 1 else 0,
                 use_all=0, r_layer=1, pmax=3, r_batch=1)
    return {"name": f"tiny-{seed}", "cluster": cl, "model": md, "search": se}


def deep_tiny(variant=0):
    """Deep pipelines for the lane-per-stage kernels (16 < P <= 32 and
    32 < P <= 64): 4 A100 + 4 H100 nodes of 8 GPUs, a small 64-layer model,
    pipeline depths 17..32 per type (MIXED pipelines reach 34..64 stages),
    long steady regimes (M = 256 with b = 1).  variant 1: a100-pcie (bridge
    pairs) instead of A100 SXM, so p2p costs differ between boundaries."""
    first = presets.a100_pcie() if variant else presets.a100_sxm()
    cl = _cluster([first, presets.h100_sxm()], [4, 4], 200)
    md = _model(64, 256, 4, 4, 1024, 2, 128, 2000, True, 256)
    se = _search([1, 4], [[1, 2], [1]], [17, 20, 24, 31, 32], homo=1, mixed=1,
                 use_all=0, r_layer=1, pmax=2, r_batch=1)
    return {"name": f"deep-tiny-{variant}", "cluster": cl, "model": md, "search": se}


def four_types_tiny():
    """Four device types (A100, H100, B200, A100-PCIe), one 4-GPU node each:
    HOMO templates with up to four classes (the 4-class partition path)."""
    cl = _cluster([presets.a100_sxm(4), presets.h100_sxm(4), presets.b200(4), presets.a100_pcie(4)],
                  [1, 1, 1, 1], 200)
    md = _model(8, 256, 4, 4, 1024, 2, 128, 2000, False, 16)
    se = _search([2], [[1]] * 4, [1, 2], homo=1, mixed=0,
                 use_all=0, r_layer=0, pmax=0, r_batch=1)
    return {"name": "four-types-tiny", "cluster": cl, "model": md, "search": se}


def with_changes(cfg, **paths):
    """Copy of cfg with dotted-path overrides, e.g. ``model__global_batch=64``."""
    out = copy.deepcopy(cfg)
    for key, val in paths.items():
        node = out
        parts = key.split("__")
        for p in parts[:-1]:
            node = node[int(p)] if isinstance(node, list) else node[p]
        last = parts[-1]
        if isinstance(node, list):
            node[int(last)] = val
        else:
            node[last] = val
    return out


def with_mem_check(cfg, mem_bytes=None):
    """Copy of cfg with the memory-feasibility check on (SURVEY.md §8(f) f2,
    DESIGN.md M.1); optionally per-type capacities in bytes (plain data)."""
    out = copy.deepcopy(cfg)
    out["search"]["mem_check"] = 1
    if mem_bytes is not None:
        for t, v in zip(out["cluster"]["types"], mem_bytes):
            t["mem_bytes"] = int(v)
    out["name"] = out["name"] + "-memcheck"
    return out


def with_sync_overlap(cfg):
    """Copy of cfg with the gradient sync overlapped with the backward pass
    (DESIGN.md S.1) instead of after the barrier (C.8)."""
    out = copy.deepcopy(cfg)
    out["search"]["sync_overlap"] = 1
    out["name"] = out["name"] + "-overlap"
    return out


def with_interleave(cfg, v=2):
    """Copy of cfg with the interleaved 1F1B schedule, v model chunks per
    stage (DESIGN.md V.2)."""
    out = copy.deepcopy(cfg)
    out["search"]["interleave"] = int(v)
    out["name"] = out["name"] + f"-ilv{v}"
    return out


def with_ep_dp(cfg):
    """Copy of cfg with expert parallelism across the DP replicas of
    single-class MoE templates (DESIGN.md V.3)."""
    out = copy.deepcopy(cfg)
    out["search"]["ep_dp"] = 1
    out["name"] = out["name"] + "-epdp"
    return out


def variant_tiny(seed, moe=False):
    """A tiny workload (tiny_random's draw) with a larger global batch and more
    layers, so interleaved candidates (m mod P = 0, every chunk non-empty) and
    multi-replica EP groups are common; moe=True forces 4 experts, top-2."""
    cfg = tiny_random(seed)
    md = cfg["model"]
    md["global_batch"] = 12 * md["global_batch"]
    md["layers"] = md["layers"] + 4
    if moe:
        md["moe_experts"], md["moe_topk"] = 4, 2
    cfg["name"] = f"variant-tiny-{seed}{'-moe' if moe else ''}"
    return cfg
