"""Device/node presets — plain DATA, no arithmetic of the method.

Shared input plumbing for both the product (``paper_2508_05370_b200``) and the
test oracle (``oracle/``).  Every number here is a datasheet-style figure or a
value printed in the paper; the method's derivations (link delays, rates,
durations) are done independently on each side.

Sources
-------
* Table 4 ("Cluster specific configurations"): A100 and H100
  NVLink / PCIe bandwidths (listed bidirectional, Gbps), NIC 200 Gbps and the
  368 ns NIC processing delay.
* Jumbo frame of 9200 B for the per-hop delay formula.
* Other GPUs (V100, A100-PCIe, B200, GH200/GH200e) are synthetic
  datasheet-style presets (DESIGN.md §3 "input recipe"); parity never depends
  on their values.

Units
-----
``peak_flop_per_ns`` (dense bf16 FLOP per ns = TFLOP/s x 1000),
``hbm_bytes_per_ns`` (= GB/s), link ``gbps`` as listed (``bidir`` says whether
the listed figure is a bidirectional aggregate), ``nic_gbps`` per direction,
``nic_delay_ns`` as listed (Table 4 column) or ``9200*8/nic_gbps`` for
non-Table-4 NICs, written here as the literal integer.

Kinds (index into ``eff_flop`` / ``eff_mem``): 0 attn, 1 mlp, 2 moe, 3 emb, 4 head.
"""

NKIND = 5
EFF_FLOP = [0.5] * NKIND   # DESIGN.md reading A4: eff 0.5 for every FLOP kind
EFF_MEM = [1.0] * NKIND    # and 1.0 for memory


def _hop(gbps, bidir=True):
    return {"gbps": float(gbps), "bidir": 1 if bidir else 0}


def _all_pairs(g, kind):
    return [[-1 if i == j else kind for j in range(g)] for i in range(g)]


def _dev(name, peak, hbm, mem_gb, gpus, link_kinds, intra_kind, gpu_nic, nic_gbps, nic_delay_ns):
    return {
        "name": name,
        "peak_flop_per_ns": float(peak),
        "hbm_bytes_per_ns": float(hbm),
        "eff_flop": list(EFF_FLOP),
        "eff_mem": list(EFF_MEM),
        "mem_bytes": int(mem_gb) * (1 << 30),
        "gpus_per_node": gpus,
        "link_kinds": link_kinds,
        "intra_kind": intra_kind,
        "gpu_nic": gpu_nic,
        "nic_gbps": float(nic_gbps),
        "nic_delay_ns": int(nic_delay_ns),
    }


def a100_sxm(gpus=8):
    """Table 4 Ampere row: NVLink Gen3 4800 Gbps (bidir), PCIe Gen4 512 Gbps
    (bidir), ConnectX-6 200 Gbps, NIC delay 368 ns.  NVSwitch node: every
    GPU pair is GPU->NVSwitch->GPU (2 NVLink hops); GPU->NIC is two PCIe trips
    (PAPER.md:396)."""
    return _dev("A100", 312000, 1555, 40, gpus,
                [[_hop(4800), _hop(4800)]], _all_pairs(gpus, 0),
                [_hop(512), _hop(512)], 200, 368)


def h100_sxm(gpus=8):
    """Table 4 Hopper row: NVLink Gen4 7200, PCIe Gen5 1024, NIC 200 / 368 ns."""
    return _dev("H100", 989400, 3350, 80, gpus,
                [[_hop(7200), _hop(7200)]], _all_pairs(gpus, 0),
                [_hop(1024), _hop(1024)], 200, 368)


def b200(gpus=8):
    """Synthetic: NVLink 5 14400 Gbps bidir, PCIe Gen5 1024, NIC 400 / 184 ns."""
    return _dev("B200", 2250000, 8000, 180, gpus,
                [[_hop(14400), _hop(14400)]], _all_pairs(gpus, 0),
                [_hop(1024), _hop(1024)], 400, 184)


def v100_dgx1(gpus=8):
    """Synthetic DGX-1-like hybrid cube-mesh: same-quad pairs share one
    NVLink2 link (400 Gbps bidir), partners (i, i+4) two links (800), the
    other pairs go over two PCIe Gen3 trips (256 bidir each).  NIC 100 / 736."""
    assert gpus == 8

    def kind(i, j):
        if i == j:
            return -1
        if i // 4 == j // 4:
            return 0
        if abs(i - j) == 4:
            return 1
        return 2
    intra = [[kind(i, j) for j in range(8)] for i in range(8)]
    return _dev("V100", 125000, 900, 32, 8,
                [[_hop(400)], [_hop(800)], [_hop(256), _hop(256)]], intra,
                [_hop(256), _hop(256)], 100, 736)


def a100_pcie(gpus=8):
    """Synthetic A100-PCIe box: NVLink bridges on pairs (2k, 2k+1) (one 4800
    Gbps bidir hop), other pairs two PCIe Gen4 trips.  NIC 200 / 368."""
    def kind(i, j):
        if i == j:
            return -1
        return 0 if i // 2 == j // 2 else 1
    intra = [[kind(i, j) for j in range(gpus)] for i in range(gpus)]
    return _dev("A100P", 312000, 1555, 40, gpus,
                [[_hop(4800)], [_hop(512), _hop(512)]], intra,
                [_hop(512), _hop(512)], 200, 368)


def gh200_quad(name="GH200", hbm=4000, mem_gb=96):
    """Synthetic Grace-Hopper quad node (4 superchips): near pairs (0,1),(2,3)
    one 4800 Gbps hop, far pairs one 2400 Gbps hop; GPU->NIC crosses C2C
    (7200 bidir) then one PCIe Gen5 trip (1024).  NIC 200 / 368."""
    def kind(i, j):
        if i == j:
            return -1
        return 0 if i // 2 == j // 2 else 1
    intra = [[kind(i, j) for j in range(4)] for i in range(4)]
    return _dev(name, 989400, hbm, mem_gb, 4,
                [[_hop(4800)], [_hop(2400)]], intra,
                [_hop(7200), _hop(1024)], 200, 368)


def gh200e_quad():
    return gh200_quad("GH200e", 4900, 144)
