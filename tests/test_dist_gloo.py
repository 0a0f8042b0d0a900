"""Multi-process (world size 2, gloo, CPU) coverage of the multi-GPU sweep's
host logic: block-cyclic sharding, the all_gather of per-rank top-k lists and
the merge, against a brute-force oracle top-k.  The per-rank evaluator is the
oracle (test infrastructure) behind the same topk() signature as Sim; the
merge is a plain lexicographic merge (the device merge kernel is covered by
the GPU tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import hsim_inputs as H
from paper_2508_05370_b200.sweep import shard, shard_indices, sweep

INF = np.iinfo(np.int64).max


class OracleSim:
    """Sim-like adapter over the CPU oracle (tests only)."""

    def __init__(self, cfg):
        import oracle
        self.o = oracle.Oracle(cfg)

    def space_size(self):
        return self.o.space_size()

    def topk(self, k, n, first=0, block=0, stride=0, out=None, stream=None):
        if block:
            idx = np.array([first + (t // block) * stride + t % block for t in range(n)], dtype=np.int64)
        else:
            idx = np.arange(first, first + n, dtype=np.int64)
        t = self.o.eval_many(idx, threads=2)
        ok = np.nonzero(t >= 0)[0]
        order = np.lexsort((idx[ok], t[ok]))[:k]
        tt = np.full(k, INF, dtype=np.int64)
        ii = np.full(k, -1, dtype=np.int64)
        tt[:len(order)] = t[ok][order]
        ii[:len(order)] = idx[ok][order]
        out[0].copy_(torch.from_numpy(tt))
        out[1].copy_(torch.from_numpy(ii))
        return out


def cpu_merge(gathered, k, out):
    g = gathered.numpy()
    t = g[:, :k].ravel()
    i = g[:, k:].ravel()
    keep = i >= 0
    order = np.lexsort((i[keep], t[keep]))[:k]
    tt = np.full(k, INF, dtype=np.int64)
    ii = np.full(k, -1, dtype=np.int64)
    tt[:len(order)] = t[keep][order]
    ii[:len(order)] = i[keep][order]
    return torch.from_numpy(tt), torch.from_numpy(ii)


def _worker(rank, world, port, seed, k, block, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sim = OracleSim(H.tiny_random(seed))
        t, i = sweep(sim, k, block=block, merge=cpu_merge, device="cpu")
        q.put((rank, t.tolist(), i.tolist()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n,world,block", [(10, 2, 3), (1000, 4, 64), (5, 8, 1), (1 << 20, 8, 1 << 16), (7, 3, 100)])
def test_shards_partition_the_space(n, world, block):
    seen = []
    for r in range(world):
        first, cnt, blk, stride = shard(n, r, world, block)
        idx = shard_indices(n, r, world, block)
        assert len(idx) == cnt
        seen += idx
    assert sorted(seen) == list(range(n))


@pytest.mark.parametrize("seed,k,block", [(101, 5, 2), (103, 16, 5)])
def test_sweep_world2_gloo_matches_bruteforce(oracle_mod, seed, k, block):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, seed, k, block, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    o = oracle_mod.Oracle(H.tiny_random(seed))
    wt, wi = o.topk(k)
    for rank, t, i in res:
        assert t[:len(wt)] == list(wt) and i[:len(wi)] == list(wi), rank
        assert all(x == INF for x in t[len(wt):]) and all(x == -1 for x in i[len(wi):])
