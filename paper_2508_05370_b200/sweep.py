"""Multi-GPU sweep: the candidate space sharded block-cyclically over ranks
(one process per B200), per-rank top-k on the device, one NCCL all_gather of
the k-entry lists over NVLink, merged by the hsim_merge_topk kernel
(BASELINE.json north_star "merged by an NCCL allgather").

torch.distributed is plumbing only (process group + the one collective); the
evaluation and both top-k stages run in libhsim's kernels.  `merge` is
injectable so the host-side sharding / gather logic can be exercised on CPU
(gloo) by the tests.
"""
import torch
import torch.distributed as dist

DEFAULT_BLOCK = 1 << 16


def shard(n_space, rank, world, block=DEFAULT_BLOCK):
    """Block-cyclic shard of [0, n_space): (first, n, block, stride) for rank.
    Rank r owns blocks r, r+W, r+2W, ... of `block` consecutive indices."""
    if world == 1:
        return 0, n_space, 0, 0
    stride = world * block
    full, rem = divmod(n_space, stride)
    n = full * block + min(block, max(0, rem - rank * block))
    return rank * block, n, block, stride


def shard_indices(n_space, rank, world, block=DEFAULT_BLOCK):
    """The explicit index list of a shard (for tests and reports)."""
    first, n, blk, stride = shard(n_space, rank, world, block)
    if blk == 0:
        return list(range(first, first + n))
    return [first + (t // blk) * stride + t % blk for t in range(n)]


def _device_merge(gathered, k, out):
    from .hsim import hsim_merge_topk
    return hsim_merge_topk(gathered, k, out=out)


def sweep(sim, k, group=None, block=DEFAULT_BLOCK, stream=None, out=None, merge=None, device=None):
    """Global top-k (times, indices) over the whole space of `sim`, identical
    on every rank.  Single process when torch.distributed is not initialised.

    Everything -- the local top-k, the all_gather and the merge -- is queued on
    `stream` (default: the current stream): the NCCL collective is issued with
    `stream` as the current stream, so it waits for the local top-k."""
    import contextlib
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    first, n, blk, stride = shard(sim.space_size(), rank, world, block)
    device = device or "cuda"
    on_gpu = torch.device(device).type == "cuda"
    if on_gpu and stream is None:
        stream = torch.cuda.current_stream()
    ctx = torch.cuda.stream(stream) if on_gpu else contextlib.nullcontext()
    with ctx:
        if world == 1:
            return sim.topk(k, n=n, first=first, stream=stream, out=out)
        local = torch.empty(2 * k, dtype=torch.int64, device=device)
        sim.topk(k, n=n, first=first, block=blk, stride=stride, stream=stream, out=(local[:k], local[k:]))
        gathered = torch.empty(world * 2 * k, dtype=torch.int64, device=device)
        dist.all_gather_into_tensor(gathered, local, group=group)
        return (merge or _device_merge)(gathered.view(world, 2 * k), k, out)
