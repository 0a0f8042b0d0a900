"""Workload for compute-sanitizer (memcheck / racecheck / synccheck) over the
final kernels: every phase kernel and both top-k paths, on samples of configs
2-5, the deep-pipeline and four-type tiny spaces, the f1/f2 rows, and the
device merge.  Usage: compute-sanitizer --tool X python tools/sanitize_run.py [small]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsim_inputs as H  # noqa: E402
from paper_2508_05370_b200 import Sim  # noqa: E402
from paper_2508_05370_b200.hsim import hsim_merge_topk  # noqa: E402

small = len(sys.argv) > 1 and sys.argv[1] == "small"
n = 4096 if small else 60000
cfgs = [H.get(2), H.get(3), H.get(4), H.get(5), H.deep_tiny(1), H.four_types_tiny(),
        H.with_mem_check(H.get(2)), H.with_sync_overlap(H.get(4)),
        # f4 / f1 rows: interleaved 1F1B (K_ilv, K_sync_ilv), EP across replicas,
        # mixed-type TP groups, two gradient buckets (C.8 and S.1)
        H.with_interleave(H.get(2), 2), H.with_interleave(H.with_changes(H.deep_tiny(0), model__global_batch=7680,
                                                                         model__layers=192), 2),
        H.with_ep_dp(H.get(4)), H.with_changes(H.get(2), search__mixtp=1),
        H.with_changes(H.with_sync_overlap(H.get(2)), search__sync_buckets=2),
        H.with_changes(H.get(4), search__sync_buckets=2)]
for cfg in cfgs:
    s = Sim(cfg)
    N = s.space_size()
    m = min(n, N)
    first = (N // 3) if N > m else 0
    out = torch.empty(m, dtype=torch.int64, device="cuda")
    s.eval_batch(n=m, first=first, out=out)
    idx = torch.randint(0, N, (min(m, 3000),), device="cuda", dtype=torch.int64)
    s.eval_batch(idx=idx)
    s.topk(16, n=m, first=first)
    s.topk(100, n=m, first=first)
    s.topk(8, n=min(m, 5000), first=0, block=1000, stride=3000) if N > 15000 else None
    s.count_cells(first, min(m, 2000))  # count mode (the dedupe table is cleared by a memset there)
    s.set_dedup(False)                  # the per-(candidate, class) path too
    s.topk(16, n=min(m, 8000), first=first)
    s.set_dedup(True)
    torch.cuda.synchronize()
    print("ok", cfg["name"], m, flush=True)
lists = torch.full((4, 64), 2**63 - 1, dtype=torch.int64, device="cuda")
lists[:, 32:] = -1
lists[0, 0], lists[0, 32] = 5, 7
hsim_merge_topk(lists, 32)
hsim_merge_topk(torch.full((3, 2 * 40), -1, dtype=torch.int64, device="cuda").contiguous(), 40)
torch.cuda.synchronize()
print("ok merge")
