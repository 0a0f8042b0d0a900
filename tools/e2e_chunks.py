import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, hsim_inputs as H
from paper_2508_05370_b200 import Sim
s = Sim(H.get(2)); N = s.space_size()
ih = torch.arange(N, dtype=torch.int64).pin_memory(); oh = torch.empty(N, dtype=torch.int64).pin_memory()
for ch in (1, 2, 3, 4, 8):
    for _ in range(3): s.eval_host(ih, oh, chunks=ch)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): s.eval_host(ih, oh, chunks=ch)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(ch, round(ms, 3), 'ms', round(N / ms / 1e6, 3), 'G/s')
# pure eval range for reference
out = torch.empty(N, dtype=torch.int64, device='cuda')
e0.record()
for _ in range(20): s.eval_batch(n=N, out=out)
e1.record(); torch.cuda.synchronize(); print('eval range', e0.elapsed_time(e1)/20)
idx = ih.cuda()
e0.record()
for _ in range(20): s.eval_batch(idx=idx, out=out)
e1.record(); torch.cuda.synchronize(); print('eval idx', e0.elapsed_time(e1)/20)
