import sys; sys.path.insert(0,'.')
import torch, hsim_inputs as H
from paper_2508_05370_b200 import Sim
s=Sim(H.get(2))
for it in range(2):
    s.eval_batch(n=1000); torch.cuda.synchronize(); print("eval", s.last_launch_count(), file=sys.stderr, flush=True)
    s.topk(8, n=1000, out_ns=torch.empty(1000,dtype=torch.int64,device='cuda')); torch.cuda.synchronize(); print("topk out", s.last_launch_count(), file=sys.stderr, flush=True)
    s.topk(8, n=1000); torch.cuda.synchronize(); print("topk", s.last_launch_count(), file=sys.stderr, flush=True)
