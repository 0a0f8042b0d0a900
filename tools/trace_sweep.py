"""Timeline of one hsim_topk sweep (HSIM_TRACE=1: timing events around every launch).

  HSIM_TRACE=1 python tools/trace_sweep.py [config] [reps]   -> stderr TRACE lines of each call
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsim_inputs as H  # noqa: E402
from paper_2508_05370_b200 import Sim  # noqa: E402

cfg_n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
s = Sim(H.get(cfg_n))
for r in range(reps):
    print(f"--- call {r}", file=sys.stderr, flush=True)
    t, i = s.topk(16)
    torch.cuda.synchronize()
print("top1", t[0].item(), i[0].item())
