"""One warm-up sweep + N profiled sweeps of a BASELINE config (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsim_inputs as H  # noqa: E402
from paper_2508_05370_b200 import Sim  # noqa: E402

cfg_n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
k = int(sys.argv[3]) if len(sys.argv) > 3 else 16
s = Sim(H.get(cfg_n))
for _ in range(reps):
    t, i = s.topk(k)
torch.cuda.synchronize()
print("top1", t[0].item(), i[0].item())
