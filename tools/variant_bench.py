"""Times one library variant: full config sweep -> top-k, CUDA events (select the .so via HSIM_LIB)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsim_inputs as H  # noqa: E402
from paper_2508_05370_b200 import Sim  # noqa: E402

cfg_n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
s = Sim(H.get(cfg_n))
N = s.space_size()
for _ in range(3):
    t, i = s.topk(16)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    t, i = s.topk(16)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"{os.path.basename(os.environ.get('HSIM_LIB', 'default'))} cfg{cfg_n} {ms:.3f} ms/sweep "
      f"{N / ms * 1e3 / 1e6:.1f} M/s top1={t[0].item()}:{i[0].item()}", flush=True)
