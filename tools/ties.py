"""How many candidates tie at the smallest iteration times (top-k merge sizing)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsim_inputs as H  # noqa: E402
from paper_2508_05370_b200 import Sim  # noqa: E402

for c in [int(x) for x in sys.argv[1:]] or [2]:
    s = Sim(H.get(c))
    N = s.space_size()
    out = torch.empty(N, dtype=torch.int64, device="cuda")
    s.eval_batch(n=N, out=out)
    v = out[out >= 0]
    srt = torch.sort(v).values
    k16 = srt[15].item()
    print(f"cfg{c}: valid {v.numel()} min {srt[0].item()} 16th {k16} count<=16th {(v <= k16).sum().item()} "
          f"count==min {(v == srt[0]).sum().item()}")
