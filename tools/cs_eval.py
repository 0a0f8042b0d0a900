"""Evaluates [first, first + n) of a config through hsim_eval_batch (debug aid:
run under compute-sanitizer, or bisect a failing range)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsim_inputs as H  # noqa: E402
from paper_2508_05370_b200 import Sim  # noqa: E402

s = Sim(H.get(int(sys.argv[1])))
N = s.space_size()
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else N - first
out = torch.empty(n, dtype=torch.int64, device="cuda")
s.eval_batch(n=n, first=first, out=out)
torch.cuda.synchronize()
print("ok", first, n, out[:4].tolist())
