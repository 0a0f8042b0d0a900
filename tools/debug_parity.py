"""Debug helper: GPU vs oracle on samples of a config; prints mismatches with plans."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hsim_inputs as H  # noqa: E402
import oracle  # noqa: E402
from paper_2508_05370_b200 import Sim  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cnt = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
cfg = H.get(n)
s, o = Sim(cfg), oracle.Oracle(cfg)
pre = o.template_prefix()
ks = np.unique(np.linspace(0, len(pre) - 2, 400).astype(int))
extra = np.concatenate([pre[ks], pre[ks + 1] - 1])
idx = H.sample_indices(o.space_size(), cnt, seed=H.PARITY_SEED + n, extra=extra)
got = s.eval_batch(idx=torch.as_tensor(idx, device="cuda")).cpu().numpy()
want = o.eval_many(idx)
bad = np.nonzero(got != want)[0]
print("mismatches", len(bad), "of", len(idx))
for b in bad[:8]:
    d = s.decode(int(idx[b]))
    print(idx[b], got[b], want[b], [(len(c["stages"]), c["D"], c["subclasses"], c["mb"][:3]) for c in d["classes"]])
