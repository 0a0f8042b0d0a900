"""Per-call timings of the three candidate-list modes (range / explicit / block-cyclic),
with out_ns and top-k, config 2 (diagnostics)."""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch  # noqa: E402

import hsim_inputs as H  # noqa: E402
from paper_2508_05370_b200 import Sim  # noqa: E402

s = Sim(H.get(int(sys.argv[1]) if len(sys.argv) > 1 else 2))
N = s.space_size()
out = torch.empty(N, dtype=torch.int64, device="cuda")
idx = torch.arange(N, dtype=torch.int64, device="cuda")


def t(name, fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name:32s} {ms:.3f} ms  {N / ms / 1e6:.3f} G/s", flush=True)


t("eval range out_ns", lambda: s.eval_batch(n=N, out=out))
t("eval idx out_ns", lambda: s.eval_batch(idx=idx, out=out))
t("eval block-cyclic out_ns", lambda: s.eval_batch(n=N, block=65536, stride=65536, out=out))
t("topk16 range", lambda: s.topk(16))
t("topk16 idx", lambda: s.topk(16, idx=idx))
t("topk16 range + out_ns", lambda: s.topk(16, out_ns=out))
t("topk100 range", lambda: s.topk(100))
