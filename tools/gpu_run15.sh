#!/bin/bash
mkdir -p gpurun_out
timeout 300 python bench.py --steps 100 --warmup 5 > gpurun_out/bench15.log 2>&1; tail -1 gpurun_out/bench15.log
timeout 1800 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/gputest15.log 2>&1; tail -16 gpurun_out/gputest15.log
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py small > gpurun_out/cs15_$t.log 2>&1; tail -3 gpurun_out/cs15_$t.log
done
python - > gpurun_out/ilv15.log 2>&1 <<'PY'
import torch, hsim_inputs as H
from paper_2508_05370_b200 import Sim
def tm(name, cfg, reps=5):
    s = Sim(cfg); N = s.space_size()
    s.topk(16); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): s.topk(16)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name}: N={N} {ms:.3f} ms/sweep {N / ms / 1e6:.3f} Gcand/s  cells/sweep={s.count_cells()}")
tm("config2 default", H.get(2))
tm("config2 interleave v=2", H.with_interleave(H.get(2), 2))
tm("config2 interleave v=4", H.with_interleave(H.get(2), 4))
tm("config4 interleave v=2", H.with_interleave(H.get(4), 2))
tm("config3 interleave v=2", H.with_interleave(H.get(3), 2), reps=2)
tm("config4 ep_dp", H.with_ep_dp(H.get(4)))
tm("config2 mixtp", H.with_changes(H.get(2), search__mixtp=1))
tm("config2 overlap", H.with_sync_overlap(H.get(2)))
tm("config2 buckets", H.with_changes(H.get(2), search__sync_buckets=2))
tm("config2 buckets+overlap", H.with_changes(H.with_sync_overlap(H.get(2)), search__sync_buckets=2))
tm("config3 default", H.get(3), reps=3)
tm("config4 default", H.get(4))
tm("config5 default", H.get(5), reps=2)
PY
cat gpurun_out/ilv15.log
