"""Full-sweep top-16 timings with the pipeline dedupe on / off (configs 2-5),
plus executed-cell counts for config 2 (diagnostics)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import hsim_inputs as H  # noqa: E402
from paper_2508_05370_b200 import Sim  # noqa: E402


def sweep_ms(sim, reps):
    N = sim.space_size()
    for _ in range(2):
        sim.topk(16, n=N)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        sim.topk(16, n=N)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for n in [int(a) for a in sys.argv[1:]] or [2, 4, 3, 5]:
    sim = Sim(H.get(n))
    reps = {2: 50, 3: 10, 4: 20, 5: 2}[n]
    r = {}
    for on in (True, False):
        sim.set_dedup(on)
        r[on] = sweep_ms(sim, reps)
    t1 = sim.topk(16)[0].cpu().numpy()
    sim.set_dedup(True)
    t0 = sim.topk(16)[0].cpu().numpy()
    print(f"config {n}: N={sim.space_size()} dedupe on {r[True]:.3f} ms ({sim.space_size() / r[True] / 1e6:.3f} G/s), "
          f"off {r[False]:.3f} ms, same top-16 {bool((t0 == t1).all())}", flush=True)
    if n == 2:
        c_on = sim.count_cells()
        sim.set_dedup(False)
        c_off = sim.count_cells()
        sim.set_dedup(True)
        print(f"config 2 cells: on {c_on} off {c_off}", flush=True)
