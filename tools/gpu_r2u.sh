mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_dedup_gpu.py tests/test_parity_gpu_r2.py -x -q > gpurun_out/r2u_test.log 2>&1; tail -1 gpurun_out/r2u_test.log
for rep in 1 2; do for c in 2 4 3; do timeout 120 python tools/variant_bench.py $c 30 >> gpurun_out/r2u_var.log 2>&1; done; done; timeout 300 python tools/dedup_timing.py 5 >> gpurun_out/r2u_var.log 2>&1
cat gpurun_out/r2u_var.log
HSIM_TRACE=1 timeout 120 python tools/prof_sweep.py 2 3 > gpurun_out/r2u_trace.log 2>&1; tail -4 gpurun_out/r2u_trace.log
python - <<'PY' > gpurun_out/r2u_units.log 2>&1
import sys; sys.path.insert(0,'.')
import hsim_inputs as H
from paper_2508_05370_b200 import Sim
s=Sim(H.get(2)); s.topk(16); print('units', s.last_sync_units())
PY
cat gpurun_out/r2u_units.log
