set -x
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_split|k_final" -s 2 -c 2 -o gpurun_out/prof_dd4 python tools/prof_sweep.py 2 2 > gpurun_out/ncu_dd4.log 2>&1
python - <<'PY' > gpurun_out/syncunits.log 2>&1
import sys; sys.path.insert(0,'.')
import hsim_inputs as H
from paper_2508_05370_b200 import Sim
s=Sim(H.get(2))
for k in (1,16,32):
    s.topk(k); print(k, s.last_sync_units())
PY
cat gpurun_out/syncunits.log
