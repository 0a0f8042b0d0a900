set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/alu_peak.py --ncu > gpurun_out/alu_peak.log 2>&1; cp profiles/alu_peak_r02.json gpurun_out/ 2>/dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest1.log 2>&1; tail -3 gpurun_out/gputest1.log
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/bench1.log 2>&1; tail -2 gpurun_out/bench1.log
