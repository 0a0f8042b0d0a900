mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; tail -1 gpurun_out/fin_smoke.log
timeout 600 python bench.py --steps 100 --warmup 10 > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; cat gpurun_out/fin_bench.json
timeout 900 python -m pytest tests/test_parity_variants_gpu.py tests/test_parity_memcheck_gpu.py tests/test_parity_overlap_gpu.py tests/test_flow_gpu.py -x -q > gpurun_out/fin_gputest2.log 2>&1; tail -1 gpurun_out/fin_gputest2.log
