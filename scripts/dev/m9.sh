FSGG_TRACE=1 timeout 300 python scripts/profile_once.py C3 2 2>&1 | grep "level 12" | tail -1 > gpurun_out/trace_l12.log
FSGG_NODE_KERNEL=0 FSGG_TRACE=1 timeout 300 python scripts/profile_once.py C3 2 2>&1 | grep "level 12" | tail -1 >> gpurun_out/trace_l12.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b_c3.json 2> gpurun_out/bench_all.err
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/trace_l12.log
