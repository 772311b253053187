timeout 300 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_C4_wpt2.json 2> gpurun_out/bench_all.err
FSGG_SYM_WPT=1 timeout 300 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_C4_wpt1.json 2>> gpurun_out/bench_all.err
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b_c3.json 2>> gpurun_out/bench_all.err
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
