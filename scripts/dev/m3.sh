timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b_c3.json 2> gpurun_out/bench_all.err
FSGG_SYM_WPT=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b_c3_old.json 2>> gpurun_out/bench_all.err
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_C2.json 2>> gpurun_out/bench_all.err
tail -3 gpurun_out/pytest_gpu.log
