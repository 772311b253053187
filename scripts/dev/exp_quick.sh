# quick experiment: C3 bench line + GPU tests
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/exp_bench_c3.json 2> gpurun_out/exp_bench.err; echo bench rc=$?
FSGG_TRACE=1 python scripts/profile_once.py C3 2 2> gpurun_out/exp_trace_c3.log | tail -1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/exp_pytest.log 2>&1; echo rc=$?; tail -3 gpurun_out/exp_pytest.log
