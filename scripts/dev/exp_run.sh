# quick experiment: C3/C2 bench lines, GPU tests, one ncu capture of the root kernel
set -x
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/exp_bench_c3.json 2> gpurun_out/exp_bench.err; echo bench rc=$?
timeout 200 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/exp_bench_C2.json 2>> gpurun_out/exp_bench.err
timeout 200 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/exp_bench_C4.json 2>> gpurun_out/exp_bench.err
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/exp_pytest.log 2>&1; echo rc=$?; tail -5 gpurun_out/exp_pytest.log
mkdir -p /tmp/ncu
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:sym_wtile_kernel -c 1 -o /tmp/ncu/c3_exp python scripts/profile_once.py C3 1 > gpurun_out/ncu_exp.log 2>&1
ncu -i /tmp/ncu/c3_exp.ncu-rep --page raw --csv > gpurun_out/c3_exp_raw.csv
ncu -i /tmp/ncu/c3_exp.ncu-rep --page source --csv > gpurun_out/c3_exp_source.csv
