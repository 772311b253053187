set -x
mkdir -p /tmp/ncu
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/r2_bench_c3.json 2> gpurun_out/bench_all.err
for c in C2 C4 C5; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_$c.json 2>> gpurun_out/bench_all.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_reference_c3.json 2>> gpurun_out/bench_all.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3.csv python scripts/dev/shard_once.py --full > /dev/null 2>&1
cap() { # name regex config
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:$2 -c 1 -o /tmp/ncu/$1 python scripts/profile_once.py $3 1 > /dev/null 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
}
cap c3_wtile sym_wtile_kernel C3
cap c4_wtile sym_wtile_kernel C4
cap c3_walkf walk_fast_kernel C3
cap c3_node kde_lowd_node_kernel C3
cap c5_tcsym kde_tc_sym256 C5
python scripts/shard_projection.py --out gpurun_out/r2_shard_projection_c3.json > gpurun_out/r2_shard_projection_c3.log 2>&1
tail -3 gpurun_out/r2_pytest_gpu.log; tail -2 gpurun_out/smoke.log
