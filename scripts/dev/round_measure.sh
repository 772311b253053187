set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/r2_bench_c3.json 2> gpurun_out/bench_all.err
for c in C2 C4 C5; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_$c.json 2>> gpurun_out/bench_all.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_reference_c3.json 2>> gpurun_out/bench_all.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3.csv python scripts/dev/shard_once.py --full > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sym_tile_kernel -c 1 -o gpurun_out/c3_sym python scripts/profile_once.py C3 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sym_tile_kernel -c 1 -o gpurun_out/c4_sym python scripts/profile_once.py C4 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kde_tc_sym256 -c 1 -o gpurun_out/c5_tc python scripts/profile_once.py C5 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o gpurun_out/c3_walk python scripts/profile_once.py C3 1 > /dev/null 2>&1
python scripts/shard_projection.py --out gpurun_out/shard_proj.json > gpurun_out/shard_proj.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
