set -x
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r2_bench_c3.json 2> gpurun_out/bench_all.err
for c in C2 C4 C5; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_$c.json 2>> gpurun_out/bench_all.err; done
python scripts/shard_projection.py --out gpurun_out/shard_proj.json > gpurun_out/shard_proj.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/r2_bench_c3.json; tail -5 gpurun_out/shard_proj.log
