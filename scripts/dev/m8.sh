python scripts/shard_projection.py --out gpurun_out/shard_proj.json > gpurun_out/shard_proj.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_shard8.csv python scripts/dev/shard_once.py --world 8 > /dev/null 2>&1
python scripts/dev/shard_phases.py --world 8 --rank 1 > gpurun_out/shard_phases8.log 2>&1
tail -6 gpurun_out/shard_proj.log; cat gpurun_out/shard_phases8.log
