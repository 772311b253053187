for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --kernel-regex kns=wtile --kernel-regex kns=walk --kernel-regex kns=kde_lowd_node --print-limit 20 python scripts/dev/sanitize_small.py > gpurun_out/sanitize_$tool.log 2>&1
  tail -5 gpurun_out/sanitize_$tool.log
done
