set -x
timeout 300 python scripts/dev/e2e_phases.py > gpurun_out/e2e_phases.log 2>&1
FSGG_TRACE=1 timeout 300 python scripts/profile_once.py C3 2 > gpurun_out/trace_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3.csv python scripts/profile_once.py C3 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sym_tile_kernel -c 1 -o gpurun_out/c3_sym python scripts/profile_once.py C3 1 > /dev/null 2>&1
cat gpurun_out/e2e_phases.log
