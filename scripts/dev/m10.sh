run() { FSGG_TRACE=1 timeout 300 python scripts/profile_once.py C3 2 2>&1 | grep "level" | tail -21 | awk -v tag="$1" '{for(i=1;i<=NF;i++) if($i ~ /scan\+scatter=/) {v=$(i+1); sub("ms","",v); s+=v}} END {print tag, "scan+scatter total", s}'; }
run default16 >> gpurun_out/scan_var.log
for v in s32; do FSGG_LIB_PATH=$PWD/variants/$v/libfsgg.so run $v >> gpurun_out/scan_var.log; done
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/scan_var.log
