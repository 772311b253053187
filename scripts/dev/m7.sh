FSGG_TRACE=1 timeout 300 python scripts/profile_once.py C3 3 2>&1 | grep walks | tail -2 | sed "s/^/default12 /" >> gpurun_out/trace_walk2.log
for v in wf16 wf10; do
FSGG_LIB_PATH=$PWD/variants/$v/libfsgg.so FSGG_TRACE=1 timeout 300 python scripts/profile_once.py C3 3 2>&1 | grep walks | tail -2 | sed "s/^/$v /" >> gpurun_out/trace_walk2.log
done
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/trace_walk2.log
