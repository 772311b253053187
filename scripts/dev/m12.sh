for m in 2 4 6; do
echo "min $m" >> gpurun_out/trace_c5.log
FSGG_TIE_GEMM_MIN=$m FSGG_TRACE=1 timeout 600 python scripts/profile_once.py C5 2 2>&1 | grep "level" | tail -18 | head -9 | tail -5 | cut -c1-150 >> gpurun_out/trace_c5.log
done
cat gpurun_out/trace_c5.log
