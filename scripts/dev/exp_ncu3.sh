mkdir -p /tmp/ncu
cap() { # name regex skip
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:$2 --launch-skip $3 -c 1 -o /tmp/ncu/$1 python scripts/profile_once.py C3 1 > gpurun_out/ncu_$1.log 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/$1.ncu-rep --page source --csv > gpurun_out/$1_source.csv 2>/dev/null
}
cap c3_route12 route_kernel 12
cap c3_scatter12 scatter_kernel 12
cap c3_scan12 flags_scan_kernel 12
