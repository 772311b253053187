mkdir -p /tmp/ncu
cap() { # name regex config
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -c 1 -o /tmp/ncu/$1 python scripts/profile_once.py $3 1 > /dev/null 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/$1.ncu-rep --page source --csv > gpurun_out/$1_source.csv 2>/dev/null
}
cap c3_walkf walk_fast_kernel C3
