mkdir -p /tmp/ncu
cap() { # name regex skip
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:$2 --launch-skip $3 -c 1 -o /tmp/ncu/$1 python scripts/profile_once.py C3 1 > gpurun_out/ncu_$1.log 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/$1.ncu-rep --page source --csv > gpurun_out/$1_source.csv 2>/dev/null
}
cap c3_node kde_lowd_node_kernel 0
cap c3_blk block_lookup_kernel 4
cap c3_symrows sym_rows_kernel 0
cap c3_tiesplit tie_split_kernel 3
cap c3_edges edges_kernel 0
cap c3_rowssort rows_sort_kernel 0
cap c3_rowsfill rows_fill_kernel 0
