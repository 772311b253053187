# Prune-threshold sweep (dev): C3/C4 step time and tie counts per build, plus
# the full-size reference fingerprints (pruned mode) for each.
for v in base p44 p40 p36; do
  if [ $v = base ]; then unset FSGG_LIB_PATH; else export FSGG_LIB_PATH=$PWD/variants/$v/libfsgg.so; fi
  echo "== $v"
  PYTHONPATH=. timeout 300 python scripts/dev/quick_perf.py C3 C4 2>&1 | grep -E "it1|Error"
  timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -k "pruned" 2>&1 | tail -2
done
