mkdir -p gpurun_out
for o in 3 0 1 2 5; do
  echo "order $o"; ZOLO_DAG_ORDER=$o python tools/quick_check.py cfg3 2>&1 | grep -E "apply_filter" | tail -1 | cut -c1-120
done
for p in 8 10 5 9; do
  echo "policy $p"; ZOLO_L2_POLICY=$p python tools/quick_check.py cfg3 2>&1 | grep -E "apply_filter" | tail -1 | cut -c1-120
done
