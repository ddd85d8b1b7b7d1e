for o in 3 6 16 32 128 1; do
  echo "order $o"; ZOLO_DAG_ORDER=$o python tools/quick_check.py cfg2 cfg3 2>&1 | grep -E "apply_filter" | sed -n '2p;4p' | cut -c1-120
done
