#!/bin/bash
for st in 0 0.25 0.5 1.0; do
  echo "== stagger $st"
  ZOLO_DAG_STAGGER=$st timeout 300 python tools/quick_check.py cfg2 cfg3 2>&1 | grep -E "apply_filter|solve:" | sed -n '3,4p;7,8p'
done
