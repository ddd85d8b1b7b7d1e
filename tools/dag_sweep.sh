#!/bin/bash
for ch in 0 1; do
  echo "== chain $ch"
  ZOLO_DAG_CHAIN=$ch timeout 300 python tools/quick_check.py cfg2 cfg3 cfg1 2>&1 | grep -E "apply_filter" | sed -n '2p;4p;6p'
done
