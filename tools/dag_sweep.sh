#!/bin/bash
for lv in 2 1; do
  echo "== levels $lv"
  ZOLO_FACTOR_LEVELS=$lv timeout 300 python tools/quick_check.py cfg2 cfg1 2>&1 | grep -E "factor wall|apply_filter|vs reference" | head -6
done
