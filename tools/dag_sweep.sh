#!/bin/bash
for lib in tools/dev/lib_v2_n2b3.so; do
  echo "== lib ${lib}"
  ZOLO_DAG_V2=1 ZOLO_LIB_PATH=$lib timeout 300 python tools/quick_check.py cfg2 cfg3 2>&1 | grep -E "apply_filter|solve:" | sed -n '3,4p;7,8p'
done
