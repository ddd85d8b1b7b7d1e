#!/bin/bash
# Development sweep over DAG knobs on cfg2 (GPU box).
for h in 0 1 2 3; do
  echo "== hints $h"
  ZOLO_DAG_HINTS=$h timeout 120 python tools/quick_check.py cfg2 2>&1 | tail -1
done
