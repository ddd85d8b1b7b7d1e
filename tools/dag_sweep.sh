#!/bin/bash
# Development sweep over DAG schedule knobs on cfg2 (GPU box).
mkdir -p gpurun_out
for near in 1 2 4; do for ch in 8 16 24; do
  echo "== near $near chunk $ch"
  ZOLO_DAG_NEAR=$near ZOLO_DAG_CHUNK=$ch timeout 120 python tools/quick_check.py cfg2 2>&1 | tail -1
done; done
