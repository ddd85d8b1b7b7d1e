#!/bin/bash
# Development sweep over DAG schedule knobs on cfg2 (GPU box).
mkdir -p gpurun_out
for o in 0 1 2; do for ch in 8 16; do for leaf in 512 256; do
  echo "== order $o chunk $ch leaf $leaf"
  ZOLO_DAG_ORDER=$o ZOLO_DAG_CHUNK=$ch ND_LEAF=$leaf timeout 120 python tools/quick_check.py cfg2 2>&1 | tail -1
done; done; done
