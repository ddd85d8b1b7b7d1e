#!/bin/bash
for leaf in 192 256; do
  echo "== leaf $leaf"
  ND_LEAF=$leaf timeout 300 python tools/quick_check.py cfg3 cfg1 2>&1 | grep -E "apply_filter" | sed -n '2p;4p'
done
