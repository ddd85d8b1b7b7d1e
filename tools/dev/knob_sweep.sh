#!/bin/bash
# development: apply_filter rate of cfg2/cfg3 under DAG schedule / ND knobs (one line per setting)
cfgs=${CFGS:-cfg2}
while read -r line; do
  [ -z "$line" ] && continue
  r=$(env $line timeout 300 python tools/quick_check.py $cfgs 2>&1 | grep -E "apply_filter" | sed -n '2p;4p' | sed -E 's/.*-> ([0-9.]+) vec\/s/\1/' | tr '\n' ' ')
  echo "$line => $r"
done
