mkdir -p gpurun_out
for p in 8 9 10 4 5 6; do
  echo "policy $p"; ZOLO_L2_POLICY=$p python tools/quick_check.py cfg3 2>&1 | grep -E "apply_filter|solve:" | tail -2
done > gpurun_out/policy_cfg3.txt 2>&1
for p in 8 9 10 4 6; do
  echo "policy $p"; ZOLO_L2_POLICY=$p python tools/quick_check.py cfg2 2>&1 | grep -E "apply_filter|solve:" | tail -2
done > gpurun_out/policy_cfg2.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x -k "solves or sharding or generators" > gpurun_out/gputest_r02f.txt 2>&1
tail -3 gpurun_out/gputest_r02f.txt
