mkdir -p gpurun_out
python tools/quick_check.py cfg1 cfg2 cfg3 2>&1 | grep -E "^cfg|apply_filter" | cut -c1-140
for o in 1 4; do echo "order $o"; ZOLO_DAG_ORDER=$o python tools/quick_check.py cfg2 cfg3 2>&1 | grep -E "apply_filter" | cut -c1-140; done
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/t3_gputest.txt 2>&1
tail -3 gpurun_out/t3_gputest.txt
