python tools/quick_check.py cfg2 cfg3 2>&1 | grep -E "apply_filter" | sed -n '2p;4p' | cut -c1-130
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/t7_gputest.txt 2>&1; tail -3 gpurun_out/t7_gputest.txt
