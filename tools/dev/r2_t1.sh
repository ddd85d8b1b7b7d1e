mkdir -p gpurun_out
python tools/quick_check.py cfg2 cfg3 > gpurun_out/t1_qc.txt 2>&1
cat gpurun_out/t1_qc.txt
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/t1_gputest.txt 2>&1
tail -5 gpurun_out/t1_gputest.txt
