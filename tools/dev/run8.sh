mkdir -p gpurun_out
ZOLO_TRACE=gpurun_out/trace_cfg3.txt python tools/quick_check.py cfg3 > gpurun_out/qc3t.txt 2>&1
python tools/dag2_trace_analyze.py gpurun_out/trace_cfg3.txt > gpurun_out/trace_cfg3_summary.txt 2>&1
ZOLO_TRACE=gpurun_out/trace_cfg2.txt python tools/quick_check.py cfg2 > gpurun_out/qc2t.txt 2>&1
python tools/dag2_trace_analyze.py gpurun_out/trace_cfg2.txt > gpurun_out/trace_cfg2_summary.txt 2>&1
rm -f gpurun_out/trace_cfg3.txt gpurun_out/trace_cfg2.txt
timeout 1800 python -m pytest tests -q -m gpu -x -k "solves" > gpurun_out/gputest_r02g.txt 2>&1
tail -3 gpurun_out/gputest_r02g.txt
