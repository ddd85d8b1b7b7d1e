mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:dag2_kernel -s 4 -c 1 -f -o gpurun_out/p3_cfg3_dag2 python tools/quick_check.py cfg3 > gpurun_out/p3_ncu3.log 2>&1
ZOLO_TRACE=gpurun_out/trace_cfg3.txt python tools/quick_check.py cfg3 > gpurun_out/p3_qc3t.txt 2>&1
python tools/dag2_trace_analyze.py gpurun_out/trace_cfg3.txt > gpurun_out/p3_trace_cfg3.txt 2>&1
rm -f gpurun_out/trace_cfg3.txt
