set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-eigensolver"
python tools/quick_check.py cfg3 > gpurun_out/qc3.txt 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:dag2_kernel -s 4 -c 1 -f -o gpurun_out/r02_cfg3_dag2 python tools/quick_check.py cfg3 > gpurun_out/ncu3.log 2>&1
python tools/quick_check.py cfg2 > gpurun_out/qc2.txt 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:dag2_kernel -s 4 -c 1 -f -o gpurun_out/r02_cfg2_dag2 python tools/quick_check.py cfg2 > gpurun_out/ncu2.log 2>&1
$B > gpurun_out/b_plain.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg3.csv $B > gpurun_out/ncu_l.log 2>&1
ls -la gpurun_out/
