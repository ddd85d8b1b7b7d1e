set -x
mkdir -p gpurun_out
python tools/quick_check.py cfg3 > gpurun_out/p1_qc3.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:dag2_kernel -s 4 -c 1 -f -o gpurun_out/p1_cfg3_dag2 python tools/quick_check.py cfg3 > gpurun_out/p1_ncu3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"apply_b|update_kernel|dots_kernel|combine|next_basis|least_squares" -s 24 -c 12 -f -o gpurun_out/p1_cfg3_aux python tools/quick_check.py cfg3 > gpurun_out/p1_ncu3aux.log 2>&1
ls -la gpurun_out
