mkdir -p gpurun_out/s5
ncu --set full --clock-control none --import-source on -k regex:trailing_level -s 60 -c 2 -o gpurun_out/s5/trailing_mask python tools/dev/factor_only.py cfg3 > gpurun_out/s5/ncu_trailing_mask.log 2>&1
python tools/dev/factor_scaling.py cfg3
