mkdir -p gpurun_out/s5
ZOLO_SETUP_TIMES=1 python tools/quick_check.py cfg3 > gpurun_out/s5/setup_cfg3.txt 2>&1
ZOLO_SETUP_TIMES=1 python tools/dev/ttae_probe.py cfg3 > gpurun_out/s5/ttae_cfg3.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:apply_b -s 6 -c 1 -o gpurun_out/s5/apply_b_cfg3 python tools/quick_check.py cfg3 > gpurun_out/s5/ncu_apply_b.log 2>&1
tail -30 gpurun_out/s5/setup_cfg3.txt
