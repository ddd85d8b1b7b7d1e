mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/m2_gputest.txt 2>&1; tail -3 gpurun_out/m2_gputest.txt
python bench.py > gpurun_out/m2_bench_cfg3.json 2> gpurun_out/m2_bench_cfg3.err; tail -1 gpurun_out/m2_bench_cfg3.json | cut -c1-200
python bench.py --config cfg4s --no-cpu-baseline > gpurun_out/m2_bench_cfg4s.json 2> gpurun_out/m2_bench_cfg4s.err; tail -1 gpurun_out/m2_bench_cfg4s.json | cut -c1-200
python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/m2_bench_cfg1.json 2> gpurun_out/m2_bench_cfg1.err; tail -1 gpurun_out/m2_bench_cfg1.json | cut -c1-200
ncu --set full --import-source on --clock-control none -k regex:trailing_level -s 40 -c 2 -f -o gpurun_out/m2_cfg3_trailing python tools/quick_check.py cfg3 > gpurun_out/m2_ncu_tr.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"diag_level|panel_level" -s 40 -c 2 -f -o gpurun_out/m2_cfg3_diagpanel python tools/quick_check.py cfg3 > gpurun_out/m2_ncu_dp.log 2>&1
