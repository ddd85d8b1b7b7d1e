mkdir -p gpurun_out
python bench.py > gpurun_out/m1_bench_cfg3.json 2> gpurun_out/m1_bench_cfg3.err
tail -1 gpurun_out/m1_bench_cfg3.json | cut -c1-300
python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/m1_bench_cfg2.json 2> gpurun_out/m1_bench_cfg2.err
tail -1 gpurun_out/m1_bench_cfg2.json | cut -c1-300
ncu --set full --import-source on --clock-control none -k regex:dag2_kernel -s 8 -c 1 -f -o gpurun_out/m1_cfg2_dag2 python tools/quick_check.py cfg2 > gpurun_out/m1_ncu2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m1_launches_cfg3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-eigensolver > gpurun_out/m1_ncu_l.log 2>&1
python bench.py --config cfg5 --no-cpu-baseline > gpurun_out/m1_bench_cfg5.json 2> gpurun_out/m1_bench_cfg5.err
tail -1 gpurun_out/m1_bench_cfg5.json | cut -c1-300
