mkdir -p gpurun_out/s5
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-eigensolver > gpurun_out/s5/b_plain.json 2> gpurun_out/s5/b_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/s5/launches_cfg3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-eigensolver > gpurun_out/s5/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dag2_kernel -s 4 -c 1 -o gpurun_out/s5/dag2_cfg3 python tools/quick_check.py cfg3 > gpurun_out/s5/ncu_dag2.log 2>&1
ls -la gpurun_out/s5 | tail -5
