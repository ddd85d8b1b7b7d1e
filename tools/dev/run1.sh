set -x
mkdir -p gpurun_out
(nproc; lscpu | head -30; free -g; cat /sys/fs/cgroup/cpu.max 2>/dev/null; nvidia-smi) > gpurun_out/host_info.txt 2>&1
timeout 900 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3_r02a.json 2> gpurun_out/bench_cfg3_r02a.err
timeout 600 python tools/dev/cfg3_gtol.py > gpurun_out/gtol.txt 2>&1
