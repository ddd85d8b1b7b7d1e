set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gputest_r02c.txt 2>&1
tail -15 gpurun_out/gputest_r02c.txt
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err
tail -3 gpurun_out/bench_r02c.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02c.json 2> gpurun_out/bench_ref_r02c.err
tail -3 gpurun_out/bench_ref_r02c.err
