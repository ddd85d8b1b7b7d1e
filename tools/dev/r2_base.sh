set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2b_smi.txt
timeout 2400 python -m pytest tests -q -m gpu -x --durations=25 > gpurun_out/r2b_gputest.txt 2>&1
tail -30 gpurun_out/r2b_gputest.txt
timeout 1200 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
tail -3 gpurun_out/r2b_bench.json
timeout 1800 python bench.py --impl reference > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err
tail -3 gpurun_out/r2b_ref.json
