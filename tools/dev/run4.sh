set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --durations=25 > gpurun_out/gputest_r02d.txt 2>&1
tail -45 gpurun_out/gputest_r02d.txt
