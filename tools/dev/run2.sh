set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gputest_r02b.txt 2>&1
tail -5 gpurun_out/gputest_r02b.txt
timeout 900 python tools/dev/refine_probe.py cfg3 > gpurun_out/refine_cfg3.txt 2>&1
cat gpurun_out/refine_cfg3.txt
