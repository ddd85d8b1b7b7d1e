bash tools/dev/ab.sh "w8 cs" "cfg1 cfg2 cfg3"
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/t4_gputest.txt 2>&1
tail -3 gpurun_out/t4_gputest.txt
