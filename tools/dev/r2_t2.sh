bash tools/dev/ab.sh "$1" "$2"
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/t2_gputest.txt 2>&1
tail -5 gpurun_out/t2_gputest.txt
