for v in head t3s4 t3s3 t3s4; do echo "== $v"; ZOLO_LIB_PATH=tools/dev/variants/libzolo_$v.so timeout 300 python tools/quick_check.py cfg2 cfg3 2>&1 | grep -E "^cfg|Error" | cut -c1-130; done
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/fac4_gputest.txt 2>&1; tail -3 gpurun_out/fac4_gputest.txt
