for v in t3s4 pan t3s4 pan; do echo "== $v"; ZOLO_LIB_PATH=tools/dev/variants/libzolo_$v.so timeout 300 python tools/quick_check.py cfg2 cfg3 2>&1 | grep -E "^cfg|Error" | cut -c1-130; done
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/fac5_gputest.txt 2>&1; tail -3 gpurun_out/fac5_gputest.txt
