for v in head tr3 head tr3; do echo "== $v"; ZOLO_LIB_PATH=tools/dev/variants/libzolo_$v.so python tools/quick_check.py cfg2 cfg3 2>&1 | grep -E "^cfg|apply_filter" | cut -c1-130; done
ZOLO_LIB_PATH=tools/dev/variants/libzolo_tr3.so timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/fac_gputest.txt 2>&1; tail -3 gpurun_out/fac_gputest.txt
