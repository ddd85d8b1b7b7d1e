for v in db2; do echo "== $v"; ZOLO_LIB_PATH=tools/dev/variants/libzolo_$v.so timeout 300 python tools/quick_check.py cfg2 cfg3 2>&1 | grep -E "^cfg|apply_filter|Error" | cut -c1-130; done
