mkdir -p gpurun_out/s5
for v in work xhalf xquart work xhalf; do
  echo "== $v"; ZOLO_LIB_PATH=tools/dev/variants/libzolo_$v.so python tools/dev/probe_time.py cfg3 2>&1 | tail -1
done
