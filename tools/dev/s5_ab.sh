mkdir -p gpurun_out/s5
for rep in 1 2; do
for v in head new; do
  if [ $v = head ]; then export ZOLO_LIB_PATH=tools/dev/variants/libzolo_head.so; else unset ZOLO_LIB_PATH; fi
  ZOLO_SETUP_TIMES=1 python tools/dev/ttae_probe.py cfg3 > gpurun_out/s5/ab_${v}_$rep.txt 2>&1
  echo "== $v $rep"; grep -E "apply_filter|total=" gpurun_out/s5/ab_${v}_$rep.txt
done
done
