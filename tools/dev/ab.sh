# usage: bash tools/dev/ab.sh "<variant names>" "<configs>"  -> gpurun_out/ab_<variant>.txt
mkdir -p gpurun_out
for v in $1; do
  ZOLO_LIB_PATH=tools/dev/variants/libzolo_$v.so python tools/quick_check.py $2 > gpurun_out/ab_$v.txt 2>&1
  echo "== $v"; grep -E "apply_filter|^cfg" gpurun_out/ab_$v.txt | sed -n '1,20p' | cut -c1-150
done
