for v in head sb0 sb1 sb2 sb3; do
ZOLO_LIB_PATH=tools/dev/variants/libzolo_$v.so ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:apply_b -s 6 -c 2 python tools/quick_check.py cfg3 > gpurun_out/spmm2_$v.txt 2>&1
echo "== $v"; grep -E "gpu__time_duration" gpurun_out/spmm2_$v.txt
done
