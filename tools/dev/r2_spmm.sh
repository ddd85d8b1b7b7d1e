mkdir -p gpurun_out
for v in base sp1 sp2 sp3; do
ZOLO_LIB_PATH=tools/dev/variants/libzolo_$v.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:apply_b -s 6 -c 3 python tools/quick_check.py cfg3 > gpurun_out/spmm_$v.txt 2>&1
echo "== $v"; grep -E "gpu__time_duration|dram__bytes" gpurun_out/spmm_$v.txt
done
