#!/bin/bash
# development: build libzolo_b200.so with extra compile flags into tools/dev/variants/libzolo_<name>.so
# usage: tools/dev/build_variant.sh <name> "<nvcc flags>"   (load with ZOLO_LIB_PATH=<path>)
set -e
name=$1; extra=$2
R=$(cd "$(dirname "$0")/../.." && pwd)
S=$R/paper_1701_08935_b200/csrc
B=/tmp/zolo_variant_$name
mkdir -p $B $R/tools/dev/variants
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -I$R/include $extra"
for f in factor trsm krylov capi driver shard; do $NV -c $S/$f.cu -o $B/$f.o & done
for f in host design symbolic; do g++ -std=c++17 -O3 -fPIC -c $S/$f.cpp -o $B/$f.o & done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/tools/dev/variants/libzolo_$name.so $B/*.o -lcudart -ldl
echo built tools/dev/variants/libzolo_$name.so
