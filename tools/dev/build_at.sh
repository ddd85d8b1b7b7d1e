#!/bin/bash
# development: build libzolo_b200.so from a source tree (a git revision or the working tree) with
# extra nvcc flags into tools/dev/variants/libzolo_<name>.so (load with ZOLO_LIB_PATH=<path>)
# usage: tools/dev/build_at.sh <name> <git-rev|WORK> "<nvcc flags>"
set -e
name=$1; rev=$2; extra=$3
R=$(cd "$(dirname "$0")/../.." && pwd)
B=/tmp/zolo_variant_$name
rm -rf $B; mkdir -p $B/src $R/tools/dev/variants
if [ "$rev" = WORK ]; then mkdir -p $B/src/paper_1701_08935_b200; cp -r $R/paper_1701_08935_b200/csrc $B/src/paper_1701_08935_b200/; cp -r $R/include $B/src/;
else (cd $R && git archive $rev paper_1701_08935_b200/csrc include | tar -x -C $B/src); fi
S=$B/src/paper_1701_08935_b200/csrc
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -I$B/src/include $extra"
for f in $S/*.cu; do $NV -c $f -o $B/$(basename $f .cu).o & done
for f in $S/*.cpp; do g++ -std=c++17 -O3 -fPIC -pthread $(echo "$extra" | grep -o "\-D[A-Z0-9_]*=[0-9]*") -c $f -o $B/$(basename $f .cpp).o & done
wait
for f in $S/*.cu $S/*.cpp; do o=$B/$(basename ${f%.*}).o; [ -f $o ] || { echo "missing $o"; exit 1; }; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/tools/dev/variants/libzolo_$name.so $B/*.o -lcudart -ldl
echo built tools/dev/variants/libzolo_$name.so
