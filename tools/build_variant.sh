#!/bin/bash
# tools/build_variant.sh NAME SRC_DIR [cluster_header] : build an A/B variant of the C-ABI
# library from the sources in SRC_DIR (a copy of csrc/) into
# paper_2312_01121_b200/libsto_b200_NAME.so; load it with STO_LIB=libsto_b200_NAME.so
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; SRC=$2
W=$(mktemp -d); mkdir -p $W/csrc $W/include
cp $SRC/*.cu $SRC/*.cuh $SRC/*.cpp $W/csrc/; cp $ROOT/include/sto.h $W/include/
[ -n "$3" ] && cp $3 $W/csrc/sto_cluster_kernel.cuh
sed -i "s#\"../../include/sto.h\"#\"../include/sto.h\"#" $W/csrc/sto_b200.cu $W/csrc/sto_io.cpp
cd $W/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -shared \
  -o $ROOT/paper_2312_01121_b200/libsto_b200_$NAME.so sto_b200.cu sto_io.cpp -lcudart
rm -rf $W
