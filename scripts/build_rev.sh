#!/bin/bash
# build libvmps.so of git revision $1 into $2 (A/B comparisons via VMPS_LIB)
set -e
REV=$1; OUT=$2
T=$(mktemp -d)
git -C /root/repo archive $REV paper_2605_27147_b200/csrc include | tar -x -C $T
cd $T/paper_2605_27147_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr -cudart static -shared -o $OUT *.cu
rm -rf $T
