#!/bin/bash
# build the working tree's libvmps.so with extra nvcc flags ($1, e.g. "-DVMPS_DESC4_ANCHOR=16") into $2
set -e
[ -n "$2" ] || { echo "usage: build_def.sh FLAGS OUT.so" >&2; exit 2; }
cd /root/repo/paper_2605_27147_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr -cudart static $1 -shared -o $2 *.cu
