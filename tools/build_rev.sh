#!/bin/bash
# Build libmrv.so of a git revision into exp/<name>.so (A/B experiments only).
#   bash tools/build_rev.sh <rev> <name>
set -e
rev=$1; name=$2
d=exp/src_$name; rm -rf $d; mkdir -p $d
git archive $rev include paper_2604_23960_b200/csrc | tar -x -C $d
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
  -shared -cudart static -o exp/$name.so $d/paper_2604_23960_b200/csrc/kernels.cu $d/paper_2604_23960_b200/csrc/scene.cpp
echo exp/$name.so
