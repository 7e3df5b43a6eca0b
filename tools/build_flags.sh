#!/bin/bash
# Build libgsr.so from the WORKING TREE with extra nvcc flags into
# paper_2503_11731_b200/libgsr_<name>.so, for A/B sweeps with GSR_DEV_LIB.
# usage: tools/build_flags.sh <name> [-DKNOB=value ...]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
cd $ROOT/paper_2503_11731_b200/csrc
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared -cudart static \
  "$@" -o "$ROOT/paper_2503_11731_b200/libgsr_$name.so" abi.cu project.cu sort.cu render.cu decode.cu route.cu backward.cu
echo "$ROOT/paper_2503_11731_b200/libgsr_$name.so"
