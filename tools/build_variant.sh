#!/bin/bash
# Build libgsr.so from the csrc of a git revision (or a directory) into
# paper_2503_11731_b200/libgsr_<name>.so, for A/B sweeps with GSR_DEV_LIB.
# usage: tools/build_variant.sh <name> <git-rev>
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; rev=$2
tmp=$(mktemp -d)
mkdir -p $tmp/paper_2503_11731_b200/csrc $tmp/include
git -C "$ROOT" archive "$rev" paper_2503_11731_b200/csrc include | tar -x -C $tmp
cd $tmp/paper_2503_11731_b200/csrc
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared -cudart static \
  -o "$ROOT/paper_2503_11731_b200/libgsr_$name.so" *.cu
rm -rf $tmp
echo "$ROOT/paper_2503_11731_b200/libgsr_$name.so"
