#!/bin/bash
# Build compile-time variants of libpasgal_bcc.so for parameter sweeps (experiments only).
# usage: tools/build_variants.sh NAME "-DPG_WCH_U=16" ...
set -e
cd "$(dirname "$0")/.."
OUT=paper_2404_17101_b200/lib/variants
mkdir -p $OUT
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  d=$(mktemp -d)
  for f in bcc gen sort adj bfs vgc capi; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $defs \
      -c paper_2404_17101_b200/csrc/$f.cu -o $d/$f.o &
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/lib_$name.so $d/*.o
  rm -rf $d
  echo built $OUT/lib_$name.so
done
